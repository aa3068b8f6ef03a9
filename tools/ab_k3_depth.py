"""K3 (compressed) GLUP/s per fused depth t on 600^3 and 512^3, with an oracle-free
cross-check: in-place vs stash storage must be bit-identical."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1006_3148_b200 as sp
L = sp._lib.load()
for dims in [(600, 600, 600), (512, 512, 512)]:
    for t in (2, 3, 4):
        out = {}
        for stash in (1, 0):
            L.sp_set_tuning(10, stash)
            g = sp.create_grid(*dims, pad=4, init="random", seed=42, lo=-1.0, hi=1.0)
            cfg = sp.PipelineConfig(spec=sp.BlockSpec(dims[0], 8, 8), t=t, grid_mode="compressed")
            sp.run_pipelined(g, cfg, 4)
            best = max(sp.run_pipelined(g, cfg, 12).mlups / 1e3 for _ in range(3))
            out[stash] = (best, g.data.clone())
            del g
        same = torch.equal(out[0][1], out[1][1])
        print(f"{dims} t={t}: stash {out[1][0]:.1f}  in place {out[0][0]:.1f} GLUP/s  identical={same}", flush=True)
L.sp_set_tuning(10, 0)
