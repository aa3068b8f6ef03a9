"""K3 (compressed, t=4) GLUP/s on a few grid shapes; SP200_TUNE selects variants."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1006_3148_b200 as sp
for dims in [(300, 300, 600), (256, 256, 256), (512, 512, 512), (600, 600, 600), (1024, 1024, 256), (400, 400, 400)]:
    g = sp.create_grid(*dims, pad=4, init="random", seed=42, lo=-1.0, hi=1.0)
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(dims[0], 8, 8), t=4, grid_mode="compressed")
    sp.run_pipelined(g, cfg, 4)
    best = max(sp.run_pipelined(g, cfg, 16).mlups / 1e3 for _ in range(3))
    print(f"{dims}: {best:.1f} GLUP/s", flush=True)
    del g
