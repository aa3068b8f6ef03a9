import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1006_3148_b200 as sp
L = sp._lib.load()
dims = tuple(int(v) for v in sys.argv[1].split(","))
npass = int(sys.argv[2])
cfg = sp.PipelineConfig(spec=sp.BlockSpec(dims[0], 8, 8), t=4, grid_mode="compressed")
res = []
for stash in (1, 0):
    L.sp_set_tuning(10, stash)
    g = sp.create_grid(*dims, pad=4, init="random", seed=100, lo=-1.0, hi=1.0)
    eng = sp.PipelineEngine(cfg, g)
    out = []
    for k in range(npass):
        eng.run_pass(1 if k % 2 == 0 else -1)
        out.append(g.interior_numpy().copy())
    res.append(out)
for k in range(npass):
    a, b = res[0][k], res[1][k]
    bad = np.argwhere(a != b)
    print("pass", k, "mismatch", len(bad))
    if len(bad):
        z, y, x = bad[:, 0], bad[:, 1], bad[:, 2]
        print("  z planes:", np.unique(z)[:40], "count", len(np.unique(z)))
        print("  y range:", y.min(), y.max(), " x range:", x.min(), x.max())
        print("  y/26 tiles:", np.unique(y // 26)[:30])
        break
# the same through run_pipelined (faces trusted between passes)
res = []
for stash in (1, 0):
    L.sp_set_tuning(10, stash)
    g = sp.create_grid(*dims, pad=4, init="random", seed=100, lo=-1.0, hi=1.0)
    sp.run_pipelined(g, cfg, npass)
    res.append(g.interior_numpy().copy())
bad = np.argwhere(res[0] != res[1])
print("run_pipelined", npass, "passes: mismatch", len(bad))
if len(bad):
    z, y, x = bad[:, 0], bad[:, 1], bad[:, 2]
    print("  z planes:", np.unique(z)[:40], "count", len(np.unique(z)))
    print("  y range:", y.min(), y.max(), " x range:", x.min(), x.max())
