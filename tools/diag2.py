import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1006_3148_b200 as sp
L = sp._lib.load()
dims = (600, 600, 600)
cfg = sp.PipelineConfig(spec=sp.BlockSpec(dims[0], 8, 8), t=4, grid_mode="compressed")
res = []
for stash in (1, 0):
    L.sp_set_tuning(10, stash)
    g = sp.create_grid(*dims, pad=4, init="random", seed=100, lo=-1.0, hi=1.0)
    eng = sp.PipelineEngine(cfg, g)
    eng.run_pass(1)
    eng.run_pass(-1)
    res.append(g.interior_numpy().copy())
a, b = res
bad = np.argwhere(a != b)
z, y, x = bad[:, 0], bad[:, 1], bad[:, 2]
print("n", len(bad))
print("unique y:", np.unique(y)[:80])
print("unique x:", np.unique(x))
zs = np.unique(z)
print("z min max", zs.min(), zs.max())
for yy in np.unique(y)[:6]:
    m = bad[y == yy]
    print("y", yy, "z range", m[:, 0].min(), m[:, 0].max(), "x", np.unique(m[:, 2]))
# per tile row: first bad z
for ty in range(0, 12):
    m = bad[(y // 26) == ty]
    if len(m):
        print("ty", ty, "count", len(m), "z", m[:, 0].min(), m[:, 0].max(), "y%26", np.unique(m[:, 1] % 26))
