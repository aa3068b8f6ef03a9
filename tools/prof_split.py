import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1006_3148_b200 as sp
L = sp._lib.load()
L.sp_set_tuning(9, int(os.environ.get("LAYOUT", "4")))
n = 512
g = sp.create_grid(n, n, n, init="random", seed=42)
h = g.copy()
for r in range(6):
    sp.fused_sweeps(g if r % 2 == 0 else h, h if r % 2 == 0 else g, 4)
torch.cuda.synchronize()
