"""A/B of fused depths beyond SP_MAX_FUSED (A/B build only):
    SP200_LIB=paper_1006_3148_b200/libsp200_ab.so python tools/ab_depth.py
Bit-exact check of T=5 / T=8 against the oracle, then GLUP/s of 100 sweeps
of C2 (512^3) in passes of 4, 5 and 8 fused sweeps (and t=8 as two launches
of 4, the product's schedule)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
import paper_1006_3148_b200 as sp

for dims in [(90, 61, 30), (130, 70, 24)]:
    d0 = oracle.make_storage(*dims, init="random", seed=7, ring=0.5)
    for t in (5,):
        exp = oracle.interior(oracle.sweeps(d0, dims, t), *dims)
        g = sp.create_grid(*dims, init="random", seed=7, ring=0.5)
        dst = g.copy()
        sp.fused_sweeps(g, dst, t)
        print(f"check dims={dims} t={t}: {'OK' if np.array_equal(dst.interior_numpy(), exp) else 'MISMATCH'}",
              flush=True)

n = 512
g = sp.create_grid(n, n, n, init="random", seed=42)
bufs = [g, g.copy()]


def plan(total, t):
    k = -(-total // t)
    b, e = divmod(total, k)
    return [b + (1 if i < e else 0) for i in range(k)]


for name, depths in [("t=4", plan(100, 4)), ("t=5", plan(100, 5)), 
                     ("t=8 as 2x4", [c for h in plan(100, 8) for c in sp.split_levels(h, 4)])]:
    for rep in range(2):
        for i, c in enumerate(depths):
            sp.fused_sweeps(bufs[i % 2], bufs[1 - i % 2], c)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for rep in range(3):
        for i, c in enumerate(depths):
            sp.fused_sweeps(bufs[i % 2], bufs[1 - i % 2], c)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    print(f"time {name} n={n}: {ms:.3f} ms per 100 sweeps, {n ** 3 * 100 / ms / 1e6:.1f} GLUP/s "
          f"(depths {sorted(set(depths))})", flush=True)
