"""A/B the two-grid K2 layouts (sp_set_tuning key 9: 0 lane pairs, 1 column
layout, 2 column layout with level-1 shuffles): bit-exact check against the
oracle on ragged shapes and live z ranges, then GLUP/s per fused depth.

    python tools/ab_layout.py --layouts 0,1,2 --ts 2,3,4 --n 512
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
import paper_1006_3148_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--layouts", default="0,1,2")
ap.add_argument("--ts", default="2,3,4")
ap.add_argument("--n", default="512")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--no-check", action="store_true")
ap.add_argument("--tune", default="", help="extra sp_set_tuning pairs, e.g. 0=64")
a = ap.parse_args()
L = sp._lib.load()
for kv in filter(None, a.tune.split(",")):
    k, v = kv.split("=")
    L.sp_set_tuning(int(k), int(v))
lays = [int(c) for c in a.layouts.split(",")]
ts = [int(t) for t in a.ts.split(",")]

bad_total = 0
if not a.no_check:
    shapes = [(90, 61, 30), (130, 130, 20), (37, 100, 17), (64, 5, 9), (70, 200, 12), (1, 1, 1),
              (33, 31, 3), (200, 97, 40)]
    for dims in shapes:
        d0 = oracle.make_storage(*dims, init="random", seed=7, ring=0.5)
        for t in ts:
            exp = oracle.interior(oracle.sweeps(d0, dims, t), *dims)
            for c in lays:
                for loader in (0, 1):
                    L.sp_set_tuning(9, c)
                    L.sp_set_tuning(1, loader)
                    g = sp.create_grid(*dims, init="random", seed=7, ring=0.5)
                    dst = g.copy()
                    sp.fused_sweeps(g, dst, t)
                    ok = np.array_equal(dst.interior_numpy(), exp)
                    nz = dims[2]
                    zlo, zhi = min(1, nz - 1), max(nz - 1, 1)
                    dst2 = g.copy()
                    dst2.data.fill_(-3.0)
                    sp.fused_sweeps(g, dst2, t, zlo, zhi)
                    got2 = dst2.interior_numpy()
                    ok2 = np.array_equal(got2[zlo:zhi], exp[zlo:zhi]) and np.all(got2[:zlo] == -3.0) \
                        and np.all(got2[zhi:] == -3.0)
                    if not (ok and ok2):
                        bad_total += 1
                        bad = np.argwhere(dst.interior_numpy() != exp)
                        print(f"MISMATCH dims={dims} t={t} layout={c} loader={loader}: "
                              f"full={ok} range={ok2} first bad (z,y,x) {bad[:4].tolist()} count {len(bad)}",
                              flush=True)
    L.sp_set_tuning(1, 0)
    print(f"check done: {bad_total} mismatching cases", flush=True)

for n in [int(x) for x in a.n.split(",")]:
    g = sp.create_grid(n, n, n, init="random", seed=42)
    h = g.copy()
    bufs = [g, h]
    for t in ts:
        for c in lays:
            L.sp_set_tuning(9, c)
            for r in range(3):
                sp.fused_sweeps(bufs[r % 2], bufs[1 - r % 2], t)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for r in range(a.reps):
                sp.fused_sweeps(bufs[r % 2], bufs[1 - r % 2], t)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / a.reps
            print(f"time t={t} layout={c} n={n}: {ms:.3f} ms/pass, {n ** 3 * t / ms / 1e6:.1f} GLUP/s",
                  flush=True)
    del g, h, bufs
    torch.cuda.empty_cache()
