"""A/B a K2 kernel variant (sp_set_tuning key 2 = levels*16 + cfg index):
bit-exact check against the oracle on ragged shapes, then GLUP/s on 512^3.

    python tools/ab_cfg.py --cfgs 0,4 --ts 2,3,4
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
ap.add_argument("--cfgs", default="0,4")
ap.add_argument("--ts", default="2,3,4")
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--no-check", action="store_true")
ap.add_argument("--debug", type=int, default=0, help="sp_set_tuning key 4 (profiling builds)")
ap.add_argument("--tune", default="", help="extra sp_set_tuning pairs, e.g. 6=1")
a = ap.parse_args()
L = sp._lib.load()
L.sp_set_tuning(4, a.debug)
for kv in filter(None, a.tune.split(",")):
    k, v = kv.split("=")
    L.sp_set_tuning(int(k), int(v))
cfgs = [int(c) for c in a.cfgs.split(",")]
ts = [int(t) for t in a.ts.split(",")]

if not a.no_check:
    shapes = [(90, 61, 30), (130, 130, 20), (37, 100, 17), (64, 5, 9), (70, 200, 12), (1, 1, 1)]
    for dims in shapes:
        d0 = oracle.make_storage(*dims, init="random", seed=7, ring=0.5)
        for t in ts:
            exp = oracle.interior(oracle.sweeps(d0, dims, t), *dims)
            for c in cfgs:
                L.sp_set_tuning(2, t * 16 + c)
                g = sp.create_grid(*dims, init="random", seed=7, ring=0.5)
                dst = g.copy()
                sp.fused_sweeps(g, dst, t)
                ok = np.array_equal(dst.interior_numpy(), exp)
                # live z range (distributed ghost shrink)
                nz = dims[2]
                zlo, zhi = min(1, nz - 1), max(min(nz - 1, nz), 1)
                dst2 = g.copy()
                dst2.data.fill_(-3.0)
                sp.fused_sweeps(g, dst2, t, zlo, zhi)
                ok2 = np.array_equal(dst2.interior_numpy()[zlo:zhi], exp[zlo:zhi])
                print(f"check dims={dims} t={t} cfg={c}: {'OK' if ok and ok2 else 'MISMATCH'}", flush=True)
                if not (ok and ok2):
                    bad = np.argwhere(dst.interior_numpy() != exp)
                    print("  first bad (z,y,x):", bad[:5].tolist(), "count", len(bad))
    L.sp_set_tuning(2, 0)

n = a.n
g = sp.create_grid(n, n, n, init="random", seed=42)
h = g.copy()
bufs = [g, h]
for t in ts:
    for c in cfgs:
        L.sp_set_tuning(2, t * 16 + c)
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
        print(f"time t={t} cfg={c} n={n}: {ms:.3f} ms/pass, {n ** 3 * t / ms / 1e6:.1f} GLUP/s", flush=True)
