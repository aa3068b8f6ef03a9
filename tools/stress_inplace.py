"""Stress the in-place K3 pass (--t 2..4): the same passes with the band-stash path
(tuning key 10 = 1) must leave bit-identical storage, pass after pass, on
shapes with one and several rounds of tiles, with and without another stream
keeping some SMs busy (so tiles of one pass start at different times and the
progress waits actually run).

    python tools/stress_inplace.py --reps 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1006_3148_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--passes", type=int, default=4)
ap.add_argument("--t", type=int, default=4)
a = ap.parse_args()
L = sp._lib.load()

SHAPES = [(600, 600, 160), (700, 500, 120), (1000, 300, 100), (300, 1000, 90), (1200, 1200, 48),
          (130, 90, 300), (59, 27, 500), (2000, 64, 64), (64, 2000, 64)]
bad = 0
total = 0
side = torch.cuda.Stream()
for dims in SHAPES:
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(dims[0], 8, 8), t=a.t, grid_mode="compressed")
    for rep in range(a.reps):
        for disturb in (False, True):
            res = []
            for stash in (1, 0):
                L.sp_set_tuning(10, stash)
                g = sp.create_grid(*dims, pad=4, init="random", seed=100 + rep, lo=-1.0, hi=1.0)
                eng = sp.PipelineEngine(cfg, g)
                snaps = []
                if disturb and not stash:
                    # a plain sweep loop on another stream takes SMs away at random times
                    d = sp.create_grid(256, 256, 256, init="random", seed=1)
                    e = d.copy()
                    with torch.cuda.stream(side):
                        for _ in range(40):
                            sp.reference_sweep(d, e)
                            d, e = e, d
                for k in range(a.passes):
                    eng.run_pass(1 if k % 2 == 0 else -1)
                    snaps.append(g.data.clone())
                torch.cuda.synchronize()
                res.append(snaps)
            for k, (x, y) in enumerate(zip(*res)):
                total += 1
                if not torch.equal(x, y):
                    bad += 1
                    print(f"MISMATCH dims={dims} rep={rep} disturb={disturb} pass={k}: "
                          f"{int((x != y).sum())} cells differ", flush=True)
    print(f"dims={dims}: ok so far ({total - bad}/{total})", flush=True)
L.sp_set_tuning(10, 0)
print(f"stress done: {bad} mismatching passes of {total}")
sys.exit(1 if bad else 0)
