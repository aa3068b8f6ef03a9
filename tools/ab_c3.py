"""A/B the K3 band epilogue (sp_set_tuning key 6: 0 = in-pass last-arriver
unstash, 1 = separate k_unstash_* launches): C3 digest check, then GLUP/s.

    python tools/ab_c3.py --modes 0,1 --n 600 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1006_3148_b200 as sp

C3_DIGEST = "7933b08499ca106efc89cf070a608c49373b7594086ebb49a0cbd68c38230d35"

ap = argparse.ArgumentParser()
ap.add_argument("--modes", default="0,1")
ap.add_argument("--n", type=int, default=600)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--zchunk", type=int, default=0)
a = ap.parse_args()
L = sp._lib.load()
L.sp_set_tuning(0, a.zchunk)
for m in [int(v) for v in a.modes.split(",")]:
    L.sp_set_tuning(6, m)
    g = sp.create_grid(a.n, a.n, a.n, pad=4, init="random", seed=42, lo=-1.0, hi=1.0)
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(a.n, 30, 30), t=4, grid_mode="compressed")
    st = sp.run_pipelined(g, cfg, 16)
    dig = g.checksum() if a.n == 600 else None
    ok = "n/a" if dig is None else ("OK" if dig == C3_DIGEST else "MISMATCH " + dig)
    best = 0.0
    for _ in range(a.reps):
        st = sp.run_pipelined(g, cfg, 16)
        best = max(best, st.mlups / 1e3)
    print(f"mode={m} n={a.n}: digest {ok}; best {best:.1f} GLUP/s over {a.reps} x 64 sweeps", flush=True)
    del g
    torch.cuda.empty_cache()
if a.n == 600 and "0" in a.modes:
    # bounds: debug 16 = every band plane in place (timing only, wrong
    # results), 32 = every band plane stashed (the epilogue copies it all)
    L.sp_set_tuning(6, 0)
    for dbg in (16, 32):
        L.sp_set_tuning(4, dbg)
        g = sp.create_grid(a.n, a.n, a.n, pad=4, init="random", seed=42, lo=-1.0, hi=1.0)
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(a.n, 30, 30), t=4, grid_mode="compressed")
        best = 0.0
        for _ in range(a.reps):
            best = max(best, sp.run_pipelined(g, cfg, 16).mlups / 1e3)
        print(f"debug={dbg}: best {best:.1f} GLUP/s", flush=True)
        del g
    L.sp_set_tuning(4, 0)
