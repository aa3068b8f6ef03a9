"""Time the C3 compressed solve (K3) and check its digest; SP200_LIB selects an
alternative build for A/B timing.

    python tools/ab_c3.py --n 600 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1006_3148_b200 as sp

C3_DIGEST = "7933b08499ca106efc89cf070a608c49373b7594086ebb49a0cbd68c38230d35"

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=600)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--zchunk", type=int, default=0)
ap.add_argument("--maxfused", type=int, default=4, help="levels per K3 launch (a pass of 4 = 4/maxfused launches)")
a = ap.parse_args()
sp.PipelineEngine.max_fused = a.maxfused
L = sp._lib.load()
L.sp_set_tuning(0, a.zchunk)
g = sp.create_grid(a.n, a.n, a.n, pad=4, init="random", seed=42, lo=-1.0, hi=1.0)
cfg = sp.PipelineConfig(spec=sp.BlockSpec(a.n, 30, 30), t=4, grid_mode="compressed")
sp.run_pipelined(g, cfg, 16)
ok = "n/a" if a.n != 600 else ("OK" if g.checksum() == C3_DIGEST else "MISMATCH " + g.checksum())
best = 0.0
for _ in range(a.reps):
    best = max(best, sp.run_pipelined(g, cfg, 16).mlups / 1e3)
print(f"C3 n={a.n}: digest {ok}; best {best:.1f} GLUP/s over {a.reps} x 64 sweeps", flush=True)
