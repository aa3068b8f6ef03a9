"""Run a few fused launches of one depth on the C2 grid (for ncu captures)."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1006_3148_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--t", type=int, default=4)
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cfg", type=int, default=0)
ap.add_argument("--zc", type=int, default=0)
ap.add_argument("--debug", type=int, default=0)
a = ap.parse_args()
L = sp._lib.load()
L.sp_set_tuning(2, a.t * 16 + a.cfg)
L.sp_set_tuning(0, a.zc)
L.sp_set_tuning(4, a.debug)
g = sp.create_grid(a.n, a.n, a.n, init="random", seed=42)
h = g.copy()
bufs = [g, h]
for r in range(a.reps):
    sp.fused_sweeps(bufs[r % 2], bufs[1 - r % 2], a.t)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for r in range(a.reps):
    sp.fused_sweeps(bufs[r % 2], bufs[1 - r % 2], a.t)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / a.reps
print(f"t={a.t} cfg={a.cfg} zc={a.zc} dbg={a.debug} n={a.n}: {ms:.3f} ms/launch, {a.n**3*a.t/ms/1e6:.1f} GLUP/s")
