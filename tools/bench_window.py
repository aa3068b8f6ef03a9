"""Time the apply_window seam (k_window, the path of every non-fusable pass
and direct apply_window callers) against the plain sweep K1 on 512^3:
    python tools/bench_window.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1006_3148_b200 as sp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = sp.create_grid(n, n, n, init="random", seed=42)
h = g.copy()
win = ((0, n), (0, n), (0, n))


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


peak = 6551.7
ms = timed(lambda: sp.apply_window(g.data, h.data, win, g.offset, h.offset))
print(f"apply_window two-grid {n}^3: {ms:.3f} ms, {n**3 / ms / 1e6:.1f} GLUP/s, "
      f"{n**3 * 16 / ms / 1e6 / peak:.3f} of the 16 B/LUP HBM roofline")
ms = timed(lambda: sp.apply_window(g.data, g.data, ((0, n), (0, n), (0, n - 2)), g.offset, g.offset - 1) if False else None)
g2 = sp.create_grid(n, n, n, pad=1, init="random", seed=42)
ms = timed(lambda: sp.apply_window(g2.data, g2.data, win, g2.offset, g2.offset - 1))
print(f"apply_window shifted in place (scratch + unstage) {n}^3: {ms:.3f} ms, {n**3 / ms / 1e6:.1f} GLUP/s")
ms = timed(lambda: sp.reference_sweep(g, h))
print(f"reference_sweep (K1) {n}^3: {ms:.3f} ms, {n**3 / ms / 1e6:.1f} GLUP/s")
