"""Diagnostic: run each fused depth / loader in its own process and compare
with the oracle (isolates sticky CUDA faults)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def one(levels, loader, dims):
    import numpy as np, torch
    import oracle, paper_1006_3148_b200 as sp
    L = sp._lib.load()
    L.sp_set_tuning(1, 1 if loader == "cpasync" else 0)
    d0 = oracle.make_storage(*dims, init="random", seed=7, ring=0.75)
    src = sp.Grid3.from_numpy(*dims, 0, d0)
    dst = src.copy()
    sp.fused_sweeps(src, dst, levels)
    torch.cuda.synchronize()
    exp = oracle.interior(oracle.sweeps(d0, dims, levels), *dims)
    got = dst.interior_numpy()
    bad = np.flatnonzero(got != exp)
    return f"mismatch {bad.size} first {np.unravel_index(bad[0], got.shape) if bad.size else None}" if bad.size else "ok"

if __name__ == "__main__":
    if len(sys.argv) > 1:
        lv, ld = int(sys.argv[1]), sys.argv[2]
        dims = tuple(int(v) for v in sys.argv[3].split("x"))
        try:
            print(lv, ld, dims, one(lv, ld, dims), flush=True)
        except Exception as e:
            print(lv, ld, dims, "ERROR", repr(e)[:300], flush=True)
        sys.exit(0)
    for dims in ("60x60x60", "13x9x6", "130x70x20"):
        for ld in ("tma", "cpasync"):
            for lv in (1, 2, 3, 4):
                subprocess.run([sys.executable, __file__, str(lv), ld, dims], timeout=120)
