"""CPU ORACLE — test / baseline infrastructure, never the product.

A NumPy + threads restatement of the reference's pipelined temporal-blocking
scheduler (/root/reference/pkg/src/stencilpipe/pipeline.py), used only as the
`cpu_baseline` timing of bench.py (run_pipelined with
n=1, T=1, d_l=1, d_u=3, block (nx,32,32), relaxed sync, on t threads) and in
tests/test_oracle.py against the plain sweeps.  The reference itself is pure
Python and cannot travel to the GPU box, so this restatement stands in for it.

Schedule (sp/pipeline.py:212-221, 285-312, 363-395):
  * the interior is cut into blocks (sp/grid.py:187-206), visited in
    lexicographic order (z outermost);
  * thread g applies levels g*T+1 .. g*T+T to each block; the window of level
    u is the block shifted by -u on every axis (forward pass), clamped to the
    interior, so the windows of one level still tile the interior;
  * relaxed sync (Eq. 3): thread g starts block k only when its
    predecessor has finished d_l more blocks, and stays at most d_u blocks
    ahead of its successor; the last block bumps by d_u + 1 (wind-down);
  * two-grid: level lvl reads grids[(lvl-1) % 2] and writes grids[lvl % 2].
NumPy's element-wise ufuncs release the GIL, which is what lets the threads
run concurrently.
"""

from __future__ import annotations

import threading
import time

from . import apply_window


def _bounds(bases, delta, n):
    out = [0]
    for b in bases[1:]:
        out.append(min(max(b + delta, 0), n))
    out.append(n)
    return out


def pipelined_pass_two_grid(grids, n, t, block, levels_done=0, T=1, d_l=1, d_u=3, off=1):
    """One forward pass of h = t*T levels over a two-grid pair of storage
    arrays (numpy, (z, y, x)); returns the index of the grid holding the
    result.  n = (nx, ny, nz), block = (bx, by, bz)."""
    nx, ny, nz = n
    bx, by, bz = block
    bases = [list(range(0, nx, bx)), list(range(0, ny, by)), list(range(0, nz, bz))]
    blocks = [(ix, iy, iz) for iz in range(len(bases[2])) for iy in range(len(bases[1]))
              for ix in range(len(bases[0]))]
    h = t * T
    tables = {u: [_bounds(bases[ax], -u, n[ax]) for ax in range(3)] for u in range(1, h + 1)}
    counters = [0] * t
    errors = []

    def level(k, u):
        ix, iy, iz = blocks[k]
        bxs, bys, bzs = tables[u]
        win = ((bxs[ix], bxs[ix + 1]), (bys[iy], bys[iy + 1]), (bzs[iz], bzs[iz + 1]))
        if any(lo >= hi for lo, hi in win):
            return
        lvl = levels_done + u
        apply_window(grids[(lvl - 1) % 2], grids[lvl % 2], win, off, off)

    def worker(g):
        try:
            total = len(blocks)
            for k in range(total):
                if g > 0:
                    while counters[g - 1] - counters[g] < d_l:
                        time.sleep(0)
                for i in range(1, T + 1):
                    level(k, g * T + i)
                if k == total - 1:
                    counters[g] += d_u + 1
                else:
                    counters[g] += 1
                    if g < t - 1:
                        while counters[g] - counters[g + 1] > d_u:
                            time.sleep(0)
        except BaseException as exc:  # surface to the caller
            errors.append(exc)
            counters[g] += 1 << 40

    threads = [threading.Thread(target=worker, args=(g,), daemon=True) for g in range(t)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    return (levels_done + h) % 2
