"""GPU: out-of-bounds write detection without a sanitizer.  Every grid and
the K3 stash live in the middle of a larger buffer filled with a canary
pattern; after K1, K2 (all depths, both loaders, z-chunks, live ranges),
K3 (both directions, depths 1-4), the window seam, faces and ring kernels,
the guard regions must be untouched and the results must still match the
oracle bit for bit."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

sp = pytest.importorskip("paper_1006_3148_b200")
from paper_1006_3148_b200.kernel import compressed_pass  # noqa: E402

GUARD = 1 << 16  # doubles on each side (512 KB)
CANARY = -7.25e300


def guarded(shape):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), CANARY, dtype=torch.float64, device="cuda")
    return buf, buf[GUARD:GUARD + n].view(shape)


def intact(buf, n):
    return bool(torch.all(buf[:GUARD] == CANARY)) and bool(torch.all(buf[GUARD + n:] == CANARY))


def guarded_grid(nx, ny, nz, pad=0, **kw):
    src = sp.create_grid(nx, ny, nz, pad=pad, **kw)
    buf, view = guarded(tuple(src.data.shape))
    view.copy_(src.data)
    g = sp.Grid3(nx, ny, nz, pad, data=view)
    g.boundary_faces = src.boundary_faces
    return buf, g


@pytest.mark.parametrize("dims", [(70, 37, 21), (64, 32, 16), (5, 3, 2), (130, 66, 9)])
def test_two_grid_kernels_stay_in_bounds(dims):
    L = sp._lib.load()
    for force in (0, 1):
        L.sp_set_tuning(1, force)
        try:
            ba, a = guarded_grid(*dims, init="random", seed=1, ring=0.5)
            bb, b = guarded_grid(*dims, init="random", seed=1, ring=0.5)
            d = oracle.make_storage(*dims, init="random", seed=1, ring=0.5)
            sp.reference_sweep(a, b)
            levels, cur, oth = 1, b, a
            for t in (2, 3, 4):
                sp.fused_sweeps(cur, oth, t)
                levels += t
                cur, oth = oth, cur
            n = a.data.numel()
            assert intact(ba, n) and intact(bb, n)
            exp = oracle.interior(oracle.sweeps(d, dims, levels), *dims)
            assert_bitwise(cur.interior_numpy(), exp)
            sp.fused_sweeps(a, b, 4, 1, max(2, dims[2] - 1))
            sp.apply_window(a.data, a.data, ((0, dims[0]), (0, dims[1]), (0, dims[2])), a.offset, a.offset)
            sp.copy_ring(a, b)
            assert sp.rings_equal(a, b)
            assert intact(ba, n) and intact(bb, n)
        finally:
            L.sp_set_tuning(1, 0)


@pytest.mark.parametrize("t,dims", [(4, (66, 35, 24)), (3, (61, 29, 19)), (2, (130, 70, 12)),
                                    (1, (20, 9, 7))])
def test_compressed_kernels_stay_in_bounds(t, dims):
    bg, g = guarded_grid(*dims, pad=t, init="random", seed=3, lo=-1.0, hi=1.0)
    n = g.data.numel()
    nbytes = int(sp._lib.load().sp_compressed_workspace(dims[0], dims[1], dims[2], t))
    wbuf = torch.full((max(nbytes, 256) // 8 + 2 * GUARD + 1,), CANARY, dtype=torch.float64, device="cuda")
    ws = wbuf[GUARD:GUARD + max(nbytes, 256) // 8 + 1].view(torch.uint8)
    d = oracle.make_storage(*dims, pad=t, init="random", seed=3, lo=-1.0, hi=1.0)
    for p, direction in enumerate((1, -1, 1, -1)):
        compressed_pass(g, t, direction, g.alignment, ws)
        g.alignment += t * direction
    assert intact(bg, n)
    assert bool(torch.all(wbuf[:GUARD] == CANARY))
    assert bool(torch.all(wbuf[GUARD + max(nbytes, 256) // 8 + 1:] == CANARY))
    exp = oracle.interior(oracle.sweeps(oracle.make_storage(*dims, init="random", seed=3, lo=-1.0, hi=1.0),
                                        dims, 4 * t), *dims)
    assert_bitwise(g.interior_numpy(), exp)


def test_compressed_workspace_covers_every_layout():
    """sp_compressed_workspace is the worst case over the stored-tile parities
    a launch may pick (the parity changes the tile count and so the z-chunk
    count); a launch given less than its own layout needs fails with
    ValueError instead of writing past the stash (512^3, t=1, pad 1: the case
    where the parities pick different chunk counts)."""
    n, t = 512, 1
    bg, g = guarded_grid(n, n, n, pad=t, init="random", seed=9, lo=-1.0, hi=1.0)
    nbytes = int(sp._lib.load().sp_compressed_workspace(n, n, n, t))
    words = max(nbytes, 256) // 8 + 1
    wbuf = torch.full((words + 2 * GUARD,), CANARY, dtype=torch.float64, device="cuda")
    ws = wbuf[GUARD:GUARD + words].view(torch.uint8)
    d = oracle.make_storage(n, n, n, pad=t, init="random", seed=9, lo=-1.0, hi=1.0)
    with pytest.raises(ValueError):
        compressed_pass(g, t, 1, g.alignment, ws[:64])
    for direction in (1, -1):
        compressed_pass(g, t, direction, g.alignment, ws)
        g.alignment += t * direction
    assert intact(bg, g.data.numel())
    assert bool(torch.all(wbuf[:GUARD] == CANARY)) and bool(torch.all(wbuf[GUARD + words:] == CANARY))
    a = oracle.make_storage(n, n, n, init="random", seed=9, lo=-1.0, hi=1.0)
    exp = oracle.interior(oracle.sweeps(a, (n, n, n), 2), n, n, n)
    assert_bitwise(g.interior_numpy(), exp)


@pytest.mark.parametrize("t", [2, 3, 4])
def test_in_place_workspace_is_small_and_guarded(t):
    """The in-place K3 pass (t = 2..4) needs its progress counters and the z
    stash of the z-chunked tiles only: sp_compressed_workspace_for returns
    that size for the array (far below the band stash), a launch inside
    canaries with exactly that many bytes touches nothing outside and is
    bit-exact, and a smaller workspace fails with ValueError."""
    n = (300, 290, 70)
    L = sp._lib.load()
    bg, g = guarded_grid(*n, pad=4, init="random", seed=9, lo=-1.0, hi=1.0)
    ex, ey, _ = g.extents
    from paper_1006_3148_b200.kernel import _ptr
    small = int(L.sp_compressed_workspace_for(_ptr(g.data), ex, ey, n[0], n[1], n[2], t))
    worst = int(L.sp_compressed_workspace(n[0], n[1], n[2], t))
    assert 0 < small <= worst
    L.sp_set_tuning(7, 1)   # whole columns only: counters, no z stash
    try:
        tiny = int(L.sp_compressed_workspace_for(_ptr(g.data), ex, ey, n[0], n[1], n[2], t))
    finally:
        L.sp_set_tuning(7, 0)
    assert tiny < 64 * 1024 and tiny < worst // 50
    words = small // 8 + 1
    wbuf = torch.full((words + 2 * GUARD,), CANARY, dtype=torch.float64, device="cuda")
    ws = wbuf[GUARD:GUARD + words].view(torch.uint8)[:small]
    with pytest.raises(ValueError):
        compressed_pass(g, t, 1, g.alignment, ws[:128])
    for direction in (1, -1):
        compressed_pass(g, t, direction, g.alignment, ws)
        g.alignment += t * direction
    assert intact(bg, g.data.numel())
    assert bool(torch.all(wbuf[:GUARD] == CANARY)) and bool(torch.all(wbuf[GUARD + words:] == CANARY))
    a = oracle.make_storage(*n, init="random", seed=9, lo=-1.0, hi=1.0)
    exp = oracle.interior(oracle.sweeps(a, n, 2 * t), *n)
    assert_bitwise(g.interior_numpy(), exp)
