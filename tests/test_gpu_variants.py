"""Every K2 kernel instance the dispatcher can select (sp_set_tuning key 2:
levels*16 + index), including the tall-tile defaults and the two-CTA cluster
variant (index 4: DSMEM halo rows through st.async), bit-exact against the
oracle on ragged shapes and over live z ranges.  The alternative instances
exist only in A/B builds (-DSP200_AB=1, tools/build_variant.py); in the
product library every index selects the default instance, which these tests
then cover on the same shapes."""

import numpy as np
import pytest

import oracle
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

sp = pytest.importorskip("paper_1006_3148_b200")

SHAPES = [(90, 61, 30), (130, 130, 20), (37, 100, 17), (64, 5, 9), (70, 200, 12)]


@pytest.fixture
def lib():
    L = sp._lib.load()
    yield L
    for t in range(1, 5):
        L.sp_set_tuning(2, t * 16)
    L.sp_set_tuning(6, 0)
    L.sp_set_tuning(7, 0)


@pytest.mark.parametrize("levels,idx", [(lv, i) for lv in (2, 3, 4) for i in range(6)] +
                         [(4, 6)] +                                   # WP: level 0 from the stage ring
                         [(1, i) for i in range(8)])   # 0, 5-7: k_temporal<1> tiles; 1-4: k_sweep1
def test_kernel_variants(lib, levels, idx):
    assert lib.sp_set_tuning(2, levels * 16 + idx) == 0
    for dims in SHAPES:
        d0 = oracle.make_storage(*dims, init="random", seed=11, ring=0.5)
        exp = oracle.interior(oracle.sweeps(d0, dims, levels), *dims)
        g = sp.create_grid(*dims, init="random", seed=11, ring=0.5)
        dst = g.copy()
        sp.fused_sweeps(g, dst, levels)
        assert_bitwise(dst.interior_numpy(), exp)
        zlo, zhi = 1, dims[2] - 2
        dst2 = g.copy()
        dst2.data.fill_(-3.0)
        sp.fused_sweeps(g, dst2, levels, zlo, zhi)
        got = dst2.interior_numpy()
        assert_bitwise(got[zlo:zhi], exp[zlo:zhi])
        assert np.all(got[:zlo] == -3.0) and np.all(got[zhi:] == -3.0)


@pytest.mark.parametrize("two_launch,balanced", [(0, 0), (1, 0), (0, 1)])
def test_split_grid_pass(lib, two_launch, balanced):
    """K2 pass with more tiles than SMs: one split grid (full columns, then
    z-chunk CTAs; default), two launches (tuning key 6), or one column plus
    an equal piece of the remaining columns per CTA, pieces crossing tile
    boundaries (tuning key 7)."""
    assert lib.sp_set_tuning(6, two_launch) == 0
    assert lib.sp_set_tuning(7, balanced) == 0
    dims = (700, 500, 40)   # 13 x 20 = 260 tiles at T=4 > 148 SMs
    d0 = oracle.make_storage(*dims, init="random", seed=3, ring=0.5)
    exp = oracle.interior(oracle.sweeps(d0, dims, 4), *dims)
    g = sp.create_grid(*dims, init="random", seed=3, ring=0.5)
    dst = g.copy()
    sp.fused_sweeps(g, dst, 4)
    assert_bitwise(dst.interior_numpy(), exp)


@pytest.mark.parametrize("t", [2, 3, 4])
@pytest.mark.parametrize("mode", ["in_place", "whole_columns", "chunks_of_8", "stash"])
@pytest.mark.parametrize("dims,pad", [((700, 500, 40), 4), ((90, 61, 30), 4), ((130, 130, 20), 5),
                                       ((64, 9, 12), 4), ((300, 290, 70), 4)])
def test_compressed_in_place_and_stash(lib, mode, dims, pad, t):
    """K3 at t=2..4.  The default pass stores everything in place: per-tile
    progress counters, tiles taken in dependency order; whole multiples of
    the SM count march full columns, the remaining tiles follow in a second
    launch as z-chunks decoupled by a z stash (260 tiles on the first shape).
    Tuning key 7 = 1: whole columns only; key 8: chunk length; key 10 = 1:
    the band stash and the unstash kernels.  Forward and backward passes,
    bit-exact against the oracle after every pass."""
    key, val = {"in_place": (7, 0), "whole_columns": (7, 1), "chunks_of_8": (8, 8), "stash": (10, 1)}[mode]
    assert lib.sp_set_tuning(key, val) == 0
    try:
        d0 = oracle.make_storage(*dims, init="random", seed=5, lo=-1.0, hi=1.0)
        g = sp.create_grid(*dims, pad=pad, init="random", seed=5, lo=-1.0, hi=1.0)
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(dims[0], 8, 8), t=t, grid_mode="compressed")
        eng = sp.PipelineEngine(cfg, g)
        for k in range(1, 4):
            eng.run_pass(1 if k % 2 == 1 else -1)
            exp = oracle.interior(oracle.sweeps(d0, dims, t * k), *dims)
            assert_bitwise(g.interior_numpy(), exp)
    finally:
        lib.sp_set_tuning(key, 0)


@pytest.mark.parametrize("layout", [6, 7, 8])
def test_tmem_state_layouts(lib, layout):
    """k_tm: K2 at t=4 with the level values parked in tensor memory between
    steps (tuning key 9 = 6: 12 warps, 64 x 48 region; 7: 8 warps, R = 6;
    8: the 64 x 32 region), bit-exact on ragged shapes and live z ranges."""
    assert lib.sp_set_tuning(9, layout) == 0
    try:
        for dims in SHAPES + [(700, 500, 24)]:
            d0 = oracle.make_storage(*dims, init="random", seed=11, ring=0.5)
            exp = oracle.interior(oracle.sweeps(d0, dims, 4), *dims)
            g = sp.create_grid(*dims, init="random", seed=11, ring=0.5)
            dst = g.copy()
            sp.fused_sweeps(g, dst, 4)
            assert_bitwise(dst.interior_numpy(), exp)
            zlo, zhi = 1, dims[2] - 2
            dst2 = g.copy()
            dst2.data.fill_(-3.0)
            sp.fused_sweeps(g, dst2, 4, zlo, zhi)
            got = dst2.interior_numpy()
            assert_bitwise(got[zlo:zhi], exp[zlo:zhi])
            assert np.all(got[:zlo] == -3.0) and np.all(got[zhi:] == -3.0)
    finally:
        lib.sp_set_tuning(9, 0)
