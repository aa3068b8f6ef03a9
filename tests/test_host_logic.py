"""CPU: host-side API parity of the drop-in (mirrors the host-logic parts of
pkg/tests/test_pipeline.py:51-124 and test_grid.py): config validation, Eq. 3
helpers, block plans, level splitting and the fusability rule."""

import types

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1006_3148_b200.grid import BlockSpec, decompose_blocks, next_block
from paper_1006_3148_b200.pipeline import (
    EffectiveDistances,
    PipelineConfig,
    PipelineEngine,
    SyncCounters,
    estimate_max_distance,
    may_advance,
    split_levels,
)


def _grid(nx, ny, nz):
    return types.SimpleNamespace(nx=nx, ny=ny, nz=nz)


def _counters(values):
    c = SyncCounters(len(values))
    for i, v in enumerate(values):
        c.bump(i, v)
    return c


def test_config_validation_matches_reference():
    spec = BlockSpec(12, 4, 4)
    for kw in (dict(d_l=0), dict(d_l=2, d_u=1), dict(t=0), dict(n=0), dict(T=0), dict(d_t=-1),
               dict(sync_mode="sometimes"), dict(grid_mode="bogus")):
        with pytest.raises(ValueError):
            PipelineConfig(spec=spec, **kw)
    cfg = PipelineConfig(spec=spec, n=2, t=3, T=2)
    assert cfg.threads == 6 and cfg.h == 12


def test_may_advance_eq3():
    # sp/pipeline.py:133-141 — predecessor >= d_l ahead, successor <= d_u behind
    dist = EffectiveDistances(d_l=(1, 1, 1), d_u=(2, 2, 2))
    assert may_advance(_counters([5, 4, 3]), 1, dist)
    assert not may_advance(_counters([4, 4, 3]), 1, dist)
    assert not may_advance(_counters([9, 7, 4]), 1, dist)
    assert may_advance(_counters([0, 0, 0]), 0, dist)
    with pytest.raises(IndexError):
        may_advance(_counters([1]), 3, dist)


def test_team_delay_distances():
    cfg = PipelineConfig(spec=BlockSpec(4, 4, 4), n=2, t=2, d_l=1, d_u=3, d_t=2)
    d = EffectiveDistances.from_config(cfg)
    assert d.d_l == (1, 1, 3, 1)
    assert d.d_u == (3, 5, 3, 3)


def test_estimate_max_distance():
    assert estimate_max_distance(8e6, 4, BlockSpec(120, 20, 20)) == 5
    assert estimate_max_distance(24e6, 8, BlockSpec(120, 20, 20)) == 7
    assert estimate_max_distance(1000, 4, BlockSpec(120, 20, 20)) == 0
    with pytest.raises(ValueError):
        estimate_max_distance(8e6, 0, BlockSpec(10, 10, 10))


def test_blockspec_and_plans():
    g = _grid(7, 7, 7)
    with pytest.raises(ValueError):
        BlockSpec(8, 1, 1).validate(g)
    plan = decompose_blocks(g, BlockSpec(7, 3, 3), 1)
    assert plan.total_blocks == 9
    assert plan.blocks[-1] == ((0, 6, 6), (7, 1, 1))
    bwd = decompose_blocks(g, BlockSpec(7, 3, 3), -1)
    assert bwd.blocks == list(reversed(plan.blocks))
    assert next_block(plan, 9) is None
    with pytest.raises(ValueError):
        next_block(plan, -1)
    with pytest.raises(ValueError):
        decompose_blocks(g, BlockSpec(7, 3, 3), 2)


@settings(max_examples=60, deadline=None)
@given(nx=st.integers(1, 40), ny=st.integers(1, 40), nz=st.integers(1, 40),
       bx=st.integers(1, 40), by=st.integers(1, 40), bz=st.integers(1, 40))
def test_block_plan_tiles_interior(nx, ny, nz, bx, by, bz):
    spec = BlockSpec(min(bx, nx), min(by, ny), min(bz, nz))
    plan = decompose_blocks(_grid(nx, ny, nz), spec, 1)
    assert sum(sx * sy * sz for _, (sx, sy, sz) in plan.blocks) == nx * ny * nz


@pytest.mark.parametrize("h,mf,exp", [(1, 4, [1]), (4, 4, [4]), (5, 4, [3, 2]), (8, 4, [4, 4]),
                                      (9, 4, [3, 3, 3]), (16, 4, [4, 4, 4, 4]), (6, 2, [2, 2, 2])])
def test_split_levels(h, mf, exp):
    assert split_levels(h, mf) == exp
    assert sum(split_levels(h, mf)) == h


def test_fusable_rule():
    """Fusing levels is exact iff x/y live ranges are full and z ranges shrink
    by >= 1 per level (or touch the ring) — the distributed live bounds of
    sp/halo.py:278-289 qualify, arbitrary windows do not."""
    eng = PipelineEngine.__new__(PipelineEngine)
    eng.dims = (10, 10, 20)
    eng.physical_sides = {ax: (True, True) for ax in range(3)}
    full = {u: [(0, 10), (0, 10), (0, 20)] for u in range(1, 5)}
    assert eng._fusable(full, 4)
    shrink = {u: [(0, 10), (0, 10), (u, 20 - u)] for u in range(1, 5)}
    assert eng._fusable(shrink, 4)
    flat_inner = {u: [(0, 10), (0, 10), (2, 18)] for u in range(1, 5)}
    assert not eng._fusable(flat_inner, 4)
    xwin = {u: [(1, 9), (0, 10), (0, 20)] for u in range(1, 5)}
    assert not eng._fusable(xwin, 4)
    # x/y sides owned by a neighbour may shrink (ghost cells); physical may not
    xshrink = {u: [(u, 10 - u), (0, 10 - u), (0, 20)] for u in range(1, 5)}
    assert not eng._fusable(xshrink, 4)
    eng.physical_sides = {0: (False, False), 1: (True, False), 2: (True, True)}
    assert eng._fusable(xshrink, 4)
    assert not eng._fusable({u: [(1, 9), (0, 10 - u), (0, 20)] for u in range(1, 5)}, 4)
