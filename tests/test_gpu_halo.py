"""GPU: the z-slab distributed data path on one device.  Every rank's
RankRuntime (GPU grids, fused K2 passes with shrinking live ranges) runs in
this process; the halo messages of the plan are delivered by device copies
instead of NCCL (the transport itself is covered by the gloo tests).  The
assembled result must equal the undecomposed oracle bit for bit."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

sp = pytest.importorskip("paper_1006_3148_b200")
from paper_1006_3148_b200 import halo  # noqa: E402


def _box(g, box):
    (xl, xh), (yl, yh), (zl, zh) = box
    o = g.offset
    return g.data[zl + o:zh + o, yl + o:yh + o, xl + o:xh + o]


def _emulate(dc):
    rts = halo.run_distributed_inprocess(dc)
    for rt in rts:
        assert rt.timings["compute_s"] > 0 and rt.timings["mlups"] > 0
    return halo.assemble_global(rts)


@pytest.mark.parametrize("topo,gd,h,mode,cycles,ring", [
    ((1, 1, 2), (40, 40, 40), 2, "two_grid", 2, None),
    ((1, 1, 2), (40, 40, 40), 4, "two_grid", 3, 1.0),
    ((1, 1, 4), (24, 24, 64), 4, "two_grid", 3, None),
    ((1, 1, 3), (18, 20, 36), 2, "two_grid", 3, None),
    ((1, 1, 2), (130, 70, 40), 4, "two_grid", 2, 0.5),
    ((1, 1, 2), (40, 40, 40), 4, "compressed", 2, None),
    ((2, 2, 1), (40, 40, 40), 2, "two_grid", 2, None),
    ((2, 1, 1), (48, 20, 20), 4, "two_grid", 2, 1.0),
    ((2, 2, 2), (24, 24, 24), 2, "two_grid", 3, None),
    ((2, 1, 2), (32, 16, 32), 2, "compressed", 2, None),
])
def test_zslab_gpu_equals_oracle(topo, gd, h, mode, cycles, ring, golden):
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(8, 8, 8), t=h, grid_mode=mode)
    dc = halo.DistConfig(topo=halo.RankTopology(*topo), cfg=cfg, cycles=cycles, global_dims=gd,
                         mode="strong", seed=42, ring=ring)
    g = _emulate(dc)
    d0 = oracle.make_storage(*gd, init="random", seed=42, ring=ring)
    exp = oracle.interior(oracle.sweeps(d0, gd, h * cycles), *gd)
    assert_bitwise(g.interior_numpy(), exp)


def test_golden_distributed_digests(golden):
    for name, c in golden["distributed"].items():
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(c["global_dims"][0], 10, 10), t=c["h"],
                                grid_mode=c["mode"])
        dc = halo.DistConfig(topo=halo.RankTopology(*c["topo"]), cfg=cfg, cycles=c["cycles"],
                             global_dims=tuple(c["global_dims"]), mode="strong", seed=c["seed"])
        assert _emulate(dc).checksum() == c["digest"], name


@pytest.mark.slow
def test_c4_weak_scaling_p2_window_oracle():
    """BASELINE configs[3] at P=2 (1024^2 x 2048, ring 1.0, t=4, 40 sweeps),
    every rank on this GPU; boxes straddling the rank boundary and touching
    the physical faces checked with the light-cone window oracle."""
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(64, 32, 32), t=4)
    dc = halo.DistConfig(topo=halo.RankTopology(1, 1, 2), cfg=cfg, cycles=10,
                         per_rank_dims=(1024, 1024, 1024), mode="weak", seed=42, ring=1.0)
    g = _emulate(dc)
    gd = dc.resolved_global()
    for box in (((0, 48), (480, 528), (1016, 1032)), ((990, 1024), (0, 40), (2040, 2048)),
                ((500, 540), (1000, 1024), (0, 12))):
        exp = oracle.window_oracle(gd, 42, box, 40, ring=1.0)
        (xl, xh), (yl, yh), (zl, zh) = box
        assert_bitwise(g.interior_view()[zl:zh, yl:yh, xl:xh].cpu().numpy(), exp)


@pytest.mark.parametrize("topo", [(2, 1, 1), (2, 2, 1), (2, 2, 2), (1, 1, 2)])
def test_general_topologies_take_the_fused_path(topo):
    """Neighbour-owned x/y sides shrink like z: every rank's pass runs the
    fused kernels, not the per-level windows."""
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(8, 8, 8), t=4)
    subs = halo.decompose_domain((32, 32, 32), halo.RankTopology(*topo), halo.HaloSpec(4))
    for s in subs:
        rt = halo.RankRuntime(s, cfg, None)
        assert rt.engine._fusable(rt.engine._lives(4), 4)
        assert rt.engine.run_pass(1).kernel_launches == 1
