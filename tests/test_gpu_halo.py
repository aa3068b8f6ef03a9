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


def _global_box(rts, box):
    """Values of a global box (half-open x, y, z) gathered from the ranks'
    owned blocks, as a (z, y, x) numpy array (no global assembly: the C4 P=8
    and C5 grids do not fit twice in HBM)."""
    (xl, xh), (yl, yh), (zl, zh) = box
    out = np.full((zh - zl, yh - yl, xh - xl), np.nan)
    for rt in rts:
        c = rt.sub.topo.coords(rt.sub.rank)
        o = [c[ax] * rt.sub.owned[ax] for ax in range(3)]
        lo = [max(b[0], o[ax]) for ax, b in enumerate(box)]
        hi = [min(b[1], o[ax] + rt.sub.owned[ax]) for ax, b in enumerate(box)]
        if any(l >= h for l, h in zip(lo, hi)):
            continue
        v = rt.owned_view()[lo[2] - o[2]:hi[2] - o[2], lo[1] - o[1]:hi[1] - o[1], lo[0] - o[0]:hi[0] - o[0]]
        out[lo[2] - zl:hi[2] - zl, lo[1] - yl:hi[1] - yl, lo[0] - xl:hi[0] - xl] = v.cpu().numpy()
    assert not np.isnan(out).any()
    return out


def _free():
    import gc
    gc.collect()
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_c4_p8_window_anchor():
    """BASELINE configs[3] at P=8 (1024 x 1024 x 8192 global, ring 1.0, t=4,
    40 sweeps = 10 exchange cycles), all eight ranks on this GPU (~140 GB of
    HBM): the box x[0,64) y[480,544) z[4090,4102), which straddles the rank
    3 / rank 4 boundary and touches the x = 0 face, equals the light-cone
    window oracle and the SURVEY.md Appendix A digest."""
    _free()
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(64, 32, 32), t=4)
    dc = halo.DistConfig(topo=halo.RankTopology(1, 1, 8), cfg=cfg, cycles=10,
                         per_rank_dims=(1024, 1024, 1024), mode="weak", seed=42, ring=1.0)
    rts = halo.run_distributed_inprocess(dc)
    box = ((0, 64), (480, 544), (4090, 4102))
    got = _global_box(rts, box)
    del rts
    _free()
    exp = oracle.window_oracle(dc.resolved_global(), 42, box, 40, ring=1.0)
    assert_bitwise(got, exp)
    assert oracle.digest(got) == "a41a391e1e10d10e75712d66f0877ab928897586835a4527693d705d7eb1e7fc"


@pytest.mark.slow
def test_c5_strong_window_anchors():
    """BASELINE configs[4] (2048^3 global, ring 0.0, 32 sweeps) as four z-slabs
    with ghost depth / exchange interval t=8 (4 cycles of two fused 4-level
    launches each), all ranks on this GPU (~143 GB): the SURVEY.md Appendix A
    window anchors, each also recomputed with the window oracle."""
    _free()
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(64, 32, 32), t=8)
    dc = halo.DistConfig(topo=halo.RankTopology(1, 1, 4), cfg=cfg, cycles=4,
                         global_dims=(2048, 2048, 2048), mode="strong", seed=42)
    rts = halo.run_distributed_inprocess(dc)
    boxes = {((1000, 1064), (1000, 1064), (1000, 1048)):
             "9d1b69d342fb981b618cdb6041268d07e7e45c3a732479fe394d1924a3788586",
             ((0, 48), (0, 48), (0, 48)):
             "5974e85c6c4706831f80dd497bc1af0abe95df36bff1aed9468d7fb01d42db69"}
    got = {box: _global_box(rts, box) for box in boxes}
    del rts
    _free()
    for box, dg in boxes.items():
        exp = oracle.window_oracle((2048, 2048, 2048), 42, box, 32)
        assert_bitwise(got[box], exp)
        assert oracle.digest(got[box]) == dg, box


@pytest.mark.parametrize("topo_dims,h", [
    ((2, 1, 1), 2), ((2, 2, 1), 2), ((2, 2, 2), 2),
    ((3, 2, 1), 1), ((2, 2, 2), 4), ((3, 3, 3), 4), ((3, 3, 3), 2),
])
def test_rank_id_fill_ownership_oracle(topo_dims, h):
    """pkg/tests/test_halo.py:144-180 on the device: after one exchange
    (sp_pack_boxes / sp_unpack_boxes per axis phase, x -> y -> z forwarding)
    every local cell, halos included, holds its owner's rank id — edge and
    corner halos arrive by forwarding, with no diagonal messages."""
    topo = halo.RankTopology(*topo_dims)
    n_per = 12 if max(topo_dims) < 3 else 18
    gd = tuple(n_per * p for p in topo_dims)
    subs = halo.decompose_domain(gd, topo, halo.HaloSpec(h))
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(4, 4, 4), t=h)
    rts = []
    for sub in subs:
        rt = halo.RankRuntime(sub, cfg, None, init="constant", value=0.0)
        ob = sub.owned_box()
        rt.sub.grid.interior_view()[ob[2][0]:ob[2][1], ob[1][0]:ob[1][1], ob[0][0]:ob[0][1]] = float(sub.rank)
        rts.append(rt)
    launches = sp._lib.launch_count()
    halo.exchange_inprocess(rts)
    # one pack and one unpack launch per rank and phase with messages
    phases = sum(len({m.axis for m in rt.plan.messages}) for rt in rts)
    assert sp._lib.launch_count() - launches == 2 * phases
    for rt in rts:
        sub = rt.sub
        mx, my, mz = sub.local_dims
        gz = (sub.global_origin[2] + np.arange(mz))[:, None, None] // sub.owned[2]
        gy = (sub.global_origin[1] + np.arange(my))[None, :, None] // sub.owned[1]
        gx = (sub.global_origin[0] + np.arange(mx))[None, None, :] // sub.owned[0]
        owner = gx + topo.px * (gy + topo.py * gz)
        assert_bitwise(rt.sub.grid.interior_numpy(), owner.astype(np.float64))


@pytest.mark.parametrize("topo_dims", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
@pytest.mark.parametrize("h,mode", [(2, "two_grid"), (2, "compressed"), (4, "two_grid"), (4, "compressed")])
def test_acceptance_2_distributed_oracle(topo_dims, h, mode, oracle_cache):
    """Acceptance criterion #2 (pkg/tests/test_acceptance.py:94-115): the
    assembled distributed result equals 2h reference sweeps for every
    required topology and halo width, 60^3, seed 42, two cycles (n=1, t=2,
    T=1|2, block 15x10x10)."""
    t, T = (2, 1) if h == 2 else (2, 2)
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(15, 10, 10), n=1, t=t, T=T, d_l=1, d_u=3, grid_mode=mode)
    assert cfg.h == h
    dc = halo.DistConfig(topo=halo.RankTopology(*topo_dims), cfg=cfg, cycles=2,
                         global_dims=(60, 60, 60), mode="strong", seed=42)
    assert_bitwise(_emulate(dc).interior_numpy(), oracle_cache.after_sweeps(60, 42, 2 * h))
