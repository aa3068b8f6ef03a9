"""CPU, world_size 2-3 over gloo: the distributed driver (decomposition, live
bounds, x->y->z halo exchange with torch.distributed P2P, direction
alternation, gather) against the undecomposed oracle (mirrors
pkg/tests/test_halo.py:144-263 and acceptance #2).  The per-rank compute is a
CPU stand-in built from the oracle (the GPU engine is covered by the -m gpu
tests); everything else is the product code path."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

from paper_1006_3148_b200 import halo
from paper_1006_3148_b200.pipeline import PipelineConfig
from paper_1006_3148_b200.grid import BlockSpec


class _HostGrid:
    """Storage + frame of one rank's grid on the CPU (test stand-in)."""

    def __init__(self, data, pad, alignment=0):
        self.data = data
        self.pad = pad
        self.alignment = alignment

    @property
    def origin(self):
        return self.pad + 1

    @property
    def offset(self):
        return self.origin - self.alignment


class OracleEngine:
    """CPU stand-in with PipelineEngine's interface and the reference's level
    semantics (sp/pipeline.py:301-335): per level, the live window of level u
    is updated from level u-1 (two grids alternate, or one grid shifted)."""

    def __init__(self, cfg, grids, live_bounds, physical_sides):
        self.cfg = cfg
        self.grids = list(grids) if isinstance(grids, (list, tuple)) else [grids]
        self.live = live_bounds
        self.phys = physical_sides
        self.levels_done = 0
        self.faces = None

    def current_grid(self):
        if self.cfg.grid_mode == "compressed":
            return self.grids[0]
        return self.grids[self.levels_done % 2]

    def run_pass(self, direction, boundary=None):
        h = self.cfg.h
        if self.cfg.grid_mode == "two_grid":
            for u in range(1, h + 1):
                lvl = self.levels_done + u
                src, dst = self.grids[(lvl - 1) % 2], self.grids[lvl % 2]
                win = tuple(self.live(ax, u) for ax in range(3))
                (xl, xh), (yl, yh), (zl, zh) = win
                if u == h and boundary is not None and zh - zl > boundary[0] + boundary[1]:
                    # PipelineEngine's boundary-first protocol: the planes the
                    # exchange sends are final, the exchange is posted, then the
                    # interior planes are computed while it is in flight
                    blo, bhi, post = boundary
                    sd, dd = src.data.numpy(), dst.data.numpy()
                    if blo:
                        oracle.apply_window(sd, dd, ((xl, xh), (yl, yh), (zl, zl + blo)), src.offset, src.offset)
                    if bhi:
                        oracle.apply_window(sd, dd, ((xl, xh), (yl, yh), (zh - bhi, zh)), src.offset, src.offset)
                    post(dst.data, dst.offset)
                    oracle.apply_window(sd, dd, ((xl, xh), (yl, yh), (zl + blo, zh - bhi)), src.offset,
                                        src.offset)
                    self.levels_done += h
                    self.posted_inside = True
                    return
                oracle.apply_window(src.data.numpy(), dst.data.numpy(), win, src.offset, src.offset)
        else:
            g = self.grids[0]
            d = g.data.numpy()
            a0 = g.alignment
            s = 1 if direction == 1 else -1
            dims = self._dims
            for u in range(1, h + 1):
                so = g.origin - (a0 + s * (u - 1))
                do = g.origin - (a0 + s * u)
                win = tuple(self.live(ax, u) for ax in range(3))
                if u == 1:
                    self._faces_at(d, so, dims, full=True)
                oracle.apply_window(d, d, win, so, do)
                self._faces_at(d, do, dims, full=False, win=win)
            g.alignment = a0 + s * h
        self.levels_done += h
        if boundary is not None:
            cur = self.current_grid()
            boundary[2](cur.data, cur.offset)

    # Dirichlet faces at a frame, physical sides only (sp/pipeline.py:427-447)
    def _faces_at(self, d, off, dims, full, win=None):
        nx, ny, nz = dims
        f = self.faces
        spans = [(0, nx), (0, ny), (0, nz)] if full else [win[0], win[1], win[2]]
        for ax in range(3):
            for side in (0, 1):
                if not self.phys[ax][side]:
                    continue
                pos = off + (-1 if side == 0 else dims[ax])
                (xl, xh), (yl, yh), (zl, zh) = spans
                if ax == 0:
                    d[zl + off:zh + off, yl + off:yh + off, pos] = f[(0, side)][zl:zh, yl:yh]
                elif ax == 1:
                    d[zl + off:zh + off, pos, xl + off:xh + off] = f[(1, side)][zl:zh, xl:xh]
                else:
                    d[pos, yl + off:yh + off, xl + off:xh + off] = f[(2, side)][yl:yh, xl:xh]


def _make_rank(dc, rank):
    gd = dc.resolved_global()
    subs = halo.decompose_domain(gd, dc.topo, halo.HaloSpec(dc.cfg.h))
    sub = subs[rank]
    mx, my, mz = sub.local_dims
    pad = dc.cfg.h if dc.cfg.grid_mode == "compressed" else 0
    d = np.zeros(oracle.storage_shape(mx, my, mz, pad))
    o = pad + 1
    d[o:o + mz, o:o + my, o:o + mx] = oracle.global_field_box(
        gd, dc.seed, tuple((sub.global_origin[a], sub.global_origin[a] + (mx, my, mz)[a]) for a in range(3)))
    faces = {(0, 0): d[o:o + mz, o:o + my, o - 1].copy(), (0, 1): d[o:o + mz, o:o + my, o + mx].copy(),
             (1, 0): d[o:o + mz, o - 1, o:o + mx].copy(), (1, 1): d[o:o + mz, o + my, o:o + mx].copy(),
             (2, 0): d[o - 1, o:o + my, o:o + mx].copy(), (2, 1): d[o + mz, o:o + my, o:o + mx].copy()}
    g = _HostGrid(torch.from_numpy(d), pad)
    grids = g if dc.cfg.grid_mode == "compressed" else (g, _HostGrid(torch.from_numpy(d.copy()), pad))

    def factory(cfg, grids, live_bounds, physical_sides):
        e = OracleEngine(cfg, grids, live_bounds, physical_sides)
        e._dims = (mx, my, mz)
        e.faces = faces
        return e

    return halo.RankRuntime(sub, dc.cfg, None, engine_factory=factory, grids=grids)


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        topo = halo.RankTopology(*case["topo"])
        cfg = PipelineConfig(spec=BlockSpec(*case["spec"]), t=case["h"], grid_mode=case["mode"])
        dc = halo.DistConfig(topo=topo, cfg=cfg, cycles=case["cycles"],
                             global_dims=tuple(case["global_dims"]), mode="strong", seed=case["seed"])
        rt = _make_rank(dc, rank)
        rt.check_config_hash(halo.config_digest(cfg, dc.resolved_global(), dc.cycles, dc.seed))
        for c in range(dc.cycles):
            rt.cycle(c)
        full = halo.gather_owned(rt)
        if case["topo"][:2] == (1, 1) and case["mode"] == "two_grid":
            # z-slab two-grid cycles post the exchange from inside the pass
            assert rt.timings.get("overlapped_cycles") == dc.cycles
        if rank == 0:
            np.save(out, full)
            with open(out + ".json", "w") as f:
                json.dump(rt.timings, f)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    dict(topo=(1, 1, 2), global_dims=(20, 18, 24), h=2, mode="two_grid", cycles=3, seed=42, spec=(20, 6, 6)),
    dict(topo=(1, 1, 2), global_dims=(16, 16, 32), h=4, mode="two_grid", cycles=2, seed=7, spec=(16, 8, 8)),
    dict(topo=(1, 1, 3), global_dims=(12, 10, 36), h=2, mode="two_grid", cycles=3, seed=5, spec=(12, 5, 6)),
    dict(topo=(1, 1, 2), global_dims=(20, 20, 24), h=2, mode="compressed", cycles=2, seed=42, spec=(20, 10, 6)),
    dict(topo=(2, 1, 1), global_dims=(24, 12, 12), h=2, mode="two_grid", cycles=2, seed=3, spec=(12, 6, 6)),
    dict(topo=(1, 2, 1), global_dims=(12, 24, 12), h=3, mode="two_grid", cycles=2, seed=9, spec=(12, 6, 6)),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['topo']}-h{c['h']}-{c['mode']}")
def test_distributed_equals_undecomposed_oracle(case, tmp_path):
    world = int(np.prod(case["topo"]))
    out = str(tmp_path / "full.npy")
    mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    gd = tuple(case["global_dims"])
    d0 = oracle.make_storage(*gd, init="random", seed=case["seed"])
    exp = oracle.interior(oracle.sweeps(d0, gd, case["h"] * case["cycles"]), *gd)
    assert np.array_equal(got, exp)
    t = json.load(open(out + ".json"))
    for key in ("compute_s", "pack_s", "transfer_s", "unpack_s", "messages", "bytes"):
        assert key in t


def _owner_worker(rank, world, port, topo_dims, h, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        topo = halo.RankTopology(*topo_dims)
        n_per = 12 if max(topo_dims) < 3 else 18
        gd = tuple(n_per * p for p in topo_dims)
        sub = halo.decompose_domain(gd, topo, halo.HaloSpec(h))[rank]
        mx, my, mz = sub.local_dims
        d = torch.zeros(oracle.storage_shape(mx, my, mz), dtype=torch.float64)
        ob = sub.owned_box()
        d[1 + ob[2][0]:1 + ob[2][1], 1 + ob[1][0]:1 + ob[1][1], 1 + ob[0][0]:1 + ob[0][1]] = float(rank)
        halo.exchange_multilayer_halos(sub, halo.build_halo_plan(sub), data=d, offset=1)
        gz = (sub.global_origin[2] + np.arange(mz))[:, None, None] // sub.owned[2]
        gy = (sub.global_origin[1] + np.arange(my))[None, :, None] // sub.owned[1]
        gx = (sub.global_origin[0] + np.arange(mx))[None, None, :] // sub.owned[0]
        owner = (gx + topo.px * (gy + topo.py * gz)).astype(np.float64)
        ok = np.array_equal(d.numpy()[1:1 + mz, 1:1 + my, 1:1 + mx], owner)
        with open(f"{out}.{rank}", "w") as f:
            f.write("ok" if ok else "bad")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("topo_dims,h", [((2, 2, 2), 4), ((3, 2, 1), 1), ((2, 2, 1), 2)])
def test_rank_id_fill_ownership_oracle_gloo(topo_dims, h, tmp_path):
    """pkg/tests/test_halo.py:144-180 across processes: one exchange over
    gloo and every halo cell (edges and corners by forwarding) holds its
    owner's rank id."""
    world = int(np.prod(topo_dims))
    out = str(tmp_path / "owner")
    mp.start_processes(_owner_worker, args=(world, _free_port(), topo_dims, h, out), nprocs=world,
                       join=True, start_method="spawn")
    assert all(open(f"{out}.{r}").read() == "ok" for r in range(world))


def test_halo_plan_geometry_zslab():
    subs = halo.decompose_domain((64, 64, 96), halo.RankTopology(1, 1, 3), halo.HaloSpec(4))
    mid = subs[1]
    assert mid.local_dims == (64, 64, 32 + 8)
    plan = halo.build_halo_plan(mid)
    assert [(m.axis, m.side) for m in plan.messages] == [(2, 0), (2, 1)]
    lo, hi = plan.messages
    assert lo.send_box[2] == (4, 8) and lo.recv_box[2] == (0, 4)
    assert hi.send_box[2] == (32, 36) and hi.recv_box[2] == (36, 40)
    assert lo.nbytes == 64 * 64 * 4 * 8
    live = halo.live_bounds_for(mid, PipelineConfig(spec=BlockSpec(8, 8, 8), t=4))
    assert [live(2, u) for u in (1, 2, 3, 4)] == [(1, 39), (2, 38), (3, 37), (4, 36)]
    assert live(0, 3) == (0, 64)


def test_decomposition_errors_and_topology():
    with pytest.raises(ValueError):
        halo.decompose_domain((10, 10, 10), halo.RankTopology(1, 1, 3), halo.HaloSpec(1))
    with pytest.raises(ValueError):
        halo.decompose_domain((8, 8, 8), halo.RankTopology(1, 1, 2), halo.HaloSpec(4))
    with pytest.raises(ValueError):
        halo.RankTopology(0, 1, 1)
    topo = halo.RankTopology(3, 2, 2)
    for r in range(topo.ranks):
        assert topo.rank_of(*topo.coords(r)) == r
    assert topo.neighbor(0, 2, 0) is None and topo.neighbor(0, 2, 1) == 6
