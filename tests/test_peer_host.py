"""Host logic of the fused peer-memory halo delivery (no GPU): where a rank's
send planes land in each z neighbour's grid, the counter protocol's pass
phases, and the transport's scope checks."""

import pytest

from paper_1006_3148_b200 import halo
from paper_1006_3148_b200.pipeline import PipelineConfig, _drive
from paper_1006_3148_b200.grid import BlockSpec


@pytest.mark.parametrize("p,nz,h", [(2, 40, 4), (3, 48, 3), (4, 64, 4), (3, 72, 8), (2, 20, 1)])
def test_mirror_zshift_matches_the_plan(p, nz, h):
    subs = halo.decompose_domain((16, 16, nz), halo.RankTopology(1, 1, p), halo.HaloSpec(h))
    for s in subs:
        plan = halo.build_halo_plan(s)
        for m in plan.messages:
            nb = subs[m.neighbor]
            zs = halo.mirror_zshift(s, nb, m.side)
            (a, b) = m.send_box[2]
            theirs = [q for q in halo.build_halo_plan(nb).messages if q.side == 1 - m.side][0]
            assert (a + zs, b + zs) == theirs.recv_box[2]
            # the planes are the neighbour's ghost layers, in global z the sender's owned planes
            ga = s.global_origin[2] + a
            gb = nb.global_origin[2] + a + zs
            assert ga == gb
            assert b - a == h


def test_mirror_zshift_rejects_non_neighbours():
    subs = halo.decompose_domain((16, 16, 48), halo.RankTopology(1, 1, 3), halo.HaloSpec(2))
    with pytest.raises(halo.TransportError):
        halo.mirror_zshift(subs[0], subs[2], 1)
    with pytest.raises(halo.TransportError):
        halo.mirror_zshift(subs[0], subs[1], 0)  # rank 0 has no low neighbour


def test_p2p_scope_checks():
    cfg = PipelineConfig(spec=BlockSpec(8, 8, 8), t=2)
    subs = halo.decompose_domain((16, 16, 16), halo.RankTopology(2, 1, 1), halo.HaloSpec(2))
    with pytest.raises(ValueError):
        halo.RankRuntime(subs[0], cfg, transport="p2p")
    zs = halo.decompose_domain((16, 16, 16), halo.RankTopology(1, 1, 2), halo.HaloSpec(2))
    comp = PipelineConfig(spec=BlockSpec(8, 8, 8), t=2, grid_mode="compressed")
    with pytest.raises(ValueError):
        halo.RankRuntime(zs[0], comp, transport="p2p")
    with pytest.raises(ValueError):
        halo.RankRuntime(zs[0], cfg, transport="tcp")


class _Rec:
    """Stands in for a RankRuntime: records the counter protocol."""

    def __init__(self, has_lo, has_hi, h):
        self.log = []

        class S:
            pass
        self.sub = S()
        self.sub.has_nb = ((False, False), (False, False), (has_lo, has_hi))
        self.sub.h = h

    def _wait(self, v):
        self.log.append(("wait", v))

    def _signal(self, v):
        self.log.append(("signal", v))


def test_counter_protocol_values():
    """Pass k: wait 2k, signal 2k+1, (interior), wait 2k+1, stores, signal
    2k+2 — each wait only needs the neighbour's earlier signals."""
    r = _Rec(True, True, 4)
    for k in range(3):
        b = halo.FusedZHalo(r, k)
        assert (b.blo, b.bhi) == (4, 4)
        b.begin()
        b.chunks_done()
        b.before_stores()
        b.end()
    assert r.log == [(op, v) for k in range(3) for op, v in
                     (("wait", 2 * k), ("signal", 2 * k + 1), ("wait", 2 * k + 1), ("signal", 2 * k + 2))]
    # a rank's n-th wait never exceeds what the neighbour signalled before its own n-th wait
    sig, waits = 0, []
    for op, v in r.log:
        if op == "wait":
            assert v <= sig
        else:
            sig = v
    assert halo.FusedZHalo(_Rec(False, True, 3), 0).blo == 0


def test_drive_returns_generator_value():
    def g():
        yield
        yield
        return 7
    assert _drive(g()) == 7
