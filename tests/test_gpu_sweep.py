"""GPU parity: K0 seeded fill and K1 plain sweep through the C ABI, bit-exact
against the reference's own pins and the reference-generated golden digests
(mirrors pkg/tests/test_kernel.py and test_grid.py)."""

import numpy as np
import pytest
import torch

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

sp = pytest.importorskip("paper_1006_3148_b200")


def _sweeps(g0, count):
    a, b = g0.copy(), g0.copy()
    for _ in range(count):
        sp.reference_sweep(a, b)
        a, b = b, a
    return a


def _case_grid(c):
    return sp.create_grid(c["nx"], c["ny"], c["nz"], pad=c["pad"], init=c["init"],
                          value=c["value"], seed=c["seed"], ring=c["ring"], lo=c["lo"], hi=c["hi"])


def test_field_pins(golden):
    g = sp.create_grid(60, 60, 60, init="random", seed=42)
    assert g.checksum() == golden["pins"]["FIELD_60_SEED42"]
    assert sp.seeded_field_checksum(600, 600, 600, 42) == golden["pins"]["FIELD_600_SEED42"]


def test_ref_60_8_pin(golden):
    g = sp.create_grid(60, 60, 60, init="random", seed=42)
    assert _sweeps(g, 8).checksum() == golden["pins"]["REF_60_SEED42_8SWEEPS"]


@pytest.mark.parametrize("loader", ["tma", "cpasync"])
def test_golden_sweep_cases_every_sweep(golden, loader):
    L = sp._lib.load()
    L.sp_set_tuning(1, 1 if loader == "cpasync" else 0)
    try:
        for name, c in golden["sweeps"].items():
            g0 = _case_grid(c)
            assert g0.checksum() == c["init_digest"], name
            a, b = g0.copy(), g0.copy()
            for s in range(1, c["sweeps"] + 1):
                sp.reference_sweep(a, b)
                a, b = b, a
                assert a.checksum() == c["digests"][str(s)], (name, s)
    finally:
        L.sp_set_tuning(1, 0)


def test_ring_copied_including_edges_and_corners():
    import oracle
    n = (13, 9, 6)
    d = oracle.make_storage(*n, init="random", seed=3)
    d2 = d.copy()
    # distinct ring values everywhere in a, garbage in b
    rng = np.random.default_rng(0)
    shell = np.ones_like(d, dtype=bool)
    shell[1:-1, 1:-1, 1:-1] = False
    d[shell] = rng.random(shell.sum())
    a = sp.Grid3.from_numpy(*n, 0, d)
    b = sp.Grid3.from_numpy(*n, 0, np.full_like(d2, 7.0))
    sp.reference_sweep(a, b)
    out = b.to_numpy()
    assert_bitwise(out[shell], d[shell])
    ref = np.zeros_like(d)
    oracle.reference_sweep(d, ref, *n, 1)
    assert_bitwise(out, ref)


def test_cell_known_answers():
    g = sp.create_grid(3, 3, 3, init="constant", value=3.0)
    assert sp.stencil_update_cell(g, 1, 1, 1) == 3.0
    g = sp.create_grid(3, 3, 3, init="constant", value=0.0)
    g.data[g.index(0, 1, 1)] = 1.0
    assert sp.stencil_update_cell(g, 1, 1, 1) == 1.0 / 6.0
    g = sp.create_grid(3, 3, 3, init="constant", value=0.0)
    vals = {(0, 1, 1): 1.0, (2, 1, 1): 2.0, (1, 0, 1): 3.0,
            (1, 2, 1): 4.0, (1, 1, 0): 5.0, (1, 1, 2): 6.0}
    for cell, v in vals.items():
        g.data[g.index(*cell)] = v
    assert sp.stencil_update_cell(g, 1, 1, 1) == 3.5
    with pytest.raises(IndexError):
        sp.stencil_update_cell(g, 3, 0, 0)


def test_constant_fixed_point_and_impulse():
    g = sp.create_grid(6, 6, 6, init="constant", value=1.0)
    assert torch.all(_sweeps(g, 3).interior_view() == 1.0)
    g = sp.create_grid(4, 4, 4, init="impulse")
    b = g.copy()
    sp.reference_sweep(g, b)
    iv = b.interior_numpy()
    assert iv[2, 2, 2] == 0.0
    assert len(np.argwhere(iv == 1.0 / 6.0)) == 6
    assert iv.sum() == 6 * (1.0 / 6.0)


def test_errors_match_reference():
    a = sp.create_grid(4, 4, 4)
    b = sp.create_grid(4, 4, 5)
    with pytest.raises(ValueError):
        sp.reference_sweep(a, b)
    c = sp.create_grid(4, 4, 4, pad=1)
    c.alignment = 1
    with pytest.raises(ValueError):
        sp.reference_sweep(a, c)
    with pytest.raises(ValueError):
        sp.create_grid(0, 4, 4)
    with pytest.raises(ValueError):
        sp.create_grid(4, 4, 4, pad=-1)
    with pytest.raises(ValueError):
        sp.create_grid(4, 4, 4, init="bogus")


def test_maximum_principle_and_linearity():
    g = sp.create_grid(8, 8, 8, init="random", seed=5)
    lo, hi = g.data.min().item(), g.data.max().item()
    iv = _sweeps(g, 4).interior_view()
    assert iv.min().item() >= lo and iv.max().item() <= hi
    for alpha in (0.5, 2.0, 8.0):
        g = sp.create_grid(8, 8, 8, init="random", seed=9)
        s = g.copy()
        s.data *= alpha
        s.capture_boundary_faces()
        assert_bitwise(_sweeps(s, 2).interior_numpy(), _sweeps(g, 2).interior_numpy() * alpha)


def test_blocked_sweep_equals_reference():
    """spatial_blocked_sweep (sp/kernel.py:114-125) against the oracle's
    reference sweep, storage including the copied ring (tests/test_kernel.py:104-126)."""
    import oracle
    for n, spec in ((6, (6, 6, 6)), (60, (60, 20, 20)), (7, (7, 3, 3)), (33, (5, 7, 11))):
        g = sp.create_grid(n, n, n, init="random", seed=4, ring=0.75)
        b2 = sp.create_grid(n, n, n, init="constant", value=-2.0)
        sp.spatial_blocked_sweep(g, b2, sp.BlockSpec(*spec))
        d0 = oracle.make_storage(n, n, n, init="random", seed=4, ring=0.75)
        d1 = np.full_like(d0, -2.0)
        oracle.reference_sweep(d0, d1, n, n, n, 1)
        assert_bitwise(b2.to_numpy(), d1)
    with pytest.raises(ValueError):
        sp.spatial_blocked_sweep(g, b2, sp.BlockSpec(0, 1, 1))


def test_apply_window_seam_matches_oracle():
    import oracle
    n = (11, 10, 9)
    d = oracle.make_storage(*n, pad=2, init="random", seed=21, ring=0.25)
    g = sp.Grid3.from_numpy(*n, 2, d)
    dst = torch.full_like(g.data, -1.0)
    ref = np.full_like(d, -1.0)
    win = ((1, 8), (2, 10), (0, 5))
    sp.apply_window(g.data, dst, win, 3, 3)
    oracle.apply_window(d, ref, win, 3, 3)
    assert_bitwise(dst.cpu().numpy(), ref)
    # shifted in place (compressed frame move), scratch path
    d2 = d.copy()
    oracle.apply_window(d2, d2, ((0, 11), (0, 10), (0, 9)), 3, 2)
    sp.apply_window(g.data, g.data, ((0, 11), (0, 10), (0, 9)), 3, 2)
    assert_bitwise(g.to_numpy(), d2)


def test_snapshot_roundtrip(tmp_path):
    g = sp.create_grid(7, 6, 5, init="random", seed=3)
    p = tmp_path / "s.bin"
    sp.write_snapshot(g, p)
    raw = p.read_bytes()
    assert raw.startswith(b"7 6 5\n")
    h = sp.read_snapshot(p)
    assert_bitwise(h.interior_numpy(), g.interior_numpy())


def test_large_config_c1(golden):
    c = golden["configs"]["C1"]
    g = sp.create_grid(*c["n"], init="random", seed=c["seed"], ring=c["ring"])
    assert g.checksum() == c["init_digest"]
    assert _sweeps(g, c["sweeps"]).checksum() == c["digest"]


def test_layout_extents_alignment_and_faces():
    """Storage layout of sp/grid.py:47-120: extents include pad, x fastest,
    logical (i,j,k) at pad+1-alignment+(k,j,i), faces captured per axis."""
    g = sp.create_grid(4, 4, 4, pad=2, init="constant", value=1.0)
    assert tuple(g.data.shape) == (8, 8, 8) and bool(torch.all(g.data == 1.0))
    g = sp.create_grid(5, 4, 3, pad=0)
    assert g.data.stride() == (6 * 7, 7, 1)
    g = sp.create_grid(6, 6, 6, pad=2, init="random", seed=3)
    before = g.interior_numpy().copy()
    g.alignment = 1  # frame moves one cell toward lower storage indices
    assert g.index(0, 0, 0) == (2, 2, 2)
    g.data[2:8, 2:8, 2:8] = torch.from_numpy(before).cuda()
    assert_bitwise(g.interior_numpy(), before)
    g.capture_boundary_faces()
    assert g.boundary_faces[("x", 0)].shape == (6, 6)
    assert g.boundary_faces[("z", 1)].shape == (6, 6)


def test_snapshots_are_byte_identical_across_runs(tmp_path):
    """Acceptance #8 (tests/test_acceptance.py:266-280): two identical runs
    produce byte-identical snapshots; the snapshot equals the oracle's."""
    import oracle
    outs = []
    for k in range(2):
        g = sp.create_grid(37, 29, 23, init="random", seed=99, ring=0.5)
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(37, 8, 8), t=3)
        st = sp.run_pipelined((g, g.copy()), cfg, 3)
        path = tmp_path / f"snap{k}.bin"
        sp.write_snapshot(st.result, path)
        outs.append(path.read_bytes())
    assert outs[0] == outs[1]
    d0 = oracle.make_storage(37, 29, 23, init="random", seed=99, ring=0.5)
    exp = oracle.interior(oracle.sweeps(d0, (37, 29, 23), 9), 37, 29, 23)
    assert outs[0] == b"37 29 23\n" + exp.astype("<f8").tobytes()


def test_no_cpu_fallback_without_library(monkeypatch):
    """The product path fails loudly when the CUDA library is missing."""
    from paper_1006_3148_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load("/nonexistent/libsp200.so")


def test_rings_equal_sees_faces_edges_and_corners():
    a = sp.create_grid(9, 7, 5, pad=1, init="random", seed=5, ring=0.25)
    b = a.copy()
    assert sp.rings_equal(a, b)
    o = a.offset
    for cell in ((o - 1, o + 2, o + 3), (o + 5, o - 1, o - 1), (o - 1, o - 1, o + 9),
                 (o + 2, o + 3, o + 9)):
        c = a.copy()
        c.data[cell] += 1.0
        assert not sp.rings_equal(a, c), cell
    c = a.copy()
    c.data[o + 2, o + 3, o + 4] += 1.0  # interior cells do not count
    assert sp.rings_equal(a, c)
    d = sp.create_grid(9, 7, 5, pad=1, init="random", seed=5, ring=0.0)
    sp.copy_ring(a, d)
    assert sp.rings_equal(a, d)
