"""CPU: pin the oracle (C and NumPy restatements) against the reference's own
frozen digests and the fixtures generated from the reference itself."""

import numpy as np
import pytest

import oracle
from conftest import assert_bitwise


def test_splitmix_c_equals_numpy():
    for start, count, seed in ((0, 1000, 42), (123456789, 777, 7), (2**40, 64, 2**63 + 5)):
        assert_bitwise(oracle.c_splitmix64_unit(start, count, seed),
                       oracle.splitmix64_unit(start, count, seed))


def test_field_60_pin(golden):
    d = oracle.make_storage(60, 60, 60, init="random", seed=42)
    assert oracle.digest(oracle.interior(d, 60, 60, 60)) == golden["pins"]["FIELD_60_SEED42"]


def test_field_600_pin_streamed(golden):
    import hashlib
    h = hashlib.sha256()
    slab = 600 * 600
    for k in range(600):
        h.update(oracle.c_splitmix64_unit(k * slab, slab, 42).astype("<f8").tobytes())
    assert h.hexdigest() == golden["pins"]["FIELD_600_SEED42"]


def test_ref_60_8_sweeps_pin_numpy_and_c(golden):
    d0 = oracle.make_storage(60, 60, 60, init="random", seed=42)
    res = oracle.sweeps(d0, (60, 60, 60), 8)
    assert oracle.digest(oracle.interior(res, 60, 60, 60)) == golden["pins"]["REF_60_SEED42_8SWEEPS"]
    a, b = d0.copy(), d0.copy()
    out = oracle.c_sweeps(a, b, (60, 60, 60), 8)
    assert oracle.digest(oracle.interior(out, 60, 60, 60)) == golden["pins"]["REF_60_SEED42_8SWEEPS"]


def _case_storage(c):
    return oracle.make_storage(c["nx"], c["ny"], c["nz"], pad=c["pad"], init=c["init"],
                               value=c["value"], seed=c["seed"], ring=c["ring"],
                               lo=c["lo"], hi=c["hi"])


def test_golden_sweep_cases_numpy(golden):
    for name, c in golden["sweeps"].items():
        d0 = _case_storage(c)
        n = (c["nx"], c["ny"], c["nz"])
        assert oracle.digest(oracle.interior(d0, *n, pad=c["pad"])) == c["init_digest"], name
        a, b = d0.copy(), d0.copy()
        off = c["pad"] + 1
        for s in range(1, c["sweeps"] + 1):
            oracle.reference_sweep(a, b, *n, off)
            a, b = b, a
            assert oracle.digest(oracle.interior(a, *n, pad=c["pad"])) == c["digests"][str(s)], (name, s)


def test_golden_sweep_cases_c(golden):
    for name, c in golden["sweeps"].items():
        d0 = _case_storage(c)
        n = (c["nx"], c["ny"], c["nz"])
        out = oracle.c_sweeps(d0.copy(), d0.copy(), n, c["sweeps"], pad=c["pad"])
        assert oracle.digest(oracle.interior(out, *n, pad=c["pad"])) == c["digests"][str(c["sweeps"])], name


def test_c_oracle_matches_numpy_with_alignment_frames():
    # pad 3, alignment 2: frame offset 2
    n = (9, 8, 7)
    d0 = oracle.make_storage(*n, pad=3, init="random", seed=19, alignment=2, ring=0.5)
    r1 = oracle.sweeps(d0, n, 5, pad=3, alignment=2)
    r2 = oracle.c_sweeps(d0.copy(), d0.copy(), n, 5, pad=3, alignment=2)
    assert_bitwise(oracle.interior(r2, *n, pad=3, alignment=2), oracle.interior(r1, *n, pad=3, alignment=2))


def test_apply_window_shifted_in_place_equals_two_grid():
    # sp/kernel.py:41-44: whole window before store makes the shifted write safe
    n = (6, 6, 6)
    d = oracle.make_storage(*n, pad=2, init="random", seed=33)
    ref = oracle.sweeps(d, n, 1, pad=2)
    o = 3
    oracle.apply_window(d, d, ((0, 6), (0, 6), (0, 6)), o, o - 1)
    assert_bitwise(d[o - 1:o + 5, o - 1:o + 5, o - 1:o + 5], oracle.interior(ref, *n, pad=2))


def test_window_oracle_matches_full_run():
    G = (30, 28, 26)
    S = 5
    d0 = oracle.make_storage(*G, init="random", seed=11, ring=1.0)
    full = oracle.interior(oracle.sweeps(d0, G, S), *G)
    for box in (((10, 20), (8, 16), (9, 14)), ((0, 7), (0, 5), (0, 4)), ((22, 30), (20, 28), (20, 26))):
        got = oracle.window_oracle(G, 11, box, S, ring=1.0)
        (xl, xh), (yl, yh), (zl, zh) = box
        assert_bitwise(got, full[zl:zh, yl:yh, xl:xh])


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_config_digests_c_oracle(golden, name):
    """The BASELINE config digests (computed with the reference's own
    run_pipelined) reproduced by the C restatement."""
    c = golden.get("configs", {}).get(name)
    if c is None:
        pytest.skip("config digest not generated")
    n = tuple(c["n"])
    d0 = oracle.make_storage(*n, pad=c["pad"], init="random", seed=c["seed"], ring=c["ring"],
                             lo=c["lo"], hi=c["hi"])
    assert oracle.digest(oracle.interior(d0, *n, pad=c["pad"])) == c["init_digest"]
    out = oracle.c_sweeps(d0, d0.copy(), n, c["sweeps"], pad=c["pad"])
    assert oracle.digest(oracle.interior(out, *n, pad=c["pad"])) == c["digest"]


@pytest.mark.parametrize("t,block,dims", [(4, (20, 6, 6), (20, 18, 24)), (2, (13, 5, 4), (13, 11, 9)),
                                          (3, (8, 8, 8), (16, 16, 16))])
def test_pipelined_restatement_equals_sweeps(t, block, dims):
    """The threaded restatement of the reference's pipelined scheduler
    (bench.py's second CPU baseline) equals t plain sweeps bit for bit."""
    from oracle.pipelined import pipelined_pass_two_grid
    d0 = oracle.make_storage(*dims, init="random", seed=3, ring=0.5)
    grids = [d0.copy(), d0.copy()]
    which = pipelined_pass_two_grid(grids, dims, t, block)
    which = pipelined_pass_two_grid(grids, dims, t, block, levels_done=t)
    exp = oracle.interior(oracle.sweeps(d0, dims, 2 * t), *dims)
    assert np.array_equal(oracle.interior(grids[which], *dims), exp)
