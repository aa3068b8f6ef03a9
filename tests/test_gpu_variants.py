"""Every K2 kernel instance the dispatcher can select (sp_set_tuning key 2:
levels*16 + index), including the tall-tile defaults and the two-CTA cluster
variant (index 4: DSMEM halo rows through st.async), bit-exact against the
oracle on ragged shapes and over live z ranges."""

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
    for t in range(2, 5):
        L.sp_set_tuning(2, t * 16)


@pytest.mark.parametrize("levels", [2, 3, 4])
@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4, 5])
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
