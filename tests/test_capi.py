"""CPU: the C-ABI library loads, exports every symbol include/sp200.h declares,
and rejects invalid geometry without touching the GPU."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

from paper_1006_3148_b200 import _lib

HEADER = os.path.join(ROOT, "include", "sp200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*\*?\s*(sp_\w+)\s*\(", text, re.M)))


def test_header_lists_the_python_exports():
    assert set(_declared()) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.sp_version() >= 10000


def test_invalid_geometry_is_einval_without_gpu():
    L = _lib.load()
    p = ctypes.c_void_p(16)
    # null pointers
    assert L.sp_sweep(None, None, 10, 10, 10, 8, 8, 8, 1, 1, None) == _lib.SP_EINVAL
    # frame does not fit
    assert L.sp_sweep(p, ctypes.c_void_p(32), 10, 10, 10, 9, 8, 8, 1, 1, None) == _lib.SP_EINVAL
    assert b"frame" in L.sp_last_error()
    # aliasing rejected
    assert L.sp_temporal(p, p, 10, 10, 10, 8, 8, 8, 1, 2, 0, 8, None) == _lib.SP_EINVAL
    # fused depth out of range
    assert L.sp_temporal(p, ctypes.c_void_p(32), 10, 10, 10, 8, 8, 8, 1, 9, 0, 8, None) == _lib.SP_EUNSUP
    # shifted in-place window without scratch
    assert L.sp_apply_window(p, p, 10, 10, 10, 0, 4, 0, 4, 0, 4, 2, 1, None, None) == _lib.SP_EINVAL
    # empty window is a no-op
    assert L.sp_apply_window(p, p, 10, 10, 10, 3, 3, 0, 4, 0, 4, 2, 1, None, None) == _lib.SP_OK


def test_check_maps_codes_to_reference_exceptions():
    L = _lib.load()
    rc = L.sp_sweep(None, None, 10, 10, 10, 8, 8, 8, 1, 1, None)
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_tuning_and_tma_query():
    L = _lib.load()
    assert L.sp_tma_eligible(514, 514) == 1
    assert L.sp_tma_eligible(9, 9) == 0  # 72-byte rows: cp.async loader
    assert L.sp_set_tuning(0, 0) == 0
    assert L.sp_set_tuning(2, 1 * 16 + 0) == 0
    assert L.sp_set_tuning(99, 0) == _lib.SP_EINVAL
    assert L.sp_launch_count(0) >= 0
    # A/B keys documented in include/sp200.h: accepted and reset to defaults
    for key in (1, 5, 6, 7, 8):
        assert L.sp_set_tuning(key, 1) == 0
        assert L.sp_set_tuning(key, 0) == 0
    assert L.sp_set_tuning(2, 0 * 16) == _lib.SP_EINVAL   # levels outside [1, 4]


def test_sp200_tune_env_hook():
    """SP200_TUNE applies tuning pairs when the library loads (A/B runs of
    bench.py); a malformed pair fails loudly."""
    import subprocess
    import sys
    code = ("import paper_1006_3148_b200._lib as l; l.load(); print('ok')")
    env = dict(os.environ, SP200_TUNE="6=1,8=64")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout
    env["SP200_TUNE"] = "99=1"
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=ROOT)
    assert r.returncode != 0 and "SP200_TUNE" in r.stderr
