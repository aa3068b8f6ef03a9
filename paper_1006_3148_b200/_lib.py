"""ctypes binding of libsp200.so (include/sp200.h).

The library is built in-tree (``python -m paper_1006_3148_b200._build`` or
``__graft_entry__.build()``).  There is no CPU fallback: importing the compute
entry points without the library or without a CUDA device raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SP200_LIB selects another in-tree build (kernel A/B experiments in tools/)
LIB_PATH = os.environ.get("SP200_LIB") or os.path.join(HERE, "libsp200.so")

SP_OK = 0
SP_EINVAL = -1
SP_EUNSUP = -2
SP_ECUDA = -3
SP_ERANGE = -4
SP_MAX_FUSED = 4

# every symbol include/sp200.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "sp_version", "sp_last_error", "sp_launch_count", "sp_fill_seeded",
    "sp_fill_constant", "sp_sweep", "sp_apply_window", "sp_window_gather",
    "sp_copy_ring", "sp_rings_equal", "sp_write_faces", "sp_temporal", "sp_compressed_workspace", "sp_compressed_workspace_for",
    "sp_compressed", "sp_set_tuning", "sp_tma_eligible", "sp_temporal_mirror", "sp_ipc_handle",
    "sp_ipc_open", "sp_ipc_close", "sp_signal", "sp_wait", "sp_pack_boxes", "sp_unpack_boxes",
)
SP_MAX_BOXES = 8


class SpBox(ctypes.Structure):
    """sp_box_t: half-open storage box + its contiguous device buffer."""
    _fields_ = [("x0", ctypes.c_int64), ("x1", ctypes.c_int64), ("y0", ctypes.c_int64),
                ("y1", ctypes.c_int64), ("z0", ctypes.c_int64), ("z1", ctypes.c_int64),
                ("buf", ctypes.c_void_p)]

_lib = None


class Sp200Error(RuntimeError):
    """A CUDA-side failure reported by libsp200 (SP_ECUDA / SP_EUNSUP)."""


def _declare(L):
    i64, i32, dp, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p
    u64, f64 = ctypes.c_uint64, ctypes.c_double
    sig = {
        "sp_version": ([], i32),
        "sp_last_error": ([], ctypes.c_char_p),
        "sp_launch_count": ([i32], i64),
        "sp_fill_seeded": ([dp, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64,
                            u64, f64, f64, f64, vp], i32),
        "sp_fill_constant": ([dp, i64, f64, vp], i32),
        "sp_sweep": ([dp, dp, i64, i64, i64, i64, i64, i64, i64, i32, vp], i32),
        "sp_apply_window": ([dp, dp, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, dp, vp],
                            i32),
        "sp_window_gather": ([dp, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, dp, vp], i32),
        "sp_copy_ring": ([dp, dp, i64, i64, i64, i64, i64, i64, i64, vp], i32),
        "sp_rings_equal": ([dp, dp, i64, i64, i64, i64, i64, i64, i64, ctypes.POINTER(i32), vp], i32),
        "sp_write_faces": ([dp, i64, i64, i64, i64, i64, i64, i64, ctypes.POINTER(dp), i32, vp], i32),
        "sp_temporal": ([dp, dp, i64, i64, i64, i64, i64, i64, i64, i32, i64, i64, vp], i32),
        "sp_compressed_workspace": ([i64, i64, i64, i32], i64),
        "sp_compressed_workspace_for": ([dp, i64, i64, i64, i64, i64, i32], i64),
        "sp_compressed": ([dp, i64, i64, i64, i64, i64, i64, i64, i32, i32, i64, i64, vp, i64,
                           ctypes.POINTER(dp), i32, vp], i32),
        "sp_set_tuning": ([i32, i64], i32),
        "sp_temporal_mirror": ([dp, dp, i64, i64, i64, i64, i64, i64, i64, i32, i64, i64, dp, i64, i64,
                                vp], i32),
        "sp_ipc_handle": ([vp, ctypes.c_char_p, ctypes.POINTER(i64)], i32),
        "sp_ipc_open": ([ctypes.c_char_p, ctypes.POINTER(vp)], i32),
        "sp_ipc_close": ([vp], i32),
        "sp_signal": ([vp, ctypes.c_uint32, vp], i32),
        "sp_wait": ([vp, ctypes.c_uint32, vp], i32),
        "sp_tma_eligible": ([i64, i64], i32),
        "sp_pack_boxes": ([dp, i64, i64, i64, i32, ctypes.POINTER(SpBox), vp], i32),
        "sp_unpack_boxes": ([dp, i64, i64, i64, i32, ctypes.POINTER(SpBox), vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(
                f"libsp200.so not found at {path}; build it with "
                "`python -m paper_1006_3148_b200._build` (there is no CPU fallback)")
        L = ctypes.CDLL(path)
        _declare(L)
        # A/B experiments only: SP200_TUNE="key=value,..." (sp_set_tuning)
        for kv in filter(None, os.environ.get("SP200_TUNE", "").split(",")):
            k, v = kv.split("=")
            if L.sp_set_tuning(int(k), int(v)) != SP_OK:
                raise ValueError(f"SP200_TUNE: bad pair {kv!r}")
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map an sp200 status code to the reference's exception types."""
    if rc == SP_OK:
        return
    msg = load().sp_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == SP_EINVAL:
        raise ValueError(msg)
    if rc == SP_ERANGE:
        raise IndexError(msg)
    raise Sp200Error(msg)


# Ring-write epoch: bumped by every wrapper whose kernel may store Dirichlet
# ring cells through a raw pointer (torch's tensor version counters do not see
# those writes).  kernel.rings_equal caches verdicts under it.
_ring_epoch = 0


def rings_touched() -> None:
    global _ring_epoch
    _ring_epoch += 1


def ring_epoch() -> int:
    return _ring_epoch


def launch_count(reset: bool = False) -> int:
    return int(load().sp_launch_count(1 if reset else 0))
