"""Jacobi updates on cells, windows and whole grids — B200 kernels.

Mirrors sp/kernel.py (/root/reference/pkg/src/stencilpipe/kernel.py).  Every
path runs an sp200 CUDA kernel with the reference's per-cell summation order
(x-low, x-high, y-low, y-high, z-low, z-high, then multiply by fl(1/6)), so
the results are bitwise identical to the reference sweep.
"""

from __future__ import annotations

import ctypes
import weakref

import torch

from . import _lib
from .grid import FACE_KEYS, BlockSpec, Grid3, _ptr, _stream

SIXTH = 1.0 / 6.0  # sp/kernel.py:16
AXES = ("x", "y", "z")


def _ext(t: torch.Tensor):
    ez, ey, ex = t.shape
    return ex, ey, ez


def _check_storage(t: torch.Tensor, name: str):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
            and t.dim() == 3 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous 3D float64 CUDA tensor")


def stencil_update_cell(grid: Grid3, i: int, j: int, k: int) -> float:
    """Single cell update (sp/kernel.py:21-29); IndexError outside the interior."""
    if not (0 <= i < grid.nx and 0 <= j < grid.ny and 0 <= k < grid.nz):
        raise IndexError(f"cell {(i, j, k)} outside interior {grid.shape}")
    out = torch.empty(1, dtype=torch.float64, device=grid.data.device)
    ex, ey, ez = grid.extents
    _lib.check(_lib.load().sp_window_gather(
        _ptr(grid.data), ex, ey, ez, i, i + 1, j, j + 1, k, k + 1, grid.offset, _ptr(out),
        _stream()), "stencil_update_cell")
    return float(out.item())


def window_is_empty(window) -> bool:
    return any(lo >= hi for lo, hi in window)


def apply_window(src: torch.Tensor, dst: torch.Tensor, window, src_off: int,
                 dst_off: int) -> None:
    """Update one rectangular window of logical cells (sp/kernel.py:36-58).

    src/dst are storage tensors (Grid3.data); they may alias: a shifted
    in-place update is computed into a temporary before the store, exactly as
    the reference's NumPy buffer."""
    _check_storage(src, "src")
    _check_storage(dst, "dst")
    if src.shape != dst.shape:
        raise ValueError("src and dst storage shapes differ")
    (xl, xh), (yl, yh), (zl, zh) = window
    if xl >= xh or yl >= yh or zl >= zh:
        return
    ex, ey, ez = _ext(src)
    scratch = None
    if src.data_ptr() == dst.data_ptr() and src_off != dst_off:
        scratch = torch.empty((zh - zl) * (yh - yl) * (xh - xl), dtype=torch.float64,
                              device=src.device)
    _lib.rings_touched()
    _lib.check(_lib.load().sp_apply_window(
        _ptr(src), _ptr(dst), ex, ey, ez, xl, xh, yl, yh, zl, zh, src_off, dst_off,
        _ptr(scratch) if scratch is not None else None, _stream()), "apply_window")


def write_ring_strips(dst: torch.Tensor, faces: dict, window, dst_off: int, sides,
                      dims) -> None:
    """Dirichlet strips next to a window in a displaced frame (sp/kernel.py:61-82)."""
    (xl, xh), (yl, yh), (zl, zh) = window
    do = dst_off
    nx, ny, nz = dims
    for axis, side in sides:
        vals = faces[(axis, side)]
        if axis == "x":
            p = (-1 if side == 0 else nx) + do
            dst[zl + do:zh + do, yl + do:yh + do, p] = vals[zl:zh, yl:yh]
        elif axis == "y":
            p = (-1 if side == 0 else ny) + do
            dst[zl + do:zh + do, p, xl + do:xh + do] = vals[zl:zh, xl:xh]
        else:
            p = (-1 if side == 0 else nz) + do
            dst[p, yl + do:yh + do, xl + do:xh + do] = vals[yl:yh, xl:xh]


def write_faces(grid: Grid3, dst_off: int, side_mask: int = 63) -> None:
    """All (enabled) Dirichlet faces of `grid` at frame offset dst_off, one kernel."""
    ex, ey, ez = grid.extents
    faces = grid.face_pointers()
    mask = 0
    for n, key in enumerate(FACE_KEYS):
        if (side_mask >> n) & 1 and grid.boundary_faces.get(key) is not None:
            mask |= 1 << n
    _lib.rings_touched()
    _lib.check(_lib.load().sp_write_faces(
        _ptr(grid.data), ex, ey, ez, grid.nx, grid.ny, grid.nz, dst_off,
        ctypes.cast(faces, ctypes.POINTER(ctypes.c_void_p)), mask, _stream()), "write_faces")


def copy_ring(a: Grid3, b: Grid3) -> None:
    """Copy the one-cell shell of A onto B (sp/kernel.py:85-96)."""
    ex, ey, ez = a.extents
    _lib.rings_touched()
    _lib.check(_lib.load().sp_copy_ring(_ptr(a.data), _ptr(b.data), ex, ey, ez, a.nx, a.ny,
                                        a.nz, a.offset, _stream()), "copy_ring")
    note_rings_equal(a, b)


# Verdicts of rings_equal, keyed by both storages' pointers, frame offsets and
# torch version counters plus the library's ring-write epoch: any write that
# could change a shell (torch in-place ops, or an sp200 kernel that stores ring
# cells) changes the key, so a cached verdict is never stale.  Calls that make
# the shells equal by construction (copy_ring, reference_sweep, Grid3.copy)
# record True without a device round trip.
_RING_CACHE: dict = {}


def _ring_key(a: Grid3, b: Grid3):
    if a.data.data_ptr() > b.data.data_ptr():
        a, b = b, a
    return (id(a.data), id(b.data), a.data.data_ptr(), b.data.data_ptr(), a.offset, b.offset,
            tuple(a.data.shape), tuple(b.data.shape), a.data._version, b.data._version,
            _lib.ring_epoch())


def _ring_lookup(a: Grid3, b: Grid3):
    """Cached verdict, or None.  Entries hold weak references to both storage
    tensors: a tensor freed and replaced by a new one at the same address
    (the caching allocator reuses blocks) never matches an old entry."""
    hit = _RING_CACHE.get(_ring_key(a, b))
    if hit is None:
        return None
    wa, wb, verdict = hit
    if {id(wa()), id(wb())} != {id(a.data), id(b.data)}:
        return None
    return verdict


def _ring_store(a: Grid3, b: Grid3, verdict: bool) -> None:
    if len(_RING_CACHE) > 256:
        _RING_CACHE.clear()
    _RING_CACHE[_ring_key(a, b)] = (weakref.ref(a.data), weakref.ref(b.data), verdict)


def note_rings_equal(a: Grid3, b: Grid3) -> None:
    _ring_store(a, b, True)


def rings_equal(a: Grid3, b: Grid3) -> bool:
    """True when A and B hold equal one-cell shells (faces, edges, corners)
    at their frame — the precondition for fusing two-grid levels.  Waits only
    for the current stream (the verdict comes back through host-mapped
    memory, not a copy engine)."""
    if a.data.shape != b.data.shape or a.offset != b.offset:
        return False
    hit = _ring_lookup(a, b)
    if hit is not None:
        return hit
    ex, ey, ez = a.extents
    eq = ctypes.c_int(0)
    _lib.check(_lib.load().sp_rings_equal(_ptr(a.data), _ptr(b.data), ex, ey, ez, a.nx, a.ny,
                                          a.nz, a.offset, ctypes.byref(eq), _stream()), "rings_equal")
    _ring_store(a, b, bool(eq.value))
    return bool(eq.value)


def reference_sweep(a: Grid3, b: Grid3) -> None:
    """One plain Jacobi sweep: B.interior = stencil(A), B.ring = A.ring
    (sp/kernel.py:99-111) — K1, the streaming sweep with the fused ring copy."""
    if a.shape != b.shape:
        raise ValueError(f"grid shapes differ: {a.shape} vs {b.shape}")
    if a.alignment != b.alignment:
        raise ValueError("reference_sweep requires equal alignments")
    if a.data.shape != b.data.shape:
        raise ValueError("grid storage extents differ (pad mismatch)")
    if a.data.data_ptr() == b.data.data_ptr():
        raise ValueError("reference_sweep needs two distinct grids")
    ex, ey, ez = a.extents
    _lib.rings_touched()
    _lib.check(_lib.load().sp_sweep(_ptr(a.data), _ptr(b.data), ex, ey, ez, a.nx, a.ny, a.nz,
                                    a.offset, 1, _stream()), "reference_sweep")
    note_rings_equal(a, b)


def spatial_blocked_sweep(a: Grid3, b: Grid3, spec: BlockSpec) -> None:
    """Reference sweep traversed block by block (sp/kernel.py:114-125).  On the
    GPU the CTA tiling is the blocking; block order cannot change per-cell
    arithmetic, so this is K1 after validating the block spec."""
    if a.shape != b.shape:
        raise ValueError(f"grid shapes differ: {a.shape} vs {b.shape}")
    spec.validate(a)
    ex, ey, ez = a.extents
    _lib.rings_touched()
    _lib.check(_lib.load().sp_sweep(_ptr(a.data), _ptr(b.data), ex, ey, ez, a.nx, a.ny, a.nz,
                                    a.offset, 1, _stream()), "spatial_blocked_sweep")
    note_rings_equal(a, b)


def fused_sweeps(src: Grid3, dst: Grid3, levels: int, zlo: int = 0, zhi: int | None = None) -> None:
    """K2: `levels` (1..4) sweeps in one HBM pass, src -> dst interior (two-grid
    pipeline semantics: rings untouched, read from src)."""
    if src.data.shape != dst.data.shape or src.shape != dst.shape:
        raise ValueError("grid geometry differs")
    ex, ey, ez = src.extents
    _lib.check(_lib.load().sp_temporal(
        _ptr(src.data), _ptr(dst.data), ex, ey, ez, src.nx, src.ny, src.nz, src.offset,
        int(levels), int(zlo), int(src.nz if zhi is None else zhi), _stream()), "fused_sweeps")


def fused_sweeps_mirror(src: Grid3, dst: Grid3, levels: int, zlo: int, zhi: int, mirror_ptr: int,
                        mirror_ez: int, mirror_zshift: int) -> None:
    """fused_sweeps whose stored planes [zlo, zhi) also go to a peer rank's grid
    (device pointer `mirror_ptr` with the same x/y storage extents, `mirror_ez`
    planes) at storage plane z + zshift: the z-slab halo delivery fused into
    the pass (sp/halo.py:239-271 for topology (1,1,P))."""
    if src.data.shape != dst.data.shape or src.shape != dst.shape:
        raise ValueError("grid geometry differs")
    ex, ey, ez = src.extents
    _lib.check(_lib.load().sp_temporal_mirror(
        _ptr(src.data), _ptr(dst.data), ex, ey, ez, src.nx, src.ny, src.nz, src.offset,
        int(levels), int(zlo), int(zhi), ctypes.c_void_p(int(mirror_ptr)), int(mirror_ez),
        int(mirror_zshift), _stream()), "fused_sweeps_mirror")


def compressed_pass(grid: Grid3, levels: int, direction: int, src_alignment: int,
                    workspace: torch.Tensor, zlo: int = 0, zhi: int | None = None,
                    side_mask: int = 63) -> None:
    """K3: `levels` (1..4) in-place shifted updates of a compressed grid in one
    HBM pass, frame a -> a +/- levels (sp/pipeline.py:309-312), then the
    Dirichlet faces at the new frame (sp/kernel.py:61-82)."""
    ex, ey, ez = grid.extents
    faces = grid.face_pointers()
    mask = 0
    for n, key in enumerate(FACE_KEYS):
        if (side_mask >> n) & 1 and grid.boundary_faces.get(key) is not None:
            mask |= 1 << n
    _lib.rings_touched()
    _lib.check(_lib.load().sp_compressed(
        _ptr(grid.data), ex, ey, ez, grid.nx, grid.ny, grid.nz, grid.origin - src_alignment,
        int(direction), int(levels), int(zlo), int(grid.nz if zhi is None else zhi),
        _ptr(workspace), workspace.numel() * workspace.element_size(), ctypes.cast(faces, ctypes.POINTER(ctypes.c_void_p)), mask, _stream()),
        "compressed_pass")


def compressed_workspace(grid: Grid3, levels: int, depth: int | None = None) -> torch.Tensor:
    """Workspace for a K3 pass of this grid over `depth` planes (default nz):
    the progress counters of the in-place pass, or the band stash."""
    ex, ey, _ = grid.extents
    n = int(_lib.load().sp_compressed_workspace_for(_ptr(grid.data), ex, ey, grid.nx, grid.ny,
                                                    grid.nz if depth is None else depth, int(levels)))
    return torch.empty(max(n, 256), dtype=torch.uint8, device=grid.data.device)
