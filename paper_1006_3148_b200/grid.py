"""Device-resident 3D grid storage, seeded init, block plans and snapshots.

Mirrors the reference module sp/grid.py (/root/reference/pkg/src/stencilpipe/
grid.py) with the storage moved into B200 HBM: `Grid3.data` is a CUDA
float64 torch tensor of shape (z, y, x) = n + 2 + pad per axis, x fastest
(sp/grid.py:3-8, 117-121), so every index expression of the reference
(`g.data[g.index(i, j, k)]`, `g.interior_view()`) works unchanged.  All fills
run as sp200 kernels (K0); there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

BOUNDARY = 1  # fixed Dirichlet ring width, one layer per side (sp/grid.py:18)

FACE_KEYS = (("x", 0), ("x", 1), ("y", 0), ("y", 1), ("z", 0), ("z", 1))


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1006_3148_b200 runs on a CUDA device (B200, sm_100a); no CUDA device is "
            "visible and there is no CPU fallback")
    _lib.load()
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


class Grid3:
    """Padded 3D double grid in HBM (sp/grid.py:47-120).

    Logical interior cells are (i, j, k) with 0 <= i < nx etc.; the Dirichlet
    ring sits at logical -1 and n per axis.  ``alignment`` in [0, pad] is the
    current shift of the logical origin toward lower storage indices: logical
    cell c of axis a lives at storage index ``pad + BOUNDARY + c - alignment``.
    """

    def __init__(self, nx, ny, nz, pad=0, data=None, alignment=0, device=None):
        if min(nx, ny, nz) < 1:
            raise ValueError(f"grid dimensions must be >= 1, got {(nx, ny, nz)}")
        if pad < 0:
            raise ValueError(f"pad must be >= 0, got {pad}")
        self.nx, self.ny, self.nz = nx, ny, nz
        self.pad = pad
        self.alignment = alignment
        ext = lambda n: n + 2 * BOUNDARY + pad
        shape = (ext(nz), ext(ny), ext(nx))
        if data is None:
            dev = _device(device)
            data = torch.empty(shape, dtype=torch.float64, device=dev)
            _lib.rings_touched()
            _lib.check(_lib.load().sp_fill_constant(_ptr(data), data.numel(), 0.0, _stream()),
                       "Grid3")
        else:
            if isinstance(data, np.ndarray):
                data = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).to(_device(device))
            if tuple(data.shape) != shape:
                raise ValueError(f"storage shape {tuple(data.shape)} != {shape}")
            if data.dtype != torch.float64 or not data.is_cuda or not data.is_contiguous():
                raise ValueError("Grid3 storage must be a contiguous float64 CUDA tensor")
        self.data = data
        self.boundary_faces = {}

    # -- geometry (sp/grid.py:127-145) ---------------------------------------
    @property
    def origin(self) -> int:
        """Storage index of logical cell 0 at alignment 0 (same per axis)."""
        return self.pad + BOUNDARY

    @property
    def offset(self) -> int:
        """Storage index of logical cell 0 at the current alignment."""
        return self.origin - self.alignment

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    @property
    def extents(self):
        """Storage extents (ex, ey, ez)."""
        ez, ey, ex = self.data.shape
        return ex, ey, ez

    def index(self, i, j, k):
        o = self.offset
        return (o + k, o + j, o + i)

    def interior_view(self) -> torch.Tensor:
        o = self.offset
        return self.data[o:o + self.nz, o:o + self.ny, o:o + self.nx]

    def capture_boundary_faces(self):
        """The six Dirichlet face layers (interior extent), sp/grid.py:94-107."""
        o = self.offset
        nx, ny, nz = self.nx, self.ny, self.nz
        d = self.data
        self.boundary_faces = {
            ("x", 0): d[o:o + nz, o:o + ny, o - 1].clone(),
            ("x", 1): d[o:o + nz, o:o + ny, o + nx].clone(),
            ("y", 0): d[o:o + nz, o - 1, o:o + nx].clone(),
            ("y", 1): d[o:o + nz, o + ny, o:o + nx].clone(),
            ("z", 0): d[o - 1, o:o + ny, o:o + nx].clone(),
            ("z", 1): d[o + nz, o:o + ny, o:o + nx].clone(),
        }

    def copy(self) -> "Grid3":
        g = Grid3(self.nx, self.ny, self.nz, self.pad, data=self.data.clone(),
                  alignment=self.alignment)
        g.boundary_faces = {k: v.clone() for k, v in self.boundary_faces.items()}
        from .kernel import note_rings_equal
        note_rings_equal(self, g)  # a clone's shell equals ours
        return g

    def checksum(self) -> str:
        """SHA-256 of the interior, LE f8, (z,y,x) order (sp/grid.py:115-120)."""
        return interior_digest(self.interior_view())

    # -- host transfer helpers (not in the reference: its data is host memory)
    def to_numpy(self) -> np.ndarray:
        return self.data.cpu().numpy()

    def interior_numpy(self) -> np.ndarray:
        return self.interior_view().cpu().numpy()

    @classmethod
    def from_numpy(cls, nx, ny, nz, pad, array, alignment=0, capture=True) -> "Grid3":
        g = cls(nx, ny, nz, pad, data=torch.from_numpy(np.ascontiguousarray(array)).to(_device()),
                alignment=alignment)
        if capture:
            g.capture_boundary_faces()
        return g

    def face_pointers(self):
        """(c_void_p * 6) array of the device faces in FACE_KEYS order."""
        arr = (ctypes.c_void_p * 6)()
        for n, key in enumerate(FACE_KEYS):
            f = self.boundary_faces.get(key)
            arr[n] = f.data_ptr() if f is not None else None
        return arr


def interior_digest(view: torch.Tensor, chunk_planes: int = 64) -> str:
    """SHA-256 of a (z,y,x) tensor as little-endian f8, plane by plane."""
    h = hashlib.sha256()
    nz = view.shape[0]
    for k0 in range(0, nz, chunk_planes):
        blk = view[k0:k0 + chunk_planes].contiguous().cpu().numpy()
        h.update(blk.astype("<f8", copy=False).tobytes())
    return h.hexdigest()


def fill_shell(g: Grid3, value: float) -> None:
    """Set the full one-cell shell (faces, edges, corners) at the current frame."""
    o, nx, ny, nz = g.offset, g.nx, g.ny, g.nz
    d = g.data
    zl, zh, yl, yh, xl, xh = o - 1, o + nz, o - 1, o + ny, o - 1, o + nx
    d[zl, yl:yh + 1, xl:xh + 1] = value
    d[zh, yl:yh + 1, xl:xh + 1] = value
    d[zl:zh + 1, yl, xl:xh + 1] = value
    d[zl:zh + 1, yh, xl:xh + 1] = value
    d[zl:zh + 1, yl:yh + 1, xl] = value
    d[zl:zh + 1, yl:yh + 1, xh] = value


def fill_seeded(g: Grid3, seed: int, global_dims=None, global_origin=(0, 0, 0),
                lo: float = 0.0, hi: float = 1.0, shell: float = 0.0) -> None:
    """K0: interior from the global SplitMix64 field (sp/grid.py:21-30,
    138-143; sp/halo.py:132-147), every other stored cell = `shell`."""
    ex, ey, ez = g.extents
    gd = global_dims or g.shape
    _lib.rings_touched()
    _lib.check(_lib.load().sp_fill_seeded(
        _ptr(g.data), ex, ey, ez, g.offset, g.nx, g.ny, g.nz,
        global_origin[0], global_origin[1], global_origin[2], gd[0], gd[1], gd[2],
        ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), lo, hi, shell, _stream()), "fill_seeded")


def create_grid(nx, ny, nz, pad=0, init="constant", value=0.0, seed=0, *, ring=None,
                lo=0.0, hi=1.0, device=None) -> Grid3:
    """Allocate and fill a grid (sp/grid.py:123-147).

    init rules (as the reference):
      "constant" -- every stored cell (interior and ring) equals ``value``
      "impulse"  -- all zero except a 1.0 at the interior center cell
      "random"   -- interior from the seeded generator, ring zero
    Keyword extensions for the BASELINE configs: ``ring``
    sets the one-cell shell to a constant after the fill; ``(lo, hi)`` remaps
    the random interior to lo + (hi - lo) * u (``(-1, 1)`` is exact).
    """
    if init not in ("constant", "impulse", "random"):
        raise ValueError(f"unknown init rule {init!r}")
    g = Grid3(nx, ny, nz, pad, device=device)
    L = _lib.load()
    if init == "constant":
        _lib.rings_touched()
        _lib.check(L.sp_fill_constant(_ptr(g.data), g.data.numel(), float(value), _stream()))
    elif init == "impulse":
        g.data[g.index(nx // 2, ny // 2, nz // 2)] = 1.0
    else:
        fill_seeded(g, seed, lo=lo, hi=hi, shell=0.0 if ring is None else float(ring))
    if ring is not None and init != "random":
        fill_shell(g, float(ring))
    g.capture_boundary_faces()
    return g


def seeded_field_checksum(nx: int, ny: int, nz: int, seed: int, chunk_planes: int = 64) -> str:
    """SHA-256 of the seeded field (sp/grid.py:33-44), generated on the GPU."""
    g = Grid3(nx, ny, nz, 0)
    fill_seeded(g, seed)
    return interior_digest(g.interior_view(), chunk_planes)


# ---------------------------------------------------------------------------
# block plans (sp/grid.py:150-215) — host-side scheduling metadata.  On the
# GPU the CTA tiling replaces them; they remain for API parity and validation.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class BlockSpec:
    """Block edge lengths in cells, (bx, by, bz)."""
    bx: int
    by: int
    bz: int

    def validate(self, grid: Grid3):
        for b, n, name in ((self.bx, grid.nx, "bx"), (self.by, grid.ny, "by"),
                           (self.bz, grid.nz, "bz")):
            if not 1 <= b <= n:
                raise ValueError(f"{name}={b} outside [1, {n}]")


@dataclass
class BlockPlan:
    bases: tuple
    sizes: tuple
    direction: int
    blocks: list = field(default_factory=list)

    @property
    def total_blocks(self) -> int:
        return len(self.blocks)


def decompose_blocks(grid: Grid3, spec: BlockSpec, direction: int = 1) -> BlockPlan:
    """Tile the interior with blocks; last block per axis may be truncated."""
    spec.validate(grid)
    if direction not in (1, -1):
        raise ValueError(f"direction must be +1 or -1, got {direction}")
    xb = list(range(0, grid.nx, spec.bx))
    yb = list(range(0, grid.ny, spec.by))
    zb = list(range(0, grid.nz, spec.bz))
    blocks = [((x, y, z), (min(spec.bx, grid.nx - x), min(spec.by, grid.ny - y),
                           min(spec.bz, grid.nz - z)))
              for z in zb for y in yb for x in xb]
    if direction == -1:
        blocks.reverse()
    return BlockPlan(bases=(xb, yb, zb), sizes=(grid.nx, grid.ny, grid.nz),
                     direction=direction, blocks=blocks)


def next_block(plan: BlockPlan, counter: int):
    if counter < 0:
        raise ValueError("block counter must be >= 0")
    if counter >= plan.total_blocks:
        return None
    return plan.blocks[counter]


# ---------------------------------------------------------------------------
# snapshots (sp/grid.py:218-236): ASCII "nx ny nz\n" + raw LE f8 interior
# ---------------------------------------------------------------------------

def write_snapshot(grid: Grid3, path) -> None:
    with open(path, "wb") as f:
        f.write(f"{grid.nx} {grid.ny} {grid.nz}\n".encode("ascii"))
        iv = grid.interior_view()
        for k0 in range(0, grid.nz, 64):
            f.write(iv[k0:k0 + 64].contiguous().cpu().numpy().astype("<f8", copy=False).tobytes())


def read_snapshot(path) -> Grid3:
    with open(path, "rb") as f:
        header = f.readline().decode("ascii").split()
        nx, ny, nz = (int(v) for v in header)
        raw = f.read(nx * ny * nz * 8)
    if len(raw) != nx * ny * nz * 8:
        raise ValueError(f"snapshot {path} truncated")
    g = Grid3(nx, ny, nz, pad=0)
    g.interior_view().copy_(torch.from_numpy(
        np.frombuffer(raw, dtype="<f8").reshape(nz, ny, nx).copy()))
    g.capture_boundary_faces()
    return g
