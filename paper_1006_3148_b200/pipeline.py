"""Temporally blocked solve on the B200: PipelineEngine / run_pipelined.

Mirrors sp/pipeline.py (/root/reference/pkg/src/stencilpipe/pipeline.py).
The reference executes one pass of h = n*t*T update levels with n*t CPU
threads that trail each other through cache-sized blocks (Eq. 3 relaxed
counters).  Here the same pass is executed by fused CUDA kernels:

* two_grid: K2 (`sp_temporal`) fuses up to MAX_FUSED levels per HBM pass; a
  pass of h levels runs as ceil(h / MAX_FUSED) fused launches alternating the
  two grids.  The reference puts level `lvl` in grids[lvl % 2]
  (sp/pipeline.py:301-308); after the pass the engine rebinds the two storage
  tensors so that grids[(levels_done) % 2] — `current_grid()` — holds the
  result.  The non-current grid holds an earlier level (scratch), not
  necessarily level h-1 as in the reference.
* compressed: one array, level u written one cell diagonally shifted
  (sp/pipeline.py:309-312), Dirichlet faces re-materialised at the shifted
  frames (sp/pipeline.py:324-335, 427-447).

The result depends only on the total number of updates, which is
what makes fusing any number of levels per kernel exact.  The CPU thread
machinery (SyncCounters, EffectiveDistances, may_advance) is kept as plain
host logic for API parity; it is not used on the GPU path.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import _lib
from .grid import BlockSpec, Grid3, decompose_blocks
from .kernel import (apply_window, compressed_pass, compressed_workspace, fused_sweeps, rings_equal,
                     write_faces, write_ring_strips)

MAX_FUSED = _lib.SP_MAX_FUSED


class PipelineDeadlock(RuntimeError):
    """No counter made progress within the watchdog budget (sp/pipeline.py:34)."""


@dataclass
class PipelineConfig:
    """Tunables of the pipelined scheme (sp/pipeline.py:42-86).

    n teams of t threads, T updates per thread per block; h = n*t*T updates
    per pass.  On the GPU, h is the pass depth; d_l/d_u/d_t/sync_mode/jitter/
    pin_threads describe the CPU schedule and are validated but not used.
    """
    spec: BlockSpec
    n: int = 1
    t: int = 1
    T: int = 1
    d_l: int = 1
    d_u: int = 3
    d_t: int = 0
    sync_mode: str = "relaxed"
    grid_mode: str = "two_grid"
    watchdog_s: float = 30.0
    pin_threads: bool = False
    jitter_prob: float = 0.0
    jitter_max_s: float = 0.0
    jitter_seed: int = 0

    def __post_init__(self):
        if min(self.n, self.t, self.T) < 1:
            raise ValueError("n, t, T must all be >= 1")
        if self.d_l < 1:
            raise ValueError("d_l must be >= 1")
        if self.d_u < self.d_l:
            raise ValueError("d_u must be >= d_l")
        if self.d_t < 0:
            raise ValueError("d_t must be >= 0")
        if self.sync_mode not in ("relaxed", "barrier"):
            raise ValueError(f"unknown sync_mode {self.sync_mode!r}")
        if self.grid_mode not in ("two_grid", "compressed"):
            raise ValueError(f"unknown grid_mode {self.grid_mode!r}")

    @property
    def threads(self) -> int:
        return self.n * self.t

    @property
    def h(self) -> int:
        return self.n * self.t * self.T


class SyncCounters:
    """Per-thread monotone block counters (sp/pipeline.py:89-110); host logic."""

    def __init__(self, count: int):
        self.count = count
        self._slots = [0] * count

    def get(self, i: int) -> int:
        return self._slots[i]

    def bump(self, i: int, amount: int = 1) -> None:
        self._slots[i] += amount

    def reset(self) -> None:
        self._slots = [0] * self.count

    def snapshot(self):
        return list(self._slots)


@dataclass(frozen=True)
class EffectiveDistances:
    """Per-thread (d_l, d_u) after the team delay (sp/pipeline.py:113-130)."""
    d_l: tuple
    d_u: tuple

    @classmethod
    def from_config(cls, cfg: PipelineConfig) -> "EffectiveDistances":
        nt = cfg.threads
        dl, du = [], []
        for g in range(nt):
            team_front = (g % cfg.t == 0)
            team_rear = (g % cfg.t == cfg.t - 1)
            dl.append(cfg.d_l + (cfg.d_t if team_front and g != 0 else 0))
            du.append(cfg.d_u + (cfg.d_t if team_rear and g != nt - 1 else 0))
        return cls(d_l=tuple(dl), d_u=tuple(du))


def may_advance(c: SyncCounters, i: int, dist: EffectiveDistances) -> bool:
    """Eq. 3 progress conditions (sp/pipeline.py:133-141)."""
    if not 0 <= i < c.count:
        raise IndexError(f"thread index {i} out of range")
    ok_pred = i == 0 or c.get(i - 1) - c.get(i) >= dist.d_l[i]
    ok_succ = i == c.count - 1 or c.get(i) - c.get(i + 1) <= dist.d_u[i]
    return ok_pred and ok_succ


def estimate_max_distance(cache_bytes: float, t: int, spec: BlockSpec) -> int:
    """sp/pipeline.py:144-152."""
    volume = spec.bx * spec.by * spec.bz
    if volume <= 0:
        raise ValueError("block volume must be positive")
    if t < 1 or cache_bytes <= 0:
        raise ValueError("t and cache_bytes must be positive")
    return int(cache_bytes // (t * volume * 8))


@dataclass
class RunStats:
    """Outcome of a pipelined run (sp/pipeline.py:155-186).  Spin/gap fields
    describe the CPU schedule and stay at their neutral values on the GPU;
    `kernel_launches` counts the sp200 kernels the run issued."""
    wall_seconds: float = 0.0
    mlups: float = 0.0
    updates_total: int = 0
    passes: int = 0
    block_updates: int = 0
    spin_iterations_total: int = 0
    per_thread_spins: list = field(default_factory=list)
    pred_gap_min: int | None = None
    pred_violations: int = 0
    succ_gap_max: int | None = None
    counters_final: list = field(default_factory=list)
    result: Grid3 | None = None
    kernel_launches: int = 0

    def merge_pass(self, other: "RunStats") -> None:
        self.passes += other.passes
        self.block_updates += other.block_updates
        self.spin_iterations_total += other.spin_iterations_total
        if not self.per_thread_spins:
            self.per_thread_spins = [0] * len(other.per_thread_spins)
        for i, s in enumerate(other.per_thread_spins):
            self.per_thread_spins[i] += s
        self.pred_violations += other.pred_violations
        self.counters_final = other.counters_final
        self.kernel_launches += other.kernel_launches


def _default_live(axis_len):
    return lambda u: (0, axis_len)


def split_levels(h: int, max_fused: int = MAX_FUSED) -> list:
    """Balanced chunks of at most max_fused levels (e.g. 8 -> [4, 4], 5 -> [3, 2])."""
    n = -(-h // max_fused)
    base, extra = divmod(h, n)
    return [base + (1 if k < extra else 0) for k in range(n)]


class PipelineEngine:
    """Executes passes over one compressed grid or a two-grid pair on the GPU
    (sp/pipeline.py:230-519).  live_bounds(ax, u) -> (lo, hi) restricts level
    u to a logical range (distributed driver, sp/halo.py:278-289);
    physical_sides marks faces carrying a Dirichlet ring (compressed mode)."""

    max_fused = MAX_FUSED

    def __init__(self, cfg: PipelineConfig, grids, live_bounds=None, physical_sides=None):
        self.cfg = cfg
        if isinstance(grids, Grid3):
            grids = (grids,)
        self.grids = list(grids)
        if cfg.grid_mode == "two_grid":
            if len(self.grids) != 2:
                raise ValueError("two_grid mode needs a grid pair")
            if self.grids[0].shape != self.grids[1].shape:
                raise ValueError("grid pair shapes differ")
            if self.grids[0].data.shape != self.grids[1].data.shape:
                raise ValueError("grid pair storage extents differ")
        else:
            if len(self.grids) != 1:
                raise ValueError("compressed mode uses a single grid")
        g = self.grids[0]
        cfg.spec.validate(g)
        self.dims = g.shape
        if live_bounds is None:
            lives = [_default_live(n) for n in self.dims]
            self.live_bounds = lambda ax, u: lives[ax](u)
            self._default_live = True
        else:
            self.live_bounds = live_bounds
            self._default_live = False
        if physical_sides is None:
            physical_sides = {ax: (True, True) for ax in range(3)}
        self.physical_sides = physical_sides
        self.levels_done = 0
        self.passes_done = 0
        # (storage pointer, alignment) of the face ring the last fused
        # compressed pass wrote; trusted only while run_pipelined drives
        self._faces_frame = None
        self._faces_trusted = False
        self._rings_equal = None
        self._plans = None

    # -- API parity: block plans (sp/pipeline.py:257-266), built lazily ------
    @property
    def plan_fwd(self):
        if self._plans is None:
            self._plans = (decompose_blocks(self.grids[0], self.cfg.spec, 1),
                           decompose_blocks(self.grids[0], self.cfg.spec, -1))
        return self._plans[0]

    @property
    def plan_bwd(self):
        self.plan_fwd
        return self._plans[1]

    def _total_blocks(self) -> int:
        s = self.cfg.spec
        nx, ny, nz = self.dims
        return (-(-nx // s.bx)) * (-(-ny // s.by)) * (-(-nz // s.bz))

    def current_grid(self) -> Grid3:
        if self.cfg.grid_mode == "compressed":
            return self.grids[0]
        return self.grids[self.levels_done % 2]

    # -- helpers --------------------------------------------------------------
    def _lives(self, h):
        return {u: [tuple(self.live_bounds(ax, u)) for ax in range(3)] for u in range(1, h + 1)}

    def _fusable(self, lives, h) -> bool:
        """Fusing levels is exact when each level's live range is the previous
        level's range shrunk by at least one cell per side, or keeps touching
        the ring on that side: every live cell of the last level then depends
        only on live cells of the levels before it, which the fused kernels
        compute from the same level-0 data in the same order.  The kernels
        store z only inside the last level's live range but whole x/y rows, so
        an x/y side may shrink only where a neighbour owns it (the distributed
        live bounds of sp/halo.py:278-289): those cells are ghosts that the
        halo exchange overwrites.  Physical x/y sides must stay full."""
        dims = self.dims
        phys = self.physical_sides
        for u in range(1, h + 1):
            for ax in range(3):
                lo, hi = lives[u][ax]
                if ax < 2:
                    if phys[ax][0] and lo != 0:
                        return False
                    if phys[ax][1] and hi != dims[ax]:
                        return False
                if u >= 2:
                    plo, phi = lives[u - 1][ax]
                    if not ((lo - 1 >= plo) or (lo == 0 and plo == 0)):
                        return False
                    if not ((hi + 1 <= phi) or (hi == dims[ax] and phi == dims[ax])):
                        return False
        return True

    def _check_rings_equal(self) -> bool:
        if self._rings_equal is None:
            a, b = self.grids
            self._rings_equal = rings_equal(a, b)
        return self._rings_equal

    # -- passes ---------------------------------------------------------------
    def _pass_two_grid(self, direction, boundary=None):
        return _drive(self._pass_two_grid_steps(direction, boundary))

    def _pass_two_grid_steps(self, direction, boundary=None):
        """Generator form of the two-grid pass: with a fused peer boundary it
        yields once, right before the wait that precedes the boundary stores,
        so a driver can run every rank's first phase before any second phase
        (run_distributed_inprocess); the return value is the launch count."""
        cfg = self.cfg
        h = cfg.h
        lives = self._lives(h)
        L0 = self.levels_done
        if not (self._fusable(lives, h) and self._check_rings_equal()):
            if boundary is not None and getattr(boundary, "fused", False):
                raise ValueError("peer halo delivery needs fused two-grid passes")
            # exact per-level emulation: level lvl reads grids[(lvl-1)%2] and
            # writes grids[lvl%2] over its live range (sp/pipeline.py:301-323)
            for u in range(1, h + 1):
                lvl = L0 + u
                src, dst = self.grids[(lvl - 1) % 2], self.grids[lvl % 2]
                apply_window(src.data, dst.data, tuple(lives[u]), src.offset, src.offset)
            if boundary is not None:
                # the halo exchange is posted after the pass (run_pass contract)
                dst = self.grids[(L0 + h) % 2]
                boundary[2](dst.data, dst.offset)
            return h
        cur, other = self.grids[L0 % 2], self.grids[(L0 + 1) % 2]
        u0 = 0
        launches = 0
        chunks = split_levels(h, self.max_fused)
        peer = boundary is not None and getattr(boundary, "fused", False)
        if peer:
            boundary.begin()  # neighbours' previous pass delivered our ghost planes
        for n, c in enumerate(chunks):
            zlo, zhi = lives[u0 + c][2]
            last = n == len(chunks) - 1
            if last and peer:
                # fused peer delivery: the interior first, then the boundary
                # planes, stored locally and into the neighbours' ghost planes
                boundary.chunks_done()
                blo, bhi = boundary.blo, boundary.bhi
                if zhi - bhi > zlo + blo:
                    fused_sweeps(cur, other, c, zlo + blo, zhi - bhi)
                    launches += 1
                yield
                boundary.before_stores()
                if blo:
                    boundary.store(0, cur, other, c, zlo, zlo + blo)
                    launches += 1
                if bhi:
                    boundary.store(1, cur, other, c, zhi - bhi, zhi)
                    launches += 1
                boundary.end()
            elif last and boundary is not None and zhi - zlo > boundary[0] + boundary[1]:
                # boundary-first: the planes the halo exchange sends are
                # finished first, the exchange is posted, and the interior
                # planes are computed while the transfer is in flight
                blo, bhi, post = boundary
                if blo:
                    fused_sweeps(cur, other, c, zlo, zlo + blo)
                    launches += 1
                if bhi:
                    fused_sweeps(cur, other, c, zhi - bhi, zhi)
                    launches += 1
                post(other.data, other.offset)
                fused_sweeps(cur, other, c, zlo + blo, zhi - bhi)
                launches += 1
            else:
                fused_sweeps(cur, other, c, zlo, zhi)
                launches += 1
                if last and boundary is not None:
                    boundary[2](other.data, other.offset)
            cur, other = other, cur
            u0 += c
        target = self.grids[(L0 + h) % 2]
        if cur is not target:
            # rebind storage so grids[(L0+h)%2] holds the newest level
            a, b = self.grids
            a.data, b.data = b.data, a.data
            a.boundary_faces, b.boundary_faces = b.boundary_faces, a.boundary_faces
        return launches

    def _pass_compressed(self, direction):
        cfg = self.cfg
        h = cfg.h
        g = self.grids[0]
        a0 = g.alignment
        s = 1 if direction == 1 else -1
        mask = 0
        for n, (axis, side) in enumerate((("x", 0), ("x", 1), ("y", 0), ("y", 1), ("z", 0), ("z", 1))):
            if self.physical_sides["xyz".index(axis)][side]:
                mask |= 1 << n
        # _write_full_ring (sp/pipeline.py:427-447) at the pass's source frame.
        # Inside run_pipelined the previous fused pass already left the faces
        # at exactly this frame (no caller code runs in between), so the
        # rewrite would store the same values again.
        if not (self._faces_trusted and self._faces_frame == (g.data.data_ptr(), a0)):
            write_faces(g, g.origin - a0, mask)
        self._faces_frame = None
        lives = self._lives(h)
        if self._fusable(lives, h):
            # K3: fused in-place passes; each leaves the faces at its new frame
            u0, a = 0, a0
            launches = 1
            for c in split_levels(h, self.max_fused):
                zlo, zhi = lives[u0 + c][2]
                ws = self._workspace(c, zhi - zlo)
                compressed_pass(g, c, direction, a, ws, zlo, zhi, mask)
                launches += 2
                a += s * c
                u0 += c
            self._faces_frame = (g.data.data_ptr(), a)
            return launches
        sides = [(name, side) for ax, name in enumerate("xyz") for side in (0, 1)
                 if self.physical_sides[ax][side]]
        for u in range(1, h + 1):
            so = g.origin - (a0 + s * (u - 1))
            do = g.origin - (a0 + s * u)
            win = tuple(lives[u])
            apply_window(g.data, g.data, win, so, do)
            write_ring_strips(g.data, g.boundary_faces, win, do, sides, self.dims)
        return 2 * h + 1

    def _workspace(self, levels, depth):
        ws = getattr(self, "_ws", {})
        if (levels, depth) not in ws:
            ws[(levels, depth)] = compressed_workspace(self.grids[0], levels, depth)
            self._ws = ws
        return ws[(levels, depth)]

    def run_pass(self, direction: int, boundary=None) -> RunStats:
        """One team sweep: every interior cell receives h updates
        (sp/pipeline.py:451-519).  Stream-ordered: the kernels are enqueued on
        the current CUDA stream; results are visible to later stream work.

        `boundary` = (planes_low, planes_high, post): two-grid fused passes
        finish the lowest / highest z planes of the last level first and call
        post(storage, offset) before computing the rest (used by the z-slab
        driver to overlap the halo exchange with interior compute).  Without
        the fused path, post is called after the pass.  A FusedZHalo boundary
        (halo.py) instead stores the boundary planes into the neighbours'
        grids from the pass itself."""
        return _drive(self.run_pass_steps(direction, boundary))

    def run_pass_steps(self, direction: int, boundary=None):
        """Generator form of run_pass (see _pass_two_grid_steps)."""
        cfg = self.cfg
        if direction not in (1, -1):
            raise ValueError("direction must be +1 or -1")
        a0 = self.grids[0].alignment
        if cfg.grid_mode == "compressed":
            pad = self.grids[0].pad
            if direction == 1 and a0 + cfg.h > pad:
                raise ValueError(
                    f"forward pass needs alignment+h <= pad ({a0}+{cfg.h} > {pad})")
            if direction == -1 and a0 - cfg.h < 0:
                raise ValueError(
                    f"backward pass needs alignment >= h ({a0} < {cfg.h})")
            launches = self._pass_compressed(direction)
        else:
            launches = yield from self._pass_two_grid_steps(direction, boundary)
        self.levels_done += cfg.h
        self.passes_done += 1
        if cfg.grid_mode == "compressed":
            self.grids[0].alignment = a0 + (cfg.h if direction == 1 else -cfg.h)
        stats = RunStats(passes=1, kernel_launches=launches)
        stats.per_thread_spins = [0] * cfg.threads
        stats.block_updates = self._total_blocks() * cfg.threads
        return stats


def _drive(gen):
    """Run a pass generator to completion and return its value."""
    try:
        while True:
            next(gen)
    except StopIteration as stop:
        return stop.value


def team_sweep(grids, cfg: PipelineConfig, direction: int = 1) -> RunStats:
    """A single pass on a fresh engine (sp/pipeline.py:522-524)."""
    return PipelineEngine(cfg, grids).run_pass(direction)


def run_pipelined(grids, cfg: PipelineConfig, total_passes: int) -> RunStats:
    """Alternate forward/backward passes (sp/pipeline.py:527-548).  Compressed
    mode needs an even number of passes and pad >= h.  Synchronises the
    current stream at both ends so wall_seconds / mlups cover the GPU work;
    work on other streams (e.g. host transfers of the next input) keeps
    running."""
    engine = PipelineEngine(cfg, grids)
    engine._faces_trusted = True
    if cfg.grid_mode == "compressed":
        if total_passes % 2 != 0:
            raise ValueError("compressed mode needs an even number of passes")
        if engine.grids[0].pad < cfg.h:
            raise ValueError(
                f"compressed mode needs pad >= h ({engine.grids[0].pad} < {cfg.h})")
    stats = RunStats()
    stream = torch.cuda.current_stream()
    stream.synchronize()
    t0 = time.perf_counter()
    for p in range(total_passes):
        direction = 1 if p % 2 == 0 else -1
        stats.merge_pass(engine.run_pass(direction))
    stream.synchronize()
    stats.wall_seconds = time.perf_counter() - t0
    nx, ny, nz = engine.dims
    stats.updates_total = nx * ny * nz * cfg.h * total_passes
    stats.mlups = stats.updates_total / max(stats.wall_seconds, 1e-12) / 1e6
    stats.result = engine.current_grid()
    return stats
