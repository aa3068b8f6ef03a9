"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box):

    python tests/golden/make_golden.py            # small cases (seconds)
    python tests/golden/make_golden.py --big      # + BASELINE configs C1..C4 (minutes, ~20 GB RAM)

Every digest is SHA-256 of the interior in (z, y, x) storage order as
little-endian f8 — the convention of Grid3.checksum (sp/grid.py:115-120) and
pkg/tests/test_kernel.py:71-75.  The file records, for each case, how it was
produced so the GPU tests can rebuild the identical input on the device.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def _digest(iv) -> str:
    h = hashlib.sha256()
    for k in range(iv.shape[0]):
        h.update(np.ascontiguousarray(iv[k]).astype("<f8").tobytes())
    return h.hexdigest()


def _ref():
    sys.path.insert(0, REF)
    import stencilpipe  # noqa: F401  (read-only import of the reference)
    return stencilpipe


def make_input(sp, nx, ny, nz, seed, pad=0, init="random", value=0.0, ring=None,
               lo=0.0, hi=1.0):
    """Build a reference Grid3 for one case (SURVEY.md §8a a3 recipe)."""
    g = sp.create_grid(nx, ny, nz, pad=pad, init=init, value=value, seed=seed)
    if (lo, hi) != (0.0, 1.0):
        iv = g.interior_view()
        iv[...] = lo + (hi - lo) * iv
    if ring is not None:
        o = g.origin - g.alignment
        d = g.data
        zl, zh, yl, yh, xl, xh = o - 1, o + nz, o - 1, o + ny, o - 1, o + nx
        d[zl, yl:yh + 1, xl:xh + 1] = ring
        d[zh, yl:yh + 1, xl:xh + 1] = ring
        d[zl:zh + 1, yl, xl:xh + 1] = ring
        d[zl:zh + 1, yh, xl:xh + 1] = ring
        d[zl:zh + 1, yl:yh + 1, xl] = ring
        d[zl:zh + 1, yl:yh + 1, xh] = ring
    g.capture_boundary_faces()
    return g


def ref_sweeps(sp, g0, count):
    a, b = g0.copy(), g0.copy()
    for _ in range(count):
        sp.reference_sweep(a, b)
        a, b = b, a
    return a


# (name, nx, ny, nz, seed, pad, init, value, ring, lo, hi, sweeps)
SWEEP_CASES = [
    ("cube7_s4", 7, 7, 7, 4, 0, "random", 0.0, None, 0.0, 1.0, 3),
    ("odd5x4x3_s11", 5, 4, 3, 11, 0, "random", 0.0, None, 0.0, 1.0, 5),
    ("tiny1x1x1", 1, 1, 1, 3, 0, "random", 0.0, None, 0.0, 1.0, 2),
    ("thin1x9x4", 1, 9, 4, 5, 0, "random", 0.0, 0.5, 0.0, 1.0, 3),
    ("rect13x9x6_s2", 13, 9, 6, 2, 0, "random", 0.0, None, 0.0, 1.0, 4),
    ("rect33x17x9_s7", 33, 17, 9, 7, 0, "random", 0.0, 1.0, 0.0, 1.0, 2),
    ("cube24_s42", 24, 24, 24, 42, 0, "random", 0.0, None, 0.0, 1.0, 8),
    ("cube16_s21", 16, 16, 16, 21, 0, "random", 0.0, None, 0.0, 1.0, 8),
    ("cube20_s13", 20, 20, 20, 13, 0, "random", 0.0, None, 0.0, 1.0, 16),
    ("pad2_12x10x8_s3", 12, 10, 8, 3, 2, "random", 0.0, None, 0.0, 1.0, 3),
    ("ring1_30x26x22_s9", 30, 26, 22, 9, 0, "random", 0.0, 1.0, 0.0, 1.0, 6),
    ("sym_37x35x41_s6", 37, 35, 41, 6, 1, "random", 0.0, 0.25, -1.0, 1.0, 9),
    ("wide130x70x20_s8", 130, 70, 20, 8, 0, "random", 0.0, 1.0, 0.0, 1.0, 12),
    ("impulse4", 4, 4, 4, 0, 0, "impulse", 0.0, None, 0.0, 1.0, 1),
    ("impulse9", 9, 9, 9, 0, 0, "impulse", 0.0, None, 0.0, 1.0, 4),
    ("const6", 6, 6, 6, 0, 0, "constant", 1.0, None, 0.0, 1.0, 3),
    ("cube60_s42", 60, 60, 60, 42, 0, "random", 0.0, None, 0.0, 1.0, 8),
    ("cube64_s1_ring1", 64, 64, 64, 1, 0, "random", 0.0, 1.0, 0.0, 1.0, 24),
]

# pipelined cases: (name, n, seed, mode, n_, t, T, d_u, sync, passes, spec)
PIPE_CASES = [
    ("pipe_degenerate", 24, 42, "two_grid", 1, 1, 1, 3, "relaxed", 4, (24, 8, 8)),
    ("pipe_t3", 60, 42, "two_grid", 1, 3, 1, 3, "relaxed", 1, (60, 20, 20)),
    ("pipe_compressed_h16", 24, 42, "compressed", 2, 4, 2, 3, "relaxed", 2, (24, 8, 8)),
    ("pipe_lockstep", 24, 42, "two_grid", 1, 4, 1, 1, "relaxed", 2, (24, 8, 8)),
    ("pipe_shape_h8", 20, 13, "compressed", 1, 8, 1, 3, "relaxed", 2, (20, 5, 5)),
    ("pipe_t2_two_grid", 60, 42, "two_grid", 1, 2, 1, 3, "barrier", 2, (60, 20, 20)),
    ("pipe_t4_compressed", 60, 42, "compressed", 1, 4, 1, 3, "relaxed", 2, (60, 20, 20)),
    ("pipe_t3_compressed", 33, 5, "compressed", 1, 3, 1, 3, "relaxed", 4, (33, 11, 11)),
    ("pipe_t8_two_grid", 40, 2, "two_grid", 1, 8, 1, 3, "relaxed", 3, (40, 10, 10)),
]

# distributed z-slab cases (1,1,P) plus one general topology for the host logic
DIST_CASES = [
    ("dist_z2_h2_two", (1, 1, 2), (40, 40, 40), 2, "two_grid", 2),
    ("dist_z2_h4_comp", (1, 1, 2), (40, 40, 40), 4, "compressed", 2),
    ("dist_z4_h4_two", (1, 1, 4), (24, 24, 64), 4, "two_grid", 3),
    ("dist_z3_h2_two", (1, 1, 3), (18, 20, 36), 2, "two_grid", 3),
    ("dist_z2_h1_two", (1, 1, 2), (20, 20, 20), 1, "two_grid", 4),
]


def small(sp, out):
    g = sp.create_grid(60, 60, 60, init="random", seed=42)
    out["pins"] = {
        # frozen by the reference's own tests
        "FIELD_60_SEED42": "fa5b509457fd250fd0d2ee349ead4cba2ee3e0371553af4166dc21d1d8690112",
        "FIELD_600_SEED42": "b283cb61c807d14afd4610377cdbd48706393fad39dfa3b9827629cb4c5ac88c",
        "REF_60_SEED42_8SWEEPS": "5f3b56d7c9c1dd077ed2bdbd74898718695a950104ceb329990231fe103d6d15",
    }
    assert g.checksum() == out["pins"]["FIELD_60_SEED42"]
    cases = {}
    for (name, nx, ny, nz, seed, pad, init, value, ring, lo, hi, sw) in SWEEP_CASES:
        g0 = make_input(sp, nx, ny, nz, seed, pad, init, value, ring, lo, hi)
        res = ref_sweeps(sp, g0, sw)
        per = {}
        a, b = g0.copy(), g0.copy()
        for s in range(1, sw + 1):
            sp.reference_sweep(a, b)
            a, b = b, a
            per[s] = _digest(a.interior_view())
        assert per[sw] == _digest(res.interior_view())
        cases[name] = dict(nx=nx, ny=ny, nz=nz, seed=seed, pad=pad, init=init, value=value,
                           ring=ring, lo=lo, hi=hi, sweeps=sw,
                           init_digest=_digest(g0.interior_view()),
                           digests={str(k): v for k, v in per.items()})
    assert cases["cube60_s42"]["digests"]["8"] == out["pins"]["REF_60_SEED42_8SWEEPS"]
    out["sweeps"] = cases

    pipes = {}
    for (name, n, seed, mode, n_, t, T, d_u, sync, passes, spec) in PIPE_CASES:
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(*spec), n=n_, t=t, T=T, d_l=1, d_u=d_u,
                                sync_mode=sync, grid_mode=mode)
        if mode == "compressed":
            g = sp.create_grid(n, n, n, pad=cfg.h, init="random", seed=seed)
            st = sp.run_pipelined(g, cfg, passes)
            assert st.result.alignment == 0
        else:
            a = sp.create_grid(n, n, n, init="random", seed=seed)
            st = sp.run_pipelined((a, a.copy()), cfg, passes)
        total = cfg.h * passes
        d = _digest(st.result.interior_view())
        assert d == _digest(ref_sweeps(sp, sp.create_grid(n, n, n, init="random", seed=seed),
                                       total).interior_view())
        pipes[name] = dict(n=n, seed=seed, mode=mode, nteams=n_, t=t, T=T, d_u=d_u,
                           sync=sync, passes=passes, spec=list(spec), h=cfg.h,
                           sweeps=total, digest=d)
    out["pipelined"] = pipes

    dists = {}
    from stencilpipe.halo import DistConfig, RankTopology, assemble_global, run_distributed_inprocess
    for (name, topo, gd, h, mode, cycles) in DIST_CASES:
        t, T = (h, 1)
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(gd[0], 10, 10), n=1, t=t, T=T,
                                grid_mode=mode)
        dist = DistConfig(topo=RankTopology(*topo), cfg=cfg, cycles=cycles, global_dims=gd,
                          mode="strong", seed=42)
        rts = run_distributed_inprocess(dist)
        asm = assemble_global(rts)
        d = _digest(asm.interior_view())
        ref = ref_sweeps(sp, sp.create_grid(*gd, init="random", seed=42), h * cycles)
        assert d == _digest(ref.interior_view())
        dists[name] = dict(topo=list(topo), global_dims=list(gd), h=h, mode=mode,
                           cycles=cycles, seed=42, sweeps=h * cycles, digest=d)
    out["distributed"] = dists


def big(sp, out, which):
    """BASELINE configs.  C2/C4 sweeps run through the
    reference's own multi-threaded run_pipelined (bitwise equal to the plain
    sweep by the reference's contract)."""
    cfgs = out.setdefault("configs", {})

    def pipelined(g, t, passes, mode, nx, bx=32):
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(nx, bx, bx), n=1, t=t, T=1, d_l=1, d_u=3,
                                grid_mode=mode)
        if mode == "compressed":
            return sp.run_pipelined(g, cfg, passes)
        return sp.run_pipelined((g, g.copy()), cfg, passes)

    if "C1" in which:
        t0 = time.time()
        g = make_input(sp, 128, 128, 128, 42, ring=1.0)
        init = _digest(g.interior_view())
        res = ref_sweeps(sp, g, 10)
        cfgs["C1"] = dict(n=[128, 128, 128], seed=42, ring=1.0, lo=0.0, hi=1.0, pad=0,
                          sweeps=10, init_digest=init, digest=_digest(res.interior_view()),
                          how="reference_sweep x10")
        print("C1", time.time() - t0, flush=True)
    if "C2" in which:
        t0 = time.time()
        g = make_input(sp, 512, 512, 512, 42, ring=0.0)
        init = _digest(g.interior_view())
        st = pipelined(g, 4, 25, "two_grid", 512)
        cfgs["C2"] = dict(n=[512, 512, 512], seed=42, ring=0.0, lo=0.0, hi=1.0, pad=0,
                          sweeps=100, init_digest=init, digest=_digest(st.result.interior_view()),
                          how="run_pipelined two_grid t=4 x25 passes")
        print("C2", time.time() - t0, flush=True)
        del g, st
    if "C3" in which:
        t0 = time.time()
        g = make_input(sp, 600, 600, 600, 42, pad=4, ring=0.0, lo=-1.0, hi=1.0)
        init = _digest(g.interior_view())
        st = pipelined(g, 4, 16, "compressed", 600, bx=30)
        assert st.result.alignment == 0
        cfgs["C3"] = dict(n=[600, 600, 600], seed=42, ring=0.0, lo=-1.0, hi=1.0, pad=4,
                          sweeps=64, init_digest=init, digest=_digest(st.result.interior_view()),
                          how="run_pipelined compressed t=4 x16 passes")
        print("C3", time.time() - t0, flush=True)
        del g, st
    if "C4" in which:
        t0 = time.time()
        g = make_input(sp, 1024, 1024, 1024, 42, ring=1.0)
        init = _digest(g.interior_view())
        st = pipelined(g, 8, 5, "two_grid", 1024)
        cfgs["C4_P1"] = dict(n=[1024, 1024, 1024], seed=42, ring=1.0, lo=0.0, hi=1.0, pad=0,
                             sweeps=40, init_digest=init,
                             digest=_digest(st.result.interior_view()),
                             how="run_pipelined two_grid t=8 x5 passes")
        print("C4", time.time() - t0, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", default="", help="comma list of C1,C2,C3,C4")
    ap.add_argument("--skip-small", action="store_true")
    args = ap.parse_args()
    sp = _ref()
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out = json.load(f)
    out["_generator"] = ("tests/golden/make_golden.py: reference stencilpipe "
                         "imported read-only from /root/reference/pkg/src")
    if not args.skip_small:
        small(sp, out)
    if args.big:
        big(sp, out, set(args.big.split(",")))
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
