"""Benchmark of the B200 FP64 7-point Jacobi hot path (BASELINE.json metric).

Workloads (BASELINE.json configs, seeded synthetic grids, seed 42):
  N=1   configs[1] "C2": 512^3 interior in 514^3 storage, two grids (2.2 GB),
        U[0,1), ring 0.0, 100 sweeps.  One step = the 100-sweep solve.
  N>1   configs[3] "C4" weak scaling (torchrun, one process per GPU): a
        1024^3 interior per GPU as z-slabs of a 1024 x 1024 x 1024N grid,
        U[0,1), ring 1.0, t=4 with 4-deep ghost planes exchanged over NCCL
        once per fused pass, 40 sweeps.  One step = the 40-sweep solve.
        Extra leg: configs[4] "C5" strong scaling, 2048^3 global over the N
        GPUs, t in {1, 4, 8}, 32 sweeps.  (`--slab` runs C4 at N=1 through the
        same distributed driver.)

Metric: GLUP/s = interior cells x sweeps / time (the reference's LUP
accounting, sp/pipeline.py:545; owned cells only in distributed runs,
sp/halo.py:388-392).  Inputs (2.2 GB / 17 GB per GPU) are larger than L2
(126 MB), so no explicit flush is needed between steps.

--impl reference: the reference CPU path (the oracle's C port of
reference_sweep, all host threads) on the same workload config; at N=1 each
step is the whole 100-sweep C2 solve, for N>1 a bounded sample (stated in
cpu_baseline.sample).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GLUP/s FP64 3D 7-pt Jacobi at 1/2/4/8 B200; % of HBM roofline (B/LUP)"
UNIT = "GLUP/s"
SEED = 42
# BASELINE configs[1] (C2) and configs[3] (C4, per GPU), configs[4] (C5, global)
C2 = dict(n=(512, 512, 512), sweeps=100, ring=0.0)
C4 = dict(n=(1024, 1024, 1024), sweeps=40, ring=1.0, t=4)
C5 = dict(n=(2048, 2048, 2048), sweeps=32, ring=0.0, ts=(1, 4, 8))


def workload(ws: int, slab: bool) -> dict:
    """The workload both arms report in `config` (identical dicts)."""
    if not slab:
        return {"workload": "C2: 512^3 FP64 7-pt Jacobi, two grids (2.2 GB), U[0,1) seed 42, "
                            "ring 0.0, 100 sweeps",
                "grid": list(C2["n"]), "sweeps_per_step": C2["sweeps"], "parallelism": "single GPU",
                "l2_flush": "not needed: 2.2 GB working set > 126 MB L2"}
    nx, ny, nz = C4["n"]
    return {"workload": (f"C4 weak scaling: {nx}^3 interior per GPU, z-slabs of {nx}x{ny}x{nz * ws}, "
                         f"U[0,1) seed 42, ring 1.0, t=4, 4-deep ghosts, 40 sweeps"),
            "grid": [nx, ny, nz * ws], "sweeps_per_step": C4["sweeps"],
            "parallelism": f"z-slab x{ws}",
            "l2_flush": "not needed: 17 GB per GPU working set > 126 MB L2"}


def host_threads() -> int:
    """Host threads this process may run on (the CPU baselines use all)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_info() -> dict:
    """Host CPU facts for the cpu_baseline."""
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "sched_getaffinity": aff}


# ---------------------------------------------------------------------------
# clocks sampler (NVML thread during the timed region; nvidia-smi as the fallback)
# ---------------------------------------------------------------------------

class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        # NVML in a thread (20 ms period, no process start-up inside a
        # sub-second timed region); nvidia-smi -lms 100 as the fallback
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            rows, stop = [], threading.Event()

            def sample():
                while not stop.is_set():
                    try:
                        rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                     pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM),
                                     pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:
                        pass
                    stop.wait(0.02)

            th = threading.Thread(target=sample, daemon=True)
            th.start()
            self.nvml = (pynvml, rows, stop, th)
            return
        except Exception:
            self.nvml = None
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.nvml is not None:
            pynvml, rows, stop, th = self.nvml
            stop.set()
            th.join(timeout=2)
            try:
                pynvml.nvmlShutdown()
            except Exception:
                pass
            if not rows:
                return None
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted({n for n, b in bits.items() for r in rows if r[2] & b})
            return {"sm_mhz": statistics.median(r[0] for r in rows),
                    "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                    "samples": len(rows), "source": "nvml, 20 ms"}
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, name in enumerate(names):
                if r[5 + k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle's C port of reference_sweep, and
# the oracle's NumPy restatement of the reference's own ufunc sequence
# ---------------------------------------------------------------------------

def _cpu_child(target_s: float, n, max_sweeps: int, numpy_sweeps: int) -> int:
    """Child of cpu_rate: time the reference CPU path on an n-grid in a
    process without torch or a CUDA context; print one JSON line.
      port:  the oracle's C restatement of reference_sweep (sp/kernel.py:99-111),
             OpenMP over z on every host thread, for ~target_s seconds;
      numpy: the oracle's NumPy restatement (the reference's own ufunc order,
             sp/kernel.py:51-58), single-threaded, `numpy_sweeps` sweeps."""
    import numpy as np
    import oracle
    d = oracle.make_storage(*n, init="random", seed=SEED)
    a, b = d, d.copy()
    threads = oracle.lib().or_max_threads()
    oracle.c_sweeps(a, b, n, 1, threads=threads)  # first touch, thread pool
    a, b = b, a
    done = 0
    t0 = time.perf_counter()
    while done < max_sweeps:
        oracle.c_sweeps(a, b, n, 1, threads=threads)
        a, b = b, a
        done += 1
        if time.perf_counter() - t0 >= target_s:
            break
    dt = time.perf_counter() - t0
    out = {"rate": n[0] * n[1] * n[2] * done / dt / 1e9, "threads": threads, "done": done, "dt": dt}
    if numpy_sweeps > 0:
        off = 1
        t1 = time.perf_counter()
        for _ in range(numpy_sweeps):
            oracle.reference_sweep(a, b, *n, off)
            a, b = b, a
        dtn = time.perf_counter() - t1
        out["numpy"] = {"rate": n[0] * n[1] * n[2] * numpy_sweeps / dtn / 1e9, "sweeps": numpy_sweeps,
                        "dt": dtn}
        # the reference's pipelined temporal blocking (run_pipelined with n=1,
        # t=4, T=1, d_l=1, d_u=3, block (nx, 32, 32), relaxed sync): t threads
        # running NumPy windows, one pass of 4 sweeps (oracle/pipelined.py)
        from oracle.pipelined import pipelined_pass_two_grid
        grids = [a, b]
        t2 = time.perf_counter()
        pipelined_pass_two_grid(grids, n, 4, (n[0], 32, 32))
        dtp = time.perf_counter() - t2
        out["pipelined"] = {"rate": n[0] * n[1] * n[2] * 4 / dtp / 1e9, "threads": 4, "dt": dtp}
    print(json.dumps(out))
    return 0


def cpu_rate(n, target_s: float = 12.0, max_sweeps: int = 100, numpy_sweeps: int = 2):
    """Time the reference CPU path in a separate process (the bench process
    holds torch's thread pool, a CUDA context and the clock sampler; inside it
    the OpenMP sweep measured about half its rate).  Returns the cpu_baseline
    dict."""
    # every host core (torchrun exports OMP_NUM_THREADS=1 to each rank)
    env = dict(os.environ, OMP_NUM_THREADS=str(host_threads()))
    # NumPy leg on one core: no BLAS threads (element-wise ufuncs are single-threaded anyway)
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-child", str(target_s),
                          "--cpu-n", ",".join(map(str, n)), "--cpu-numpy-sweeps", str(numpy_sweeps)],
                         capture_output=True, text=True, check=True, env=env).stdout
    r = json.loads(out.strip().splitlines()[-1])
    g = "x".join(map(str, n))
    sample = (f"{r['done']} reference sweeps of a {g} grid (oracle C port of reference_sweep, "
              f"sp/kernel.py:99-111, OpenMP over z, {r['threads']} threads) in {r['dt']:.1f} s, "
              f"separate process")
    cb = {"value": r["rate"], "unit": UNIT, "cores": r["threads"], "kind": "port", "sample": sample,
          "host": host_info()}
    if "numpy" in r:
        cb["numpy_reference_sweep_1core"] = {
            "value": r["numpy"]["rate"], "unit": UNIT, "cores": 1,
            "sample": (f"{r['numpy']['sweeps']} sweeps of the {g} grid through the oracle's NumPy "
                       f"restatement of reference_sweep (the reference's ufunc sequence, "
                       f"sp/kernel.py:51-58) in {r['numpy']['dt']:.1f} s")}
    if "pipelined" in r:
        cb["numpy_run_pipelined_t4"] = {
            "value": r["pipelined"]["rate"], "unit": UNIT, "cores": r["pipelined"]["threads"],
            "sample": (f"one pass of 4 sweeps of the {g} grid through the oracle's threaded NumPy "
                       f"restatement of the reference's pipelined temporal blocking (run_pipelined with "
                       f"n=1, t=4, T=1, d_l=1, d_u=3, block ({n[0]},32,32), relaxed sync; "
                       f"sp/pipeline.py:363-395, 527-548) in {r['pipelined']['dt']:.1f} s")}
    return cb


def run_reference_arm(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    slab = ws > 1 or args.slab
    cfg = workload(ws, slab)
    if slab:
        # bounded sample: one rank's 1024^3 slab (ring 1.0), a few sweeps per step
        n = C4["n"]
        sps = args.ref_sweeps_per_step or 2
        d = oracle.make_storage(*n, init="random", seed=SEED, ring=C4["ring"])
        what = (f"{sps} reference sweeps per step of one rank's {n[0]}^3 C4 slab (ring 1.0); "
                f"a CPU sweep's rate does not depend on the sweep count or the rank")
    else:
        n = C2["n"]
        sps = args.ref_sweeps_per_step or C2["sweeps"]
        d = oracle.make_storage(*n, init="random", seed=SEED)
        what = f"{sps} reference sweeps of the 512^3 C2 grid per step" + (
            " (the whole C2 solve)" if sps == C2["sweeps"] else "")
    a, b = d, d.copy()
    threads = host_threads()  # all of them, whatever OMP_NUM_THREADS torchrun set
    for _ in range(args.warmup):
        oracle.c_sweeps(a, b, n, sps, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.c_sweeps(a, b, n, sps, threads=threads)
    dt = time.perf_counter() - t0
    value = n[0] * n[1] * n[2] * sps * args.steps / dt / 1e9
    sample = (f"{what} (oracle C port of reference_sweep, sp/kernel.py:99-111; OpenMP over z, "
              f"{threads} threads); the reference itself is pure Python/NumPy and does not "
              f"travel to the GPU box, so this is its restatement ('port')")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, seed 42)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def plan_depths(total: int, t: int):
    """Fused-pass depths summing to `total` with passes of at most t."""
    n = -(-total // t)
    base, extra = divmod(total, n)
    return [base + (1 if k < extra else 0) for k in range(n)]


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class LaunchTimer:
    """CUDA events around every fused launch on the launching stream."""

    def __init__(self):
        import torch
        self.torch = torch
        self.ev = []

    def start(self, depth):
        s = self.torch.cuda.Event(enable_timing=True)
        s.record()
        self.ev.append([depth, s, None])

    def stop(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev[-1][2] = e

    def stats(self):
        ms = [s.elapsed_time(e) for _, s, e in self.ev]
        return ms, [d for d, _, _ in self.ev]


def _pin(t):
    """Pinned host copy target; pageable if the host cannot pin that much."""
    try:
        return t.pin_memory(), True
    except RuntimeError:
        return t, False


def e2e_pipelined(units, host_in, host_out, steps, warmup, all_ranks_max):
    """Steps through the public API with host buffers: every step copies its
    input from pinned host memory (H2D stream), solves (compute stream) and
    copies the result back to pinned host memory (D2H stream).  Steps are
    pipelined over len(units) device solve units, as a serving loop would
    run them: the H2D of step i+1 and the D2H of step i-1 overlap step i.
    unit.load(host) / unit.solve() / unit.result() -> device tensor."""
    import torch
    NP = len(units)
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def run(count, e0=None, e1=None):
        loaded, freed = [None] * (count + 1), [None] * NP

        def h2d(i):
            with torch.cuda.stream(s_h2d):
                if freed[i % NP] is not None:
                    s_h2d.wait_event(freed[i % NP])
                units[i % NP].load(host_in)
                ev = torch.cuda.Event()
                ev.record(s_h2d)
                loaded[i] = ev

        if e0 is not None:
            e0.record(s_h2d)
        h2d(0)
        for i in range(count):
            if i + 1 < count:
                h2d(i + 1)
            u = units[i % NP]
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(loaded[i])
                u.solve()
                done = torch.cuda.Event()
                done.record(s_cmp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(done)
                host_out.copy_(u.result(), non_blocking=True)
                fr = torch.cuda.Event()
                fr.record(s_d2h)
                freed[i % NP] = fr
        if e1 is not None:
            e1.record(s_d2h)
        torch.cuda.synchronize()

    run(max(1, warmup))
    all_ranks_max(None)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    run(steps, e0, e1)
    return all_ranks_max(e0.elapsed_time(e1)) / steps


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1006_3148_b200 as sp
    from paper_1006_3148_b200 import _lib

    ws, rank, local = _dist()
    if args.dist_backend == "gloo":
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    slab = ws > 1 or args.slab
    if slab:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # path check only: several ranks on one GPU, halos staged through host memory
            dist.init_process_group("gloo")
    L = _lib.load()
    peak, peak_src = _peaks()

    def barrier_sync():
        if slab:
            dist.barrier()
        torch.cuda.synchronize()

    def all_max(ms):
        """Barrier + max over ranks of a device-timed interval (None: barrier only)."""
        torch.cuda.synchronize()
        if not slab:
            return ms
        t = torch.tensor([0.0 if ms is None else ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg_line = workload(ws, slab)
    # --- the solve of this rank ------------------------------------------------
    if slab:
        from paper_1006_3148_b200 import halo
        solver = halo.SlabSolver.weak(per_rank=C4["n"], seed=SEED, ring=C4["ring"], depth=args.t,
                                      transport=args.transport)
        sweeps = C4["sweeps"]
        cells_rank = solver.owned_cells
        passes_per_step = sweeps // solver.dist_cfg.cfg.h

        def step(timer=None):
            solver.run_sweeps(sweeps)

        grid_bytes = solver.storage_bytes()
    else:
        g0 = sp.create_grid(*C2["n"], init="random", seed=SEED)
        a, b = g0, g0.copy()
        sweeps = C2["sweeps"]
        cells_rank = C2["n"][0] * C2["n"][1] * C2["n"][2]
        grid_bytes = a.data.numel() * 8
        depths = plan_depths(sweeps, args.t)
        passes_per_step = len(depths)
        bufs = [a, b]

        def step(timer=None):
            cur = 0
            for c in depths:
                if timer is not None:
                    timer.start(c)
                sp.fused_sweeps(bufs[cur], bufs[1 - cur], c)
                if timer is not None:
                    timer.stop()
                cur = 1 - cur

    # --- warmup + timed region ------------------------------------------------
    for _ in range(args.warmup):
        step()
    clocks = Clocks(local)
    barrier_sync()
    clocks.start()
    L.sp_launch_count(1)
    timer = LaunchTimer()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier_sync()
    ev0.record()
    for _ in range(args.steps):
        step(None if slab else timer)
    ev1.record()
    barrier_sync()
    launches = int(L.sp_launch_count(0))
    clk = clocks.stop()
    elapsed_ms = all_max(ev0.elapsed_time(ev1))
    value = cells_rank * sweeps * ws * args.steps / (elapsed_ms / 1e3) / 1e9

    # roofline of the dominant kernel: one fused pass = one read + one write
    # of every cell it owns (16 B/LUP / depth x depth levels)
    if slab:
        # the slab pass (boundary launches + interior launch + NCCL exchange)
        # is timed as a whole: a conservative launch time
        avg_ms = elapsed_ms / args.steps / passes_per_step
        dom_depth = args.t
        alg_bytes = 16.0 * cells_rank
    else:
        ms, ds = timer.stats()
        dom_depth = max(set(ds), key=ds.count) if ds else args.t
        dom = [m for m, d in zip(ms, ds) if d == dom_depth]
        avg_ms = (sum(dom) / len(dom)) if dom else elapsed_ms / args.steps / passes_per_step
        alg_bytes = 16.0 * cells_rank
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pt = json.load(f)
            key = f"k_temporal_T{dom_depth}" + ("_C4" if slab else "")
            traffic = pt.get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    extra = {}
    # The fused pass is not HBM-bound: report the FP64 pipe it runs against.
    # Peak = 64 FP64 lanes/clk/SM x SMs x max SM clock; "useful" counts 6
    # flops per LUP, "executed" adds the overlapped-tile recompute.
    props = torch.cuda.get_device_properties(local)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:
        mhz = 1965.0
    fp64_peak = 64 * props.multi_processor_count * mhz * 1e6 / 1e12
    nn = C4["n"][0] if slab else C2["n"][0]
    if dom_depth > 1:
        cy = {2: 48, 3: 36, 4: 32}.get(dom_depth, 32)
        ox, oy = 64 - 2 * (dom_depth - 1), cy - 2 * (dom_depth - 1)
        redundancy = (-(-nn // ox) * 64) * (-(-nn // oy) * cy) / nn ** 2
    else:
        redundancy = 1.0
    useful = value / ws * 6 / 1e3
    extra["compute_roofline"] = {
        "bound": "issue latency + LSU data pipe (not HBM, not FP64)", "fp64_unit": "TFLOP/s (per GPU)",
        "fp64_peak": fp64_peak, "fp64_achieved_useful": useful, "fp64_frac_useful": useful / fp64_peak,
        "executed_lup_per_lup": redundancy, "fp64_frac_executed": useful * redundancy / fp64_peak,
        "note": ("6 DADD/DMUL per LUP, no FMA (bit-exact order). ncu K2 T=4 (profiles/r02_ncu_k2_t4.txt): "
                 "LSU data pipe 68.5 % of peak (shared LD 64 M + ST 21 M + SHFL 37 M wavefronts per pass; "
                 "SHFL.32 and LDS share that pipe at 1 wavefront per clock per SM, profiles/r02_mio_bench.txt), "
                 "FP64 pipe 38 %, issue 40 % at 8 warps/SM (254 registers); top stalls: fixed-latency "
                 "dependency 1.17, short scoreboard 0.80, barrier 0.53 per issue")}

    if rank == 0 and not slab and not args.quick:
        extra.update(_single_gpu_legs(sp, torch, bufs, peak, args))

    if slab and not args.quick:
        del solver
        torch.cuda.empty_cache()
        extra["C5_strong"] = _c5_strong(sp, torch, dist, ws, all_max)

    # --- e2e through the public API with host buffers --------------------------
    e2e = None
    if not args.quick:
        e2e = _e2e(sp, torch, dist, ws, slab, args, all_max, grid_bytes)

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_rate(C4["n"] if slab else C2["n"], args.cpu_seconds,
                       numpy_sweeps=0 if slab else 2)

    if slab:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (seeded SplitMix64 U[0,1), seed 42; ring 1.0)" if slab else
                     "synthetic (seeded SplitMix64 U[0,1), seed 42; ring 0.0)"),
            "config": cfg_line,
            "impl_config": {"fused_depth": args.t, "halo_transport": args.transport if slab else None,
                            "kernel": f"k_temporal<T={dom_depth}>"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"k_temporal<T={dom_depth}> (per fused pass)"
                                   + (" incl. boundary launches and the NCCL exchange" if slab else ""),
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_ms,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        if slab:
            line["per_gpu_glups"] = value / ws
        line.update(extra)
        print(json.dumps(line), flush=True)
    if slab:
        dist.destroy_process_group()
    return 0


def _single_gpu_legs(sp, torch, bufs, peak, args):
    """N=1 extras: per-depth GLUP/s on C2, C3 compressed, C4 and C5 on one GPU."""
    extra = {}
    n3 = C2["n"][0] ** 3
    per = {}
    for t in (1, 2, 3, 4):
        d_t = plan_depths(C2["sweeps"], t)
        cur = 0
        for rep in range(2):
            for c in d_t:
                sp.fused_sweeps(bufs[cur], bufs[1 - cur], c)
                cur = 1 - cur
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for rep in range(3):
            for c in d_t:
                sp.fused_sweeps(bufs[cur], bufs[1 - cur], c)
                cur = 1 - cur
        e1.record()
        torch.cuda.synchronize()
        ms_t = e0.elapsed_time(e1) / 3
        glups = n3 * C2["sweeps"] / (ms_t / 1e3) / 1e9
        per[str(t)] = {"glups": glups, "ms_per_solve": ms_t, "hbm_roofline_glups": peak / (16.0 / t),
                       "frac_of_hbm_roofline": glups * (16.0 / t) / peak}
    # t=8 as BASELINE configs[1] states it: passes of 8 sweeps (12 x 8 + 1 x 4),
    # each pass two fused launches of 4 (SP_MAX_FUSED), the same kernels as t=4
    d8 = [c for h in ([8] * 12 + [4]) for c in sp.split_levels(h, sp.MAX_FUSED)]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    cur = 0
    torch.cuda.synchronize()
    e0.record()
    for rep in range(3):
        for c in d8:
            sp.fused_sweeps(bufs[cur], bufs[1 - cur], c)
            cur = 1 - cur
    e1.record()
    torch.cuda.synchronize()
    ms_t = e0.elapsed_time(e1) / 3
    glups = n3 * C2["sweeps"] / (ms_t / 1e3) / 1e9
    per["8"] = {"glups": glups, "ms_per_solve": ms_t, "hbm_roofline_glups": peak / 2.0,
                "frac_of_hbm_roofline": glups * 2.0 / peak,
                "note": "passes of 8 sweeps run as two fused launches of 4 (DESIGN.md §8: no depth-8 kernel)"}
    extra["per_depth"] = per
    extra["plain_sweep_glups"] = per["1"]["glups"]
    extra["fused_vs_plain"] = per[str(args.t)]["glups"] / per["1"]["glups"]
    # C3: compressed single-array grid, 600^3 (pad 4), U[-1,1), 64 sweeps at
    # t=4 through run_pipelined (K3 in-place passes), one timed solve
    g3 = sp.create_grid(600, 600, 600, pad=4, init="random", seed=SEED, lo=-1.0, hi=1.0)
    cfg3 = sp.PipelineConfig(spec=sp.BlockSpec(600, 30, 30), t=4, grid_mode="compressed")
    sp.run_pipelined(g3, cfg3, 2)  # warm-up (alignment returns to 0)
    st3 = sp.run_pipelined(g3, cfg3, 16)
    extra["C3_compressed"] = {"glups": st3.mlups / 1e3, "sweeps": 64, "wall_s": st3.wall_seconds,
                              "frac_of_hbm_roofline": st3.mlups / 1e3 * 4.0 / peak,
                              "config": "600^3 in 606^3 (pad 4), t=4 x16 passes, in place"}
    del g3
    # C4 at P=1: the per-GPU block of the weak-scaling runs (1024^3, ring 1.0,
    # t=4, 40 sweeps) through run_pipelined, device-timed
    torch.cuda.empty_cache()
    a4 = sp.create_grid(*C4["n"], init="random", seed=SEED, ring=C4["ring"])
    b4 = a4.copy()
    cfg4 = sp.PipelineConfig(spec=sp.BlockSpec(C4["n"][0], 32, 32), t=C4["t"])
    sp.run_pipelined((a4, b4), cfg4, 2)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    sp.run_pipelined((a4, b4), cfg4, C4["sweeps"] // C4["t"])
    e1.record()
    torch.cuda.synchronize()
    ms4 = e0.elapsed_time(e1)
    extra["C4_single_gpu"] = {"glups": C4["n"][0] ** 3 * C4["sweeps"] / (ms4 / 1e3) / 1e9, "ms": ms4,
                              "config": "1024^3, ring 1.0, t=4, 40 sweeps (the per-GPU C4 block)"}
    # the N>1 lines run C4 weak scaling: their per-GPU rate compares with this
    # one-GPU C4 block, not with the C2 headline of this line
    extra["weak_scaling_baseline"] = {"per_gpu_glups": extra["C4_single_gpu"]["glups"],
                                      "workload": "C4 block at P=1 (1024^3, ring 1.0, t=4, 40 sweeps)",
                                      "compare_with": "per_gpu_glups of the N>1 lines"}
    del a4, b4
    # C5 on one GPU: 2048^3 global, two 2050^3 grids = 137.8 GB of HBM,
    # 32 sweeps at t=1/4/8, device-timed with CUDA events
    torch.cuda.empty_cache()
    if torch.cuda.mem_get_info()[0] >= 140e9:
        n5 = C5["n"][0]
        a5 = sp.create_grid(n5, n5, n5, init="random", seed=SEED)
        b5 = a5.copy()
        c5 = {"hbm_gb_resident": 2 * a5.data.numel() * 8 / 1e9, "sweeps": C5["sweeps"],
              "config": "2048^3 in 2050^3, two grids, U[0,1) seed 42, ring 0.0, 32 sweeps"}
        for t5 in C5["ts"]:
            cfg5 = sp.PipelineConfig(spec=sp.BlockSpec(n5, 32, 32), t=t5)
            sp.run_pipelined((a5, b5), cfg5, 1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            sp.run_pipelined((a5, b5), cfg5, C5["sweeps"] // t5)
            e1.record()
            torch.cuda.synchronize()
            ms5 = e0.elapsed_time(e1)
            c5[f"t{t5}"] = {"glups": n5 ** 3 * C5["sweeps"] / (ms5 / 1e3) / 1e9, "ms": ms5}
        c5["glups"] = c5["t4"]["glups"]
        extra["C5_single_gpu"] = c5
        del a5, b5
        torch.cuda.empty_cache()
    else:
        extra["C5_single_gpu"] = {"skipped": "needs 140 GB of free HBM"}
    return extra


def _c5_strong(sp, torch, dist, ws, all_max):
    """BASELINE configs[4]: 2048^3 global as z-slabs over the ws GPUs, 32
    sweeps at ghost depth / exchange interval t in {1, 4, 8}; device-timed,
    max over ranks."""
    from paper_1006_3148_b200 import halo
    out = {"config": "2048^3 global, z-slabs over the GPUs, U[0,1) seed 42, ring 0.0, 32 sweeps",
           "scaling": "strong"}
    n5 = C5["n"]
    if n5[2] % ws:
        out["skipped"] = f"2048 planes do not split over {ws} ranks"
        return out
    for t in C5["ts"]:
        solver = halo.SlabSolver.strong(n5, seed=SEED, ring=C5["ring"], depth=t)
        solver.run_sweeps(2 * t)  # warm-up
        all_max(None)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        solver.run_sweeps(C5["sweeps"])
        e1.record()
        torch.cuda.synchronize()
        ms = all_max(e0.elapsed_time(e1))
        out[f"t{t}"] = {"glups": n5[0] * n5[1] * n5[2] * C5["sweeps"] / (ms / 1e3) / 1e9, "ms": ms,
                        "exchanges": C5["sweeps"] // t}
        del solver
        torch.cuda.empty_cache()
    out["glups"] = max(out[f"t{t}"]["glups"] for t in C5["ts"])
    return out


def _pcie_duplex(torch, host_in, host_out, dev, all_max) -> float:
    """GB/s each way with an H2D and a D2H of one grid in flight together
    (the e2e steady state), best of three; max over ranks of the time."""
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    scratch = torch.empty_like(dev)
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a.wait_event(e0)
        b.wait_event(e0)
        with torch.cuda.stream(a):
            scratch.copy_(host_in, non_blocking=True)
            ea = torch.cuda.Event(enable_timing=True)
            ea.record(a)
        with torch.cuda.stream(b):
            host_out.copy_(dev, non_blocking=True)
            eb = torch.cuda.Event(enable_timing=True)
            eb.record(b)
        torch.cuda.synchronize()
        ms = max(e0.elapsed_time(ea), e0.elapsed_time(eb))
        ms = all_max(ms)
        best = ms if best is None else min(best, ms)
    del scratch
    return host_in.numel() * 8 / (best / 1e3) / 1e9


def _e2e(sp, torch, dist, ws, slab, args, all_max, grid_bytes):
    """The same metric through the public API with host buffers (see
    e2e_pipelined): N=1 run_pipelined on C2; N>1 the z-slab driver on C4,
    every rank loading its local grid and returning its result grid."""
    import numpy as np
    # a serving loop's throughput: at least 40 steps, so the first H2D and the
    # last D2H (which no solve can overlap) are amortised like in a long run
    steps = max(40, args.steps)
    if slab:
        from paper_1006_3148_b200 import halo

        class Unit:
            def __init__(self):
                self.s = halo.SlabSolver.weak(per_rank=C4["n"], seed=SEED, ring=C4["ring"], depth=args.t,
                                              transport=args.transport)

            def load(self, host):
                self.s.load(host)

            def solve(self):
                self.s.run_sweeps(C4["sweeps"])

            def result(self):
                return self.s.current().data

        units = [Unit(), Unit()]
        host_in, pinned = _pin(units[0].s.current().data.cpu())
        host_out, _ = _pin(torch.empty_like(host_in, device="cpu"))
        cells, sweeps = units[0].s.owned_cells * ws, C4["sweeps"]
        api = ("pinned host local grid -> SlabSolver.load (H2D stream) -> 10 RankRuntime cycles with "
               "NCCL z-halo exchange (compute stream) -> result grid -> pinned host (D2H stream); "
               "steps pipelined over two solve units per rank; time = max over ranks")
    else:
        n = C2["n"]
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(n[0], 32, 32), t=args.t)

        class Unit:
            def __init__(self):
                self.a, self.b = sp.Grid3(*n, 0), sp.Grid3(*n, 0)
                self.res = None

            def load(self, host):
                self.a.data.copy_(host, non_blocking=True)

            def solve(self):
                sp.copy_ring(self.a, self.b)  # the partner grid needs the same ring
                # 100 sweeps exactly: passes of t, then the remainder as one pass
                full, rem = divmod(C2["sweeps"], cfg.h)
                st = sp.run_pipelined((self.a, self.b), cfg, full)
                self.res = st.result
                if rem:
                    cfg_r = sp.PipelineConfig(spec=cfg.spec, t=rem)
                    other = self.b if self.res is self.a else self.a
                    st = sp.run_pipelined((self.res, other), cfg_r, 1)
                    self.res = st.result

            def result(self):
                return self.res.data

        units = [Unit() for _ in range(3)]
        g0 = sp.create_grid(*n, init="random", seed=SEED)
        host_in, pinned = _pin(g0.data.cpu())
        host_out, _ = _pin(torch.empty_like(host_in, device="cpu"))
        del g0
        cells, sweeps = n[0] * n[1] * n[2], C2["sweeps"]
        api = ("pinned host grid -> Grid3.data.copy_ (H2D stream) -> run_pipelined (compute stream) "
               "-> result.data -> pinned host (D2H stream); steps pipelined over three device grid pairs")
    ms = e2e_pipelined(units, host_in, host_out, steps, max(1, args.warmup), all_max)
    # the read-back must be the solve's result (last unit's grid)
    last = units[(steps - 1) % len(units)].result()
    assert torch.equal(host_out, last.cpu())
    pcie = _pcie_duplex(torch, host_in, host_out, last, all_max)
    value = cells * sweeps / (ms / 1e3) / 1e9
    # e2e roofline: one grid each way per step over this box's PCIe link with
    # both directions busy (the solve hides under the transfers)
    ceiling = cells * sweeps / (grid_bytes / (pcie * 1e9)) / 1e9
    e2e = {"value": value, "unit": UNIT,
           "h2d_bytes_per_step": grid_bytes, "d2h_bytes_per_step": grid_bytes,
           "ms_per_step": ms, "sweeps": sweeps, "pinned_host": pinned, "api": api,
           "steps": steps, "fill_drain": "included: first H2D and last D2H inside the timed region",
           "roofline": {"bound": "pcie (H2D and D2H concurrently)", "link_gbs_each_way": pcie,
                        "ceiling": ceiling, "frac": value / ceiling,
                        "how": "one pinned grid H2D and one D2H at once on two streams, "
                               "best of 3, measured on this box before the e2e leg's teardown"}}
    assert np.isfinite(e2e["value"])
    del units
    torch.cuda.empty_cache()
    return e2e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--t", type=int, default=4, help="fused sweeps per HBM pass (1..4)")
    ap.add_argument("--quick", action="store_true", help="skip the extra legs and e2e")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-child", type=float, default=None, help=argparse.SUPPRESS)
    ap.add_argument("--cpu-n", default="512,512,512", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-numpy-sweeps", type=int, default=2, help=argparse.SUPPRESS)
    ap.add_argument("--ref-sweeps-per-step", type=int, default=0,
                    help="reference arm: sweeps per step (0 = the workload's, C2: 100; C4: 2-sweep sample)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help=argparse.SUPPRESS)  # gloo: N>1 path check with all ranks on one GPU
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="z-slab halo delivery for N>1: NCCL P2P, or the fused peer-memory stores")
    ap.add_argument("--slab", action="store_true",
                    help="run the C4 distributed z-slab workload even on one GPU")
    args = ap.parse_args()
    if args.cpu_child is not None:
        return _cpu_child(args.cpu_child, tuple(int(v) for v in args.cpu_n.split(",")), 100,
                          args.cpu_numpy_sweeps)
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
