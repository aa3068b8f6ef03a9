"""Time pinned H2D, D2H, both at once, and H2D/D2H concurrent with a K2 solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1006_3148_b200 as sp

n = 512
g = sp.create_grid(n, n, n, init="random", seed=42)
h_in = torch.empty(tuple(g.data.shape), dtype=torch.float64).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
d1 = torch.empty_like(g.data)
d2 = torch.empty_like(g.data)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
nb = g.data.numel() * 8


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d2, non_blocking=True)


def both():
    h2d(); d2h()


a, b = g, g.copy()
cfg = sp.PipelineConfig(spec=sp.BlockSpec(n, 32, 32), t=4)


def solve():
    with torch.cuda.stream(s3):
        sp.run_pipelined((a, b), cfg, 25)


def all3():
    h2d(); d2h(); solve()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("h2d+d2h", both), ("solve", solve), ("all3", all3)):
    ms = timed(fn)
    print(f"{name:10s} {ms:8.2f} ms  ({nb / ms / 1e6:.1f} GB/s per direction)" if name in ("h2d", "d2h", "h2d+d2h") else f"{name:10s} {ms:8.2f} ms")

# timeline of one round: events at the start/end of each stream's work
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t0.record()
ev = {}
for name, st, fn in (("h2d", s1, lambda: d1.copy_(h_in, non_blocking=True)),
                     ("d2h", s2, lambda: h_out.copy_(d2, non_blocking=True))):
    with torch.cuda.stream(st):
        st.wait_event(t0)
        e_a = torch.cuda.Event(enable_timing=True); e_a.record(st)
        fn()
        e_b = torch.cuda.Event(enable_timing=True); e_b.record(st)
        ev[name] = (e_a, e_b)
with torch.cuda.stream(s3):
    s3.wait_event(t0)
    e_a = torch.cuda.Event(enable_timing=True); e_a.record(s3)
    cur, oth = a, b
    for _ in range(25):
        sp.fused_sweeps(cur, oth, 4)
        cur, oth = oth, cur
    e_b = torch.cuda.Event(enable_timing=True); e_b.record(s3)
    ev["kernels"] = (e_a, e_b)
torch.cuda.synchronize()
for k, (e_a, e_b) in ev.items():
    print(f"timeline {k:8s} start {t0.elapsed_time(e_a):7.2f} ms  end {t0.elapsed_time(e_b):7.2f} ms")


def timeline(label, body):
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t0.record()
    ev = {}
    for name, st, fn in (("h2d", s1, lambda: d1.copy_(h_in, non_blocking=True)),
                         ("d2h", s2, lambda: h_out.copy_(d2, non_blocking=True))):
        with torch.cuda.stream(st):
            st.wait_event(t0)
            e_a = torch.cuda.Event(enable_timing=True); e_a.record(st)
            fn()
            e_b = torch.cuda.Event(enable_timing=True); e_b.record(st)
            ev[name] = (e_a, e_b)
    with torch.cuda.stream(s3):
        s3.wait_event(t0)
        e_a = torch.cuda.Event(enable_timing=True); e_a.record(s3)
        h0 = time.perf_counter()
        body()
        h1 = time.perf_counter()
        e_b = torch.cuda.Event(enable_timing=True); e_b.record(s3)
        ev["compute"] = (e_a, e_b)
    torch.cuda.synchronize()
    print(label, " ".join(f"{k}=[{t0.elapsed_time(x):.2f},{t0.elapsed_time(y):.2f}]" for k, (x, y) in ev.items()),
          f"host {1e3 * (h1 - h0):.2f} ms")


timeline("run_pipelined", lambda: sp.run_pipelined((a, b), cfg, 25))
eng = sp.PipelineEngine(cfg, (a, b))
timeline("engine.run_pass x25", lambda: [eng.run_pass(1 if p % 2 == 0 else -1) for p in range(25)])
timeline("new engine only", lambda: sp.PipelineEngine(cfg, (a, b))._check_rings_equal())
