"""PCIe probe for the e2e leg: pinned H2D / D2H of one 514^3 grid (1.086 GB),
alone and concurrent, whole or chunked over several streams, with the host
buffers allocated after pinning the process to the GPU's NUMA-local CPUs or not.

    python tools/pcie_probe2.py [--local]
"""
import os
import subprocess
import sys
import time

import torch

local = "--local" in sys.argv
if local:
    # CPUs the driver reports as local to GPU 0 (nvidia-smi topo -m "CPU Affinity")
    out = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
    line = [l for l in out.splitlines() if l.startswith("GPU0")][0].split()
    aff = [c for c in line if "-" in c and c[0].isdigit()]
    cpus = set()
    for part in aff[0].split(","):
        lo, hi = part.split("-")
        cpus.update(range(int(lo), int(hi) + 1))
    os.sched_setaffinity(0, cpus)
    print("affinity", aff[0], flush=True)

n = 514 ** 3
nb = n * 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
h_in.fill_(1.0)
h_out.fill_(0.0)
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
ss = [torch.cuda.Stream() for _ in range(8)]


def run(dirs, chunks, nstreams, reps=4):
    def once():
        k = 0
        step = -(-n // chunks)
        for c in range(chunks):
            sl = slice(c * step, min(n, (c + 1) * step))
            for d in dirs:
                s = ss[k % nstreams] if d == "h2d" else ss[4 + k % nstreams]
                with torch.cuda.stream(s):
                    if d == "h2d":
                        d_in[sl].copy_(h_in[sl], non_blocking=True)
                    else:
                        h_out[sl].copy_(d_out[sl], non_blocking=True)
            k += 1
    once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        once()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    return ms, nb / ms / 1e6


for dirs in (("h2d",), ("d2h",), ("h2d", "d2h")):
    for chunks, nst in ((1, 1), (8, 1), (8, 2), (32, 4)):
        ms, gbs = run(dirs, chunks, nst)
        print(f"{'+'.join(dirs):8s} chunks={chunks:3d} streams/dir={nst}: {ms:7.2f} ms  {gbs:6.1f} GB/s per direction", flush=True)
