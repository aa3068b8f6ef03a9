"""K1 plain sweep: GLUP/s per block of 50 back-to-back sweeps over 400 sweeps
(does the rate decay with time, or is it a property of the launch pattern?)."""
import os, sys, subprocess, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1006_3148_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = sp.create_grid(n, n, n, init="random", seed=42)
a, b = g, g.copy()
bufs = [a, b]
for i in range(20):
    sp.fused_sweeps(bufs[i % 2], bufs[1 - i % 2], 1)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
ev[0].record()
k = 0
for blk in range(8):
    for _ in range(50):
        sp.fused_sweeps(bufs[k % 2], bufs[1 - k % 2], 1)
        k += 1
    ev[blk + 1].record()
torch.cuda.synchronize()
for blk in range(8):
    ms = ev[blk].elapsed_time(ev[blk + 1])
    print(f"block {blk}: {n**3 * 50 / (ms / 1e3) / 1e9:.1f} GLUP/s ({ms / 50 * 1e3:.1f} us/sweep)")
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,temperature.gpu,temperature.memory,power.draw,clocks_throttle_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)
