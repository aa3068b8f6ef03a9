"""Small runs of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): K0, K1 (TMA and cp.async), K2 at T=2..4 with z-chunks and live
ranges, K3 both directions, the window seam, faces, ring copy/compare."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1006_3148_b200 as sp

L = sp._lib.load()
for force in (0, 1):
    L.sp_set_tuning(1, force)
    g = sp.create_grid(70, 37, 21, init="random", seed=1, ring=0.5)
    h = g.copy()
    sp.reference_sweep(g, h)
    for t in (2, 3, 4):
        sp.fused_sweeps(g, h, t)
        sp.fused_sweeps(g, h, t, 3, 17)
L.sp_set_tuning(1, 0)
L.sp_set_tuning(0, 5)
g = sp.create_grid(67, 40, 30, init="random", seed=2)
sp.fused_sweeps(g, g.copy(), 4)
L.sp_set_tuning(0, 0)
c = sp.create_grid(66, 35, 24, pad=4, init="random", seed=3, lo=-1.0, hi=1.0)
cfg = sp.PipelineConfig(spec=sp.BlockSpec(66, 8, 8), t=4, grid_mode="compressed")
sp.run_pipelined(c, cfg, 2)
cfg = sp.PipelineConfig(spec=sp.BlockSpec(66, 8, 8), t=3, grid_mode="compressed")
sp.run_pipelined(c, cfg, 2)
sp.apply_window(g.data, g.data, ((1, 60), (2, 30), (0, 20)), g.offset, g.offset - 1)
assert sp.rings_equal(g, g)
sp.copy_ring(g, g.copy())
torch.cuda.synchronize()
print("sanitize cases done")
