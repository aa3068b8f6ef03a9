import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_1006_3148_b200 as sp
L = sp._lib.load()
n = 600
g = sp.create_grid(n, n, n, pad=4, init="random", seed=42, lo=-1.0, hi=1.0)
cfg = sp.PipelineConfig(spec=sp.BlockSpec(n, 30, 30), t=4, grid_mode="compressed")
for zc in (0, 60, 100, 150, 200, 300, 600, 0):
    L.sp_set_tuning(0, zc)
    sp.run_pipelined(g, cfg, 2)
    st = sp.run_pipelined(g, cfg, 8)
    print(f"zc={zc}: {st.mlups/1e3:.1f} GLUP/s")
L.sp_set_tuning(0, 0)
