"""Time the C3 compressed solve (K3) for a few fused depths, and K2 at the same size."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1006_3148_b200 as sp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 16
fuse = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "4").split(",")]
for mf in fuse:
    sp.PipelineEngine.max_fused = mf
    g = sp.create_grid(n, n, n, pad=4, init="random", seed=42, lo=-1.0, hi=1.0)
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(n, 30, 30), t=4, grid_mode="compressed")
    sp.run_pipelined(g, cfg, 2)
    st = sp.run_pipelined(g, cfg, passes)
    print(f"C3 n={n} max_fused={mf}: {st.mlups/1e3:.1f} GLUP/s ({st.wall_seconds*1e3:.2f} ms, {passes} passes)")
    del g
    a = sp.create_grid(n, n, n, init="random", seed=42)
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(n, 30, 30), t=4)
    sp.run_pipelined((a, a.copy()), cfg, 2)
    st = sp.run_pipelined((a, a.copy()), cfg, passes)
    print(f"K2 two-grid n={n} max_fused={mf}: {st.mlups/1e3:.1f} GLUP/s")
