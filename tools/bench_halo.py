"""Time the halo pack/unpack kernels (k_boxes: sp_pack_boxes /
sp_unpack_boxes) on one exchange of a general topology, all ranks on this
GPU: bytes moved per exchange (each message packed once and unpacked once:
16 B per halo cell of HBM traffic) over the device time.
    python tools/bench_halo.py [per_rank_n] [h]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1006_3148_b200 as sp
from paper_1006_3148_b200 import halo

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
h = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for topo in ((2, 1, 1), (2, 2, 1), (2, 2, 2)):
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(8, 8, 8), t=h)
    gd = tuple(n * p for p in topo)
    subs = halo.decompose_domain(gd, halo.RankTopology(*topo), halo.HaloSpec(h))
    rts = [halo.RankRuntime(s, cfg, None, init="constant", value=1.0) for s in subs]
    halo.exchange_inprocess(rts)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    s.record()
    for _ in range(reps):
        halo.exchange_inprocess(rts)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    nbytes = sum(m.nbytes for rt in rts for m in rt.plan.messages)
    print(f"topology {topo}, {n}^3 per rank, h={h}: {len(rts)} ranks, {nbytes / 1e6:.1f} MB of messages, "
          f"{ms:.3f} ms per exchange, {2 * nbytes / ms / 1e6:.0f} GB/s of pack+unpack traffic "
          f"(read + write each: {4 * nbytes / ms / 1e6:.0f} GB/s HBM)", flush=True)
    del rts
    torch.cuda.empty_cache()
