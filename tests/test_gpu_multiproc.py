"""GPU, two processes on cuda:0: the distributed driver with the real GPU
PipelineEngine in every rank (fused K2/K3 passes with shrinking live ranges,
RankRuntime.cycle with the boundary-first split that posts the z exchange from
inside the pass) over a host-staged gloo transport between the processes.
The assembled result must equal the undecomposed oracle bit for bit.

No rank waits on another's GPU work: the messages cross through host memory
and gloo, so each process's stream only runs its own kernels
(B200_PROFILING.md: ranks on one GPU must not wait on each other's kernels).
NCCL between devices is the same code path with device buffers
(halo.start_zslab_exchange / exchange_multilayer_halos)."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1006_3148_b200 as sp
        from paper_1006_3148_b200 import halo
        cfg = sp.PipelineConfig(spec=sp.BlockSpec(*case.get("spec", (8, 8, 8))), t=case.get("t", case["h"]),
                                T=case.get("T", 1), grid_mode=case["mode"])
        dc = halo.DistConfig(topo=halo.RankTopology(*case["topo"]), cfg=cfg, cycles=case["cycles"],
                             global_dims=tuple(case["global_dims"]), mode="strong", seed=case["seed"],
                             ring=case.get("ring"))
        rt = halo.run_rank(dc, rank)
        assert isinstance(rt.engine, sp.PipelineEngine) and rt.engine.grids[0].data.is_cuda
        full = halo.gather_owned(rt)
        timings = dict(rt.timings)
        timings["launches"] = sp._lib.launch_count()
        if rank == 0:
            np.save(out, full)
        with open(f"{out}.{rank}.json", "w") as f:
            json.dump(timings, f)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    dict(topo=(1, 1, 2), global_dims=(40, 36, 48), h=4, mode="two_grid", cycles=3, seed=42, ring=1.0),
    dict(topo=(1, 1, 2), global_dims=(70, 33, 40), h=2, mode="two_grid", cycles=4, seed=7),
    dict(topo=(1, 1, 3), global_dims=(24, 20, 48), h=3, mode="two_grid", cycles=3, seed=5),
    dict(topo=(1, 1, 2), global_dims=(30, 30, 32), h=4, mode="compressed", cycles=2, seed=42),
    dict(topo=(2, 1, 1), global_dims=(48, 20, 20), h=4, mode="two_grid", cycles=2, seed=3, ring=0.5),
    dict(topo=(1, 2, 1), global_dims=(20, 48, 16), h=2, mode="two_grid", cycles=3, seed=9),
]


# acceptance criterion #2 (pkg/tests/test_acceptance.py:94-158) over gloo:
# the 12 topology / halo / mode cases at 60^3, seed 42, two cycles, each rank
# a separate process with the GPU engine (the reference's in-process threads
# plus its 2-rank TCP loopback run, in one matrix)
for _topo in ((2, 1, 1), (2, 2, 1), (2, 2, 2)):
    for _h, _mode in ((2, "two_grid"), (2, "compressed"), (4, "two_grid"), (4, "compressed")):
        CASES.append(dict(topo=_topo, global_dims=(60, 60, 60), h=_h, t=2, T=1 if _h == 2 else 2,
                          mode=_mode, cycles=2, seed=42, spec=(15, 10, 10)))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['topo']}-h{c['h']}-{c['mode']}-{c['global_dims'][0]}")
def test_two_process_gpu_engine_equals_oracle(case, tmp_path):
    world = int(np.prod(case["topo"]))
    out = str(tmp_path / "full.npy")
    mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    gd = tuple(case["global_dims"])
    d0 = oracle.make_storage(*gd, init="random", seed=case["seed"], ring=case.get("ring"))
    exp = oracle.interior(oracle.sweeps(d0, gd, case["h"] * case["cycles"]), *gd)
    assert np.array_equal(got, exp)
    for r in range(world):
        t = json.load(open(f"{out}.{r}.json"))
        assert t["launches"] > 0 and t["messages"] > 0
        if case["topo"][:2] == (1, 1) and case["mode"] == "two_grid":
            # every cycle posted its exchange from inside the pass
            assert t.get("overlapped_cycles") == case["cycles"], t
