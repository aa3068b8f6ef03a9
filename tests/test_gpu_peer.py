"""GPU: the fused peer-memory halo delivery of z-slab runs (transport "p2p").

Every rank runs in this process (one stream, phase-interleaved cycles); the
last fused pass of each cycle stores its boundary planes into the neighbours'
ghost planes (sp_temporal_mirror) and the ranks order their passes through
the stream-ordered counters (sp_signal / sp_wait), the protocol one process
per GPU runs over NVLink.  The assembled result must equal the undecomposed
oracle bit for bit.  The IPC mapping itself is checked across two processes
(no rank waits on another there)."""

import ctypes
import multiprocessing as mp

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

sp = pytest.importorskip("paper_1006_3148_b200")
from paper_1006_3148_b200 import _lib, halo  # noqa: E402


def _run_p2p(topo, gd, h, cycles, ring=None):
    cfg = sp.PipelineConfig(spec=sp.BlockSpec(8, 8, 8), t=h)
    dc = halo.DistConfig(topo=halo.RankTopology(*topo), cfg=cfg, cycles=cycles, global_dims=gd,
                         mode="strong", seed=42, ring=ring)
    rts = halo.run_distributed_inprocess(dc, transport="p2p")
    g = halo.assemble_global(rts)
    d0 = oracle.make_storage(*gd, init="random", seed=42, ring=ring)
    exp = oracle.interior(oracle.sweeps(d0, gd, h * cycles), *gd)
    assert_bitwise(g.interior_numpy(), exp)
    return rts


@pytest.mark.parametrize("topo,gd,h,cycles,ring", [
    ((1, 1, 2), (40, 40, 40), 4, 3, None),
    ((1, 1, 2), (40, 40, 40), 2, 4, 1.0),
    ((1, 1, 3), (36, 20, 48), 3, 3, None),
    ((1, 1, 4), (24, 24, 64), 4, 3, 0.5),
    ((1, 1, 2), (130, 70, 40), 4, 2, None),
    ((1, 1, 2), (40, 40, 40), 1, 5, None),      # plain sweep: mirrored by a copy after the launch
    ((1, 1, 2), (40, 40, 48), 6, 2, None),      # two fused chunks per pass (4 + 2)
    ((1, 1, 3), (30, 30, 72), 8, 2, 1.0),       # two chunks of 4
])
def test_p2p_zslab_equals_oracle(topo, gd, h, cycles, ring):
    rts = _run_p2p(topo, gd, h, cycles, ring)
    for rt in rts:
        nbs = sum(rt.sub.has_nb[2])
        assert rt.timings.get("messages", 0) == nbs * cycles
        # counters: two phases per pass, written by each neighbour
        flags = rt.flags.cpu().tolist()
        for side in rt.links:
            assert flags[side] == 2 * cycles


def test_p2p_cpasync_copy_fallback():
    L = _lib.load()
    try:
        L.sp_set_tuning(1, 1)  # cp.async loader: planes mirrored by a copy after the pass
        _run_p2p((1, 1, 2), (40, 40, 40), 4, 2)
    finally:
        L.sp_set_tuning(1, 0)


@pytest.mark.parametrize("kernels", [0, 1])
def test_signal_wait_one_stream(kernels):
    """sp_signal / sp_wait on one stream, stream memory operations (the
    cross-GPU path) and the kernel fallback: the wait releases on the value
    written earlier in the stream, and the counter compares cyclically."""
    L = _lib.load()
    L.sp_set_tuning(5, kernels)
    try:
        flag = torch.zeros(4, dtype=torch.int32, device="cuda")
        out = torch.zeros(8, dtype=torch.float64, device="cuda")
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        fp = ctypes.c_void_p(flag.data_ptr() + 4)
        for v in (1, 2, 7):
            _lib.check(L.sp_signal(fp, v, s))
            _lib.check(L.sp_wait(fp, v, s))
            _lib.check(L.sp_wait(fp, v - 1, s))
            _lib.check(L.sp_fill_constant(ctypes.c_void_p(out.data_ptr()), 8, float(v), s))
        torch.cuda.synchronize()
        assert flag.cpu().tolist() == [0, 7, 0, 0]
        assert torch.all(out == 7.0)
    finally:
        L.sp_set_tuning(5, 0)


def test_mirror_planes_and_bounds():
    dims = (70, 33, 30)
    g = sp.create_grid(*dims, init="random", seed=3, ring=0.25)
    dst = g.copy()
    peer = torch.full((20,) + tuple(g.data.shape[1:]), -7.0, dtype=torch.float64, device="cuda")
    zlo, zhi, zs = 10, 16, -8  # storage planes 11..16 -> peer planes 3..8
    sp.kernel.fused_sweeps_mirror(g, dst, 4, zlo, zhi, peer.data_ptr(), peer.shape[0], zs)
    torch.cuda.synchronize()
    off = g.offset
    o = off  # interior x/y of the mirrored planes equal the local result
    got = peer[zlo + off + zs:zhi + off + zs, o:o + dims[1], o:o + dims[0]]
    ref = dst.data[zlo + off:zhi + off, o:o + dims[1], o:o + dims[0]]
    assert torch.equal(got, ref)
    d0 = oracle.make_storage(*dims, init="random", seed=3, ring=0.25)
    exp = oracle.interior(oracle.sweeps(d0, dims, 4), *dims)
    assert_bitwise(dst.interior_numpy()[zlo:zhi], exp[zlo:zhi])
    # nothing outside those planes was touched
    keep = torch.ones(peer.shape[0], dtype=torch.bool)
    keep[zlo + off + zs:zhi + off + zs] = False
    assert torch.all(peer[keep] == -7.0)
    with pytest.raises(ValueError):
        sp.kernel.fused_sweeps_mirror(g, dst, 4, zlo, zhi, peer.data_ptr(), peer.shape[0], 10)


def _ipc_child(handle, offset, n, q):
    try:
        import ctypes as ct
        import torch as th
        from paper_1006_3148_b200 import _lib as lib
        th.cuda.set_device(0)
        L = lib.load()
        p = ct.c_void_p()
        lib.check(L.sp_ipc_open(handle, ct.byref(p)), "open")
        ptr = p.value + offset
        lib.check(L.sp_fill_constant(ct.c_void_p(ptr), n, 2.5, None), "fill")
        th.cuda.synchronize()
        lib.check(L.sp_ipc_close(p), "close")
        q.put("ok")
    except Exception as e:  # reported to the parent
        q.put(repr(e))


def test_ipc_handle_across_processes():
    L = _lib.load()
    base = torch.zeros(4096, dtype=torch.float64, device="cuda")
    view = base[1000:2000]  # an interior pointer: handle of the allocation + offset
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _lib.check(L.sp_ipc_handle(ctypes.c_void_p(view.data_ptr()), buf, ctypes.byref(off)))
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ipc_child, args=(buf.raw, off.value, view.numel(), q))
    p.start()
    msg = q.get(timeout=240)
    p.join(timeout=60)
    assert msg == "ok", msg
    b = base.cpu().numpy()
    assert np.all(b[1000:2000] == 2.5) and np.all(b[:1000] == 0) and np.all(b[2000:] == 0)
