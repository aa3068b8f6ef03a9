"""Measure the bandwidth parameters of paper_1006_3148_b200/data/b200.model.

The reference's machine files (sp/perfmodel.py, sp/data/*.model) hold STREAM
copy bandwidth (m_s) and the bandwidth of the update loop a[i] += 1 in memory
by one core (m_um1), in the outer cache by one core (m_uc1) and by all cores
sharing it (m_ucmax).  On B200 the "core" is an SM and the shared outer cache
is the 126 MB L2.  Bytes counted are read + write, as in the reference.

    python tools/measure_b200_model.py      (needs a GPU; compiles a tiny kernel)
"""
import json

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <torch/extension.h>
#include <ATen/cuda/CUDAContext.h>
__global__ void upd(double *a, long n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
            a[i] += 1.0;
}
void update(torch::Tensor a, int blocks, int reps) {
    upd<<<blocks, 1024, 0, at::cuda::getCurrentCUDAStream()>>>(a.data_ptr<double>(), a.numel(), reps);
}
"""
CPP = "void update(torch::Tensor a, int blocks, int reps);"


def main():
    mod = load_inline("b200_update", cpp_sources=CPP, cuda_sources=SRC, functions=["update"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"],
                      verbose=False)
    sms = torch.cuda.get_device_properties(0).multi_processor_count

    def rate(nbytes, blocks, reps):
        a = torch.zeros(nbytes // 8, dtype=torch.float64, device="cuda")
        mod.update(a, blocks, reps)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 0.0
        for _ in range(5):
            e0.record()
            mod.update(a, blocks, reps)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 2 * a.numel() * 8 * reps / (e0.elapsed_time(e1) / 1e3))
        return best

    src = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    dst.copy_(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m_s = 0.0
    for _ in range(5):
        e0.record()
        dst.copy_(src)
        e1.record()
        torch.cuda.synchronize()
        m_s = max(m_s, 2 * src.numel() * 8 / (e0.elapsed_time(e1) / 1e3))
    out = {
        "m_s": m_s,
        "m_um1": rate(2 << 30, 4 * sms, 1),
        "m_um1_one_sm": rate(256 << 20, 1, 1),
        "m_uc1": rate(8 << 20, 1, 20),
        "m_ucmax": rate(48 << 20, 4 * sms, 50),
        "sms": sms,
        "sm_clock_hz": torch.cuda.get_device_properties(0).clock_rate * 1e3
        if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else None,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
