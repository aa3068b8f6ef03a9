// Copy-engine probe: device-to-device 3D box copies (cudaMemcpy3DAsync) of a
// z-slab of a 606^3 FP64 grid, alone and concurrent with an SM-saturating
// kernel, to size a K3 variant that stages slab outputs and copies them back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ce_probe tools/ce_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void busy(double *p, int iters) {
    double v = p[threadIdx.x];
    for (int i = 0; i < iters; ++i) v = v * 1.0000001 + 1e-9;
    if (v == 42.0) p[threadIdx.x] = v;
}

int main() {
    const size_t E = 606, N = 600, SL = 150;
    double *grid, *tmp;
    cudaMalloc(&grid, E * E * E * 8);
    cudaMalloc(&tmp, E * E * SL * 8);
    cudaMemset(grid, 0, E * E * E * 8);
    cudaMemset(tmp, 0, E * E * SL * 8);
    cudaStream_t s0, s1;
    cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaMemcpy3DParms m = {};
    m.srcPtr = make_cudaPitchedPtr(tmp, E * 8, E, E);
    m.dstPtr = make_cudaPitchedPtr(grid, E * 8, E, E);
    m.srcPos = make_cudaPos(5 * 8, 5, 0);
    m.dstPos = make_cudaPos(1 * 8, 1, 200);
    m.extent = make_cudaExtent(N * 8, N, SL);
    m.kind = cudaMemcpyDeviceToDevice;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) cudaMemcpy3DAsync(&m, s1);
    cudaStreamSynchronize(s1);
    cudaEventRecord(a, s1);
    for (int r = 0; r < 10; ++r) cudaMemcpy3DAsync(&m, s1);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = 2.0 * N * N * SL * 8;
    printf("3D copy alone: %.3f ms per slab, %.1f GB/s (read+write)\n", ms / 10, bytes / (ms / 10 * 1e-3) / 1e9);
    // contiguous 1D copy of the same bytes
    cudaEventRecord(a, s1);
    for (int r = 0; r < 10; ++r) cudaMemcpyAsync(grid, tmp, N * N * SL * 8, cudaMemcpyDeviceToDevice, s1);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("1D copy alone: %.3f ms, %.1f GB/s\n", ms / 10, bytes / (ms / 10 * 1e-3) / 1e9);
    // concurrent with a kernel holding every SM
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    busy<<<sms * 4, 256, 0, s0>>>(tmp, 2000000);
    cudaEventRecord(a, s1);
    for (int r = 0; r < 10; ++r) cudaMemcpy3DAsync(&m, s1);
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("3D copy under a busy kernel: %.3f ms per slab, %.1f GB/s\n", ms / 10, bytes / (ms / 10 * 1e-3) / 1e9);
    cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
