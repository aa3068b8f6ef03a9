// Microbenchmarks for the fused-stencil design: FP64 add latency/throughput,
// 64-bit shuffle and shared-memory throughput on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o mb tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dadd(double *out, double a, int n, long long *cyc) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = __dadd_rn(x, a);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
__global__ void thr_dadd(double *out, double a, int n) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = a * (k + 1);
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = __dadd_rn(x[k], a);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void thr_shfl(double *out, double a, int n) {
    double x0 = a + threadIdx.x, x1 = a * 2, x2 = a * 3, x3 = a * 4;
    for (int i = 0; i < n; ++i) {
        x0 = __shfl_up_sync(0xffffffffu, x0, 1);
        x1 = __shfl_down_sync(0xffffffffu, x1, 1);
        x2 = __shfl_up_sync(0xffffffffu, x2, 1);
        x3 = __shfl_down_sync(0xffffffffu, x3, 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

__global__ void thr_lds(double *out, int n) {
    __shared__ double s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i;
    __syncthreads();
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) {
        acc0 += s[(idx + i) & 2047];
        acc1 += s[(idx + i + 32) & 2047];
        acc2 += s[(idx + i + 64) & 2047];
        acc3 += s[(idx + i + 96) & 2047];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    long long *cyc;
    cudaMalloc(&out, 1 << 26);
    cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int n = 1 << 14;
    lat_dadd<<<1, 32>>>(out, 1e-9, n, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)c / (n * 16.0));

    float ms;
    for (int warps : {4, 8, 16, 32}) {
        int blocks = sms, threads = warps * 32;
        n = 1 << 12;
        thr_dadd<8><<<blocks, threads>>>(out, 1e-9, n);
        cudaEventRecord(e0);
        thr_dadd<8><<<blocks, threads>>>(out, 1e-9, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * n * 8;
        printf("DADD throughput (%2d warps/SM, ILP 8): %.1f Gop/s = %.1f ops/clk/SM @1.9GHz\n", warps,
               ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.9e9);
    }
    for (int warps : {8, 16, 32}) {
        int blocks = sms, threads = warps * 32;
        n = 1 << 12;
        thr_shfl<<<blocks, threads>>>(out, 1.0, n);
        cudaEventRecord(e0);
        thr_shfl<<<blocks, threads>>>(out, 1.0, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double shfl = (double)blocks * warps * n * 4 * 2;  // warp-level SHFL.32 instructions
        printf("SHFL 64-bit (%2d warps/SM): %.2f SHFL.32 warp-instr/clk/SM\n", warps,
               shfl / (ms * 1e-3) / sms / 1.9e9);
        thr_lds<<<blocks, threads>>>(out, n);
        cudaEventRecord(e0);
        thr_lds<<<blocks, threads>>>(out, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double lds = (double)blocks * warps * n * 4;
        printf("LDS.64 (%2d warps/SM): %.2f warp-instr/clk/SM (%.0f B/clk/SM)\n", warps,
               lds / (ms * 1e-3) / sms / 1.9e9, lds * 256 / (ms * 1e-3) / sms / 1.9e9);
    }
    return 0;
}
