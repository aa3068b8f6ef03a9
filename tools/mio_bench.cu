// MIO throughput on sm_100a: 64-bit shuffles vs shared-memory loads, per SM
// per SM clock (clock64 around the loop), 8 warps per SM as in k_temporal.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mio tools/mio_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ILP = 8;

// mode 0: SHFL of doubles (2 SHFL.32 each); 1: LDS.64 contiguous; 2: LDS.128;
// 3: LDS.64 at 16-byte lane stride (4-way conflict); 4: SHFL + LDS.64 mixed 1:1
template <int MODE>
__global__ void k(double *out, int n, long long *cyc) {
    __shared__ __align__(16) double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = threadIdx.x + j;
    const int lane = threadIdx.x & 31;
    int base = (threadIdx.x >> 5) * 64;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            if (MODE == 0) {
                x[j] = __shfl_down_sync(0xffffffffu, x[j], 1) + 1.0;
            } else if (MODE == 1) {
                x[j] += s[(base + lane + 32 * j + i) & 4095];
            } else if (MODE == 2) {
                const double2 v = *reinterpret_cast<const double2 *>(&s[(base + 2 * lane + 64 * j + 2 * i) & 4094]);
                x[j] += v.x + v.y;
            } else if (MODE == 3) {
                x[j] += s[(base + 2 * lane + 1 + 64 * j + i) & 4095];
            } else {
                if (j & 1) x[j] = __shfl_down_sync(0xffffffffu, x[j], 1) + 1.0;
                else x[j] += s[(base + lane + 32 * j + i) & 4095];
            }
        }
    }
    long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char *name, int warps, double *out, long long *cyc, int sms) {
    int n = 2048;
    k<MODE><<<sms, warps * 32>>>(out, n, cyc);
    k<MODE><<<sms, warps * 32>>>(out, n, cyc);
    cudaDeviceSynchronize();
    long long c[1024];
    cudaMemcpy(c, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += c[i];
    avg /= sms;
    double ops = (double)warps * n * ILP;  // warp-level ops per SM
    printf("%-28s warps/SM %2d: %.3f warp-ops/clk/SM\n", name, warps, ops / avg);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    long long *cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 8 * 1024);
    for (int w : {8, 16}) {
        run<0>("SHFL double (2x SHFL.32)", w, out, cyc, sms);
        run<1>("LDS.64 contiguous", w, out, cyc, sms);
        run<2>("LDS.128 contiguous", w, out, cyc, sms);
        run<3>("LDS.64 16B stride", w, out, cyc, sms);
        run<4>("SHFL dbl + LDS.64 1:1", w, out, cyc, sms);
    }
    return 0;
}
