// TMEM as per-thread scratch on sm_100a: tcgen05.st / tcgen05.ld (32x32b.x32)
// throughput per SM clock with 4..16 warps, alone and mixed with 64-bit
// shuffles, LDS and DADD (does the TMEM path share the LSU data pipe?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

#define R32(v, o) \
    "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]), \
    "=r"(v[o + 6]), "=r"(v[o + 7]), "=r"(v[o + 8]), "=r"(v[o + 9]), "=r"(v[o + 10]), "=r"(v[o + 11]), \
    "=r"(v[o + 12]), "=r"(v[o + 13]), "=r"(v[o + 14]), "=r"(v[o + 15]), "=r"(v[o + 16]), "=r"(v[o + 17]), \
    "=r"(v[o + 18]), "=r"(v[o + 19]), "=r"(v[o + 20]), "=r"(v[o + 21]), "=r"(v[o + 22]), "=r"(v[o + 23]), \
    "=r"(v[o + 24]), "=r"(v[o + 25]), "=r"(v[o + 26]), "=r"(v[o + 27]), "=r"(v[o + 28]), "=r"(v[o + 29]), \
    "=r"(v[o + 30]), "=r"(v[o + 31])
#define W32(v, o) \
    "r"(v[o + 0]), "r"(v[o + 1]), "r"(v[o + 2]), "r"(v[o + 3]), "r"(v[o + 4]), "r"(v[o + 5]), \
    "r"(v[o + 6]), "r"(v[o + 7]), "r"(v[o + 8]), "r"(v[o + 9]), "r"(v[o + 10]), "r"(v[o + 11]), \
    "r"(v[o + 12]), "r"(v[o + 13]), "r"(v[o + 14]), "r"(v[o + 15]), "r"(v[o + 16]), "r"(v[o + 17]), \
    "r"(v[o + 18]), "r"(v[o + 19]), "r"(v[o + 20]), "r"(v[o + 21]), "r"(v[o + 22]), "r"(v[o + 23]), \
    "r"(v[o + 24]), "r"(v[o + 25]), "r"(v[o + 26]), "r"(v[o + 27]), "r"(v[o + 28]), "r"(v[o + 29]), \
    "r"(v[o + 30]), "r"(v[o + 31])

__device__ __forceinline__ void tm_ld32(uint32_t *v, uint32_t a) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : R32(v, 0)
        : "r"(a));
}
__device__ __forceinline__ void tm_st32(uint32_t a, const uint32_t *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31};"
        :
        : W32(v, 0), "r"(a)
        : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: st x32 + wait, ld x32 + wait (round trip, dependent)
//      1: ld only (2 independent x32 loads per iteration, one wait)
//      2: st only
//      3: round trip + 16 64-bit shuffles per iteration
//      4: round trip + 32 dependent-free DADDs per iteration
//      5: 16 64-bit shuffles only;  6: 32 DADDs only
//      7: st at the top, 32 DADDs, ld at the bottom of the previous slot (software-pipelined use)
template <int MODE>
__global__ void k(double *out, int n, long long *cyc, int cols_per_warpslot) {
    __shared__ uint32_t tbase_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tbase_s;
    // warp w owns lanes 32 (w % 4) .., columns (w / 4) * cols_per_warpslot ..
    const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * cols_per_warpslot);

    uint32_t v[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = threadIdx.x * 64 + j;
    double d[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) d[j] = threadIdx.x + j;
    tm_st32(ta, v);
    tm_st32(ta + 32, v + 32);
    tm_wait_st();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (MODE == 0 || MODE == 3 || MODE == 4) {
            tm_st32(ta, v);
            tm_wait_st();
            tm_ld32(v, ta);
            tm_wait_ld();
            v[0] += 1;
        }
        if (MODE == 1) {
            tm_ld32(v, ta);
            tm_ld32(v + 32, ta + 32);
            tm_wait_ld();
            v[0] += v[33];
        }
        if (MODE == 2) {
            tm_st32(ta, v);
            tm_st32(ta + 32, v + 32);
            tm_wait_st();
            v[0] += 1;
            v[32] += 1;
        }
        if (MODE == 3 || MODE == 5) {
#pragma unroll
            for (int j = 0; j < 16; ++j) d[j] = __shfl_down_sync(0xffffffffu, d[j], 1) + 1.0;
        }
        if (MODE == 4 || MODE == 6) {
#pragma unroll
            for (int j = 0; j < 16; ++j) d[j] = __dadd_rn(d[j], 1.0);
#pragma unroll
            for (int j = 0; j < 16; ++j) d[j] = __dadd_rn(d[j], 0.5);
        }
        if (MODE == 7) {
            // values produced last iteration are stored; values stored two
            // iterations ago are loaded; DADDs in between
            tm_st32(ta + (i & 1) * 32, v);
            tm_ld32(v + 32, ta + ((i & 1) ^ 1) * 32);
#pragma unroll
            for (int j = 0; j < 16; ++j) d[j] = __dadd_rn(d[j], 1.0);
#pragma unroll
            for (int j = 0; j < 16; ++j) d[j] = __dadd_rn(d[j], 0.5);
            tm_wait_ld();
            tm_wait_st();
            v[0] += v[32];
        }
    }
    long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int j = 0; j < 64; ++j) acc += v[j];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc += d[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int MODE>
void run(const char *name, int warps, double bytes_per_iter_thread, double *out, long long *cyc, int sms) {
    const int n = 4096;
    const int slots = (warps + 3) / 4;
    const int cps = 512 / slots >= 64 ? 64 : 512 / slots;
    k<MODE><<<sms, warps * 32>>>(out, n, cyc, cps);
    k<MODE><<<sms, warps * 32>>>(out, n, cyc, cps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    static long long c[1024];
    cudaMemcpy(c, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += c[i];
    avg /= sms;
    printf("%-44s warps/SM %2d: %8.1f clk/iter", name, warps, avg / n);
    if (bytes_per_iter_thread > 0) printf("  %7.1f TMEM B/clk/SM", bytes_per_iter_thread * warps * 32 * n / avg);
    printf("\n");
}

int main() {
    int sms = 148;
    double *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(double) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    for (int w : {4, 8, 12, 16}) {
        run<0>("st x32 -> wait -> ld x32 -> wait (128+128 B)", w, 256, out, cyc, sms);
        run<1>("ld 2 x x32 (256 B)", w, 256, out, cyc, sms);
        run<2>("st 2 x x32 (256 B)", w, 256, out, cyc, sms);
        run<5>("16 SHFL.64 only", w, 0, out, cyc, sms);
        run<3>("round trip + 16 SHFL.64", w, 256, out, cyc, sms);
        run<6>("32 DADD only", w, 0, out, cyc, sms);
        run<4>("round trip + 32 DADD", w, 256, out, cyc, sms);
        run<7>("pipelined st/ld x32 around 32 DADD", w, 256, out, cyc, sms);
    }
    return 0;
}
