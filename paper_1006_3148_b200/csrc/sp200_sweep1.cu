// K1: the plain streaming sweep (reference_sweep) with the fused ring copy.
//
// One kernel template covers both: K1 is the depth-1 instance (plus the fused
// Dirichlet-ring copy of reference_sweep), K2 fuses T = 2..4 sweeps per HBM
// pass.  Design (B200-first):
//
//  * A CTA owns an x-y tile and marches along z over a chunk of planes.  The
//    level-0 input planes are staged by TMA (cp.async.bulk.tensor.3d, one
//    elected thread, mbarrier completion) into an S-deep ring of shared-memory
//    stages; a cp.async loader replaces TMA when the row pitch is not a
//    multiple of 16 bytes.
//  * Level u (1..T) is computed by the same thread for the same cells as level
//    u-1, so the z-neighbour chain stays in registers: per cell and level the
//    thread keeps the pending partial sum S = (((x-1 + x+1) + y-1) + y+1) + z-1
//    and the previous plane's value; the +z+1 term and the x fl(1/6) finish the
//    cell one plane later — exactly the reference order (sp/kernel.py:51-57).
//  * In-plane neighbours of level u-1 come from shared memory: level u-1
//    publishes each plane into a double-buffered smem plane, read by level u
//    one step later (one __syncthreads per z step for all T levels).  A thread
//    owns R consecutive rows of one column, so y-neighbours inside its rows
//    come from registers.
//  * Overlapped (ghost-zone) tiling: the CTA computes a CX x CY region at
//    every level; the valid output shrinks by one cell per side per level, so
//    the stored tile is (CX-2(T-1)) x (CY-2(T-1)).  Cells outside the interior
//    (Dirichlet ring) keep their input value at every level.
#include "sp200_internal.h"
#if SP200_AB  // A/B only: the first K1, superseded by the depth-1 k_temporal
#include <string.h>

#include <algorithm>

#include "sp200_device.cuh"
#include "sp200_internal.h"

namespace sp200 {
namespace k1 {

struct TParams {
    const double *src;
    double *dst;
    int64_t ex, ey, ez;
    int nx, ny, nz, off;
    int tiles_x, ntiles;
    int zlo, zhi, zc;
};

template <int T, int WX, int CY, int R, int S>
struct KCfg {
    static constexpr int CX = WX * 32;
    static constexpr int PX = CX + 2, PY = CY + 2;  // region + 1-cell halo
    // Stages hold CX+4 columns starting at an even x: TMA boxes must start on
    // a 16-byte boundary, so an odd box origin is moved one column left and
    // read back with a one-column shift (sh).
    static constexpr int SPX = CX + 4;
    static constexpr int SPLANE = SPX * PY;
    static constexpr int SPLANE_AL = (SPLANE + 15) & ~15;  // 128-byte aligned stages
    static constexpr int PLANE_AL = (PX * PY + 15) & ~15;   // level planes
    static constexpr int NT = WX * 32 * (CY / R);
    static constexpr int OX = CX - 2 * (T - 1), OY = CY - 2 * (T - 1);
    static constexpr int NLEV = (T > 1) ? 2 * (T - 1) : 0;
    static constexpr size_t SMEM =
        ((size_t)S * SPLANE_AL + (size_t)NLEV * PLANE_AL) * sizeof(double) + 8 * S;
    static_assert(CY % R == 0, "rows per thread must divide CY");
    static_assert(OX > 0 && OY > 0, "tile too small for the fused depth");
};

template <int T, int WX, int CY, int R, int S, bool TMA, bool RING>
__global__ void __launch_bounds__(KCfg<T, WX, CY, R, S>::NT, 1)
    k_sweep1(const TParams p, const __grid_constant__ CUtensorMap tmap) {
    using C = KCfg<T, WX, CY, R, S>;
    constexpr int PX = C::PX, SPX = C::SPX, SPLANE = C::SPLANE, SPLANE_AL = C::SPLANE_AL,
                  PLANE_AL = C::PLANE_AL, NT = C::NT;

    extern __shared__ __align__(128) double sm[];
    double *stage = sm;
    double *lev = sm + S * SPLANE_AL;
    uint64_t *bar = reinterpret_cast<uint64_t *>(lev + C::NLEV * PLANE_AL);

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int i = (warp % WX) * 32 + lane;  // region column
    const int j0 = (warp / WX) * R;         // first region row

    const int tile = blockIdx.x % p.ntiles, chunk = blockIdx.x / p.ntiles;
    const int x0 = (tile % p.tiles_x) * C::OX, y0 = (tile / p.tiles_x) * C::OY;
    const int z0 = p.zlo + chunk * p.zc;
    const int z1 = min(z0 + p.zc, p.zhi);
    const int rx0 = x0 - (T - 1), ry0 = y0 - (T - 1);

    const int x = rx0 + i;
    const bool x_in = (x >= 0) && (x < p.nx);
    const bool x_out = (i >= T - 1) && (i < T - 1 + C::OX) && (x < p.nx);
    bool y_in[R], y_out[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int jr = j0 + r, y = ry0 + jr;
        y_in[r] = (y >= 0) && (y < p.ny);
        y_out[r] = (jr >= T - 1) && (jr < T - 1 + C::OY) && (y < p.ny);
    }

    const int nload = (z1 - z0) + 2 * T;      // level-0 planes z0-T .. z1+T-1
    const int nsteps = (z1 - z0) + 3 * T - 1;  // level T emits plane z0+s-3T+1 at step s
    const int bx0 = rx0 - 1 + p.off, by0 = ry0 - 1 + p.off;
    const int sh = bx0 & 1;  // stage column of storage x = bx0
    const int bxs = bx0 - sh;

    auto issue = [&](int s) {
        const int si = s % S;
        const int zs = z0 - T + s + p.off;
        if constexpr (TMA) {
            mbar_arrive_expect_tx(&bar[si], SPLANE * 8);
            tma_load_3d(stage + si * SPLANE_AL, &tmap, &bar[si], bxs, by0, zs);
        } else {
            double *dstage = stage + si * SPLANE_AL;
            const bool zok = (zs >= 0) && (zs < p.ez);
            for (int q = tid; q < SPLANE; q += NT) {
                const int gx = bxs + q % SPX, gy = by0 + q / SPX;
                const bool inb = zok && gx >= 0 && gx < p.ex && gy >= 0 && gy < p.ey;
                const double *g = inb ? p.src + ((int64_t)zs * p.ey + gy) * p.ex + gx : p.src;
                cp_async_8(dstage + q, g, inb ? 8u : 0u);
            }
            cp_async_commit();
        }
    };

    if constexpr (TMA) {
        if (tid == 0) {
            tma_prefetch_desc(&tmap);
#pragma unroll
            for (int si = 0; si < S; ++si) mbar_init(&bar[si], 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (tid == 0)
            for (int s = 0; s < S - 1; ++s)
                if (s < nload) issue(s);
    } else {
        for (int s = 0; s < S - 1; ++s) {
            if (s < nload) issue(s);
            else cp_async_commit();
        }
    }

    // per level (index u-1): pending partial sum, previous plane value, and the
    // last published value (input of level u+1)
    double Sp[T][R], Wl[T][R], Pub[T][R];
#pragma unroll
    for (int u = 0; u < T; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) Sp[u][r] = Wl[u][r] = Pub[u][r] = 0.0;

    const bool ring_tile = RING && (x0 == 0 || y0 == 0 || x0 + C::OX >= p.nx || y0 + C::OY >= p.ny);
    const int64_t pz = p.ex * p.ey;

    for (int s = 0; s < nsteps; ++s) {
        const int si = s % S;
        if constexpr (TMA) {
            if (s < nload) mbar_wait(&bar[si], (uint32_t)((s / S) & 1));
            __syncthreads();
            if (tid == 0 && s + S - 1 < nload) issue(s + S - 1);
        } else {
            cp_async_wait<S - 2>();
            __syncthreads();
            if (s + S - 1 < nload) issue(s + S - 1);
            else cp_async_commit();
        }
        const double *cur = stage + si * SPLANE_AL + sh;

        if constexpr (RING) {
            // fused _copy_ring (sp/kernel.py:85-96): shell cells of this tile's box
            const int P0 = z0 - T + s;
            const bool zring = (P0 == -1 && z0 == 0) || (P0 == p.nz && z1 == p.nz);
            const bool zmid = (P0 >= z0) && (P0 < z1);
            if (s < nload && (zring || (zmid && ring_tile))) {
                double *drow = p.dst + (int64_t)(P0 + p.off) * pz;
                for (int q = tid; q < PX * C::PY; q += NT) {
                    const int qx = q % PX, qy = q / PX;
                    const int gx = rx0 - 1 + qx, gy = ry0 - 1 + qy;
                    if (gx < -1 || gx > p.nx || gy < -1 || gy > p.ny) continue;
                    const bool shell = zring || gx == -1 || gx == p.nx || gy == -1 || gy == p.ny;
                    if (shell) drow[(int64_t)(gy + p.off) * p.ex + gx + p.off] = cur[qy * SPX + qx];
                }
            }
        }

#pragma unroll
        for (int u = T; u >= 1; --u) {
            const int pin = z0 - T + s - 2 * (u - 1);  // level u-1 plane consumed now
            const int pout = pin - 1;                  // level u plane finished now
            const bool z_in = (pout >= 0) && (pout < p.nz);
            const double *B = (u == 1) ? cur : lev + ((u - 2) * 2 + ((s - 1) & 1)) * PLANE_AL;
            const int pitch = (u == 1) ? SPX : PX;
            double w[R];
#pragma unroll
            for (int r = 0; r < R; ++r)
                w[r] = (u == 1) ? B[(j0 + r + 1) * pitch + i + 1] : Pub[u - 2][r];
            const double cm = B[j0 * pitch + i + 1];
            const double cp = B[(j0 + R + 1) * pitch + i + 1];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double xm = B[(j0 + r + 1) * pitch + i];
                const double xp = B[(j0 + r + 1) * pitch + i + 2];
                const double ym = (r == 0) ? cm : w[r - 1];
                const double yp = (r == R - 1) ? cp : w[r + 1];
                const double n = dadd(dadd(dadd(xm, xp), ym), yp);
                const double outv = (x_in && y_in[r] && z_in)
                                        ? dmul(dadd(Sp[u - 1][r], w[r]), 1.0 / 6.0)
                                        : Wl[u - 1][r];
                Sp[u - 1][r] = dadd(n, Wl[u - 1][r]);
                Wl[u - 1][r] = w[r];
                if (u < T) {
                    Pub[u - 1][r] = outv;
                    lev[((u - 1) * 2 + (s & 1)) * PLANE_AL + (j0 + r + 1) * PX + i + 1] = outv;
                } else if (x_out && y_out[r] && pout >= z0 && pout < z1) {
                    st_stream(p.dst + (int64_t)(pout + p.off) * pz +
                                  (int64_t)(ry0 + j0 + r + p.off) * p.ex + (x + p.off),
                              outv);
                }
            }
        }
    }
    if constexpr (!TMA) cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}


template <int T, int WX, int CY, int R, int S>
static int launch_cfg(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                      int64_t nx, int64_t ny, int64_t nz, int64_t off, int64_t zlo, int64_t zhi,
                      bool copy_ring, cudaStream_t stream) {
    using C = KCfg<T, WX, CY, R, S>;
    const bool use_tma = !tuning().force_cpasync && tma_eligible(src, ex, ey) && encode_fn();

    TParams p;
    p.src = src;
    p.dst = dst;
    p.ex = ex;
    p.ey = ey;
    p.ez = ez;
    p.nx = (int)nx;
    p.ny = (int)ny;
    p.nz = (int)nz;
    p.off = (int)off;
    p.tiles_x = (int)((nx + C::OX - 1) / C::OX);
    const int tiles_y = (int)((ny + C::OY - 1) / C::OY);
    p.ntiles = p.tiles_x * tiles_y;
    p.zlo = (int)zlo;
    p.zhi = (int)zhi;

    void (*kern)(const TParams, const CUtensorMap);
    if constexpr (T == 1) {
        if (use_tma)
            kern = copy_ring ? k_sweep1<T, WX, CY, R, S, true, true>
                             : k_sweep1<T, WX, CY, R, S, true, false>;
        else
            kern = copy_ring ? k_sweep1<T, WX, CY, R, S, false, true>
                             : k_sweep1<T, WX, CY, R, S, false, false>;
    } else {
        if (copy_ring) return set_error(SP_EUNSUP, "ring copy is fused only into the plain sweep");
        kern = use_tma ? k_sweep1<T, WX, CY, R, S, true, false>
                       : k_sweep1<T, WX, CY, R, S, false, false>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess)
        return set_error(SP_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));

    // z-chunking: choose the chunk count minimising (waves x steps per chunk)
    const int64_t depth = zhi - zlo;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, C::SMEM);
    if (occ < 1) occ = 1;
    const int64_t slots = (int64_t)sm_count() * occ;
    int64_t zc = tuning().zchunk;
    if (zc <= 0) {
        // Chunks of 24-40 planes measured fastest on every size (512^3: 379
        // vs 355 GLUP/s for whole columns, 2048^3: 357 vs 279): concurrently
        // running CTAs re-align in z at every chunk, so their streams keep
        // hitting the same DRAM pages instead of drifting apart.
        const int64_t lmin = std::min<int64_t>(depth, 24), lmax = 40;
        double best = 1e300;
        for (int64_t c = 1; c <= 4096 && c <= depth; ++c) {
            int64_t len = (depth + c - 1) / c;
            if (len > lmax || len < lmin) continue;
            int64_t units = p.ntiles * ((depth + len - 1) / len);
            double waves = (double)((units + slots - 1) / slots);
            // partial last wave still costs a whole wave; a short chunk pays the
            // (3T-1)-step pipeline fill/drain and the 2T-plane halo reload
            double cost = waves * (double)(len + 3 * T - 1 + (T == 1 ? 1 : 0));
            if (cost < best * 0.999) {
                best = cost;
                zc = len;
            }
        }
    }
    if (zc < 1) zc = 1;
    p.zc = (int)zc;
    const int64_t nchunks = (depth + zc - 1) / zc;
    const int64_t grid = (int64_t)p.ntiles * nchunks;
    if (grid > 0x7fffffff) return set_error(SP_EUNSUP, "grid too large");

    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (use_tma) {
        cuuint64_t dims[3] = {(cuuint64_t)ex, (cuuint64_t)ey, (cuuint64_t)ez};
        cuuint64_t strides[2] = {(cuuint64_t)(ex * 8), (cuuint64_t)(ex * ey * 8)};
        cuuint32_t box[3] = {(cuuint32_t)C::SPX, (cuuint32_t)C::PY, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)src, dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(SP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    kern<<<(unsigned)grid, C::NT, C::SMEM, stream>>>(p, tmap);
    count_launch();
    return check_launch("k_sweep1");
}

}  // namespace k1

int launch_sweep1(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                  int64_t nx, int64_t ny, int64_t nz, int64_t off, int64_t zlo, int64_t zhi,
                  bool copy_ring, cudaStream_t stream) {
    const int idx = (int)tuning().cfg_index[1];
    switch (idx) {
    case 1: return k1::launch_cfg<1, 2, 32, 4, 4>(src, dst, ex, ey, ez, nx, ny, nz, off, zlo, zhi, copy_ring, stream);
    case 2: return k1::launch_cfg<1, 1, 16, 2, 8>(src, dst, ex, ey, ez, nx, ny, nz, off, zlo, zhi, copy_ring, stream);
    case 3: return k1::launch_cfg<1, 2, 16, 1, 6>(src, dst, ex, ey, ez, nx, ny, nz, off, zlo, zhi, copy_ring, stream);
    default: return k1::launch_cfg<1, 2, 16, 2, 6>(src, dst, ex, ey, ez, nx, ny, nz, off, zlo, zhi, copy_ring, stream);  // 4: A/B
    }
}

}  // namespace sp200

#endif  // SP200_AB
