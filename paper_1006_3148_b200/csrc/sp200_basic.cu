// K0 seeded fill, the generic apply_window seam, ring copy and face writes.
//
// These are the small / general-shape kernels.  The bandwidth-critical sweep
// and the temporally blocked passes live in sp200_temporal.cu.
#include <mutex>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>

#include "sp200_device.cuh"
#include "sp200_internal.h"

namespace sp200 {

// ---------------------------------------------------------------------------
// status / bookkeeping
// ---------------------------------------------------------------------------

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return SP_OK;
}

void count_launch(int n) { g_launches.fetch_add(n); }

Tuning &tuning() {
    static Tuning t;
    return t;
}

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// ---------------------------------------------------------------------------
// K0: seeded fill (sp/grid.py:21-30, 123-147; sp/halo.py:132-168)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double splitmix64_unit(uint64_t idx, uint64_t seed) {
    uint64_t z = idx * 0x9E3779B97F4A7C15ULL + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    // (z >> 11) < 2^53 converts exactly; the product by 2^-53 is exact.
    return dmul(static_cast<double>(z >> 11), 1.0 / 9007199254740992.0);
}

struct FillArgs {
    double *data;
    int64_t ex, ey, ez, off, nx, ny, nz, gx0, gy0, gz0, GX, GY, GZ;
    uint64_t seed;
    double lo, span, shell;
    int remap;
};

__global__ void k_fill_seeded(FillArgs a) {
    const int64_t total = a.ex * a.ey * a.ez;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t x = idx % a.ex;
        int64_t r = idx / a.ex;
        int64_t y = r % a.ey;
        int64_t z = r / a.ey;
        int64_t i = x - a.off, j = y - a.off, k = z - a.off;
        double v = a.shell;
        if (i >= 0 && i < a.nx && j >= 0 && j < a.ny && k >= 0 && k < a.nz) {
            int64_t gx = a.gx0 + i, gy = a.gy0 + j, gz = a.gz0 + k;
            if (gx >= 0 && gx < a.GX && gy >= 0 && gy < a.GY && gz >= 0 && gz < a.GZ) {
                uint64_t lin = (uint64_t)((gz * a.GY + gy) * a.GX + gx);
                v = splitmix64_unit(lin, a.seed);
                if (a.remap) v = dadd(a.lo, dmul(a.span, v));
            } else {
                v = 0.0;  // outside the global interior (sp/halo.py:137-141)
            }
        }
        a.data[idx] = v;
    }
}

__global__ void k_fill_constant(double *d, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        d[i] = v;
}

static int grid_for(int64_t n, int block) {
    int64_t b = (n + block - 1) / block;
    int64_t cap = (int64_t)sm_count() * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// ---------------------------------------------------------------------------
// generic window kernel (the apply_window seam, any shape / alignment)
// ---------------------------------------------------------------------------

struct WinArgs {
    const double *src;
    double *dst;          // final destination frame (or scratch)
    int64_t ex, ey;
    int64_t xl, yl, zl, wx, wy, wz;
    int64_t so;
    // destination addressing: dst + ((k+dz)*dey + (j+dy))*dex + (i+dx)
    int64_t dex, dey, dxo, dyo, dzo;
};

// One thread per (x, y) column of the window, marching a z-chunk of WZC
// planes: the z-neighbours rotate through registers (one new load per cell),
// the x/y neighbours of the current plane come through L1 from the loads of
// the adjacent threads, and the index math is 32-bit per thread, set up once.
// Replaces the first version's one-thread-per-cell form (seven loads and a
// 64-bit div/mod chain per cell).  Same summation order as every kernel.
constexpr int WBX = 32, WBY = 8, WZC = 16;

__global__ void __launch_bounds__(WBX * WBY) k_window(WinArgs a) {
    const int ii = blockIdx.x * WBX + threadIdx.x, jj = blockIdx.y * WBY + threadIdx.y;
    if (ii >= a.wx || jj >= a.wy) return;
    const int kk0 = blockIdx.z * WZC;
    const int kk1 = min((int64_t)kk0 + WZC, a.wz);
    const int64_t py = a.ex, pz = a.ex * a.ey;
    const double *c = a.src + ((a.zl + kk0 + a.so) * a.ey + (a.yl + jj + a.so)) * a.ex + (a.xl + ii + a.so);
    double *d = a.dst + ((kk0 + a.dzo) * a.dey + (jj + a.dyo)) * a.dex + (ii + a.dxo);
    const int64_t dpz = a.dex * a.dey;
    double zm = __ldg(c - pz), z0 = __ldg(c);
    for (int kk = kk0; kk < kk1; ++kk) {
        const double zp = __ldg(c + pz);
        *d = stencil7(__ldg(c - 1), __ldg(c + 1), __ldg(c - py), __ldg(c + py), zm, zp);
        zm = z0;
        z0 = zp;
        c += pz;
        d += dpz;
    }
}

static void launch_window(const WinArgs &a, cudaStream_t s) {
    dim3 grid((unsigned)((a.wx + WBX - 1) / WBX), (unsigned)((a.wy + WBY - 1) / WBY),
              (unsigned)((a.wz + WZC - 1) / WZC));
    k_window<<<grid, dim3(WBX, WBY), 0, s>>>(a);
}

// scratch (wz, wy, wx) -> dst frame: one window row per CTA row (grid-stride
// over the wy * wz rows), threads along x
__global__ void k_unstage(const double *scratch, double *dst, int64_t ex, int64_t ey,
                          int64_t xo, int64_t yo, int64_t zo, int64_t wx, int64_t wy,
                          int64_t wz) {
    const int64_t rows = wy * wz;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const int64_t kk = r / wy, jj = r - kk * wy;
        const double *s = scratch + r * wx;
        double *d = dst + ((kk + zo) * ey + (jj + yo)) * ex + xo;
        for (int64_t ii = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ii < wx;
             ii += (int64_t)gridDim.x * blockDim.x)
            d[ii] = s[ii];
    }
}

// ---------------------------------------------------------------------------
// ring copy (sp/kernel.py:85-96) and face writes (sp/pipeline.py:427-447)
// ---------------------------------------------------------------------------

// Shell cells at frame off: coords in [off-1, off+n] on all axes with at least
// one coordinate on the ring.  Enumerated as: two full z planes, then the two
// y rows of every interior z plane, then the two x columns of the remaining
// (interior z, interior y) rows.
__device__ __forceinline__ int64_t shell_index(int64_t idx, int64_t ex, int64_t ey, int64_t nx,
                                               int64_t ny, int64_t nz, int64_t off) {
    const int64_t PX = nx + 2, PY = ny + 2;
    const int64_t nzf = 2 * PX * PY, nyf = 2 * nz * PX;
    int64_t x, y, z;
    if (idx < nzf) {
        int64_t f = idx / (PX * PY), r = idx % (PX * PY);
        z = f ? off + nz : off - 1;
        y = off - 1 + r / PX;
        x = off - 1 + r % PX;
    } else if (idx < nzf + nyf) {
        int64_t q = idx - nzf;
        int64_t f = q / (nz * PX), r = q % (nz * PX);
        z = off + r / PX;
        y = f ? off + ny : off - 1;
        x = off - 1 + r % PX;
    } else {
        int64_t q = idx - nzf - nyf;
        int64_t f = q / (nz * ny), r = q % (nz * ny);
        z = off + r / ny;
        y = off + r % ny;
        x = f ? off + nx : off - 1;
    }
    return (z * ey + y) * ex + x;
}

__global__ void k_copy_ring(const double *a, double *b, int64_t ex, int64_t ey, int64_t nx,
                            int64_t ny, int64_t nz, int64_t off) {
    const int64_t total = 2 * (nx + 2) * (ny + 2) + 2 * nz * (nx + 2) + 2 * nz * ny;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = shell_index(idx, ex, ey, nx, ny, nz, off);
        b[p] = a[p];
    }
}

// Ring equality (the precondition of fused two-grid passes).  The verdict is
// written straight into host-mapped memory, so reading it waits only for
// this stream, never behind bulk copies queued on the copy engines.
__global__ void k_rings_equal(const double *a, const double *b, int64_t ex, int64_t ey,
                              int64_t nx, int64_t ny, int64_t nz, int64_t off,
                              volatile int *verdict) {
    const int64_t total = 2 * (nx + 2) * (ny + 2) + 2 * nz * (nx + 2) + 2 * nz * ny;
    bool same = true;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = shell_index(idx, ex, ey, nx, ny, nz, off);
        same = same && (a[p] == b[p]);
    }
    if (__any_sync(0xffffffffu, !same) && (threadIdx.x & 31) == 0) *verdict = 0;
}

struct FaceArgs {
    double *d;
    int64_t ex, ey, nx, ny, nz, off;
    const double *f[6];
    int mask;
};

// faces: (x,0),(x,1): [nz][ny]; (y,0),(y,1): [nz][nx]; (z,0),(z,1): [ny][nx]
// One face row per CTA row (blockIdx.y strides over the 2nz + 2nz + 2ny face
// rows; comparisons pick the face), threads along the row: no per-element
// 64-bit division.  The earlier flat-index form spent most of its 42 us per
// call (600^3) in the div/mod chain.
__global__ void k_write_faces(FaceArgs a) {
    const int64_t nrows = 4 * a.nz + 2 * a.ny;
    for (int64_t row = blockIdx.y; row < nrows; row += gridDim.y) {
        int face;
        int64_t r0, len, base, step;  // face-array row start, length, storage base/stride
        if (row < 2 * a.nz) {
            face = row >= a.nz;
            const int64_t z = row - face * a.nz;
            r0 = z * a.ny;
            len = a.ny;
            base = ((a.off + z) * a.ey + a.off) * a.ex + (face ? a.off + a.nx : a.off - 1);
            step = a.ex;
        } else if (row < 4 * a.nz) {
            const int64_t q = row - 2 * a.nz;
            face = 2 + (q >= a.nz);
            const int64_t z = q - (face - 2) * a.nz;
            r0 = z * a.nx;
            len = a.nx;
            base = ((a.off + z) * a.ey + ((face & 1) ? a.off + a.ny : a.off - 1)) * a.ex + a.off;
            step = 1;
        } else {
            const int64_t q = row - 4 * a.nz;
            face = 4 + (q >= a.ny);
            const int64_t y = q - (face - 4) * a.ny;
            r0 = y * a.nx;
            len = a.nx;
            base = (((face & 1) ? a.off + a.nz : a.off - 1) * a.ey + a.off + y) * a.ex + a.off;
            step = 1;
        }
        if (!((a.mask >> face) & 1)) continue;
        const double *f = a.f[face] + r0;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
             i += (int64_t)gridDim.x * blockDim.x)
            a.d[base + i * step] = f[i];
    }
}

}  // namespace sp200

using namespace sp200;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

int sp_version(void) { return 10000; }

const char *sp_last_error(void) { return g_err; }

int64_t sp_launch_count(int reset) {
    int64_t v = g_launches.load();
    if (reset) g_launches.store(0);
    return v;
}

int sp_set_tuning(int key, int64_t value) {
    Tuning &t = tuning();
    switch (key) {
    case 0: t.zchunk = value; return SP_OK;
    case 1: t.force_cpasync = value; return SP_OK;
    case 4: t.debug = value; return SP_OK;
    case 5: t.signal_kernels = value; return SP_OK;
    case 6: t.two_launch = value; return SP_OK;
    case 7: t.balanced_split = value; return SP_OK;
    case 8: t.zchunk2 = value; return SP_OK;
    case 10: t.k3_stash = value; return SP_OK;
    case 9:
        if (value < 0 || value > 15) return set_error(SP_EINVAL, "k2 layout %lld outside [0, 15]", (long long)value);
        t.k2_layout = value;
        return SP_OK;
    case 2: {
        int lv = (int)(value / 16), idx = (int)(value % 16);
        if (lv < 1 || lv > SP_MAX_FUSED) return set_error(SP_EINVAL, "bad levels in tuning");
        t.cfg_index[lv] = idx;
        return SP_OK;
    }
    default: return set_error(SP_EINVAL, "unknown tuning key %d", key);
    }
}

static int check_geom(int64_t ex, int64_t ey, int64_t ez, int64_t nx, int64_t ny, int64_t nz,
                      int64_t off) {
    if (nx < 1 || ny < 1 || nz < 1)
        return set_error(SP_EINVAL, "grid dimensions must be >= 1, got (%lld, %lld, %lld)",
                         (long long)nx, (long long)ny, (long long)nz);
    if (off < 1 || off + nx + 1 > ex || off + ny + 1 > ey || off + nz + 1 > ez)
        return set_error(SP_EINVAL, "frame offset %lld does not fit storage (%lld, %lld, %lld)",
                         (long long)off, (long long)ex, (long long)ey, (long long)ez);
    return SP_OK;
}

int sp_fill_seeded(double *data, int64_t ex, int64_t ey, int64_t ez, int64_t off, int64_t nx,
                   int64_t ny, int64_t nz, int64_t gx0, int64_t gy0, int64_t gz0, int64_t GX,
                   int64_t GY, int64_t GZ, uint64_t seed, double lo, double hi, double shell,
                   void *stream) {
    if (!data) return set_error(SP_EINVAL, "null data");
    int rc = check_geom(ex, ey, ez, nx, ny, nz, off);
    if (rc) return rc;
    FillArgs a{data, ex, ey, ez, off, nx, ny, nz, gx0, gy0, gz0, GX, GY, GZ, seed,
               lo,   hi - lo, shell, (lo != 0.0 || hi != 1.0) ? 1 : 0};
    int64_t total = ex * ey * ez;
    k_fill_seeded<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(a);
    count_launch();
    return check_launch("sp_fill_seeded");
}

int sp_fill_constant(double *data, int64_t count, double value, void *stream) {
    if (!data || count < 0) return set_error(SP_EINVAL, "bad fill arguments");
    if (count == 0) return SP_OK;
    k_fill_constant<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(data, count, value);
    count_launch();
    return check_launch("sp_fill_constant");
}

int sp_apply_window(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                    int64_t xl, int64_t xh, int64_t yl, int64_t yh, int64_t zl, int64_t zh,
                    int64_t so, int64_t dso, double *scratch, void *stream) {
    if (!src || !dst) return set_error(SP_EINVAL, "null grid");
    if (xl >= xh || yl >= yh || zl >= zh) return SP_OK;  // empty window (sp/kernel.py:47-48)
    // every read src[k+so +-1] and write dst[k+dso] must be inside storage
    if (xl + so - 1 < 0 || xh + so + 1 > ex || yl + so - 1 < 0 || yh + so + 1 > ey ||
        zl + so - 1 < 0 || zh + so + 1 > ez || xl + dso < 0 || xh + dso > ex || yl + dso < 0 ||
        yh + dso > ey || zl + dso < 0 || zh + dso > ez)
        return set_error(SP_EINVAL, "window outside storage");
    const int64_t wx = xh - xl, wy = yh - yl, wz = zh - zl;
    const bool alias = (src == dst) && (so != dso);
    if (alias && !scratch)
        return set_error(SP_EINVAL, "shifted in-place window needs a scratch buffer");
    WinArgs a;
    a.src = src;
    a.ex = ex;
    a.ey = ey;
    a.xl = xl;
    a.yl = yl;
    a.zl = zl;
    a.wx = wx;
    a.wy = wy;
    a.wz = wz;
    a.so = so;
    if (alias) {
        a.dst = scratch;
        a.dex = wx;
        a.dey = wy;
        a.dxo = a.dyo = a.dzo = 0;
    } else {
        a.dst = dst;
        a.dex = ex;
        a.dey = ey;
        a.dxo = xl + dso;
        a.dyo = yl + dso;
        a.dzo = zl + dso;
    }
    cudaStream_t s = as_stream(stream);
    launch_window(a, s);
    count_launch();
    int rc = check_launch("sp_apply_window");
    if (rc || !alias) return rc;
    const int64_t urows = wy * wz;
    dim3 ug((unsigned)((wx + 255) / 256), (unsigned)(urows < 65535 ? urows : 65535));
    k_unstage<<<ug, 256, 0, s>>>(scratch, dst, ex, ey, xl + dso, yl + dso,
                                                   zl + dso, wx, wy, wz);
    count_launch();
    return check_launch("sp_apply_window(unstage)");
}

int sp_window_gather(const double *src, int64_t ex, int64_t ey, int64_t ez, int64_t xl,
                     int64_t xh, int64_t yl, int64_t yh, int64_t zl, int64_t zh, int64_t so,
                     double *out, void *stream) {
    if (!src || !out) return set_error(SP_EINVAL, "null argument");
    if (xl >= xh || yl >= yh || zl >= zh) return SP_OK;
    if (xl + so - 1 < 0 || xh + so + 1 > ex || yl + so - 1 < 0 || yh + so + 1 > ey ||
        zl + so - 1 < 0 || zh + so + 1 > ez)
        return set_error(SP_EINVAL, "window outside storage");
    WinArgs a;
    a.src = src;
    a.ex = ex;
    a.ey = ey;
    a.xl = xl;
    a.yl = yl;
    a.zl = zl;
    a.wx = xh - xl;
    a.wy = yh - yl;
    a.wz = zh - zl;
    a.so = so;
    a.dst = out;
    a.dex = a.wx;
    a.dey = a.wy;
    a.dxo = a.dyo = a.dzo = 0;
    launch_window(a, as_stream(stream));
    count_launch();
    return check_launch("sp_window_gather");
}

int sp_copy_ring(const double *a, double *b, int64_t ex, int64_t ey, int64_t ez, int64_t nx,
                 int64_t ny, int64_t nz, int64_t off, void *stream) {
    if (!a || !b) return set_error(SP_EINVAL, "null grid");
    int rc = check_geom(ex, ey, ez, nx, ny, nz, off);
    if (rc) return rc;
    int64_t total = 2 * (nx + 2) * (ny + 2) + 2 * nz * (nx + 2) + 2 * nz * ny;
    k_copy_ring<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(a, b, ex, ey, nx, ny, nz,
                                                                      off);
    count_launch();
    return check_launch("sp_copy_ring");
}

int sp_rings_equal(const double *a, const double *b, int64_t ex, int64_t ey, int64_t ez,
                   int64_t nx, int64_t ny, int64_t nz, int64_t off, int *equal, void *stream) {
    if (!a || !b || !equal) return set_error(SP_EINVAL, "null argument");
    int rc = check_geom(ex, ey, ez, nx, ny, nz, off);
    if (rc) return rc;
    // one mapped flag per host thread: concurrent callers on other threads
    // (and their streams) never share it, so no lock is needed
    static thread_local int *host_flag = nullptr, *dev_flag = nullptr;
    if (!host_flag) {
        if (cudaHostAlloc(reinterpret_cast<void **>(&host_flag), sizeof(int), cudaHostAllocMapped) !=
                cudaSuccess ||
            cudaHostGetDevicePointer(reinterpret_cast<void **>(&dev_flag), host_flag, 0) !=
                cudaSuccess) {
            host_flag = nullptr;
            return set_error(SP_ECUDA, "mapped host flag: %s", cudaGetErrorString(cudaGetLastError()));
        }
    }
    *reinterpret_cast<volatile int *>(host_flag) = 1;
    int64_t total = 2 * (nx + 2) * (ny + 2) + 2 * nz * (nx + 2) + 2 * nz * ny;
    k_rings_equal<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(a, b, ex, ey, nx, ny, nz,
                                                                        off, dev_flag);
    count_launch();
    rc = check_launch("sp_rings_equal");
    if (rc) return rc;
    if (cudaStreamSynchronize(as_stream(stream)) != cudaSuccess)
        return set_error(SP_ECUDA, "sp_rings_equal: %s", cudaGetErrorString(cudaGetLastError()));
    *equal = *reinterpret_cast<volatile int *>(host_flag);
    return SP_OK;
}

int sp_write_faces(double *data, int64_t ex, int64_t ey, int64_t ez, int64_t nx, int64_t ny,
                   int64_t nz, int64_t off, const double *const faces[6], int side_mask,
                   void *stream) {
    if (!data || !faces) return set_error(SP_EINVAL, "null argument");
    int rc = check_geom(ex, ey, ez, nx, ny, nz, off);
    if (rc) return rc;
    FaceArgs a;
    a.d = data;
    a.ex = ex;
    a.ey = ey;
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    a.off = off;
    a.mask = side_mask & 63;
    for (int f = 0; f < 6; ++f) {
        a.f[f] = faces[f];
        if (((a.mask >> f) & 1) && !faces[f]) return set_error(SP_EINVAL, "null face %d", f);
    }
    if (!a.mask) return SP_OK;
    const int64_t len = nx > ny ? nx : ny, nrows = 4 * nz + 2 * ny;
    dim3 grid((unsigned)((len + 127) / 128), (unsigned)(nrows < 65535 ? nrows : 65535));
    k_write_faces<<<grid, 128, 0, as_stream(stream)>>>(a);
    count_launch();
    return check_launch("sp_write_faces");
}

int sp_sweep(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez, int64_t nx,
             int64_t ny, int64_t nz, int64_t off, int copy_ring, void *stream) {
    if (!src || !dst) return set_error(SP_EINVAL, "null grid");
    if (src == dst) return set_error(SP_EINVAL, "sp_sweep: src and dst must differ");
    int rc = check_geom(ex, ey, ez, nx, ny, nz, off);
    if (rc) return rc;
    return launch_temporal(src, dst, ex, ey, ez, nx, ny, nz, off, 1, 0, nz, copy_ring != 0,
                           as_stream(stream));
}

int sp_temporal(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez, int64_t nx,
                int64_t ny, int64_t nz, int64_t off, int levels, int64_t zlo, int64_t zhi,
                void *stream) {
    if (!src || !dst) return set_error(SP_EINVAL, "null grid");
    if (src == dst) return set_error(SP_EINVAL, "sp_temporal: src and dst must differ");
    int rc = check_geom(ex, ey, ez, nx, ny, nz, off);
    if (rc) return rc;
    // A/B builds also carry deeper experimental instances (T = 5, 8)
    if (levels < 1 || levels > (SP200_AB ? 8 : SP_MAX_FUSED))
        return set_error(SP_EUNSUP, "levels %d outside [1, %d]", levels, SP_MAX_FUSED);
    if (zlo < 0) zlo = 0;
    if (zhi > nz) zhi = nz;
    if (zlo >= zhi) return SP_OK;
    return launch_temporal(src, dst, ex, ey, ez, nx, ny, nz, off, levels, zlo, zhi, false,
                           as_stream(stream));
}

int sp_temporal_mirror(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                       int64_t nx, int64_t ny, int64_t nz, int64_t off, int levels, int64_t zlo,
                       int64_t zhi, double *mirror, int64_t mirror_ez, int64_t mirror_zshift,
                       void *stream) {
    if (!src || !dst || !mirror) return set_error(SP_EINVAL, "null grid");
    if (src == dst) return set_error(SP_EINVAL, "sp_temporal_mirror: src and dst must differ");
    int rc = check_geom(ex, ey, ez, nx, ny, nz, off);
    if (rc) return rc;
    if (levels < 1 || levels > SP_MAX_FUSED)
        return set_error(SP_EUNSUP, "levels %d outside [1, %d]", levels, SP_MAX_FUSED);
    if (zlo < 0) zlo = 0;
    if (zhi > nz) zhi = nz;
    if (zlo >= zhi) return SP_OK;
    // the mirrored storage planes must exist in the peer grid
    if (zlo + off + mirror_zshift < 0 || zhi + off + mirror_zshift > mirror_ez)
        return set_error(SP_EINVAL, "mirror planes [%lld, %lld) outside the peer grid (%lld planes)",
                         (long long)(zlo + off + mirror_zshift), (long long)(zhi + off + mirror_zshift),
                         (long long)mirror_ez);
    return launch_temporal_mirror(src, dst, ex, ey, ez, nx, ny, nz, off, levels, zlo, zhi, mirror,
                                  mirror_zshift, as_stream(stream));
}

int sp_tma_eligible(int64_t ex, int64_t ey) { return tma_eligible(nullptr, ex, ey) ? 1 : 0; }

int64_t sp_compressed_workspace(int64_t nx, int64_t ny, int64_t depth, int levels) {
    if (nx < 1 || ny < 1 || depth < 1 || levels < 1 || levels > SP_MAX_FUSED) return 0;
    return compressed_workspace(nx, ny, depth, levels);
}

int64_t sp_compressed_workspace_for(const double *data, int64_t ex, int64_t ey, int64_t nx, int64_t ny,
                                    int64_t depth, int levels) {
    if (nx < 1 || ny < 1 || depth < 1 || levels < 1 || levels > SP_MAX_FUSED) return 0;
    return compressed_workspace_for(data, ex, ey, nx, ny, depth, levels);
}

int sp_compressed(double *data, int64_t ex, int64_t ey, int64_t ez, int64_t nx, int64_t ny,
                  int64_t nz, int64_t src_off, int direction, int levels, int64_t zlo,
                  int64_t zhi, void *workspace, int64_t workspace_bytes,
                  const double *const faces[6], int side_mask, void *stream) {
    if (!data || !workspace) return set_error(SP_EINVAL, "null argument");
    if (direction != 1 && direction != -1) return set_error(SP_EINVAL, "direction must be +1 or -1");
    if (levels < 1 || levels > SP_MAX_FUSED)
        return set_error(SP_EUNSUP, "levels %d outside [1, %d]", levels, SP_MAX_FUSED);
    int rc = check_geom(ex, ey, ez, nx, ny, nz, src_off);
    if (rc) return rc;
    const int64_t doff = src_off - (direction > 0 ? levels : -levels);
    rc = check_geom(ex, ey, ez, nx, ny, nz, doff);
    if (rc) return set_error(SP_EINVAL, "shifted frame (offset %lld) leaves the padded storage",
                             (long long)doff);
    if (zlo < 0) zlo = 0;
    if (zhi > nz) zhi = nz;
    if (zlo < zhi) {
        rc = launch_compressed(data, ex, ey, ez, nx, ny, nz, src_off, direction, levels, zlo, zhi,
                               workspace, workspace_bytes, as_stream(stream));
        if (rc) return rc;
    }
    if (faces && side_mask) return sp_write_faces(data, ex, ey, ez, nx, ny, nz, doff, faces,
                                                  side_mask, stream);
    return SP_OK;
}

}  // extern "C"
