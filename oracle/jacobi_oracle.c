/*
 * CPU ORACLE — test infrastructure only.
 *
 * Plain-C restatement of the reference `stencilpipe` Jacobi hot path
 * (/root/reference/pkg/src/stencilpipe, pure Python + NumPy).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product path (paper_1006_3148_b200) never does.
 *
 * Parity is pinned: tests/test_oracle.py checks this code against the
 * reference's own frozen digests (FIELD_60_SEED42, FIELD_600_SEED42,
 * REF_60_SEED42_8SWEEPS from pkg/tests/test_grid.py:18-19 and
 * pkg/tests/test_kernel.py:17) and against fixtures produced by importing the
 * reference itself (tests/golden/make_golden.py).
 *
 * Arithmetic contract (sp/kernel.py:51-57 / 28-29): each cell is
 *   ((((((x-1 + x+1) + y-1) + y+1) + z-1) + z+1) * SIXTH),  SIXTH = fl(1/6)
 * in IEEE binary64 round-to-nearest; compile with -ffp-contract=off so no
 * FMA contraction changes a bit.
 *
 * Storage: one C-contiguous double array, axes (z, y, x), extents (ez, ey, ex)
 * = n + 2 + pad per axis (sp/grid.py:117-121).  Logical cell c lives at storage
 * index off + c with off = pad + 1 - alignment (sp/grid.py:136-145).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static const double SIXTH = 1.0 / 6.0; /* sp/kernel.py:16 */

/* sp/grid.py:21-30 (splitmix64_unit): values for linear indices start..start+count-1 */
void or_splitmix64_unit(uint64_t start, uint64_t count, uint64_t seed, double *out)
{
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t z = (start + i) * 0x9E3779B97F4A7C15ULL + seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z = z ^ (z >> 31);
        out[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    }
}

#define IDX(z, y, x) (((int64_t)(z) * ey + (y)) * ex + (x))

/*
 * sp/kernel.py:36-58 (apply_window).  Window is half-open in logical
 * coordinates; src_off/dst_off translate logical 0 to storage index.  The
 * whole window is computed before any store (sp/kernel.py:41-44), which makes
 * aliased, diagonally shifted in-place writes safe: when src == dst and the
 * offsets differ we go through a temporary exactly as NumPy's `buf` does.
 */
int or_apply_window(const double *src, double *dst, int64_t ez, int64_t ey, int64_t ex,
                    int64_t xl, int64_t xh, int64_t yl, int64_t yh, int64_t zl, int64_t zh,
                    int64_t so, int64_t dso, int threads)
{
    (void)ez;
    if (xl >= xh || yl >= yh || zl >= zh) return 0;
    int64_t wx = xh - xl, wy = yh - yl, wz = zh - zl;
    int alias = (src == dst) && (so != dso);
    double *buf = NULL;
    if (alias) {
        buf = (double *)malloc(sizeof(double) * (size_t)(wx * wy * wz));
        if (!buf) return -1;
    }
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (int64_t k = zl; k < zh; ++k) {
        for (int64_t j = yl; j < yh; ++j) {
            const double *c = src + IDX(k + so, j + so, so);
            const double *ym = src + IDX(k + so, j + so - 1, so);
            const double *yp = src + IDX(k + so, j + so + 1, so);
            const double *zm = src + IDX(k + so - 1, j + so, so);
            const double *zp = src + IDX(k + so + 1, j + so, so);
            double *o = alias ? buf + ((k - zl) * wy + (j - yl)) * wx - xl
                              : dst + IDX(k + dso, j + dso, dso);
            for (int64_t i = xl; i < xh; ++i) {
                double s = c[i - 1] + c[i + 1];
                s = s + ym[i];
                s = s + yp[i];
                s = s + zm[i];
                s = s + zp[i];
                o[i] = s * SIXTH;
            }
        }
    }
    if (alias) {
        for (int64_t k = zl; k < zh; ++k)
            for (int64_t j = yl; j < yh; ++j)
                memcpy(dst + IDX(k + dso, j + dso, xl + dso),
                       buf + ((k - zl) * wy + (j - yl)) * wx, sizeof(double) * (size_t)wx);
        free(buf);
    }
    return 0;
}

/* sp/kernel.py:85-96 (_copy_ring): the full one-cell shell (faces with their
 * edges and corners) of A onto B at the same frame offset `off`. */
void or_copy_ring(const double *a, double *b, int64_t ez, int64_t ey, int64_t ex,
                  int64_t nx, int64_t ny, int64_t nz, int64_t off)
{
    (void)ez;
    int64_t zl = off - 1, zh = off + nz + 1;
    int64_t yl = off - 1, yh = off + ny + 1;
    int64_t xl = off - 1, xh = off + nx + 1;
    for (int64_t z = zl; z < zh; ++z)
        for (int64_t y = yl; y < yh; ++y) {
            int zface = (z == zl || z == zh - 1), yface = (y == yl || y == yh - 1);
            if (zface || yface) {
                memcpy(b + IDX(z, y, xl), a + IDX(z, y, xl), sizeof(double) * (size_t)(xh - xl));
            } else {
                b[IDX(z, y, xl)] = a[IDX(z, y, xl)];
                b[IDX(z, y, xh - 1)] = a[IDX(z, y, xh - 1)];
            }
        }
}

/* sp/kernel.py:99-111 (reference_sweep): B.interior = stencil(A); B.ring = A.ring */
int or_reference_sweep(const double *a, double *b, int64_t ez, int64_t ey, int64_t ex,
                       int64_t nx, int64_t ny, int64_t nz, int64_t off, int threads)
{
    int rc = or_apply_window(a, b, ez, ey, ex, 0, nx, 0, ny, 0, nz, off, off, threads);
    if (rc) return rc;
    or_copy_ring(a, b, ez, ey, ex, nx, ny, nz, off);
    return 0;
}

/* `sweeps` reference sweeps alternating a, b = b, a (tests/conftest.py:20-23,
 * sp/cli.py:161-167).  Returns 0 if the result is in `a`, 1 if in `b`. */
int or_sweeps(double *a, double *b, int64_t ez, int64_t ey, int64_t ex,
              int64_t nx, int64_t ny, int64_t nz, int64_t off, int64_t sweeps, int threads)
{
    double *cur = a, *nxt = b;
    for (int64_t s = 0; s < sweeps; ++s) {
        or_reference_sweep(cur, nxt, ez, ey, ex, nx, ny, nz, off, threads);
        double *t = cur; cur = nxt; nxt = t;
    }
    return cur == a ? 0 : 1;
}

int or_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
