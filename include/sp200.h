/*
 * sp200 — C ABI of the B200-native (sm_100a) FP64 7-point Jacobi hot path.
 *
 * Drop-in boundary for the reference `stencilpipe` package (arXiv 1006.3148
 * reference, /root/reference/pkg/src/stencilpipe).  The reference has no FFI:
 * its boundary is the Python API (sp/__init__.py:4-51) plus the operator seam
 * apply_window (sp/kernel.py:36).  Each entry point below replaces one
 * reference function; the Python package paper_1006_3148_b200 binds them with
 * ctypes and keeps the reference's names, argument meaning and errors.
 *
 * Conventions
 *   - All grids are C-contiguous float64 device arrays with axes (z, y, x) and
 *     storage extents (ex, ey, ez) = n + 2 + pad per axis (sp/grid.py:117-121).
 *   - `off` = storage index of logical cell 0 on every axis
 *     (= pad + 1 - alignment, sp/grid.py:136-145).
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t;
 *     NULL = legacy default stream).  No allocation inside hot calls; no hidden
 *     global state other than the tuning table and the launch counter.
 *   - Return 0 on success, a negative SP_E* code otherwise; sp_last_error()
 *     returns a message for the calling thread.
 *   - Per-cell arithmetic is IEEE binary64 round-to-nearest in the reference
 *     order ((((((x-1 + x+1) + y-1) + y+1) + z-1) + z+1) * fl(1/6)), no FMA
 *     contraction (sp/kernel.py:51-57): results are bit-identical to the
 *     reference sweep.
 */
#ifndef SP200_H
#define SP200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_OK 0
#define SP_EINVAL (-1)   /* invalid geometry / argument (reference: ValueError) */
#define SP_EUNSUP (-2)   /* unsupported combination (e.g. levels > SP_MAX_FUSED) */
#define SP_ECUDA (-3)    /* CUDA runtime error, see sp_last_error() */
#define SP_ERANGE (-4)   /* index outside interior (reference: IndexError) */

#define SP_MAX_FUSED 4   /* max sweeps fused into one HBM pass by sp_temporal */

/* Library version (major*10000 + minor*100 + patch). */
int sp_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char *sp_last_error(void);

/* Number of kernels this library launched since the last reset (reset if
 * `reset` != 0 after reading).  Used by bench.py for "gpu_launches". */
int64_t sp_launch_count(int reset);

/*
 * Seeded fill (K0).  Replaces create_grid(init="random") (sp/grid.py:123-147)
 * and global_field_box/materialize_subdomain (sp/halo.py:132-168).
 * Every storage cell inside the local interior [0,n) (logical) gets the global
 * SplitMix64 value U[0,1) (sp/grid.py:21-30) of global cell
 * (gx0+i, gy0+j, gz0+k) with linear index (gz*GY + gy)*GX + gx, remapped to
 * lo + (hi-lo)*u (exact for (0,1) and (-1,1)); every other storage cell (ring,
 * pad) gets `shell`.
 */
int sp_fill_seeded(double *data, int64_t ex, int64_t ey, int64_t ez, int64_t off,
                   int64_t nx, int64_t ny, int64_t nz,
                   int64_t gx0, int64_t gy0, int64_t gz0,
                   int64_t GX, int64_t GY, int64_t GZ,
                   uint64_t seed, double lo, double hi, double shell, void *stream);

/* Fill `count` doubles with `value` (create_grid(init="constant"), sp/grid.py:186-187). */
int sp_fill_constant(double *data, int64_t count, double value, void *stream);

/*
 * Plain sweep (K1).  Replaces reference_sweep (sp/kernel.py:99-111):
 * dst.interior = stencil(src) and, if copy_ring, dst.ring = src.ring
 * (_copy_ring, sp/kernel.py:85-96).  Both grids share geometry and `off`.
 * src and dst must not alias.
 */
int sp_sweep(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
             int64_t nx, int64_t ny, int64_t nz, int64_t off, int copy_ring, void *stream);

/*
 * Operator seam.  Replaces apply_window (sp/kernel.py:36-58): updates the
 * half-open logical window [xl,xh)x[yl,yh)x[zl,zh), reading src at frame
 * offset `so` and writing dst at `dso`.  If src == dst and so != dso (a
 * shifted in-place update, compressed mode) the whole window is computed into
 * `scratch` (>= window volume doubles) before the store, as the reference's
 * NumPy temporary does; otherwise scratch may be NULL.
 */
int sp_apply_window(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                    int64_t xl, int64_t xh, int64_t yl, int64_t yh, int64_t zl, int64_t zh,
                    int64_t so, int64_t dso, double *scratch, void *stream);

/* Dense variant of the seam: the window's values (reading src at frame `so`)
 * are written to out[(k-zl)][(j-yl)][(i-xl)].  Used by stencil_update_cell
 * (sp/kernel.py:21-29) and the shifted in-place paths. */
int sp_window_gather(const double *src, int64_t ex, int64_t ey, int64_t ez,
                     int64_t xl, int64_t xh, int64_t yl, int64_t yh, int64_t zl, int64_t zh,
                     int64_t so, double *out, void *stream);

/* Copy the full one-cell shell of a onto b at frame `off` (_copy_ring, sp/kernel.py:85-96). */
int sp_copy_ring(const double *a, double *b, int64_t ex, int64_t ey, int64_t ez,
                 int64_t nx, int64_t ny, int64_t nz, int64_t off, void *stream);

/*
 * *equal = 1 when the 1-cell shells (faces, edges, corners) of a and b at frame
 * `off` hold equal values, else 0 — the precondition under which two-grid
 * passes may fuse levels (the reference reads the ring of the grid each
 * level alternates to, sp/pipeline.py:301-323).  Synchronises `stream` only:
 * the verdict is written into host-mapped memory, so it does not wait behind
 * bulk transfers queued on the copy engines by other streams.
 */
int sp_rings_equal(const double *a, const double *b, int64_t ex, int64_t ey, int64_t ez,
                   int64_t nx, int64_t ny, int64_t nz, int64_t off, int *equal, void *stream);

/*
 * Write Dirichlet faces at frame `off` (PipelineEngine._write_full_ring,
 * sp/pipeline.py:427-447; write_ring_strips, sp/kernel.py:61-82).  faces[0..5]
 * are device arrays in the layout of Grid3.boundary_faces (sp/grid.py:94-107):
 * (x,0),(x,1): nz*ny; (y,0),(y,1): nz*nx; (z,0),(z,1): ny*nx (C order).
 * Bit f of side_mask enables faces[f].
 */
int sp_write_faces(double *data, int64_t ex, int64_t ey, int64_t ez,
                   int64_t nx, int64_t ny, int64_t nz, int64_t off,
                   const double *const faces[6], int side_mask, void *stream);

/*
 * Temporally blocked two-grid pass (K2).  Replaces `levels` consecutive update
 * levels of PipelineEngine.run_pass in two_grid mode (sp/pipeline.py:451-519,
 * 301-308, 314-323) fused into one HBM pass: dst.interior[z in [zlo,zhi)] =
 * stencil^levels(src).  Ring cells are never written (the two-grid pipeline
 * never writes rings) and are read from src as fixed Dirichlet values at every
 * fused level.  [zlo, zhi) is the level-`levels` live z range (sp/halo.py:
 * 278-289); x and y are the full interior.  1 <= levels <= SP_MAX_FUSED.
 * src and dst must not alias.
 */
int sp_temporal(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                int64_t nx, int64_t ny, int64_t nz, int64_t off, int levels,
                int64_t zlo, int64_t zhi, void *stream);

/*
 * Compressed-grid pass (K3).  Replaces `levels` update levels of
 * PipelineEngine.run_pass in compressed mode (sp/pipeline.py:309-312, 324-335,
 * 427-447): one array, level u read at frame a0 + s*(u-1) and written at frame
 * a0 + s*u (s = +1 forward / -1 backward; frame offset = pad + 1 - alignment),
 * fused into one HBM pass frame a0 -> a0 + s*levels.  `src_off` = pad + 1 - a0.
 * Ring cells are read at the source frame (the caller writes the faces there
 * first); the faces are written at the destination frame afterwards when
 * faces != NULL.  A tile's shifted stores land in the read regions of its
 * lower (forward) or upper (backward) neighbours.  At levels 2..4 on a
 * TMA-eligible array they are stored in place: tiles are taken in dependency
 * order and a tile's stores of a plane wait until those neighbours have
 * loaded it (progress counters in `workspace`, 128 bytes per unit; tiles
 * beyond whole multiples of the SM count run as z-chunks whose first / last
 * 2*levels planes go through a z stash in `workspace`).  Otherwise the
 * outputs that would land in another tile's read region go through
 * `workspace` (a band stash) and are copied into place by a second kernel.
 * sp_compressed_workspace() returns the workspace bytes for a pass over
 * `depth` = zhi - zlo planes, the worst case over every path and tile layout
 * a launch may pick; sp_compressed_workspace_for() returns the bytes for the
 * path sp_compressed takes on this array (the in-place pass needs no x / y
 * band stash, only its counters and the small z stash).
 * sp_compressed returns SP_EINVAL when `workspace_bytes` is smaller than the
 * launch needs.
 */
int64_t sp_compressed_workspace(int64_t nx, int64_t ny, int64_t depth, int levels);
int64_t sp_compressed_workspace_for(const double *data, int64_t ex, int64_t ey, int64_t nx,
                                    int64_t ny, int64_t depth, int levels);
int sp_compressed(double *data, int64_t ex, int64_t ey, int64_t ez,
                  int64_t nx, int64_t ny, int64_t nz, int64_t src_off, int direction,
                  int levels, int64_t zlo, int64_t zhi, void *workspace,
                  int64_t workspace_bytes, const double *const faces[6], int side_mask,
                  void *stream);

/*
 * Fused pass with peer delivery (z-slab halo exchange over NVLink peer
 * memory).  Same as sp_temporal, and every plane of [zlo, zhi) it stores is
 * also stored into `mirror` — a neighbouring rank's grid with the same x/y
 * storage extents, mapped with sp_ipc_open — at storage plane
 * z + off + mirror_zshift (mirror_ez planes).  Replaces the post-pass send /
 * receive of those planes (sp/halo.py:239-271 exchange_multilayer_halos,
 * sp/transport.py:58-60 Endpoint.sendrecv) for the topology (1,1,P):
 * the kernel writes the neighbour's ghost planes while it computes them.
 */
int sp_temporal_mirror(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                       int64_t nx, int64_t ny, int64_t nz, int64_t off, int levels,
                       int64_t zlo, int64_t zhi, double *mirror, int64_t mirror_ez,
                       int64_t mirror_zshift, void *stream);

/*
 * CUDA IPC for the peer mappings (the rendezvous of sp/transport.py:194-237,
 * without a byte transport).  sp_ipc_handle writes the 64-byte handle of the
 * allocation holding `ptr` and ptr's byte offset inside it; sp_ipc_open maps a
 * handle of another process (peer access enabled on first use).
 */
int sp_ipc_handle(const void *ptr, void *handle64, int64_t *offset);
int sp_ipc_open(const void *handle64, void **ptr);
int sp_ipc_close(void *ptr);

/*
 * Stream-ordered pass counters between ranks.  sp_signal: after the stream's
 * earlier work, fence and write `value` to `flag` (typically a neighbour's
 * counter through peer memory).  sp_wait: later work on the stream waits until
 * (int32)(*flag - value) >= 0.  Stream memory operations when available, else
 * a one-thread kernel.
 */
int sp_signal(uint32_t *flag, uint32_t value, void *stream);
int sp_wait(const uint32_t *flag, uint32_t value, void *stream);

/*
 * Halo box pack / unpack for general Cartesian topologies (the strided
 * message boxes of build_halo_plan, sp/halo.py:194-229, exchanged by
 * exchange_multilayer_halos, sp/halo.py:239-271).  Box bounds are half-open
 * STORAGE indices of `grid` (extents ex, ey, ez); `buf` is the box's
 * contiguous (z, y, x)-ordered message buffer on the device.  One call
 * handles up to SP_MAX_BOXES boxes (all messages of one axis phase): pack
 * copies grid -> buf, unpack buf -> grid.
 */
#define SP_MAX_BOXES 8
typedef struct {
    int64_t x0, x1, y0, y1, z0, z1;
    double *buf;
} sp_box_t;
int sp_pack_boxes(const double *grid, int64_t ex, int64_t ey, int64_t ez, int nbox,
                  const sp_box_t *boxes, void *stream);
int sp_unpack_boxes(double *grid, int64_t ex, int64_t ey, int64_t ez, int nbox,
                    const sp_box_t *boxes, void *stream);

/* Tuning knobs (benchmarking only; results never depend on them).
 * key 0: z-chunk length for sp_sweep / sp_temporal (0 = automatic)
 * key 1: force the cp.async (non-TMA) loader when nonzero
 * key 2: tile config index per fused depth (value = levels*16 + index)
 * key 4: profiling knobs (only in builds with -DSP200_PROFILE_KNOBS=1)
 * key 5: sp_signal / sp_wait through kernels instead of stream memory ops
 * key 6: split K2 passes as two launches (full columns, then z-chunks)
 *        instead of one grid (A/B only)
 * key 7: split K2 passes as one full column plus an equal piece of the
 *        remaining columns per CTA (A/B only)
 * key 8: z-chunk length of the remaining tiles in a split K2 pass (0 = model)
 * key 9: K2 kernel layout (A/B builds only; 0 = the product's lane-pair
 *        k_temporal, 6-10 = k_tm with the pipeline state in tensor memory)
 * key 10: 1 = sp_compressed keeps the band stash and the unstash kernels at
 *        every depth instead of storing in place
 * (keys 7 and 8 also steer the in-place pass: 7 = 1 whole columns only,
 *  8 = z-chunk length of its second launch) */
int sp_set_tuning(int key, int64_t value);

/* Query: 1 if the TMA loader applies to a grid with row extent `ex`. */
int sp_tma_eligible(int64_t ex, int64_t ey);

#ifdef __cplusplus
}
#endif

#endif /* SP200_H */
