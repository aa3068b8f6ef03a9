// K1 (plain streaming sweep) and K2 (temporally blocked two-grid pass).
//
// One kernel template covers both: K1 is the depth-1 instance (plus the fused
// Dirichlet-ring copy of reference_sweep), K2 fuses T = 2..4 sweeps per HBM
// pass.  Design (B200-first):
//
//  * A CTA owns a 64-column x CY-row region of an x-y tile and marches along
//    z over a chunk of planes.  The level-0 input planes are staged by TMA
//    (cp.async.bulk.tensor.3d issued by one thread, mbarrier completion) into
//    an S-deep ring of shared-memory stages; a cp.async loader replaces TMA
//    when the row pitch is not a multiple of 16 bytes.
//  * One warp spans the 64 columns: lane l owns the column pair (2l, 2l+1) of
//    R consecutive rows and computes those cells at every fused level, so the
//    z-neighbour chain stays in registers: per cell and level the thread keeps
//    the pending partial sum S = (((x-1 + x+1) + y-1) + y+1) + z-1; the +z+1
//    term and the x fl(1/6) finish the cell one plane later — exactly the
//    reference order (sp/kernel.py:51-57), no FMA contraction.
//  * x-neighbours: the pair partner is in registers, the outer neighbours come
//    from the adjacent lanes by warp shuffle; y-neighbours inside a thread's
//    rows are registers.  Only each thread's first and last row is published
//    to shared memory (double-buffered per level) for the y-neighbours of the
//    adjacent row group — this keeps shared-memory traffic, the limiter of the
//    fused pass, near 4 wavefronts per 32 cell-updates.
//  * Overlapped (ghost-zone) tiling: the computed region shrinks by one valid
//    cell per side per level; the stored tile is OX x (CY-2(T-1)).  Cells
//    outside the interior (Dirichlet ring) keep their input value at every
//    level.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <type_traits>

#include "sp200_device.cuh"

// Profiling-only switches (sp_set_tuning key 4) that skip parts of the fused
// pass to attribute time; compiled out of the product build.
#ifndef SP200_PROFILE_KNOBS
#define SP200_PROFILE_KNOBS 0
#endif
#include "sp200_internal.h"

namespace sp200 {

// K3 in place: one progress counter per 128-byte line
constexpr int PROG_STRIDE = 32;

struct TParams {
    const double *src;
    double *dst;
    int64_t ex, ey, ez;
    int nx, ny, nz, off;
    int ox, ex0;   // stored tile width; region column of the first stored column
    int pair_store;  // 16-byte aligned column pairs in global memory
    int tiles_x, tiles_y, ntiles;
    int tile_base, tile_count;  // tiles [tile_base, tile_base+tile_count) in this launch
    // two-grid split launch: CTAs from `split` on cover tiles
    // [tile_base2, tile_base2+tile_count2) in z-chunks of zc2 planes
    int split, tile_base2, tile_count2, zc2;
    // balanced split (piece > 0): grid = `split` CTAs; CTA c marches tile c's
    // whole column, then piece c (`piece` planes) of the remaining tiles'
    // columns laid end to end (tile-major), one unit per tile it touches
    int piece;
    int zlo, zhi, zc;
    int doff;        // storage offset of logical 0 in the written frame
    int direction;   // K3: +1 forward (write shifted -T), -1 backward
    double *stash_x, *stash_y, *stash_z;  // K3 band stash
    double *mir;     // MIR: peer grid, pre-shifted so that mir + (g - dst) mirrors dst cell g
    int wx2, hy2;    // stash_x row width, stash_y rows per plane
    int debug;       // profiling only (sp_set_tuning key 4): 1 skip levels, 2 skip loads, 4 skip barrier
    int c0;          // k_col: stage column of region column 0 (2 or 3: even TMA box start)
    // K3 in place (INPLACE): every output is stored in place; a tile's stores of
    // a plane wait until the tiles that read the cells they overwrite have
    // loaded that plane (per-tile progress counters, tiles taken in
    // dependency order through a ticket)
    int *progress;            // [nslots] input planes loaded (count) per unit, then [nslots] = the ticket
    int nslots;
};

// K3 in place: wait until the neighbours' progress counters reach `need`.
// Out of line on purpose: the loop is practically never entered, but inlined
// into the step function it cost the whole kernel 7 % (C3 581 vs 621 GLUP/s
// with the loop compiled out).
__device__ __noinline__ void inplace_wait(const int *progress, int rd0, int rd1, int rd2, int need) {
    int spins = 0;
    for (;;) {
        int c = 0x7fffffff;
        if (rd0 >= 0) c = min(c, ld_acquire_s32(progress + rd0 * PROG_STRIDE));
        if (rd1 >= 0) c = min(c, ld_acquire_s32(progress + rd1 * PROG_STRIDE));
        if (rd2 >= 0) c = min(c, ld_acquire_s32(progress + rd2 * PROG_STRIDE));
        if (c >= need) return;
        if (++spins > (1 << 26)) __trap();  // a broken dependency order, never a slow neighbour
        __nanosleep(32);
    }
}

template <int T, int CY, int R, int S>
struct KCfg {
    static constexpr int CX = 64;                // region columns (one warp, 2 per lane)
    static constexpr int PY = CY + 2;            // region rows + 1-row halo each side
    static constexpr int SPX = CX + 4;           // stage / level row pitch (doubles)
    static constexpr int C0 = 2;                 // smem column of region column 0
    static constexpr int PLANE = SPX * PY;
    static constexpr int PLANE_AL = (PLANE + 15) & ~15;  // 128-byte aligned planes
    static constexpr int NT = 32 * (CY / R);
    static constexpr int OY = CY - 2 * (T - 1);
    static constexpr int NLEV = (T > 1) ? 2 * (T - 1) : 0;
    static constexpr int XBW = 2 * T + 2;        // K3 x-stash columns per tile (even)
    // mbarriers: S stage barriers, then (cluster launches) the halo-row
    // barriers rx_lo[T-1][2] and rx_hi[T-1][2]
    static constexpr int NBAR = S + 4 * (T > 1 ? T - 1 : 0);
    static constexpr size_t SMEM = (size_t)(S + NLEV) * PLANE_AL * sizeof(double) + 8 * NBAR + 16;
    // CTAs per SM the shared memory allows (1 KB per CTA is reserved by the
    // runtime); the register budget follows through __launch_bounds__
    static constexpr int MINB = (2 * (SMEM + 1024) <= 232448) ? 2 : 1;
    static_assert(CY % R == 0, "rows per thread must divide CY");
    static_assert(OY > 0, "tile too small for the fused depth");
};

template <int T, int R>
struct LState {
    double Sp[T][R][2];                     // pending partial sum of level u (index u-1)
    double W0[2][R][2];                     // level-0 own values, by step parity
    double P[T > 1 ? T - 1 : 1][2][R][2];   // outputs of levels 1..T-1, by step parity
};

template <int N>
using IC = std::integral_constant<int, N>;

__device__ __forceinline__ double2 lds2(const double *p) {
    return *reinterpret_cast<const double2 *>(p);
}
__device__ __forceinline__ void sts2(double *p, double a, double b) {
    *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}
__device__ __forceinline__ void stg2_stream(double *p, double a, double b) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(a, b));
}

// COMP: the compressed single-array pass (K3).  Reads the level-0 frame at
// p.off and writes level T into the same array at p.doff = p.off -/+ T.  A
// tile's shifted writes overlap the read regions of its lower (forward) or
// upper (backward) neighbours only inside a 2T-wide band along that edge (x,
// y, and the z-chunk edge).  Band outputs go to a side buffer (the "stash")
// and are copied into place by k_unstash after the pass; everything else is
// written in place.  No inter-CTA ordering is needed, so K3 runs on K2's
// tile-fastest schedule (the reference needs the same order-dependence only
// because its blocks run in lexicographic order, sp/grid.py:195-204).
//
// INPLACE (COMP, T >= 2, TMA): no x / y stash.  Every output is stored in
// place; the tiles run in dependency order (a ticket per CTA: ascending tiles
// forward, descending backward) and a tile's stores of a plane wait until the
// three neighbours whose read regions they land in have loaded that plane
// (per-unit progress counters in global memory, one 128-byte line each;
// thread 0 publishes after the step barrier, lane 0 of the last warp polls
// before it).  This is the paper's relaxed synchronisation (Eq. 3) between
// SMs.  ZCH: the units of the second launch, z-chunks of the tiles beyond
// whole multiples of the SM count, chunk-major; chunks are decoupled by a z
// stash (the chunk's first / last 2T planes, k_unstash_zt).
//
// CL > 1 (two-grid only): a thread-block cluster of CL CTAs stacked in y
// shares one overlapped tile of 64 x CL*CY region rows, so the ghost zone is
// paid once per cluster instead of once per CTA.  Each step the boundary
// warps push their published row of every level 1..T-1 into the adjacent
// CTA's halo row with st.async (DSMEM), completing a per-(level, parity)
// mbarrier there; only the receiving boundary warp waits, one step later.
//
// MIR (two-grid, unclustered): every level-T store is also issued to a peer
// rank's grid through NVLink peer memory (z-slab halo delivery fused into the
// pass that computes the planes, instead of a separate send/recv).
//
// WP (TMA only): level 1 reads its own level-0 values of the current and the
// previous plane from the stage ring instead of keeping them in registers
// (W0, 4R doubles per thread).  The prefetch distance drops to S-2 so the
// previous plane's stage is not refilled while it is still read.
//
// RING (depth 1, two-grid): reference_sweep's _copy_ring (sp/kernel.py:85-96)
// fused in: CTAs whose tile touches a domain face, and every CTA at the two z
// faces, copy the shell cells of their box from the stage into dst.
template <int T, int CY, int R, int S, bool TMA, bool COMP, int CL, bool MIR = false, bool WP = false,
          bool RING = false, bool XS1 = false, bool PS = false, bool INPLACE = false, bool ZCH = false>
__global__ void __launch_bounds__(KCfg<T, CY, R, S>::NT, KCfg<T, CY, R, S>::MINB)
    k_temporal(const TParams p, const __grid_constant__ CUtensorMap tmap) {
    using C = KCfg<T, CY, R, S>;
    static_assert(!RING || (T == 1 && !COMP && CL == 1 && !MIR), "RING: plain two-grid sweeps only");
    static_assert(!WP || (TMA && S >= 4), "WP: TMA loader, at least 4 stages");
    // PS (pair sync, A/B): no CTA-wide barrier per step.  Each warp syncs
    // only with the warps above and below it (named barriers over 64
    // threads; their halo rows are the only smem data warps share besides
    // the stage), and the stage ring gets per-stage "empty" mbarriers that
    // the TMA producer waits on, so a slow warp holds back its neighbours
    // and, S - PD steps later, the producer, but not the whole CTA.
    static_assert(!PS || (TMA && !COMP && CL == 1 && !RING && !WP && S >= 5), "PS: plain TMA two-grid passes");
    static_assert(!INPLACE || COMP, "INPLACE: compressed passes only");
    static_assert(!ZCH || INPLACE, "ZCH: z-chunked units of the in-place pass");
    constexpr int PD = WP ? S - 2 : (PS ? S - 3 : S - 1);  // stage prefetch distance
    constexpr int SPX = C::SPX, C0 = C::C0, PLANE = C::PLANE, PLANE_AL = C::PLANE_AL,
                  NT = C::NT;
    constexpr int NW = NT / 32;
    // stored rows of the (cluster) tile
    constexpr int OYc = CL * CY - 2 * (T - 1);
    static_assert(CL == 1 || (!COMP && T > 1), "clusters: two-grid fused passes only");

    extern __shared__ __align__(128) double sm[];
    double *stage = sm;
    double *lev = sm + S * PLANE_AL;
    uint64_t *bar = reinterpret_cast<uint64_t *>(lev + C::NLEV * PLANE_AL);

    const int tid = threadIdx.x;
    // The warp index through a shuffle is provably warp-uniform, so the row
    // predicates and per-warp addresses go to the uniform datapath.  Measured
    // per instance: K3 +7 % (stash) / +6 % (in place); K2 at 512^3 T=4 +1.0 %,
    // T=3 +2.7 %, T=2 -3.2 % (profiles/r02_s4_ab_uwarp.log), so T >= 3 only
    const int lane = tid & 31, warp = (COMP || T >= 3) ? __shfl_sync(0xffffffffu, tid >> 5, 0) : tid >> 5;
    const int i0 = 2 * lane;   // region column of this lane's first cell
    const int j0 = warp * R;   // first region row

    const int rank = (CL > 1) ? (int)cluster_ctarank() : 0;
    [[maybe_unused]] uint64_t *rx_lo = bar + S, *rx_hi = bar + S + 2 * (T - 1);
    // halo role of this warp: 1 = first warp of a CTA below another (sends
    // its first row up, receives rx_lo), 2 = last warp of a CTA above another
    [[maybe_unused]] int role = 0;
    [[maybe_unused]] uint32_t peer_base = 0;  // shared::cluster address of the peer's smem
    if constexpr (CL > 1) {
        if (warp == 0 && rank > 0) role = 1;
        else if (warp == NW - 1 && rank < CL - 1) role = 2;
        if (role) peer_base = mapa_u32(smem_u32(sm), (uint32_t)(role == 1 ? rank - 1 : rank + 1));
    }
    if constexpr (TMA || CL > 1) {
        if (tid == 0) {
            if constexpr (TMA) tma_prefetch_desc(&tmap);
#pragma unroll
            for (int si = 0; si < S; ++si) mbar_init(&bar[si], 1);
            if constexpr (PS) {
#pragma unroll
                for (int si = 0; si < S; ++si) mbar_init(&bar[C::NBAR + si], NW);
            }
            if constexpr (INPLACE) {
                // tiles are taken in dependency order: a CTA only ever waits
                // for tiles with a lower ticket, which are running or done
                reinterpret_cast<int *>(bar + C::NBAR)[0] = atomicAdd(p.progress + (int64_t)p.nslots * PROG_STRIDE, 1);
            }
            if constexpr (CL > 1) {
                // arm phase 0 of every halo barrier: 64 doubles per row
#pragma unroll
                for (int i = 0; i < 4 * (T - 1); ++i) {
                    mbar_init(&bar[S + i], 1);
                    mbar_arrive_expect_tx(&bar[S + i], 64 * 8);
                }
            }
            fence_mbar_init();
        }
        if constexpr (CL > 1) cluster_sync_all();  // peers' barriers exist before any st.async
        else __syncthreads();
    }

    LState<T, R> st;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            st.W0[0][r][c] = st.W0[1][r][c] = 0.0;
#pragma unroll
            for (int u = 0; u < T; ++u) st.Sp[u][r][c] = 0.0;
#pragma unroll
            for (int u = 0; u < (T > 1 ? T - 1 : 1); ++u) st.P[u][0][r][c] = st.P[u][1][r][c] = 0.0;
        }

    uint32_t gbase = 0;  // stage loads issued by this CTA before the current unit
    for (int unit = 0;; ++unit) {
    // one (tile, z-chunk) unit per CTA, tile-fastest so that concurrently
    // running CTAs cover neighbouring tiles at the same z range and the
    // overlapped halo reads hit L2
    const int cid = (int)(blockIdx.x / CL);
    int tile, chunk, z0, z1;
    if (COMP || CL > 1 || p.piece == 0) {
        if (unit > 0) break;
        const bool second = !COMP && cid >= p.split;
        const int ucid = second ? cid - p.split : cid;
        const int tcount = second ? p.tile_count2 : p.tile_count, uzc = second ? p.zc2 : p.zc;
        tile = (second ? p.tile_base2 : p.tile_base) + ucid % tcount;
        chunk = ucid / tcount;
        if constexpr (INPLACE) {
            // forward passes overwrite cells the lower neighbours read, so
            // tiles run in ascending order; backward passes in descending
            const int tk = reinterpret_cast<volatile int *>(bar + C::NBAR)[0];
            if constexpr (ZCH) {
                // the tiles after the `split` full columns of the first
                // launch, chunk-major: neighbours run the same chunk together
                chunk = tk / p.tile_count2;
                const int idx = p.split + tk % p.tile_count2;
                tile = p.direction > 0 ? idx : p.ntiles - 1 - idx;
            } else {
                tile = p.direction > 0 ? tk : p.ntiles - 1 - tk;
                chunk = 0;
            }
        }
        z0 = p.zlo + chunk * uzc;
        z1 = min(z0 + uzc, p.zhi);
    } else {
        chunk = 0;
        if (unit == 0) {
            tile = cid;
            z0 = p.zlo;
            z1 = p.zhi;
        } else {
            const int64_t depth = p.zhi - p.zlo;
            const int64_t lo = (int64_t)cid * p.piece, total = (int64_t)p.tile_count2 * depth;
            const int64_t t = lo / depth + (unit - 1);
            const int64_t b = max(lo, t * depth);
            const int64_t e = min(min(lo + p.piece, (t + 1) * depth), total);
            if (b >= e) break;
            tile = p.tile_base2 + (int)t;
            z0 = p.zlo + (int)(b - t * depth);
            z1 = p.zlo + (int)(e - t * depth);
        }
        // the previous unit's last step may still read the stages the
        // preload below refills
        if (unit > 0) __syncthreads();
    }
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * p.ox, y0 = ty * OYc;
    // logical coords of this CTA's region (0, 0)
    const int rx0 = x0 - p.ex0, ry0 = y0 - (T - 1) + rank * CY;

    // Dirichlet ring cells keep their value at every level; cells beyond the
    // ring are computed but never read by a kept cell, so only the ring
    // column of a lane (x = -1 or nx) and the ring rows of a warp (y = -1 or
    // ny, warp-uniform) need the select
    bool x_out[2];
    unsigned ringb = 0;  // bit 2r+c: cell (row r, column c) is a ring cell
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int xc = rx0 + i0 + c, ic = i0 + c;
        x_out[c] = (ic >= p.ex0) && (ic < p.ex0 + p.ox) && (xc < p.nx);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int y = ry0 + j0 + r;
            if (xc == -1 || xc == p.nx || y == -1 || y == p.ny) ringb |= 1u << (2 * r + c);
        }
    }
    bool y_out[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int jr = rank * CY + j0 + r, y = ry0 + j0 + r;  // jr: row of the cluster region
        y_out[r] = (jr >= T - 1) && (jr < T - 1 + OYc) && (y < p.ny);
    }
    // warps without ring cells skip the select
    // (profiling builds, p.debug bit 128: treat every warp as interior to time the ring selects; wrong results)
    const bool wint = !__any_sync(0xffffffffu, ringb != 0u) || (SP200_PROFILE_KNOBS && (p.debug & 128));
    [[maybe_unused]] const bool ring_tile =
        RING && (x0 == 0 || y0 == 0 || x0 + p.ox >= p.nx || y0 + OYc >= p.ny);

    const int nload = (z1 - z0) + 2 * T;      // level-0 planes z0-T .. z1+T-1
    const int nsteps = (z1 - z0) + 3 * T - 1;  // level T emits plane z0+s-3T+1 at step s
    // storage x of stage column 0 (even: TMA boxes start on 16-byte boundaries)
    const int bxs = rx0 + p.off - C0, bys = ry0 - 1 + p.off;
    const int64_t pz = p.ex * p.ey;
    double *dcol = p.dst + (int64_t)(ry0 + j0 + p.doff) * p.ex + (rx0 + i0 + p.doff);

    // K3 bands: outputs whose shifted store would land in a neighbour's read
    // region go to the stash (forward: the low 2T columns / rows / planes of
    // the tile unless it is the first; backward: the high 2T unless last).
    // The x band is taken in whole column pairs, so it is 2T + (ex0 & 1) wide.
    const bool fwd = p.direction > 0;
    const int sxpad = p.ex0 & 1;
    const int xo0 = rx0 + i0 - x0;  // stored-tile column of the lane's first cell
    const bool xband = COMP && !INPLACE && (fwd ? (tx > 0 && xo0 < 2 * T)
                                            : (tx < p.tiles_x - 1 && xo0 >= p.ox - 2 * T - sxpad));
    bool yb[R];
    int ky0;
    {
        const int yo = ry0 + j0 - y0;
        ky0 = fwd ? (ty - 1) * 2 * T + yo : ty * 2 * T + yo - (OYc - 2 * T);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int yo = ry0 + j0 + r - y0;
        yb[r] = COMP && !INPLACE && (fwd ? (ty > 0 && yo < 2 * T) : (ty < p.tiles_y - 1 && yo >= OYc - 2 * T));
    }
    const int nchunks = (p.zhi - p.zlo + p.zc - 1) / p.zc;
    const bool zband_chunk = COMP && (!INPLACE || ZCH) && (fwd ? chunk > 0 : chunk < nchunks - 1);
    // destinations, affine in the output plane pout and the row r:
    //   in place / x stash: ncol + pout * npz + r * nrs
    //   y stash: sy_col + (pout * hy2 + r) * srow;  z stash: sz_col + (kz * ny + r) * srow
    // stash rows are padded so that column pairs stay 16-byte aligned
    const int srow = (p.nx + 2) & ~1;
    double *ncol = dcol + (int64_t)p.doff * pz;
    int64_t npz = pz;
    int nrs = (int)p.ex;
    if (COMP && xband) {
        const int kx0 = fwd ? (tx - 1) * C::XBW + xo0 + sxpad : tx * C::XBW + xo0 - (p.ox - 2 * T - sxpad);
        ncol = p.stash_x + (int64_t)(ry0 + j0 - p.zlo * p.ny) * p.wx2 + kx0;
        npz = (int64_t)p.ny * p.wx2;
        nrs = p.wx2;
    }
    const bool npair = x_out[0] && x_out[1] && (xband || p.pair_store);
    // INPLACE: the tiles that read the cells this tile's shifted stores overwrite
    // (forward: the lower x, y and diagonal neighbours), their cached
    // progress and the relaxed loads in flight
    // The bookkeeping state lives in shared memory (bk[]: the ticket, this
    // unit's counter slot, the neighbours' slots rd, their last seen counts l,
    // the polls in flight q by step parity), touched by two threads only: in
    // registers it cost every thread a dozen of its 254 and the main loop
    // rematerialised addresses instead
    [[maybe_unused]] volatile int *bk = reinterpret_cast<volatile int *>(bar + C::NBAR);
    enum { BK_TICKET = 0, BK_SLOT = 1, BK_RD = 2, BK_L = 5 };  // rd[3], l[3]
    // polls in flight: q[parity][neighbour], 16 bytes each (cp.async.cg
    // copies the head of the neighbour's counter line here, no register held
    // while the load is in flight)
    [[maybe_unused]] volatile int *bq = reinterpret_cast<volatile int *>(
        (reinterpret_cast<uintptr_t>(bk + 8) + 15) & ~(uintptr_t)15);
    if constexpr (INPLACE) {
        int rd_y = -1, rd_x = -1, rd_d = -1;
        const int dd = fwd ? -1 : 1;
        const bool hy = fwd ? ty > 0 : ty < p.tiles_y - 1, hx = fwd ? tx > 0 : tx < p.tiles_x - 1;
        if (hy) rd_y = tile + dd * p.tiles_x;
        if (hx) rd_x = tile + dd;
        if (hx && hy) rd_d = tile + dd * p.tiles_x + dd;
        // counter slots follow the ticket order (ascending tiles forward,
        // descending backward).  ZCH: slots of this launch are (chunk,
        // position after the full columns); the full columns finished with
        // the first launch and need no wait
        auto slot = [&](int t) {
            if (t < 0) return -1;
            const int idx = fwd ? t : p.ntiles - 1 - t;
            if constexpr (ZCH) return idx < p.split ? -1 : chunk * p.tile_count2 + idx - p.split;
            return idx;
        };
        if (tid == NT - 32) {
            const int rd[3] = {slot(rd_y), slot(rd_x), slot(rd_d)};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                bk[BK_RD + k] = rd[k];
                bk[BK_L + k] = rd[k] >= 0 ? 0 : 0x7fffffff;
                bq[4 * k] = bq[4 * (3 + k)] = rd[k] >= 0 ? 0 : 0x7fffffff;
            }
        }
        if (tid == 0) bk[BK_SLOT] = slot(tile);
    }
    double *sy_col = COMP ? p.stash_y + ((int64_t)ky0 - (int64_t)p.zlo * p.hy2) * srow + rx0 + i0 + sxpad
                          : nullptr;
    double *sz_col = COMP ? p.stash_z + (int64_t)(ry0 + j0) * srow + rx0 + i0 + sxpad : nullptr;
    // per-step band tests and stash rows reduce to one compare and one
    // multiply-add each: z band = output planes zo in [zb_lo, zb_lo + 2T) of
    // the chunk, z stash plane kz = zo + kz_off
    const int zb_lo = fwd ? 0 : (z1 - z0) - 2 * T;
    const int kz_off = fwd ? (chunk - 1) * 2 * T : chunk * 2 * T - ((z1 - z0) - 2 * T);
    const int64_t ystride = (int64_t)p.hy2 * srow, zstride = (int64_t)p.ny * srow;

    auto issue = [&](int s) {
        const int si = (int)((gbase + s) % S);
        const int zs = z0 - T + s + p.off;
        if constexpr (TMA) {
            mbar_arrive_expect_tx(&bar[si], PLANE * 8);
            tma_load_3d(stage + si * PLANE_AL, &tmap, &bar[si], bxs, bys, zs);
        } else {
            double *dstage = stage + si * PLANE_AL;
            const bool zok = (zs >= 0) && (zs < p.ez);
            for (int q = tid; q < PLANE; q += NT) {
                const int gx = bxs + q % SPX, gy = bys + q / SPX;
                const bool inb = zok && gx >= 0 && gx < p.ex && gy >= 0 && gy < p.ey;
                const double *g = inb ? p.src + ((int64_t)zs * p.ey + gy) * p.ex + gx : p.src;
                cp_async_8(dstage + q, g, inb ? 8u : 0u);
            }
            cp_async_commit();
        }
    };

    if constexpr (TMA) {
        if (tid == 0 && !(SP200_PROFILE_KNOBS && (p.debug & 2)))
            for (int s = 0; s < PD; ++s)
                if (s < nload) issue(s);
    } else {
        for (int s = 0; s < S - 1; ++s) {
            if (s < nload) issue(s);
            else cp_async_commit();
        }
    }

    // All T levels advance one plane per step, deepest level first, so level u
    // reads level u-1's previous-step outputs before level u-1 overwrites its
    // older register set.  The step parity Q is a compile-time constant (the
    // loop is unrolled by two) so the register rotation is pure renaming.
    // MODE 0: every cell interior (no select); 1: static x/y Dirichlet mask;
    // 2: mask plus per-level z-ring planes (domain z ends only).
    // ZB (ZCH only): this step's level-T plane is in the chunk's z band and
    // goes to the z stash; a compile-time flag so that all other steps run the
    // code of the whole-column instance
    auto levels = [&](int s, const double *cur, const double *prv, auto Qc, auto Mc, auto Zc) {
        constexpr int Q = decltype(Qc)::value;
        constexpr int MODE = decltype(Mc)::value;
        constexpr bool ZB = decltype(Zc)::value != 0;
#pragma unroll
        for (int u = T; u >= 1; --u) {
            const int ui = (u > 1) ? u - 2 : 0;
            const int pout = z0 - T + s - 2 * u + 1;
            const bool z_ring = (pout == -1) || (pout == p.nz);
            const double *B = (u == 1) ? cur : lev + ((u - 2) * 2 + (Q ^ 1)) * PLANE_AL;
            if (u == 1) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double2 a = lds2(B + (j0 + r + 1) * SPX + C0 + i0);
                    st.W0[Q][r][0] = a.x;
                    st.W0[Q][r][1] = a.y;
                }
            }
            if constexpr (CL > 1) {
                // level u-1's boundary row of the adjacent CTA (sent at step s-1)
                if (u > 1 && s > 0 && role && !(SP200_PROFILE_KNOBS && (p.debug & 8))) {
                    uint64_t *hb = (role == 1 ? rx_lo : rx_hi) + (u - 2) * 2 + (Q ^ 1);
                    mbar_wait(hb, ((uint32_t)(s - 1) >> 1) & 1u);
                    __syncwarp();
                    if (lane == 0) mbar_arrive_expect_tx(hb, 64 * 8);  // arm the next phase
                }
            }
            const double2 cm = lds2(B + j0 * SPX + C0 + i0);
            const double2 cp = lds2(B + (j0 + R + 1) * SPX + C0 + i0);
            double *pub = lev + ((u - 1) * 2 + Q) * PLANE_AL;
            const bool store_plane = (u == T) && pout >= z0 && pout < z1;
            // K3 destinations of this level-T plane
            [[maybe_unused]] double *nrow = nullptr, *yrow = nullptr, *zrow = nullptr;
            [[maybe_unused]] bool zb = false;
            if constexpr (ZB) {
                if (u == T) zrow = sz_col + (int64_t)(pout - z0 + kz_off) * zstride;
            }
            if constexpr (COMP && !INPLACE) {
                if (u == T) {
                    nrow = ncol + (int64_t)pout * npz;
                    const int zo = pout - z0;
                    zb = zband_chunk && (unsigned)(zo - zb_lo) < (unsigned)(2 * T);
                    zrow = sz_col + (int64_t)(zo + kz_off) * zstride;
                    yrow = sy_col + (int64_t)pout * ystride;
                }
            }
            // gather the level u-1 inputs of all 2R cells first, then run the
            // five dependent adds stage by stage across all cells so that the
            // 8-cycle DADD latency is covered by independent work of this warp
            double A[R][2], xl[R], xr[R];
            [[maybe_unused]] double wp[R][2];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                A[r][0] = (u == 1) ? st.W0[Q][r][0] : st.P[ui][Q ^ 1][r][0];
                A[r][1] = (u == 1) ? st.W0[Q][r][1] : st.P[ui][Q ^ 1][r][1];
                if constexpr (WP) {
                    if (u == 1) {
                        const double2 a = lds2(prv + (j0 + r + 1) * SPX + C0 + i0);
                        wp[r][0] = a.x;
                        wp[r][1] = a.y;
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (u == 1 && !XS1) {
                    // level 0 lives in the stage: outer x-neighbours straight from
                    // smem (two 4-way-conflicted LDS.64 per row)
                    xl[r] = B[(j0 + r + 1) * SPX + C0 + i0 - 1];
                    xr[r] = B[(j0 + r + 1) * SPX + C0 + i0 + 2];
                } else if (u == 1) {
                    // XS1: shuffles (2 MIO cycles per double, like one
                    // conflict-free LDS.64), the region's outer columns -1 / 64
                    // from the stage by the two edge lanes
                    const bool edge = (lane == 0) || (lane == 31);
                    const double e = edge ? B[(j0 + r + 1) * SPX + C0 + (lane == 0 ? -1 : 64)] : 0.0;
                    const double up = __shfl_up_sync(0xffffffffu, A[r][1], 1);
                    const double dn = __shfl_down_sync(0xffffffffu, A[r][0], 1);
                    xl[r] = (lane == 0) ? e : up;
                    xr[r] = (lane == 31) ? e : dn;
                } else {
                    xl[r] = __shfl_up_sync(0xffffffffu, A[r][1], 1);
                    xr[r] = __shfl_down_sync(0xffffffffu, A[r][0], 1);
                }
            }
            double n[R][2], v[R][2];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) v[r][c] = dadd(st.Sp[u - 1][r][c], A[r][c]);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                n[r][0] = dadd(xl[r], A[r][1]);
                n[r][1] = dadd(A[r][0], xr[r]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    n[r][c] = dadd(n[r][c], (r == 0) ? (c ? cm.y : cm.x) : A[r > 0 ? r - 1 : 0][c]);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    n[r][c] = dadd(n[r][c], (r == R - 1) ? (c ? cp.y : cp.x) : A[r < R - 1 ? r + 1 : r][c]);
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const double wl = (u == 1) ? (WP ? wp[r][c] : st.W0[Q ^ 1][r][c]) : st.P[ui][Q][r][c];
                    v[r][c] = dmul(v[r][c], 1.0 / 6.0);
                    // level T values are stored only for interior cells
                    if constexpr (MODE == 1) {
                        if (u < T && ((ringb >> (2 * r + c)) & 1u)) v[r][c] = wl;
                    } else if constexpr (MODE == 2) {
                        if (u < T && (((ringb >> (2 * r + c)) & 1u) || z_ring)) v[r][c] = wl;
                    }
                    st.Sp[u - 1][r][c] = dadd(n[r][c], wl);
                    if (u < T) st.P[u < T ? u - 1 : 0][Q][r][c] = v[r][c];
                }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (u < T) {
                    if (r == 0 || r == R - 1) sts2(pub + (j0 + r + 1) * SPX + C0 + i0, v[r][0], v[r][1]);
                    if constexpr (CL > 1) {
                        // push the CTA's first (role 1) / last (role 2) region
                        // row into the adjacent CTA's halo row; the peer's
                        // shared memory has the same layout
                        if (s + 1 < nsteps && ((role == 1 && r == 0) || (role == 2 && r == R - 1))) {
                            const uint32_t prow = (uint32_t)((pub - sm) + C0) * 8u +
                                                  (role == 1 ? (uint32_t)((CY + 1) * SPX * 8) : 0u);
                            const uint32_t pbar = (uint32_t)(reinterpret_cast<char *>(
                                                      (role == 1 ? rx_hi : rx_lo) + (u - 1) * 2 + Q) -
                                                  reinterpret_cast<char *>(sm));
                            st_async_f64x2(peer_base + prow + lane * 16u, v[r][0], v[r][1], peer_base + pbar);
                        }
                    }
                } else if (store_plane && y_out[r]) {
                    if constexpr (COMP && !INPLACE) {
                        // band priority y, then z, then x (k_unstash_* skip
                        // in the same order); y and z bands are whole rows
                        double *row = nrow + (int64_t)r * nrs;
                        bool pr = npair;
                        if (yb[r]) {
                            row = yrow + (int64_t)r * srow;
                            pr = x_out[0] && x_out[1];
                        } else if (zb) {
                            row = zrow + (int64_t)r * srow;
                            pr = x_out[0] && x_out[1];
                        }
                        if (pr) {
                            stg2_stream(row, v[r][0], v[r][1]);
                        } else {
                            if (x_out[0]) st_stream(row, v[r][0]);
                            if (x_out[1]) st_stream(row + 1, v[r][1]);
                        }
                    } else {
                        double *g = dcol + (int64_t)(pout + p.doff) * pz + (int64_t)r * p.ex;
                        // ZB: the chunk's first (forward) / last (backward) 2T
                        // planes land where the chunk below / above still
                        // reads: they go to the z stash
                        if constexpr (ZB) g = zrow + (int64_t)r * srow;
                        if (x_out[0] && x_out[1] && (ZB || p.pair_store)) {
                            stg2_stream(g, v[r][0], v[r][1]);
                            if constexpr (MIR) stg2_stream(p.mir + (g - p.dst), v[r][0], v[r][1]);
                        } else {
                            if (x_out[0]) st_stream(g, v[r][0]);
                            if (x_out[1]) st_stream(g + 1, v[r][1]);
                            if constexpr (MIR) {
                                if (x_out[0]) st_stream(p.mir + (g - p.dst), v[r][0]);
                                if (x_out[1]) st_stream(p.mir + (g - p.dst) + 1, v[r][1]);
                            }
                        }
                    }
                }
            }
        }
    };

    auto one_step = [&](int s, auto Qc) {
        const int si = (int)((gbase + s) % S);
        if constexpr (TMA) {
            // One thread waits for the stage's TMA bytes; the step barrier right
            // below hands the observation to the others (the data sits in this
            // SM's shared memory once the phase has flipped).  With every thread
            // spinning on the mbarrier the pass ran 2.5 % slower at T=4
            // (789 vs 808 GLUP/s at 512^3; PS has no CTA barrier, so there all wait)
            if ((PS || tid == 0) && s < nload && !(SP200_PROFILE_KNOBS && (p.debug & 2)))
                mbar_wait(&bar[si], (uint32_t)(((gbase + s) / S) & 1));
        } else {
            cp_async_wait<S - 2>();
        }
        if constexpr (PS) {
            // even warps: upper pair first; odd warps: lower pair first, so
            // all (2k, 2k+1) pairs complete together, then the (2k+1, 2k+2)
            if (warp % 2 == 0) {
                if (warp + 1 < NW) named_sync(warp + 1, 64);
                if (warp > 0) named_sync(warp, 64);
            } else {
                named_sync(warp, 64);
                if (warp + 1 < NW) named_sync(warp + 1, 64);
            }
            if (tid == 0 && s + PD < nload) {
                const int t = s + PD;
                // the stage's previous use (step t - S) released by every warp
                if (t >= S) mbar_wait(&bar[C::NBAR + t % S], (uint32_t)(((t - S) / S) & 1));
                issue(t);
            }
        } else {
#if SP200_PROFILE_KNOBS
        if constexpr (INPLACE) {
            // test hook (p.debug bit 64): every fifth tile stalls for ~20 us
            // every 8th step, so its neighbours really have to wait for it
            if ((p.debug & 64) && tid == 0 && tile % 5 == 2 && (s & 7) == 0) __nanosleep(20000);
        }
#endif
        if constexpr (INPLACE) {
            // polled by the last warp: it covers ghost rows above the stored
            // tile and has fewer stores per step than the interior warps, so
            // the few dozen instructions here do not make it the last one at
            // the barrier
            if (tid == NT - 32) {
                // this step's level-T stores (plane index s - 2T + 1 of the
                // column) land on input plane s - 2T + 1 -/+ T of the source
                // frame: the neighbours must have loaded it.  l_* were loaded
                // one step ago (never waited on in the step that issues them).
                const int need = s - 2 * T + 1 + (fwd ? -T : T) + 1;
                // polls issued two steps ago (a counter line that another SM
                // keeps writing takes longer than one step to read)
                constexpr int QQ = decltype(Qc)::value;
                cp_async_wait<1>();  // the polls of two steps ago have landed
                const int rd0 = bk[BK_RD], rd1 = bk[BK_RD + 1], rd2 = bk[BK_RD + 2];
                if constexpr (T >= 3) {
                    // every present neighbour is polled every step (the slots
                    // of absent ones hold 0x7fffffff and are never polled)
                    if (min(bq[4 * (3 * QQ)], min(bq[4 * (3 * QQ + 1)], bq[4 * (3 * QQ + 2)])) < need)
                        inplace_wait(p.progress, rd0, rd1, rd2, need);
                    if (rd0 >= 0) cp_async_16_cg(const_cast<int *>(bq) + 4 * (3 * QQ), p.progress + rd0 * PROG_STRIDE);
                    if (rd1 >= 0) cp_async_16_cg(const_cast<int *>(bq) + 4 * (3 * QQ + 1), p.progress + rd1 * PROG_STRIDE);
                    if (rd2 >= 0) cp_async_16_cg(const_cast<int *>(bq) + 4 * (3 * QQ + 2), p.progress + rd2 * PROG_STRIDE);
                } else {
                    // T = 2 (short steps): keep the last seen counts and
                    // re-poll a neighbour only when its count runs out within
                    // three steps (487 vs 464 GLUP/s at 600^3)
                    const int rd[3] = {rd0, rd1, rd2};
                    int l[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) l[k] = max(bk[BK_L + k], bq[4 * (3 * QQ + k)]);
                    if (min(l[0], min(l[1], l[2])) < need) inplace_wait(p.progress, rd0, rd1, rd2, need);
                    const int soon = need + 3;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        bk[BK_L + k] = l[k];
                        if (rd[k] >= 0 && l[k] < soon)
                            cp_async_16_cg(const_cast<int *>(bq) + 4 * (3 * QQ + k), p.progress + rd[k] * PROG_STRIDE);
                    }
                }
                cp_async_commit();
            }
        }
        if (!(SP200_PROFILE_KNOBS && (p.debug & 4))) __syncthreads();
        // the stage was written by the async proxy and only one thread watched
        // its mbarrier: order every thread's generic reads after those writes
        // (measured free: 810 vs 808 GLUP/s)
        if constexpr (TMA) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if constexpr (TMA) {
            if (tid == 0 && s + PD < nload && !(SP200_PROFILE_KNOBS && (p.debug & 2))) issue(s + PD);
        } else {
            if (s + S - 1 < nload) issue(s + S - 1);
            else cp_async_commit();
        }
        }
        if constexpr (INPLACE) {
            // published by thread 0 after the barrier (warp 0 covers ghost
            // rows too); every counter has its own 128-byte line: counters
            // sharing a sector ran 3x slower
            if (tid == 0) {
                // input planes this tile has in shared memory: step s's, plus
                // the prefetched stages that have already landed
                if (s < nload) {
                    int done = s + 1;
                    if constexpr (TMA) {
#pragma unroll
                        // (prefetched stages count only at T = 2, whose backward
                        // passes have one plane of slack: at T >= 3 the probes cost
                        // more than the slack buys, 606 vs 570 GLUP/s at T=3)
                        for (int a = 1; a < (T <= 2 ? PD : 1); ++a) {
                            const uint32_t g = gbase + (uint32_t)(s + a);
                            if (done == s + a && s + a < nload && mbar_test_wait(&bar[g % S], (g / S) & 1u)) done = s + a + 1;
                        }
                    }
                    st_relaxed_s32(p.progress + bk[BK_SLOT] * PROG_STRIDE, done);
                } else if (s == nload) {
                    st_relaxed_s32(p.progress + bk[BK_SLOT] * PROG_STRIDE, 0x7ffffff0);
                }
            }
        }
        const double *cur = stage + si * PLANE_AL;
        if constexpr (RING) {
            // the stage holds logical plane P0 over storage columns bxs.. and
            // rows bys..; copy the shell cells of this tile's box [x0-1, x0+ox]
            // x [y0-1, y0+OY] (neighbouring tiles write the same values)
            const int P0 = z0 - T + s;
            const bool zring = (P0 == -1 && z0 == 0) || (P0 == p.nz && z1 == p.nz);
            const bool zmid = (P0 >= z0) && (P0 < z1);
            constexpr int BX = 64 + 2, BY = OYc + 2;  // box: ox <= 64 columns, OY rows, + halo
            double *drow = p.dst + (int64_t)(P0 + p.off) * pz;
            auto put = [&](int gx, int gy) {
                drow[(int64_t)(gy + p.off) * p.ex + gx + p.off] =
                    cur[(gy - (bys - p.off)) * SPX + (gx - (bxs - p.off))];
            };
            if (s < nload && zring) {
                // a z face: the whole box is shell
                for (int q = tid; q < BX * BY; q += NT) {
                    const int qy = q / BX, qx = q - qy * BX;
                    const int gx = x0 - 1 + qx, gy = y0 - 1 + qy;
                    if (qx > p.ox + 1 || gx < -1 || gx > p.nx || gy < -1 || gy > p.ny) continue;
                    put(gx, gy);
                }
            } else if (s < nload && zmid && ring_tile) {
                // interior plane: only the box's x = -1 / nx columns and
                // y = -1 / ny rows (one pass of the CTA's threads)
                for (int q = tid; q < 2 * BY + 2 * BX; q += NT) {
                    int gx, gy;
                    bool ok;
                    if (q < 2 * BY) {
                        const int side = q >= BY;
                        gx = side ? p.nx : -1;
                        gy = y0 - 1 + (q - side * BY);
                        ok = gx >= x0 - 1 && gx <= x0 + p.ox;
                    } else {
                        const int q2 = q - 2 * BY, side = q2 >= BX, qx = q2 - side * BX;
                        gy = side ? p.ny : -1;
                        gx = x0 - 1 + qx;
                        ok = qx <= p.ox + 1 && gy >= y0 - 1 && gy <= y0 + OYc;
                    }
                    if (ok && gx >= -1 && gx <= p.nx && gy >= -1 && gy <= p.ny) put(gx, gy);
                }
            }
        }
        // WP: the previous plane's stage (the current one at s = 0: that
        // step's level-1 output plane is below the valid range anyway)
        const double *prv = (WP && s > 0) ? stage + (int)((gbase + s + S - 1) % S) * PLANE_AL : cur;
        // every level's finished plane inside [0, nz): no z-ring this step
        const int pmax = z0 - T + s - 1, pmin = z0 - T + s - 2 * T + 1;
        const bool zall = (pmin >= 0) && (pmax < p.nz);
        if (SP200_PROFILE_KNOBS && (p.debug & 1)) return;  // profiling builds only
        bool zbs = false;
        if constexpr (ZCH) zbs = zband_chunk && (unsigned)(s - 3 * T + 1 - zb_lo) < (unsigned)(2 * T);
        if (ZCH && zbs) {
            if constexpr (ZCH) {
                if (wint && zall) levels(s, cur, prv, Qc, IC<0>{}, IC<1>{});
                else if (zall) levels(s, cur, prv, Qc, IC<1>{}, IC<1>{});
                else levels(s, cur, prv, Qc, IC<2>{}, IC<1>{});
            }
        } else {
            if (wint && zall) levels(s, cur, prv, Qc, IC<0>{}, IC<0>{});
            else if (zall) levels(s, cur, prv, Qc, IC<1>{}, IC<0>{});
            else levels(s, cur, prv, Qc, IC<2>{}, IC<0>{});
        }
        if constexpr (PS) {
            // this warp is done with the stage of step s
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar[C::NBAR + si]);
        }
    };

    for (int s = 0; s < nsteps; s += 2) {
        one_step(s, IC<0>{});
        if (s + 1 < nsteps) one_step(s + 1, IC<1>{});
    }
    if constexpr (!TMA) cp_async_wait<0>();
    gbase += (uint32_t)nload;
    }  // units
    // no CTA leaves while a peer may still address its shared memory
    if constexpr (CL > 1) cluster_sync_all();
}

#if SP200_AB
}  // namespace sp200
#include "sp200_tmem.cuh"
namespace sp200 {
#endif


#if SP200_AB
// ---------------------------------------------------------------------------
// K2 column layout (k_col): the two-grid fused pass with one column per lane.
//
// A warp spans the 32 columns of the region and lane l owns region column l
// of R consecutive rows; NW warps stack in y (region 32 x NW*R).  Compared
// with the lane-pair layout of k_temporal (64 x 4 per warp):
//  * y-neighbours inside a thread's R = 8 rows are registers, so the
//    published halo rows (first and last row of each warp, per level) and
//    their loads are half as many per cell;
//  * every shared-memory access is a warp-contiguous LDS.64 / STS.64
//    (256 B, 2 wavefronts, no bank conflicts), where the pair layout's
//    x-neighbour loads from the stage hit 4-way conflicts;
//  * both x-neighbours of levels >= 2 come by shuffle (one each way per
//    row); level 1 takes them from the stage (LDS) or, with XS, by shuffle
//    with the two edge lanes patched from the stage;
//  * stores are plain coalesced 8-byte stores (no pair alignment), so the
//    stored tile keeps its full width 32 - 2(T-1) at every frame parity.
// Shared memory traffic is the resource the pair layout saturates first
// (l1tex 70 %, DESIGN.md §3 K2); this layout trades part of it for shuffles.
// Same schedule, ring semantics and summation order as k_temporal.
// ---------------------------------------------------------------------------
template <int T, int R, int NW>
struct CCfg {
    static constexpr int CX = 32;
    static constexpr int CY = NW * R;
    static constexpr int SPX = CX + 4;                // stage row pitch = TMA box width
    static constexpr int PY = CY + 2;
    static constexpr int PLANE = SPX * PY;
    static constexpr int PLANE_AL = (PLANE + 15) & ~15;
    static constexpr int NT = 32 * NW;
    static constexpr int OX = CX - 2 * (T - 1);
    static constexpr int OY = CY - 2 * (T - 1);
    static constexpr int PUBR = 2 * NW + 2;           // published rows per level plane (+2 sentinels)
    static constexpr int PUB = PUBR * 32;
    static constexpr int NPUB = (T > 1) ? 2 * (T - 1) : 0;
    template <int S>
    static constexpr size_t smem() {
        return (size_t)S * PLANE_AL * 8 + (size_t)NPUB * PUB * 8 + 8 * S + 16;
    }
    static_assert(OY > 0 && OX > 0, "region too small for the fused depth");
};

template <int T, int R, int NW, int S, bool TMA, bool XS, bool MIR = false>
__global__ void __launch_bounds__(32 * NW, 1)
    k_col(const TParams p, const __grid_constant__ CUtensorMap tmap) {
    using C = CCfg<T, R, NW>;
    constexpr int SPX = C::SPX, PLANE = C::PLANE, PLANE_AL = C::PLANE_AL, NT = C::NT, PUB = C::PUB,
                  OY = C::OY;
    extern __shared__ __align__(128) double sm[];
    double *stage = sm;
    double *pub = sm + S * PLANE_AL;
    uint64_t *bar = reinterpret_cast<uint64_t *>(pub + C::NPUB * PUB);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = warp * R;  // first region row of this warp
    if constexpr (TMA) {
        if (tid == 0) {
            tma_prefetch_desc(&tmap);
#pragma unroll
            for (int si = 0; si < S; ++si) mbar_init(&bar[si], 1);
            fence_mbar_init();
        }
    }
    // sentinel rows of the published planes (the halo of the region's first
    // and last row: ghost cells, read but never feeding a kept cell)
    for (int q = tid; q < C::NPUB * 64; q += NT)
        pub[(q >> 6) * PUB + ((q & 32) ? (C::PUBR - 1) * 32 : 0) + (q & 31)] = 0.0;
    __syncthreads();

    // one (tile, z-chunk) unit per CTA, tile-fastest; CTAs from p.split on
    // cover the remaining tiles in z-chunks (see launch_col)
    const int cid = (int)blockIdx.x;
    const bool second = cid >= p.split;
    const int ucid = second ? cid - p.split : cid;
    const int tcount = second ? p.tile_count2 : p.tile_count, uzc = second ? p.zc2 : p.zc;
    const int tile = (second ? p.tile_base2 : p.tile_base) + ucid % tcount;
    const int chunk = ucid / tcount;
    const int z0 = p.zlo + chunk * uzc;
    const int z1 = min(z0 + uzc, p.zhi);
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * p.ox, y0 = ty * OY;
    const int rx0 = x0 - (T - 1), ry0 = y0 - (T - 1);  // logical coords of region (0, 0)
    const int xc = rx0 + lane;

    const bool col_ring = (xc == -1) || (xc == p.nx);
    const bool x_out = (lane >= T - 1) && (lane < T - 1 + p.ox) && (xc < p.nx);
    unsigned ringb = 0, yout = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int y = ry0 + j0 + r, jr = j0 + r;
        if (col_ring || y == -1 || y == p.ny) ringb |= 1u << r;
        if (jr >= T - 1 && jr < T - 1 + OY && y < p.ny) yout |= 1u << r;
    }
    const bool wint = !__any_sync(0xffffffffu, ringb != 0u);

    const int nload = (z1 - z0) + 2 * T;       // level-0 planes z0-T .. z1+T-1
    const int nsteps = (z1 - z0) + 3 * T - 1;  // level T emits plane z0+s-3T+1 at step s
    const int c0 = p.c0;
    const int bxs = rx0 + p.off - c0, bys = ry0 - 1 + p.off;
    const int64_t pz = p.ex * p.ey;
    double *dcol = p.dst + (int64_t)(ry0 + j0 + p.doff) * p.ex + (xc + p.doff);

    auto issue = [&](int s) {
        const int si = s % S;
        const int zs = z0 - T + s + p.off;
        if constexpr (TMA) {
            mbar_arrive_expect_tx(&bar[si], PLANE * 8);
            tma_load_3d(stage + si * PLANE_AL, &tmap, &bar[si], bxs, bys, zs);
        } else {
            double *dstage = stage + si * PLANE_AL;
            const bool zok = (zs >= 0) && (zs < p.ez);
            for (int q = tid; q < PLANE; q += NT) {
                const int gx = bxs + q % SPX, gy = bys + q / SPX;
                const bool inb = zok && gx >= 0 && gx < p.ex && gy >= 0 && gy < p.ey;
                const double *g = inb ? p.src + ((int64_t)zs * p.ey + gy) * p.ex + gx : p.src;
                cp_async_8(dstage + q, g, inb ? 8u : 0u);
            }
            cp_async_commit();
        }
    };
    if constexpr (TMA) {
        if (tid == 0)
            for (int s = 0; s < S - 1; ++s)
                if (s < nload) issue(s);
    } else {
        for (int s = 0; s < S - 1; ++s) {
            if (s < nload) issue(s);
            else cp_async_commit();
        }
    }

    // per-thread state: pending sums of levels 1..T, level-0 own values and
    // the outputs of levels 1..T-1, the last two by step parity
    double Sp[T][R], W0[2][R], P[T > 1 ? T - 1 : 1][2][R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        W0[0][r] = W0[1][r] = 0.0;
#pragma unroll
        for (int u = 0; u < T; ++u) Sp[u][r] = 0.0;
#pragma unroll
        for (int u = 0; u < (T > 1 ? T - 1 : 1); ++u) P[u][0][r] = P[u][1][r] = 0.0;
    }

    // all levels advance one plane per step, deepest first; level u finishes
    // plane z0 - T + s - 2u + 1 (MODE as in k_temporal)
    auto levels = [&](int s, const double *cur, auto Qc, auto Mc) {
        constexpr int Q = decltype(Qc)::value;
        constexpr int MODE = decltype(Mc)::value;
#pragma unroll
        for (int u = T; u >= 1; --u) {
            const int pout = z0 - T + s - 2 * u + 1;
            const bool z_ring = (pout == -1) || (pout == p.nz);
            double A[R], wl[R], xl[R], xr[R], cm, cp;
            if (u == 1) {
                const double *rp = cur + (j0 + 1) * SPX + c0 + lane;
#pragma unroll
                for (int r = 0; r < R; ++r) W0[Q][r] = rp[r * SPX];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    A[r] = W0[Q][r];
                    wl[r] = W0[Q ^ 1][r];
                }
                cm = rp[-SPX];
                cp = rp[R * SPX];
                if constexpr (XS) {
                    // edge lanes take the region's outer column from the stage
                    const bool edge = (lane == 0) || (lane == 31);
                    const double *ep = rp + (lane == 0 ? -1 : 1);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double e = edge ? ep[r * SPX] : 0.0;
                        const double up = __shfl_up_sync(0xffffffffu, A[r], 1);
                        const double dn = __shfl_down_sync(0xffffffffu, A[r], 1);
                        xl[r] = (lane == 0) ? e : up;
                        xr[r] = (lane == 31) ? e : dn;
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        xl[r] = rp[r * SPX - 1];
                        xr[r] = rp[r * SPX + 1];
                    }
                }
            } else {
                const int ui = (u > 1) ? u - 2 : 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    A[r] = P[ui][Q ^ 1][r];
                    wl[r] = P[ui][Q][r];
                }
                const double *pp = pub + (ui * 2 + (Q ^ 1)) * PUB + lane;
                cm = pp[(2 * warp) * 32];
                cp = pp[(2 * warp + 3) * 32];
                // lanes 0 / 31: the region's ghost columns, never feeding a kept cell
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    xl[r] = __shfl_up_sync(0xffffffffu, A[r], 1);
                    xr[r] = __shfl_down_sync(0xffffffffu, A[r], 1);
                }
            }
            double n[R], v[R];
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = dadd(Sp[u - 1][r], A[r]);
#pragma unroll
            for (int r = 0; r < R; ++r) n[r] = dadd(xl[r], xr[r]);
#pragma unroll
            for (int r = 0; r < R; ++r) n[r] = dadd(n[r], r == 0 ? cm : A[r > 0 ? r - 1 : 0]);
#pragma unroll
            for (int r = 0; r < R; ++r) n[r] = dadd(n[r], r == R - 1 ? cp : A[r < R - 1 ? r + 1 : 0]);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                v[r] = dmul(v[r], 1.0 / 6.0);
                if constexpr (MODE == 1) {
                    if (u < T && ((ringb >> r) & 1u)) v[r] = wl[r];
                } else if constexpr (MODE == 2) {
                    if (u < T && (((ringb >> r) & 1u) || z_ring)) v[r] = wl[r];
                }
                Sp[u - 1][r] = dadd(n[r], wl[r]);
                if (u < T) P[u < T ? u - 1 : 0][Q][r] = v[r];
            }
            if (u < T) {
                double *pw = pub + ((u - 1) * 2 + Q) * PUB + lane;
                pw[(2 * warp + 1) * 32] = v[0];
                pw[(2 * warp + 2) * 32] = v[R - 1];
            } else if (x_out && pout >= z0 && pout < z1) {
                double *g = dcol + (int64_t)(pout + p.doff) * pz;
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if ((yout >> r) & 1u) {
                        st_stream(g + (int64_t)r * p.ex, v[r]);
                        if constexpr (MIR) st_stream(p.mir + (g - p.dst) + (int64_t)r * p.ex, v[r]);
                    }
            }
        }
    };

    auto one_step = [&](int s, auto Qc) {
        const int si = s % S;
        if constexpr (TMA) {
            if (s < nload) mbar_wait(&bar[si], (uint32_t)((s / S) & 1));
        } else {
            cp_async_wait<S - 2>();
        }
        __syncthreads();
        if constexpr (TMA) {
            if (tid == 0 && s + S - 1 < nload) issue(s + S - 1);
        } else {
            if (s + S - 1 < nload) issue(s + S - 1);
            else cp_async_commit();
        }
        const double *cur = stage + si * PLANE_AL;
        const int pmax = z0 - T + s - 1, pmin = z0 - T + s - 2 * T + 1;
        const bool zall = (pmin >= 0) && (pmax < p.nz);
        if (wint && zall) levels(s, cur, Qc, IC<0>{});
        else if (zall) levels(s, cur, Qc, IC<1>{});
        else levels(s, cur, Qc, IC<2>{});
    };

    for (int s = 0; s < nsteps; s += 2) {
        one_step(s, IC<0>{});
        if (s + 1 < nsteps) one_step(s + 1, IC<1>{});
    }
    if constexpr (!TMA) cp_async_wait<0>();
}

#endif  // SP200_AB

#if SP200_AB

// ---------------------------------------------------------------------------
// K2 with split level roles (k_split, T = 4): the pair layout of k_temporal
// (lane = column pair x R=4 rows, 8 row groups of a 64 x 32 region), but two
// warps per row group: a FRONT warp runs levels 1-2 and a BACK warp levels
// 3-4 of the same cells.  The front warp hands its level-2 rows to the back
// warp through a double-buffered shared plane, which also serves as the
// level-2 halo rows (no separate level-2 publish).  Each thread keeps 5
// doubles per cell instead of 12, so the CTA holds 16 warps (4 per
// scheduler) at <= 128 registers, for 24 more shared-memory wavefronts per
// row group and step (handoff store 16 + loads 24 - the level-2 publish 8 -
// level-3 own values from registers ...).  Same schedule, level lag and
// summation order as k_temporal (results are bit-identical).
// ---------------------------------------------------------------------------
template <int S, bool TMA>
__global__ void __launch_bounds__(512, 1) k_split(const TParams p, const __grid_constant__ CUtensorMap tmap) {
    constexpr int T = 4, CY = 32, R = 4, NWR = 8;  // levels, region rows, rows per thread, row groups
    using C = KCfg<T, CY, R, S>;
    constexpr int SPX = C::SPX, C0 = C::C0, PLANE = C::PLANE, PLANE_AL = C::PLANE_AL, NT = 512;
    constexpr int OYc = CY - 2 * (T - 1);
    extern __shared__ __align__(128) double sm[];
    double *stage = sm;
    double *pub1 = sm + S * PLANE_AL;         // level-1 boundary rows, 2 parities
    double *hand = pub1 + 2 * PLANE_AL;       // level-2 rows (all), 2 parities
    double *pub3 = hand + 2 * PLANE_AL;       // level-3 boundary rows, 2 parities
    uint64_t *bar = reinterpret_cast<uint64_t *>(pub3 + 2 * PLANE_AL);

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const bool back = warp >= NWR;
    const int wr = warp & (NWR - 1);
    const int i0 = 2 * lane, j0 = wr * R;
    if constexpr (TMA) {
        if (tid == 0) {
            tma_prefetch_desc(&tmap);
#pragma unroll
            for (int si = 0; si < S; ++si) mbar_init(&bar[si], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }

    const int cid = (int)blockIdx.x;
    const bool second = cid >= p.split;
    const int ucid = second ? cid - p.split : cid;
    const int tcount = second ? p.tile_count2 : p.tile_count, uzc = second ? p.zc2 : p.zc;
    const int tile = (second ? p.tile_base2 : p.tile_base) + ucid % tcount;
    const int chunk = ucid / tcount;
    const int z0 = p.zlo + chunk * uzc, z1 = min(z0 + uzc, p.zhi);
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * p.ox, y0 = ty * OYc;
    const int rx0 = x0 - p.ex0, ry0 = y0 - (T - 1);

    bool x_out[2];
    unsigned ringb = 0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int xc = rx0 + i0 + c, ic = i0 + c;
        x_out[c] = (ic >= p.ex0) && (ic < p.ex0 + p.ox) && (xc < p.nx);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int y = ry0 + j0 + r;
            if (xc == -1 || xc == p.nx || y == -1 || y == p.ny) ringb |= 1u << (2 * r + c);
        }
    }
    bool y_out[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int jr = j0 + r, y = ry0 + j0 + r;
        y_out[r] = (jr >= T - 1) && (jr < T - 1 + OYc) && (y < p.ny);
    }
    const bool wint = !__any_sync(0xffffffffu, ringb != 0u);
    const int nload = (z1 - z0) + 2 * T;
    const int nsteps = (z1 - z0) + 3 * T - 1;
    const int bxs = rx0 + p.off - C0, bys = ry0 - 1 + p.off;
    const int64_t pz = p.ex * p.ey;
    double *dcol = p.dst + (int64_t)(ry0 + j0 + p.doff) * p.ex + (rx0 + i0 + p.doff);

    auto issue = [&](int s) {
        const int si = s % S;
        const int zs = z0 - T + s + p.off;
        if constexpr (TMA) {
            mbar_arrive_expect_tx(&bar[si], PLANE * 8);
            tma_load_3d(stage + si * PLANE_AL, &tmap, &bar[si], bxs, bys, zs);
        } else {
            double *dstage = stage + si * PLANE_AL;
            const bool zok = (zs >= 0) && (zs < p.ez);
            for (int q = tid; q < PLANE; q += NT) {
                const int gx = bxs + q % SPX, gy = bys + q / SPX;
                const bool inb = zok && gx >= 0 && gx < p.ex && gy >= 0 && gy < p.ey;
                const double *g = inb ? p.src + ((int64_t)zs * p.ey + gy) * p.ex + gx : p.src;
                cp_async_8(dstage + q, g, inb ? 8u : 0u);
            }
            cp_async_commit();
        }
    };
    if constexpr (TMA) {
        if (tid == 0)
            for (int s = 0; s < S - 1; ++s)
                if (s < nload) issue(s);
    } else {
        for (int s = 0; s < S - 1; ++s) {
            if (s < nload) issue(s);
            else cp_async_commit();
        }
    }

    // per-thread state: front = levels 1-2, back = levels 3-4
    //   Spa/Spb: pending sums of the two levels; I[2]: the input level's own
    //   values (front: level 0, back: level 2) by step parity; M[2]: the
    //   middle level's outputs (front: level 1, back: level 3) by parity
    double Spa[R][2], Spb[R][2], I[2][R][2], M[2][R][2];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) Spa[r][c] = Spb[r][c] = I[0][r][c] = I[1][r][c] = M[0][r][c] = M[1][r][c] = 0.0;

    // One level of one role: input values A (own cells, this step's newest
    // plane), wl (own cells, one plane older), halo rows cm / cp, x-neighbours
    // by shuffle (or from `xrow` when the input is the stage).
    auto level = [&](int u, double (&Sp)[R][2], double (&A)[R][2], double (&wl)[R][2], double2 cm,
                     double2 cp, const double *xrow, auto Mc, double (&out)[R][2], int s) {
        constexpr int MODE = decltype(Mc)::value;
        const int pout = z0 - T + s - 2 * u + 1;
        const bool z_ring = (pout == -1) || (pout == p.nz);
        double xl[R], xr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (xrow) {
                xl[r] = xrow[r * SPX + C0 + i0 - 1];
                xr[r] = xrow[r * SPX + C0 + i0 + 2];
            } else {
                xl[r] = __shfl_up_sync(0xffffffffu, A[r][1], 1);
                xr[r] = __shfl_down_sync(0xffffffffu, A[r][0], 1);
            }
        }
        double n[R][2], v[R][2];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) v[r][c] = dadd(Sp[r][c], A[r][c]);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            n[r][0] = dadd(xl[r], A[r][1]);
            n[r][1] = dadd(A[r][0], xr[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c)
                n[r][c] = dadd(n[r][c], (r == 0) ? (c ? cm.y : cm.x) : A[r > 0 ? r - 1 : 0][c]);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c)
                n[r][c] = dadd(n[r][c], (r == R - 1) ? (c ? cp.y : cp.x) : A[r < R - 1 ? r + 1 : r][c]);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                v[r][c] = dmul(v[r][c], 1.0 / 6.0);
                if constexpr (MODE == 1) {
                    if (u < T && ((ringb >> (2 * r + c)) & 1u)) v[r][c] = wl[r][c];
                } else if constexpr (MODE == 2) {
                    if (u < T && (((ringb >> (2 * r + c)) & 1u) || z_ring)) v[r][c] = wl[r][c];
                }
                Sp[r][c] = dadd(n[r][c], wl[r][c]);
                out[r][c] = v[r][c];
            }
        return pout;
    };

    auto one_step = [&](int s, auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        const int si = s % S;
        if constexpr (TMA) {
            if (s < nload) mbar_wait(&bar[si], (uint32_t)((s / S) & 1));
        } else {
            cp_async_wait<S - 2>();
        }
        __syncthreads();
        if constexpr (TMA) {
            if (tid == 0 && s + S - 1 < nload) issue(s + S - 1);
        } else {
            if (s + S - 1 < nload) issue(s + S - 1);
            else cp_async_commit();
        }
        const double *cur = stage + si * PLANE_AL;
        const int pmax = z0 - T + s - 1, pmin = z0 - T + s - 2 * T + 1;
        const bool zall = (pmin >= 0) && (pmax < p.nz);
        auto body = [&](auto Mc) {
            if (!back) {
                // level 2 from level 1 of the previous step (pub1[Q^1] halo rows)
                {
                    const double *B = pub1 + (Q ^ 1) * PLANE_AL;
                    const double2 cm = lds2(B + j0 * SPX + C0 + i0), cp = lds2(B + (j0 + R + 1) * SPX + C0 + i0);
                    double out[R][2];
                    level(2, Spb, M[Q ^ 1], M[Q], cm, cp, nullptr, Mc, out, s);
                    // hand all level-2 rows to the back warp (they are also its halo rows)
                    double *H = hand + Q * PLANE_AL;
#pragma unroll
                    for (int r = 0; r < R; ++r) sts2(H + (j0 + r + 1) * SPX + C0 + i0, out[r][0], out[r][1]);
                }
                // level 1 from the stage
                {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double2 a = lds2(cur + (j0 + r + 1) * SPX + C0 + i0);
                        I[Q][r][0] = a.x;
                        I[Q][r][1] = a.y;
                    }
                    const double2 cm = lds2(cur + j0 * SPX + C0 + i0), cp = lds2(cur + (j0 + R + 1) * SPX + C0 + i0);
                    level(1, Spa, I[Q], I[Q ^ 1], cm, cp, cur + (j0 + 1) * SPX, Mc, M[Q], s);
                    double *W = pub1 + Q * PLANE_AL;
                    sts2(W + (j0 + 1) * SPX + C0 + i0, M[Q][0][0], M[Q][0][1]);
                    sts2(W + (j0 + R) * SPX + C0 + i0, M[Q][R - 1][0], M[Q][R - 1][1]);
                }
            } else {
                // level 4 from level 3 of the previous step (pub3[Q^1] halo rows), stored
                {
                    const double *B = pub3 + (Q ^ 1) * PLANE_AL;
                    const double2 cm = lds2(B + j0 * SPX + C0 + i0), cp = lds2(B + (j0 + R + 1) * SPX + C0 + i0);
                    double out[R][2];
                    const int pout = level(4, Spb, M[Q ^ 1], M[Q], cm, cp, nullptr, Mc, out, s);
                    if (pout >= z0 && pout < z1) {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            if (!y_out[r]) continue;
                            double *g = dcol + (int64_t)(pout + p.doff) * pz + (int64_t)r * p.ex;
                            if (x_out[0] && x_out[1] && p.pair_store) {
                                stg2_stream(g, out[r][0], out[r][1]);
                            } else {
                                if (x_out[0]) st_stream(g, out[r][0]);
                                if (x_out[1]) st_stream(g + 1, out[r][1]);
                            }
                        }
                    }
                }
                // level 3 from the front warp's level-2 rows of the previous step
                {
                    const double *H = hand + (Q ^ 1) * PLANE_AL;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double2 a = lds2(H + (j0 + r + 1) * SPX + C0 + i0);
                        I[Q][r][0] = a.x;
                        I[Q][r][1] = a.y;
                    }
                    const double2 cm = lds2(H + j0 * SPX + C0 + i0), cp = lds2(H + (j0 + R + 1) * SPX + C0 + i0);
                    level(3, Spa, I[Q], I[Q ^ 1], cm, cp, nullptr, Mc, M[Q], s);
                    double *W = pub3 + Q * PLANE_AL;
                    sts2(W + (j0 + 1) * SPX + C0 + i0, M[Q][0][0], M[Q][0][1]);
                    sts2(W + (j0 + R) * SPX + C0 + i0, M[Q][R - 1][0], M[Q][R - 1][1]);
                }
            }
        };
        if (wint && zall) body(IC<0>{});
        else if (zall) body(IC<1>{});
        else body(IC<2>{});
    };

    for (int s = 0; s < nsteps; s += 2) {
        one_step(s, IC<0>{});
        if (s + 1 < nsteps) one_step(s + 1, IC<1>{});
    }
    if constexpr (!TMA) cp_async_wait<0>();
}

#endif  // SP200_AB

struct UnstashArgs {
    double *data;
    int64_t ex, ey;
    int nx, ny, doff, zlo, zhi, zc, nchunks, ox, oy, tiles_x, tiles_y, T2, fwd, sxpad;
    const double *sx, *sy, *sz;
    int wx2, hy2;
    int tile_lo, tile_hi;  // k_unstash_zt: the z-chunked tiles [tile_lo, tile_hi) of the in-place pass
};

__device__ __forceinline__ bool band_hit(int v, int tile, int ntiles, int o, int T2, int fwd) {
    return fwd ? (tile > 0 && v < T2) : (tile < ntiles - 1 && v >= o - T2);
}
__device__ __forceinline__ int band_pos(int k, int o, int T2, int fwd) {
    const int bt = k / T2, bo = k - bt * T2;
    return fwd ? (bt + 1) * o + bo : bt * o + o - T2 + bo;
}

// K3 epilogue: copy the stashed band outputs to their shifted frame.  The
// three stashes hold disjoint cell sets: y band first, then z band, then x
// band (the order K3 stores them).  The copies are latency-bound unless each
// thread has several loads in flight, so every thread first loads UB values,
// then stores them (measured: the one-value-per-iteration loops ran the x
// stash at a quarter of the HBM rate).
constexpr int UB = 8;

__device__ __forceinline__ void copy_row_batched(double *dst, const double *src, int n) {
    for (int b = threadIdx.x; b < n; b += UB * blockDim.x) {
        double v[UB];
#pragma unroll
        for (int i = 0; i < UB; ++i) {
            const int x = b + i * blockDim.x;
            v[i] = x < n ? __ldcs(src + x) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < UB; ++i) {
            const int x = b + i * blockDim.x;
            if (x < n) dst[x] = v[i];
        }
    }
}

// one CTA per stash row
__global__ void k_unstash_y(UnstashArgs a) {
    const int k = blockIdx.x % a.hy2, zr = blockIdx.x / a.hy2;
    const int y = band_pos(k, a.oy, a.T2, a.fwd), z = a.zlo + zr;
    if (y >= a.ny) return;
    const double *src = a.sy + (int64_t)blockIdx.x * ((a.nx + 2) & ~1) + a.sxpad;
    double *dst = a.data + ((int64_t)(z + a.doff) * a.ey + (y + a.doff)) * a.ex + a.doff;
    copy_row_batched(dst, src, a.nx);
}

__global__ void k_unstash_z(UnstashArgs a) {
    const int y = blockIdx.x % a.ny, k = blockIdx.x / a.ny;
    const int z = a.zlo + band_pos(k, a.zc, a.T2, a.fwd);
    const int ty = y / a.oy;
    if (z >= a.zhi || band_hit(y - ty * a.oy, ty, a.tiles_y, a.oy, a.T2, a.fwd)) return;
    const double *src = a.sz + (int64_t)blockIdx.x * ((a.nx + 2) & ~1) + a.sxpad;
    double *dst = a.data + ((int64_t)(z + a.doff) * a.ey + (y + a.doff)) * a.ex + a.doff;
    copy_row_batched(dst, src, a.nx);
}

// z stash of the in-place pass: only the tiles that ran as z-chunks stashed
// their chunks' first / last 2T planes, whole stored rows of the tile (no x or
// y band there); one CTA per stash row
__global__ void k_unstash_zt(UnstashArgs a) {
    const int y = blockIdx.x % a.ny, k = blockIdx.x / a.ny;
    const int z = a.zlo + band_pos(k, a.zc, a.T2, a.fwd);
    if (z >= a.zhi) return;
    const int ty = y / a.oy;
    const int t0 = max(ty * a.tiles_x, a.tile_lo), t1 = min((ty + 1) * a.tiles_x, a.tile_hi);
    if (t0 >= t1) return;
    const int xa = (t0 - ty * a.tiles_x) * a.ox, xb = min((t1 - ty * a.tiles_x) * a.ox, a.nx);
    const double *src = a.sz + (int64_t)blockIdx.x * ((a.nx + 2) & ~1) + a.sxpad;
    double *dst = a.data + ((int64_t)(z + a.doff) * a.ey + (y + a.doff)) * a.ex + a.doff;
    copy_row_batched(dst + xa, src + xa, xb - xa);
}

// x stash: CTA = UX_ROWS rows y of one plane z (blockIdx.y); thread x =
// stash column pair (tile slot bt, columns kk, kk+1 of the slot: the x band is
// stored in whole lane pairs, so a pair never straddles two slots), thread
// y + UXY*i = row i of the UB rows it copies.  Rows inside the y or z band
// belong to the other stashes and are skipped.  Pairs move as one 16-byte
// load and store (the scalar form ran at 1.8 TB/s effective, latency-bound);
// pairs with a column outside the stored tile or an odd storage x fall back
// to scalar stores.  No per-row divisions.
constexpr int UXY = 4;
constexpr int UX_ROWS = UXY * UB;
__global__ void __launch_bounds__(64 * UXY) k_unstash_x(UnstashArgs a) {
    const int zr = blockIdx.y, z = a.zlo + zr;
    {
        const int zo = zr % a.zc, chunk = zr / a.zc;
        const int zlen = min(a.zc, a.zhi - a.zlo - chunk * a.zc);
        if (a.fwd ? (chunk > 0 && zo < a.T2) : (chunk < a.nchunks - 1 && zo >= zlen - a.T2)) return;
    }
    const int y0 = blockIdx.x * UX_ROWS + threadIdx.y;
    int ty = y0 / a.oy, yo = y0 - ty * a.oy;
    const int64_t srow0 = ((int64_t)zr * a.ny + y0) * a.wx2;
    const int64_t drow0 = ((int64_t)(z + a.doff) * a.ey + (y0 + a.doff)) * a.ex + a.doff;
    unsigned live = 0;
#pragma unroll
    for (int i = 0; i < UB; ++i) {
        if (y0 + UXY * i < a.ny && !band_hit(yo, ty, a.tiles_y, a.oy, a.T2, a.fwd)) live |= 1u << i;
        yo += UXY;
        while (yo >= a.oy) {
            yo -= a.oy;
            ++ty;
        }
    }
    // stash column kk of tile slot bt holds stored-tile column lo + kk,
    // lo = -e (forward) or ox - 2T - e (backward); the forward band ends with
    // the lane pair that starts below 2T (see the x band in k_temporal)
    const int xbw = a.T2 + 2, e = a.sxpad;
    for (int c = 2 * threadIdx.x; c < a.wx2; c += 2 * blockDim.x) {
        const int bt = c / xbw, kk = c - bt * xbw;
        int xo;
        bool ok;
        if (a.fwd) {
            ok = (kk & ~1) - e < a.T2;
            xo = kk - e;
        } else {
            ok = true;
            xo = a.ox - a.T2 - e + kk;
        }
        const int x = (a.fwd ? bt + 1 : bt) * a.ox + xo;
        const bool ok0 = ok && xo >= 0 && xo < a.ox && x < a.nx;
        const bool ok1 = ok && xo + 1 >= 0 && xo + 1 < a.ox && x + 1 < a.nx;
        const bool pair = ok0 && ok1 && (((drow0 + x) & 1) == 0);
        if (!(ok0 || ok1)) continue;
        unsigned lv = live;
        double2 v[UB];
#pragma unroll
        for (int i = 0; i < UB; ++i)
            v[i] = ((lv >> i) & 1u)
                       ? __ldcs(reinterpret_cast<const double2 *>(a.sx + srow0 + (int64_t)(UXY * i) * a.wx2 + c))
                       : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < UB; ++i) {
            if (!((lv >> i) & 1u)) continue;
            double *d = a.data + drow0 + (int64_t)(UXY * i) * a.ex + x;
            if (pair) {
                *reinterpret_cast<double2 *>(d) = v[i];
            } else {
                if (ok0) d[0] = v[i].x;
                if (ok1) d[1] = v[i].y;
            }
        }
    }
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

bool tma_eligible(const void *ptr, int64_t ex, int64_t ey) {
    if ((ex * 8) % 16 != 0) return false;
    if (ptr && (reinterpret_cast<uintptr_t>(ptr) % 16) != 0) return false;
    if (ex * ey * 8 >= (int64_t(1) << 40)) return false;
    return true;
}

struct LaunchReq {
    const double *src;
    double *dst;
    int64_t ex, ey, ez, nx, ny, nz, off, doff, zlo, zhi;
    int direction;  // 0: two-grid (K1/K2); +1/-1: compressed in place (K3)
    void *ws;       // K3 workspace: the band stash
    int64_t ws_bytes;
    cudaStream_t stream;
    double *mirror = nullptr;     // two-grid: peer grid receiving every stored plane
    int64_t mirror_zshift = 0;    // storage plane z of dst -> z + zshift of mirror
    bool ring = false;            // depth 1: fused ring copy (reference_sweep)
};

template <int T, int CY, int CL = 1>
static int tile_geometry(int64_t nx, int64_t ny, int64_t off, bool aligned, int *ox, int *ex0,
                         int *tiles_x, int *tiles_y) {
    using C = KCfg<T, CY, 4, 4>;
    constexpr int OYc = CL * CY - 2 * (T - 1);
    const int par = aligned ? (int)((off - (T - 1)) & 1) : 0;
    *ox = C::CX - 2 * (T - 1) - 2 * par;
    *ex0 = (T - 1) + par;
    *tiles_x = (int)((nx + *ox - 1) / *ox);
    *tiles_y = (int)((ny + OYc - 1) / OYc);
    return par;
}

// <<<>>> for CL == 1, cudaLaunchKernelEx with a (CL, 1, 1) cluster otherwise;
// `units` counts tiles x chunks, CL CTAs each
template <int CL, typename K>
static void launch_units(K kern, int64_t units, int nt, size_t smem, cudaStream_t stream,
                         const TParams &p, const CUtensorMap &tmap) {
    if constexpr (CL == 1) {
        kern<<<(unsigned)units, nt, smem, stream>>>(p, tmap);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(units * CL), 1, 1);
        cfg.blockDim = dim3(nt, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, p, tmap);
    }
}

static int64_t pick_zchunk(int64_t depth, int64_t ntiles, int64_t slots, int T) {
    double best = 1e300;
    int64_t zc = depth;
    for (int64_t c = 1; c <= 256 && c <= depth; ++c) {
        int64_t len = (depth + c - 1) / c;
        int64_t units = ntiles * ((depth + len - 1) / len);
        double waves = (double)((units + slots - 1) / slots);
        // a partial last wave still costs a whole wave; a short chunk pays the
        // (3T-1)-step pipeline fill/drain
        double cost = waves * (double)(len + 3 * T - 1);
        if (cost < best * 0.999) {
            best = cost;
            zc = len;
        }
    }
    return zc;
}

struct CompLayout {
    int64_t zc, nchunks, nx_stash, ny_stash, nz_stash;
    int wx2, hy2;
};

// K3 geometry: z-chunks (>= 2T planes, one CTA per SM assumed so the layout is
// the same for sizing and launch) and the three band stashes.
template <int T, int CY>
static void comp_layout(int64_t nx, int64_t ny, int64_t depth, int64_t off, bool aligned,
                        CompLayout *L) {
    int ox, ex0, tx, ty;
    tile_geometry<T, CY>(nx, ny, off, aligned, &ox, &ex0, &tx, &ty);
    int64_t zc = tuning().zchunk > 0 ? tuning().zchunk
                                     : pick_zchunk(depth, (int64_t)tx * ty, sm_count(), T);
    if (zc < 2 * T) zc = std::min<int64_t>(depth, 2 * T);
    L->zc = zc;
    L->nchunks = (depth + zc - 1) / zc;
    L->wx2 = (tx - 1) * (2 * T + 2);
    L->hy2 = (ty - 1) * 2 * T;
    L->nx_stash = depth * ny * L->wx2;
    L->ny_stash = depth * L->hy2 * ((nx + 2) & ~1);
    L->nz_stash = (L->nchunks - 1) * 2 * T * ny * ((nx + 2) & ~1);
}

template <int T, int CY, int R, int S, int CL = 1, bool MIRROR = false, bool WP = false,
          bool XS1 = false, bool PS = false>
static int launch_cfg(const LaunchReq &q) {
    using C = KCfg<T, CY, R, S>;
    constexpr size_t SMEM_B = C::SMEM + (PS ? 8 * S : 0);  // + the PS empty barriers
    const bool comp = q.direction != 0;
    if constexpr (CL > 1) {
        if (comp) return launch_cfg<T, CY, R, S, 1>(q);  // K3 runs unclustered
    }
    // Pair alignment: region column 0 must sit at an even storage x (16-byte
    // aligned pairs for LDS.128 / STG.128 and the TMA box origin).  Tiles
    // start at multiples of the (even) stored width, so the parity of the
    // region origin is the same for every tile: shift it by one column when
    // needed and give up one stored column pair.
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(q.dst) | reinterpret_cast<uintptr_t>(q.src)) % 16 == 0) &&
        (q.ex % 2 == 0);
    TParams p;
    int tiles_y;
    tile_geometry<T, CY, CL>(q.nx, q.ny, q.off, aligned, &p.ox, &p.ex0, &p.tiles_x, &tiles_y);
    const bool use_tma =
        aligned && !tuning().force_cpasync && tma_eligible(q.src, q.ex, q.ey) && encode_fn();
    p.src = q.src;
    p.dst = q.dst;
    p.ex = q.ex;
    p.ey = q.ey;
    p.ez = q.ez;
    p.nx = (int)q.nx;
    p.ny = (int)q.ny;
    p.nz = (int)q.nz;
    p.off = (int)q.off;
    p.doff = (int)q.doff;
    p.direction = q.direction;
    p.pair_store = (aligned && ((q.off - q.doff) % 2 == 0)) ? 1 : 0;
    p.tiles_y = tiles_y;
    p.ntiles = p.tiles_x * tiles_y;
    p.zlo = (int)q.zlo;
    p.zhi = (int)q.zhi;
    p.stash_x = p.stash_y = p.stash_z = nullptr;
    p.progress = nullptr;
    p.nslots = 0;
    p.debug = (int)tuning().debug;
    p.wx2 = p.hy2 = 0;

    void (*kern)(const TParams, const CUtensorMap);
    p.mir = nullptr;
    if constexpr (MIRROR) {
        // fused peer stores need the TMA instance; otherwise the planes are
        // copied to the peer after the pass (same stream, DMA over NVLink)
        if (use_tma) {
            p.mir = q.mirror + q.mirror_zshift * q.ex * q.ey;
            kern = k_temporal<T, CY, R, S, true, false, 1, true>;
        } else {
            kern = k_temporal<T, CY, R, S, false, false, 1>;
        }
    } else if constexpr (CL > 1) {
        kern = use_tma ? k_temporal<T, CY, R, S, true, false, CL>
                       : k_temporal<T, CY, R, S, false, false, CL>;
    } else if (comp) {
        kern = use_tma ? k_temporal<T, CY, R, S, true, true, 1> : k_temporal<T, CY, R, S, false, true, 1>;
    } else if constexpr (PS) {
        kern = use_tma ? k_temporal<T, CY, R, S, true, false, 1, false, false, false, false, true>
                       : k_temporal<T, CY, R, S, false, false, 1>;
    } else if constexpr (XS1) {
        kern = use_tma ? k_temporal<T, CY, R, S, true, false, 1, false, false, false, true>
                       : k_temporal<T, CY, R, S, false, false, 1, false, false, false, true>;
    } else {
        kern = use_tma ? k_temporal<T, CY, R, S, true, false, 1, false, WP>
                       : k_temporal<T, CY, R, S, false, false, 1>;
        if constexpr (T == 1 && !WP) {
            if (q.ring)
                kern = use_tma ? k_temporal<T, CY, R, S, true, false, 1, false, false, true>
                               : k_temporal<T, CY, R, S, false, false, 1, false, false, true>;
        }
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_B);
    if (e != cudaSuccess)
        return set_error(SP_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));

    const int64_t depth = q.zhi - q.zlo;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, SMEM_B);
    if (occ < 1) occ = 1;
    // concurrently resident units (tiles x chunks), CL CTAs each
    int64_t slots = (int64_t)sm_count() * occ / CL;
    if constexpr (CL > 1) {
        cudaLaunchConfig_t oc = {};
        oc.gridDim = dim3((unsigned)(slots * CL), 1, 1);
        oc.blockDim = dim3(C::NT, 1, 1);
        oc.dynamicSmemBytes = SMEM_B;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        oc.attrs = at;
        oc.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &oc) == cudaSuccess && ncl > 0) slots = ncl;
        cudaGetLastError();
        if (getenv("SP200_VERBOSE")) fprintf(stderr, "sp200: T=%d CL=%d max active clusters %d\n", T, CL, ncl);
    }
    int64_t grid;
    CompLayout L;
    if (comp) {
        comp_layout<T, CY>(q.nx, q.ny, q.zhi - q.zlo, q.off, aligned, &L);
        const int64_t need = 8 * (L.nx_stash + L.ny_stash + L.nz_stash);
        if (need > q.ws_bytes)
            return set_error(SP_EINVAL, "compressed pass needs %lld workspace bytes, got %lld",
                             (long long)need, (long long)q.ws_bytes);
        p.zc = (int)L.zc;
        grid = (int64_t)p.ntiles * L.nchunks;
        char *ws = reinterpret_cast<char *>(q.ws);
        p.stash_x = reinterpret_cast<double *>(ws);
        p.stash_y = p.stash_x + L.nx_stash;
        p.stash_z = p.stash_y + L.ny_stash;
        p.wx2 = L.wx2;
        p.hy2 = L.hy2;
    } else {
        // z-chunking: choose the chunk count minimising (waves x steps per chunk)
        int64_t zc = tuning().zchunk;
        // T = 1 (plain sweep, HBM-bound): short chunks of about 12 planes
        // keep concurrently running CTAs at the same z, so their streams
        // share DRAM pages; with 15+ waves of 2 CTAs per SM the wave
        // quantisation of the model below does not matter (512^3: 8 / 12 /
        // 16 / 32 / 64 planes 387 / 393 / 385 / 373 / 345 GLUP/s; whole
        // columns 274)
        if (zc <= 0) {
            if (T == 1) {
                const int64_t c = (depth + 11) / 12;
                zc = (depth + c - 1) / c;
            } else {
                zc = pick_zchunk(depth, p.ntiles, slots, T);
            }
        }
        if (zc < 1) zc = 1;
        p.zc = (int)zc;
        grid = (int64_t)p.ntiles * ((depth + zc - 1) / zc);
    }
    p.tile_base = 0;
    p.tile_count = p.ntiles;
    p.split = 0x7fffffff;
    p.tile_base2 = p.tile_count2 = p.zc2 = 0;
    p.piece = 0;
    if (grid * CL > 0x7fffffff) return set_error(SP_EUNSUP, "grid too large");

    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (use_tma) {
        cuuint64_t dims[3] = {(cuuint64_t)q.ex, (cuuint64_t)q.ey, (cuuint64_t)q.ez};
        cuuint64_t strides[2] = {(cuuint64_t)(q.ex * 8), (cuuint64_t)(q.ex * q.ey * 8)};
        cuuint32_t box[3] = {(cuuint32_t)C::SPX, (cuuint32_t)C::PY, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)q.src, dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(SP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    if (!comp && T > 1 && tuning().zchunk <= 0 && p.ntiles >= slots) {
        // Two launches: whole slots-worth of tiles march their full column
        // (no pipeline restarts), the remaining tiles are split into z-chunks
        // so that together they fill one more wave.  Both keep neighbouring
        // tiles at the same z at the same time (L2 catches the halos).
        const int full = (int)((p.ntiles / slots) * slots);
        const int rem = p.ntiles - full;
        if (tuning().balanced_split && CL == 1 && rem > 0) {
            // every CTA: one full column, then an equal piece of the rest
            TParams a = p;
            a.tile_base = 0;
            a.tile_count = full;
            a.split = full;
            a.tile_base2 = full;
            a.tile_count2 = rem;
            a.piece = (int)(((int64_t)rem * depth + full - 1) / full);
            launch_units<CL>(kern, full, C::NT, SMEM_B, q.stream, a, tmap);
            count_launch();
            return check_launch("k_temporal");
        }
        if (!tuning().two_launch && rem > 0) {
            // one grid: the chunk CTAs follow the full-column CTAs in
            // blockIdx order, so each starts on the first SM that frees up
            // instead of behind the slowest full column (no kernel boundary)
            TParams a = p;
            a.tile_base = 0;
            a.tile_count = full;
            a.zc = (int)depth;
            a.split = full;
            a.tile_base2 = full;
            a.tile_count2 = rem;
            const int64_t zcb = tuning().zchunk2 > 0 ? std::min<int64_t>(tuning().zchunk2, depth)
                                                     : pick_zchunk(depth, rem, slots, T);
            a.zc2 = (int)zcb;
            const int64_t gb = (int64_t)rem * ((depth + zcb - 1) / zcb);
            launch_units<CL>(kern, full + gb, C::NT, SMEM_B, q.stream, a, tmap);
            count_launch();
            return check_launch("k_temporal");
        }
        TParams a = p;
        a.tile_base = 0;
        a.tile_count = full;
        a.zc = (int)depth;
        launch_units<CL>(kern, full, C::NT, SMEM_B, q.stream, a, tmap);
        count_launch();
        int rc = check_launch("k_temporal");
        if (rc || rem == 0) return rc;
        TParams b = p;
        b.tile_base = full;
        b.tile_count = rem;
        const int64_t zcb = pick_zchunk(depth, rem, slots, T);
        b.zc = (int)zcb;
        const int64_t gb = (int64_t)rem * ((depth + zcb - 1) / zcb);
        launch_units<CL>(kern, gb, C::NT, SMEM_B, q.stream, b, tmap);
        count_launch();
        return check_launch("k_temporal");
    }
    launch_units<CL>(kern, grid, C::NT, SMEM_B, q.stream, p, tmap);
    count_launch();
    int rc = check_launch("k_temporal");
    if (rc || !comp) return rc;
    UnstashArgs u;
    u.data = q.dst;
    u.ex = q.ex;
    u.ey = q.ey;
    u.nx = (int)q.nx;
    u.ny = (int)q.ny;
    u.doff = (int)q.doff;
    u.zlo = (int)q.zlo;
    u.zhi = (int)q.zhi;
    u.zc = (int)L.zc;
    u.nchunks = (int)L.nchunks;
    u.ox = p.ox;
    u.oy = C::OY;
    u.tiles_x = p.tiles_x;
    u.tiles_y = p.tiles_y;
    u.T2 = 2 * T;
    u.fwd = q.direction > 0 ? 1 : 0;
    u.sx = p.stash_x;
    u.sy = p.stash_y;
    u.sz = p.stash_z;
    u.wx2 = p.wx2;
    u.hy2 = p.hy2;
    u.sxpad = p.ex0 & 1;
    const int64_t depth_ = q.zhi - q.zlo;
    if (L.hy2 > 0) {
        k_unstash_y<<<(unsigned)(depth_ * L.hy2), 128, 0, q.stream>>>(u);
        count_launch();
    }
    if (L.nchunks > 1) {
        k_unstash_z<<<(unsigned)((L.nchunks - 1) * 2 * T * q.ny), 128, 0, q.stream>>>(u);
        count_launch();
    }
    if (L.wx2 > 0) {
        k_unstash_x<<<dim3((unsigned)((q.ny + UX_ROWS - 1) / UX_ROWS), (unsigned)depth_), dim3(64, UXY), 0,
                      q.stream>>>(u);
        count_launch();
    }
    rc = check_launch("k_unstash");
    return rc;
}




// K3 in place (T levels, TMA-eligible arrays): geometry of the two launches.
// `full` tiles (whole multiples of the SM count) march their whole column in
// the first launch; the `rem` tiles after them run in the second launch as
// z-chunks sized to fill the GPU once more, chunk-major.  Chunks of one tile
// are decoupled by a z stash (the first / last 2T planes of a chunk, copied
// into place by k_unstash_zt); x and y stay in place in both launches.
struct InplaceLayout {
    int ox, ex0, tiles_x, tiles_y, ntiles, full, rem;
    int64_t zc2, nch2, lines, nz_stash;  // progress lines (128 B each), z-stash doubles
};

template <int T, int CY>
static void inplace_layout(int64_t nx, int64_t ny, int64_t depth, int64_t off, InplaceLayout *L) {
    tile_geometry<T, CY>(nx, ny, off, true, &L->ox, &L->ex0, &L->tiles_x, &L->tiles_y);
    L->ntiles = L->tiles_x * L->tiles_y;
    const int64_t slots = sm_count();
    L->full = L->ntiles >= slots ? (int)((L->ntiles / slots) * slots) : 0;
    L->rem = L->ntiles - L->full;
    L->zc2 = depth;
    L->nch2 = 1;
    if (L->rem > 0 && !tuning().balanced_split) {
        int64_t zc = tuning().zchunk2 > 0 ? std::min<int64_t>(tuning().zchunk2, depth)
                                          : pick_zchunk(depth, L->rem, slots, T);
        if (zc < 2 * T) zc = std::min<int64_t>(depth, 2 * T);
        L->zc2 = zc;
        L->nch2 = (depth + zc - 1) / zc;
    }
    if (L->nch2 == 1) {
        // whole columns only: one launch
        L->full = L->ntiles;
        L->rem = 0;
    }
    L->lines = (L->full > 0 ? L->full + 1 : 0) + (L->rem > 0 ? (int64_t)L->rem * L->nch2 + 1 : 0);
    L->nz_stash = L->rem > 0 ? (L->nch2 - 1) * 2 * T * ny * ((nx + 2) & ~1) : 0;
}

template <int T, int CY>
static int64_t inplace_bytes(const InplaceLayout &L) {
    return L.lines * 4 * PROG_STRIDE + 8 * L.nz_stash;
}

template <int T, int CY, int R, int S>
static int launch_inplace(const LaunchReq &q) {
    using C = KCfg<T, CY, R, S>;
    InplaceLayout L;
    inplace_layout<T, CY>(q.nx, q.ny, q.zhi - q.zlo, q.off, &L);
    const int64_t need = inplace_bytes<T, CY>(L);
    if (need > q.ws_bytes)
        return set_error(SP_EINVAL, "compressed pass needs %lld workspace bytes, got %lld", (long long)need,
                         (long long)q.ws_bytes);
    TParams p;
    memset(&p, 0, sizeof(p));
    p.src = q.src;
    p.dst = q.dst;
    p.ex = q.ex;
    p.ey = q.ey;
    p.ez = q.ez;
    p.nx = (int)q.nx;
    p.ny = (int)q.ny;
    p.nz = (int)q.nz;
    p.off = (int)q.off;
    p.doff = (int)q.doff;
    p.direction = q.direction;
    p.ox = L.ox;
    p.ex0 = L.ex0;
    p.tiles_x = L.tiles_x;
    p.tiles_y = L.tiles_y;
    p.ntiles = L.ntiles;
    p.pair_store = ((q.off - q.doff) % 2 == 0) ? 1 : 0;
    p.zlo = (int)q.zlo;
    p.zhi = (int)q.zhi;
    p.debug = (int)tuning().debug;
    p.tile_count = L.ntiles;
    p.split = 0x7fffffff;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    {
        cuuint64_t dims[3] = {(cuuint64_t)q.ex, (cuuint64_t)q.ey, (cuuint64_t)q.ez};
        cuuint64_t strides[2] = {(cuuint64_t)(q.ex * 8), (cuuint64_t)(q.ex * q.ey * 8)};
        cuuint32_t box[3] = {(cuuint32_t)C::SPX, (cuuint32_t)C::PY, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)q.src, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(SP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
#if SP200_PROFILE_KNOBS
    // timing experiment (p.debug bit 1024, wrong results): store out of place
    // into a scratch array, to separate the in-place memory pattern from the
    // kernel's instruction stream
    if (tuning().debug & 1024) {
        static double *scratch = nullptr;
        static size_t scratch_n = 0;
        const size_t n = (size_t)(q.ex * q.ey * q.ez);
        if (scratch_n < n) {
            if (scratch) cudaFree(scratch);
            cudaMalloc(&scratch, n * sizeof(double));
            scratch_n = n;
        }
        p.dst = scratch;
    }
#endif
    char *ws = reinterpret_cast<char *>(q.ws);
    cudaMemsetAsync(ws, 0, (size_t)(L.lines * 4 * PROG_STRIDE), q.stream);
    int *prog = reinterpret_cast<int *>(ws);
    const int64_t depth = q.zhi - q.zlo;
    if (L.full > 0) {
        auto kern = k_temporal<T, CY, R, S, true, true, 1, false, false, false, false, false, true, false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM + 192);
        if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        TParams a = p;
        a.zc = (int)depth;
        a.progress = prog;
        a.nslots = L.full;
#if SP200_PROFILE_KNOBS
        // timing experiment (p.debug bit 2048, wrong results): the two-grid
        // instance on the same units, no tickets and no waits
        if (tuning().debug & 2048) {
            auto k2 = k_temporal<T, CY, R, S, true, false, 1>;
            cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM + 192);
            a.tile_count = L.full;
            k2<<<(unsigned)L.full, C::NT, C::SMEM + 192, q.stream>>>(a, tmap);
        } else
#endif
        kern<<<(unsigned)L.full, C::NT, C::SMEM + 192, q.stream>>>(a, tmap);
        count_launch();
        int rc = check_launch("k_temporal (in place)");
        if (rc) return rc;
        prog += (int64_t)(L.full + 1) * PROG_STRIDE;
    }
    if (L.rem > 0) {
        auto kern = k_temporal<T, CY, R, S, true, true, 1, false, false, false, false, false, true, true>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM + 192);
        if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        TParams b = p;
        b.zc = (int)L.zc2;
        b.split = L.full;
        b.tile_count2 = L.rem;
        b.progress = prog;
        b.nslots = (int)(L.rem * L.nch2);
        b.stash_z = reinterpret_cast<double *>(ws + L.lines * 4 * PROG_STRIDE);
        kern<<<(unsigned)(L.rem * L.nch2), C::NT, C::SMEM + 192, q.stream>>>(b, tmap);
        count_launch();
        int rc = check_launch("k_temporal (in place, z chunks)");
        if (rc) return rc;
        UnstashArgs u;
        memset(&u, 0, sizeof(u));
        u.data = q.dst;
        u.ex = q.ex;
        u.ey = q.ey;
        u.nx = (int)q.nx;
        u.ny = (int)q.ny;
        u.doff = (int)q.doff;
        u.zlo = (int)q.zlo;
        u.zhi = (int)q.zhi;
        u.zc = (int)L.zc2;
        u.nchunks = (int)L.nch2;
        u.ox = L.ox;
        u.oy = C::OY;
        u.tiles_x = L.tiles_x;
        u.tiles_y = L.tiles_y;
        u.T2 = 2 * T;
        u.fwd = q.direction > 0 ? 1 : 0;
        u.sz = b.stash_z;
        u.sxpad = L.ex0 & 1;
        // the z-chunked tiles in tile order: the last `rem` (forward) or the first `rem` (backward)
        u.tile_lo = q.direction > 0 ? L.full : 0;
        u.tile_hi = q.direction > 0 ? L.ntiles : L.rem;
        k_unstash_zt<<<(unsigned)((L.nch2 - 1) * 2 * T * q.ny), 128, 0, q.stream>>>(u);
        count_launch();
        return check_launch("k_unstash_zt");
    }
    return SP_OK;
}

#if SP200_AB

// Host launch of k_tm (two-grid fused passes, TMA loader, pair-aligned
// frames): launch_cfg's geometry and split schedule with the 64 x NW*R region.
template <int T, int R, int NW, int S, int NSPT>
static int launch_tm(const LaunchReq &q) {
    using C = TMCfg<T, R, NW, S, NSPT>;
    constexpr int CY = C::CY;
    TParams p;
    memset(&p, 0, sizeof(p));
    int tiles_y;
    tile_geometry<T, CY>(q.nx, q.ny, q.off, true, &p.ox, &p.ex0, &p.tiles_x, &tiles_y);
    p.src = q.src;
    p.dst = q.dst;
    p.ex = q.ex;
    p.ey = q.ey;
    p.ez = q.ez;
    p.nx = (int)q.nx;
    p.ny = (int)q.ny;
    p.nz = (int)q.nz;
    p.off = (int)q.off;
    p.doff = (int)q.doff;
    p.pair_store = ((q.off - q.doff) % 2 == 0) ? 1 : 0;
    p.tiles_y = tiles_y;
    p.ntiles = p.tiles_x * tiles_y;
    p.zlo = (int)q.zlo;
    p.zhi = (int)q.zhi;
    void (*kern)(const TParams, const CUtensorMap);
    if (q.mirror) {
        p.mir = q.mirror + q.mirror_zshift * q.ex * q.ey;
        kern = k_tm<T, R, NW, S, NSPT, true>;
    } else {
        kern = k_tm<T, R, NW, S, NSPT, false>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    const int64_t slots = sm_count();
    const int64_t depth = q.zhi - q.zlo;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    {
        cuuint64_t dims[3] = {(cuuint64_t)q.ex, (cuuint64_t)q.ey, (cuuint64_t)q.ez};
        cuuint64_t strides[2] = {(cuuint64_t)(q.ex * 8), (cuuint64_t)(q.ex * q.ey * 8)};
        cuuint32_t box[3] = {(cuuint32_t)C::SPX, (cuuint32_t)C::PY, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)q.src, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(SP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    p.tile_base = 0;
    p.tile_count = p.ntiles;
    p.split = 0x7fffffff;
    int64_t grid;
    if (tuning().zchunk <= 0 && p.ntiles >= slots) {
        // one grid: `full` tiles march their whole column, the rest follow in
        // blockIdx order as z-chunks sized to fill one more wave
        const int full = (int)((p.ntiles / slots) * slots);
        const int rem = p.ntiles - full;
        p.tile_count = full;
        p.zc = (int)depth;
        grid = full;
        if (rem > 0) {
            p.split = full;
            p.tile_base2 = full;
            p.tile_count2 = rem;
            const int64_t zcb = tuning().zchunk2 > 0 ? std::min<int64_t>(tuning().zchunk2, depth)
                                                     : pick_zchunk(depth, rem, slots, T);
            p.zc2 = (int)zcb;
            grid += (int64_t)rem * ((depth + zcb - 1) / zcb);
        }
    } else {
        int64_t zc = tuning().zchunk > 0 ? tuning().zchunk : pick_zchunk(depth, p.ntiles, slots, T);
        if (zc < 1) zc = 1;
        p.zc = (int)zc;
        grid = (int64_t)p.ntiles * ((depth + zc - 1) / zc);
    }
    if (grid > 0x7fffffff) return set_error(SP_EUNSUP, "grid too large");
    kern<<<(unsigned)grid, C::NT, C::SMEM, q.stream>>>(p, tmap);
    count_launch();
    return check_launch("k_tm");
}


// Host launch of k_split (A/B: tuning key 9 = 4): the launch_cfg geometry of
// the T=4 pair layout, 512 threads per CTA.
template <int S>
static int launch_split(const LaunchReq &q) {
    using C = KCfg<4, 32, 4, S>;
    constexpr size_t SMEM = (size_t)(S + 6) * C::PLANE_AL * 8 + 8 * S + 16;
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(q.dst) | reinterpret_cast<uintptr_t>(q.src)) % 16 == 0) && (q.ex % 2 == 0);
    TParams p;
    memset(&p, 0, sizeof(p));
    int tiles_y;
    tile_geometry<4, 32>(q.nx, q.ny, q.off, aligned, &p.ox, &p.ex0, &p.tiles_x, &tiles_y);
    const bool use_tma = aligned && !tuning().force_cpasync && tma_eligible(q.src, q.ex, q.ey) && encode_fn();
    p.src = q.src;
    p.dst = q.dst;
    p.ex = q.ex;
    p.ey = q.ey;
    p.ez = q.ez;
    p.nx = (int)q.nx;
    p.ny = (int)q.ny;
    p.nz = (int)q.nz;
    p.off = (int)q.off;
    p.doff = (int)q.doff;
    p.pair_store = (aligned && ((q.off - q.doff) % 2 == 0)) ? 1 : 0;
    p.tiles_y = tiles_y;
    p.ntiles = p.tiles_x * tiles_y;
    p.zlo = (int)q.zlo;
    p.zhi = (int)q.zhi;
    void (*kern)(const TParams, const CUtensorMap) = use_tma ? k_split<S, true> : k_split<S, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    const int64_t slots = sm_count();
    const int64_t depth = q.zhi - q.zlo;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (use_tma) {
        cuuint64_t dims[3] = {(cuuint64_t)q.ex, (cuuint64_t)q.ey, (cuuint64_t)q.ez};
        cuuint64_t strides[2] = {(cuuint64_t)(q.ex * 8), (cuuint64_t)(q.ex * q.ey * 8)};
        cuuint32_t box[3] = {(cuuint32_t)C::SPX, (cuuint32_t)C::PY, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)q.src, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(SP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    p.tile_base = 0;
    p.tile_count = p.ntiles;
    p.split = 0x7fffffff;
    int64_t grid;
    if (tuning().zchunk <= 0 && p.ntiles >= slots) {
        const int full = (int)((p.ntiles / slots) * slots);
        const int rem = p.ntiles - full;
        p.tile_count = full;
        p.zc = (int)depth;
        grid = full;
        if (rem > 0) {
            p.split = full;
            p.tile_base2 = full;
            p.tile_count2 = rem;
            const int64_t zcb = pick_zchunk(depth, rem, slots, 4);
            p.zc2 = (int)zcb;
            grid += (int64_t)rem * ((depth + zcb - 1) / zcb);
        }
    } else {
        int64_t zc = tuning().zchunk > 0 ? tuning().zchunk : pick_zchunk(depth, p.ntiles, slots, 4);
        if (zc < 1) zc = 1;
        p.zc = (int)zc;
        grid = (int64_t)p.ntiles * ((depth + zc - 1) / zc);
    }
    kern<<<(unsigned)grid, 512, SMEM, q.stream>>>(p, tmap);
    count_launch();
    return check_launch("k_split");
}

// Host launch of k_col (two-grid passes, T = 2..4): same split schedule as
// launch_cfg (full columns for one wave, the remaining tiles z-chunked).
template <int T, int R, int NW, int S, bool XS, bool MIRROR = false>
static int launch_col(const LaunchReq &q) {
    using C = CCfg<T, R, NW>;
    constexpr size_t SMEM = C::template smem<S>();
    const bool use_tma = !tuning().force_cpasync && tma_eligible(q.src, q.ex, q.ey) && encode_fn();
    TParams p;
    memset(&p, 0, sizeof(p));
    p.src = q.src;
    p.dst = q.dst;
    p.ex = q.ex;
    p.ey = q.ey;
    p.ez = q.ez;
    p.nx = (int)q.nx;
    p.ny = (int)q.ny;
    p.nz = (int)q.nz;
    p.off = (int)q.off;
    p.doff = (int)q.doff;
    p.ox = C::OX;
    p.ex0 = T - 1;
    p.tiles_x = (int)((q.nx + C::OX - 1) / C::OX);
    p.tiles_y = (int)((q.ny + C::OY - 1) / C::OY);
    p.ntiles = p.tiles_x * p.tiles_y;
    p.zlo = (int)q.zlo;
    p.zhi = (int)q.zhi;
    // region column 0 sits at storage x = tx*OX - (T-1) + off (OX even), so
    // c0 = 2 or 3 puts every tile's TMA box start on a 16-byte boundary
    p.c0 = 2 + (int)((q.off - (T - 1)) & 1);
    void (*kern)(const TParams, const CUtensorMap);
    if constexpr (MIRROR) {
        p.mir = q.mirror + q.mirror_zshift * q.ex * q.ey;
        kern = use_tma ? k_col<T, R, NW, S, true, XS, true> : k_col<T, R, NW, S, false, XS, true>;
    } else {
        kern = use_tma ? k_col<T, R, NW, S, true, XS> : k_col<T, R, NW, S, false, XS>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, SMEM);
    if (occ < 1) occ = 1;
    const int64_t slots = (int64_t)sm_count() * occ;
    const int64_t depth = q.zhi - q.zlo;

    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (use_tma) {
        cuuint64_t dims[3] = {(cuuint64_t)q.ex, (cuuint64_t)q.ey, (cuuint64_t)q.ez};
        cuuint64_t strides[2] = {(cuuint64_t)(q.ex * 8), (cuuint64_t)(q.ex * q.ey * 8)};
        cuuint32_t box[3] = {(cuuint32_t)C::SPX, (cuuint32_t)C::PY, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)q.src, dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(SP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    p.tile_base = 0;
    p.tile_count = p.ntiles;
    p.split = 0x7fffffff;
    int64_t grid;
    if (tuning().zchunk <= 0 && p.ntiles >= slots) {
        // one grid: `full` tiles march their whole column, the rest follow in
        // blockIdx order as z-chunks sized to fill one more wave
        const int full = (int)((p.ntiles / slots) * slots);
        const int rem = p.ntiles - full;
        p.tile_count = full;
        p.zc = (int)depth;
        if (rem > 0) {
            p.split = full;
            p.tile_base2 = full;
            p.tile_count2 = rem;
            const int64_t zcb = tuning().zchunk2 > 0 ? std::min<int64_t>(tuning().zchunk2, depth)
                                                     : pick_zchunk(depth, rem, slots, T);
            p.zc2 = (int)zcb;
            grid = full + (int64_t)rem * ((depth + zcb - 1) / zcb);
        } else {
            grid = full;
        }
    } else {
        int64_t zc = tuning().zchunk > 0 ? tuning().zchunk : pick_zchunk(depth, p.ntiles, slots, T);
        if (zc < 1) zc = 1;
        p.zc = (int)zc;
        grid = (int64_t)p.ntiles * ((depth + zc - 1) / zc);
    }
    if (grid > 0x7fffffff) return set_error(SP_EUNSUP, "grid too large");
    kern<<<(unsigned)grid, C::NT, SMEM, q.stream>>>(p, tmap);
    count_launch();
    return check_launch("k_col");
}

// two-grid K2 with the column layout (tuning key 9: 0 lane pairs, 1 columns
// with level-1 x-neighbours from the stage, 2 columns with level-1 shuffles)
template <bool MIRROR>
static int dispatch_col(int levels, const LaunchReq &q, bool xs) {
    switch (levels) {
    case 2: return xs ? launch_col<2, 8, 12, 4, true, MIRROR>(q) : launch_col<2, 8, 12, 4, false, MIRROR>(q);
    case 3: return xs ? launch_col<3, 6, 12, 4, true, MIRROR>(q) : launch_col<3, 6, 12, 4, false, MIRROR>(q);
    case 4: return xs ? launch_col<4, 8, 8, 4, true, MIRROR>(q) : launch_col<4, 8, 8, 4, false, MIRROR>(q);
    default: return set_error(SP_EUNSUP, "levels %d unsupported", levels);
    }
}

#endif  // SP200_AB

static int dispatch(int levels, const LaunchReq &q);

static bool uses_tma(const LaunchReq &q) {
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(q.dst) | reinterpret_cast<uintptr_t>(q.src)) % 16 == 0) &&
        (q.ex % 2 == 0);
    return aligned && !tuning().force_cpasync && tma_eligible(q.src, q.ex, q.ey) && encode_fn();
}

// Two-grid pass whose stored planes also go to a peer rank's grid: the TMA
// instances store them from the kernel (MIR); otherwise, and for the plain
// sweep, the finished planes are copied after the pass on the same stream.
static int dispatch_mirror(int levels, const LaunchReq &q) {
    int rc;
    const bool fused = levels > 1 && uses_tma(q);
    switch (fused ? levels : 0) {
    case 2: rc = launch_cfg<2, 48, 4, 4, 1, true>(q); break;
    case 3: rc = launch_cfg<3, 36, 3, 4, 1, true>(q); break;
    case 4: rc = launch_cfg<4, 32, 4, 4, 1, true>(q); break;
    default: {
        LaunchReq plain = q;
        plain.mirror = nullptr;
#if SP200_AB
        rc = (levels == 1 && tuning().cfg_index[1] >= 1 && tuning().cfg_index[1] <= 4)
                 ? launch_sweep1(q.src, q.dst, q.ex, q.ey, q.ez, q.nx, q.ny, q.nz, q.off, q.zlo, q.zhi,
                                 false, q.stream)
                 : dispatch(levels, plain);
#else
        rc = dispatch(levels, plain);
#endif
        break;
    }
    }
    if (rc || fused) return rc;
    const int64_t pz = q.ex * q.ey;
    const int64_t z0 = q.zlo + q.off;
    cudaError_t e = cudaMemcpyAsync(q.mirror + (z0 + q.mirror_zshift) * pz, q.dst + z0 * pz,
                                    (size_t)((q.zhi - q.zlo) * pz) * sizeof(double),
                                    cudaMemcpyDeviceToDevice, q.stream);
    if (e != cudaSuccess) return set_error(SP_ECUDA, "mirror copy: %s", cudaGetErrorString(e));
    return SP_OK;
}

static int dispatch(int levels, const LaunchReq &q) {
#if SP200_AB
    // A/B layouts (tuning key 9), DESIGN.md §8
    if (q.direction == 0 && levels == 4 && !q.mirror && tuning().k2_layout == 4) return launch_split<4>(q);
    if (q.direction == 0 && levels >= 2 && !q.mirror && !q.ring && tuning().k2_layout == 5) {
        switch (levels) {
        case 2: return launch_cfg<2, 48, 4, 6, 1, false, false, false, true>(q);
        case 3: return launch_cfg<3, 36, 3, 6, 1, false, false, false, true>(q);
        default: return launch_cfg<4, 32, 4, 6, 1, false, false, false, true>(q);
        }
    }
    if (q.direction == 0 && levels >= 2 && !q.mirror && tuning().k2_layout == 3) {
        switch (levels) {
        case 2: return launch_cfg<2, 48, 4, 4, 1, false, false, true>(q);
        case 3: return launch_cfg<3, 36, 3, 4, 1, false, false, true>(q);
        default: return launch_cfg<4, 32, 4, 4, 1, false, false, true>(q);
        }
    }
    if (q.direction == 0 && levels >= 2 && !q.ring && tuning().k2_layout > 0 && tuning().k2_layout < 3) {
        const bool xs = tuning().k2_layout == 2;
        return q.mirror ? dispatch_col<true>(levels, q, xs) : dispatch_col<false>(levels, q, xs);
    }
#endif
#if SP200_AB
    // k_tm: pipeline state in tensor memory (tuning key 9 = 6..10), DESIGN.md §8
    if (q.direction == 0 && levels == 4 && !q.ring && tuning().k2_layout >= 6 && uses_tma(q)) {
        if (tuning().k2_layout == 6) return launch_tm<4, 4, 12, 4, 2>(q);
        if (tuning().k2_layout == 7) return launch_tm<4, 6, 8, 4, 2>(q);
        if (tuning().k2_layout == 8) return launch_tm<4, 4, 8, 4, 0>(q);
        if (tuning().k2_layout == 9) return launch_tm<4, 4, 8, 4, 2>(q);
        if (tuning().k2_layout == 10) return launch_tm<4, 4, 8, 4, 4>(q);
    }
#endif
    if (q.mirror) return dispatch_mirror(levels, q);
    if (q.direction != 0) {
        // T = 4 (the default depth): everything stored in place, ordered by
        // per-tile progress counters; tuning key 10 = 1 keeps the band stash
        if (!tuning().k3_stash && uses_tma(q)) {
            if (levels == 4) return launch_inplace<4, 32, 4, 4>(q);
            if (levels == 3) return launch_inplace<3, 32, 4, 5>(q);
            if (levels == 2) return launch_inplace<2, 32, 4, 6>(q);
        }
        // K3: the CY = 32 instances, the geometry compressed_workspace sizes
        switch (levels) {
        case 1: return launch_cfg<1, 32, 4, 4>(q);
        case 2: return launch_cfg<2, 32, 4, 6>(q);
        case 3: return launch_cfg<3, 32, 4, 5>(q);
        case 4: return launch_cfg<4, 32, 4, 4>(q);
        default: return set_error(SP_EUNSUP, "levels %d unsupported", levels);
        }
    }
#if SP200_AB
    // A/B tile configurations (tuning key 2), built only with -DSP200_AB=1
    const int idx = (int)tuning().cfg_index[levels];
    switch (levels) {
    case 1:
        switch (idx) {
        case 5: return launch_cfg<1, 32, 4, 6>(q);
        case 6: return launch_cfg<1, 16, 2, 4>(q);
        case 7: return launch_cfg<1, 32, 4, 3>(q);
        default: break;
        }
        break;
    case 2:
        switch (idx) {
        case 1: return launch_cfg<2, 32, 4, 4>(q);
        case 2: return launch_cfg<2, 16, 2, 4>(q);
        case 3: return launch_cfg<2, 24, 2, 4>(q);
        case 4: return launch_cfg<2, 32, 4, 6, 2>(q);
        case 5: return launch_cfg<2, 32, 4, 6>(q);
        default: break;
        }
        break;
    case 3:
        switch (idx) {
        case 1: return launch_cfg<3, 32, 4, 3>(q);
        case 2: return launch_cfg<3, 16, 2, 4>(q);
        case 3: return launch_cfg<3, 24, 2, 4>(q);
        case 4: return launch_cfg<3, 32, 4, 5, 2>(q);
        case 5: return launch_cfg<3, 32, 4, 5>(q);
        default: break;
        }
        break;
    case 4:
        switch (idx) {
        case 1: return launch_cfg<4, 32, 4, 3>(q);
        case 2: return launch_cfg<4, 16, 2, 4>(q);
        case 3: return launch_cfg<4, 24, 2, 4>(q);
        case 4: return launch_cfg<4, 32, 4, 4, 2>(q);
        case 5: return launch_cfg<4, 36, 3, 4>(q);
        case 6: return launch_cfg<4, 32, 4, 5, 1, false, true>(q);  // WP: 735 vs 770 GLUP/s
        default: break;
        }
        break;
    default: break;
    }
    // a deeper fused pass than SP_MAX_FUSED: the register state (3T doubles
    // per cell) leaves T=5 at 2 rows x 2 columns per thread (12 warps, a
    // 64 x 24 region, 1.71 executed LUP per LUP at 512^3): 535 vs 782 GLUP/s
    // for T=4 (profiles/r02_ab_depth.log).  T=8 does not fit at all: 24
    // doubles per cell of register state (R=4: 384 registers) and 14
    // double-buffered level planes (333 KB of shared memory at CY=32).
    if (levels == 5) return launch_cfg<5, 24, 2, 4>(q);
#endif
    switch (levels) {
    case 1: return launch_cfg<1, 32, 4, 4>(q);
    case 2: return launch_cfg<2, 48, 4, 4>(q);  // 12 warps: 644 vs 602 GLUP/s (CY=32)
    case 3: return launch_cfg<3, 36, 3, 4>(q);  // 12 warps: 727 vs 701 GLUP/s (CY=32)
    case 4: return launch_cfg<4, 32, 4, 4>(q);  // 8 warps x 254 registers
    default: return set_error(SP_EUNSUP, "levels %d unsupported", levels);
    }
}

int launch_temporal(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                    int64_t nx, int64_t ny, int64_t nz, int64_t off, int levels, int64_t zlo,
                    int64_t zhi, bool copy_ring, cudaStream_t stream) {
    LaunchReq q{src, dst, ex, ey, ez, nx, ny, nz, off, off, zlo, zhi, 0, nullptr, 0, stream};
    // plain sweeps: the depth-1 instance of this kernel (lane pairs, 2 CTAs
    // per SM, ~12-plane z-chunks), with reference_sweep's ring copy fused in
    // when asked; tuning key 2 (levels 1, index 1-4) selects the older
    // k_sweep1 variants for A/B
#if SP200_AB
    if (levels == 1 && tuning().cfg_index[1] >= 1 && tuning().cfg_index[1] <= 4)
        return launch_sweep1(src, dst, ex, ey, ez, nx, ny, nz, off, zlo, zhi, copy_ring, stream);
#endif
    if (copy_ring && levels != 1) return set_error(SP_EUNSUP, "ring copy is fused only into the plain sweep");
    q.ring = copy_ring;
    return dispatch(levels, q);
}

int launch_temporal_mirror(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                           int64_t nx, int64_t ny, int64_t nz, int64_t off, int levels,
                           int64_t zlo, int64_t zhi, double *mirror, int64_t mirror_zshift,
                           cudaStream_t stream) {
    LaunchReq q{src, dst, ex, ey, ez, nx, ny, nz, off, off, zlo, zhi, 0, nullptr, 0, stream};
    q.mirror = mirror;
    q.mirror_zshift = mirror_zshift;
    return dispatch(levels, q);
}

// Worst case over the layouts a launch can pick: the stored-tile parity
// (par 0 / 1, from the frame offset and the pointer alignment) changes the
// tile count, and with it pick_zchunk's chunk count and all three stashes.
template <int T>
static int64_t comp_bytes_max(int64_t nx, int64_t ny, int64_t depth) {
    int64_t best = 0;
    for (int par = 0; par < 2; ++par) {
        CompLayout L;
        comp_layout<T, 32>(nx, ny, depth, (T - 1) + par, true, &L);
        best = std::max(best, L.nx_stash + L.ny_stash + L.nz_stash);
    }
    // ... and over the in-place pass's counters and z stash
    int64_t inp = 0;
    for (int par = 0; par < 2; ++par) {
        InplaceLayout L;
        inplace_layout<T, 32>(nx, ny, depth, (T - 1) + par, &L);
        inp = std::max(inp, inplace_bytes<T, 32>(L));
    }
    return std::max(8 * best, inp) + 256;
}

// The workspace of the launch sp_compressed picks for this array: the in-place
// pass (T = 4, TMA-eligible array) needs only its progress counters.
int64_t compressed_workspace_for(const double *data, int64_t ex, int64_t ey, int64_t nx, int64_t ny,
                                 int64_t depth, int levels) {
    LaunchReq q{data, const_cast<double *>(data), ex, ey, 0, nx, ny, 0, 0, 0, 0, depth, 1, nullptr, 0, nullptr};
    if (levels >= 2 && !tuning().k3_stash && data && uses_tma(q)) {
        int64_t best = 0;
        for (int par = 0; par < 2; ++par) {
            InplaceLayout L;
            switch (levels) {
            case 2: inplace_layout<2, 32>(nx, ny, depth, 1 + par, &L); best = std::max(best, inplace_bytes<2, 32>(L)); break;
            case 3: inplace_layout<3, 32>(nx, ny, depth, 2 + par, &L); best = std::max(best, inplace_bytes<3, 32>(L)); break;
            default: inplace_layout<4, 32>(nx, ny, depth, 3 + par, &L); best = std::max(best, inplace_bytes<4, 32>(L)); break;
            }
        }
        return best + 256;
    }
    return compressed_workspace(nx, ny, depth, levels);
}

int64_t compressed_workspace(int64_t nx, int64_t ny, int64_t depth, int levels) {
    switch (levels) {
    case 1: return comp_bytes_max<1>(nx, ny, depth);
    case 2: return comp_bytes_max<2>(nx, ny, depth);
    case 3: return comp_bytes_max<3>(nx, ny, depth);
    default: return comp_bytes_max<4>(nx, ny, depth);
    }
}

int launch_compressed(double *data, int64_t ex, int64_t ey, int64_t ez, int64_t nx, int64_t ny,
                      int64_t nz, int64_t src_off, int direction, int levels, int64_t zlo,
                      int64_t zhi, void *ws, int64_t ws_bytes, cudaStream_t stream) {
    const int64_t doff = src_off - (direction > 0 ? levels : -levels);
    LaunchReq q{data, data, ex, ey, ez, nx, ny, nz, src_off, doff, zlo, zhi, direction, ws, ws_bytes, stream};
    return dispatch(levels, q);
}

}  // namespace sp200
