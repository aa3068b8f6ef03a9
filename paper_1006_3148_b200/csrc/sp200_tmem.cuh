// K2 with the per-cell pipeline state in tensor memory (k_tm).
//
// k_temporal keeps 3T doubles of state per cell in registers (the pending
// partial sum of every level and two planes of every level's values), which
// caps the T=4 CTA at 8 warps x 254 registers = one 64 x 32 region per SM.
// Blackwell's tensor memory (256 KB per SM, 128 lanes x 512 32-bit columns)
// is private per lane, so a warp's lane quadrant x a column range is a
// per-thread scratch of up to 2 KB: tcgen05.st / tcgen05.ld (32x32b) move 16
// registers per instruction between it and the register file, outside the LSU
// data pipe that the shared-memory halo rows and the shuffles load
// (tools/tmem_bench.cu: 4 KB/clk/SM read, 0.9 KB/clk/SM write, overlapping
// SHFL and DADD).  k_tm parks the level values (W0, P) and the pending sums of
// the first NSPT levels there between steps, so the same registers hold a
// larger region: 64 x 48 per CTA as 12 warps x 168 registers (R = 4) or
// 8 warps x 254 registers (R = 6).  Same lane-pair layout, summation order,
// ring handling, TMA stage ring and unit schedule as k_temporal; the level
// planes in shared memory shrink to the two published rows per warp.
#pragma once

namespace sp200 {

__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One row (two doubles = 4 columns) per tcgen05.ld / tcgen05.st: a register
// quad is what an LDS.128 / STS.128 of a double2 uses already.  The x16 forms
// need 16 consecutive registers, which ptxas assembles with one move per
// register (IMAD.MOV 20 % of all instructions).
__device__ __forceinline__ void tm_ld_row(uint32_t a, double &x, double &y) {
    asm volatile(
        "{\n\t.reg .b32 a, b, c, d;\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {a, b, c, d}, [%2];\n\t"
        "mov.b64 %0, {a, b};\n\t"
        "mov.b64 %1, {c, d};\n\t}"
        : "=d"(x), "=d"(y)
        : "r"(a));
}
// R x 2 doubles of one thread <-> 4R consecutive TMEM columns of its lane
template <int R>
__device__ __forceinline__ void tm_load(uint32_t a, double (&d)[R][2]) {
#pragma unroll
    for (int r = 0; r < R; ++r) tm_ld_row(a + 4 * r, d[r][0], d[r][1]);
}
__device__ __forceinline__ void tm_st_row(uint32_t a, double x, double y) {
    asm volatile(
        "{\n\t.reg .b32 a, b, c, d;\n\t"
        "mov.b64 {a, b}, %1;\n\t"
        "mov.b64 {c, d}, %2;\n\t"
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {a, b, c, d};\n\t}" ::"r"(a),
        "d"(x), "d"(y)
        : "memory");
}
template <int R>
__device__ __forceinline__ void tm_store(uint32_t a, const double (&d)[R][2]) {
#pragma unroll
    for (int r = 0; r < R; ++r) tm_st_row(a + 4 * r, d[r][0], d[r][1]);
}
template <int T, int R, int NW, int S, int NSPT>
struct TMCfg {
    static constexpr int CX = 64;
    static constexpr int CY = NW * R;
    static constexpr int PY = CY + 2;
    static constexpr int SPX = CX + 4;
    static constexpr int C0 = 2;
    static constexpr int PLANE = SPX * PY;
    static constexpr int PLANE_AL = (PLANE + 15) & ~15;
    static constexpr int NT = 32 * NW;
    static constexpr int OY = CY - 2 * (T - 1);
    // published rows per level plane: first and last row of every warp, one
    // sentinel row at each end (the halo of the region's outer rows)
    static constexpr int PUBR = 2 * NW + 2;
    static constexpr int PUB = PUBR * CX;
    static constexpr int NLEV = 2 * (T - 1);
    static constexpr int ACOLS = 4 * R;            // TMEM columns per array of R x 2 doubles
    static constexpr int NARR = 2 * T + NSPT;      // W0[2], P[T-1][2], Sp[0 .. NSPT)
    static constexpr int NSLOT = (NW + 3) / 4;     // warps sharing a lane quadrant
    static constexpr int SLOTCOLS = (512 / NSLOT) & ~7;
    static constexpr size_t SMEM = (size_t)(S * PLANE_AL + NLEV * PUB) * sizeof(double) + 8 * S + 16;
    static_assert(NARR * ACOLS <= SLOTCOLS, "state does not fit the warp's TMEM columns");
    static_assert(NSPT >= 0 && NSPT <= T, "pending sums in TMEM");
    static_assert(OY > 0, "tile too small for the fused depth");
    static_assert(T >= 2, "fused passes only");
};

template <int T, int R, int NW, int S, int NSPT, bool MIR>
__global__ void __launch_bounds__(32 * NW, 1)
    k_tm(const TParams p, const __grid_constant__ CUtensorMap tmap) {
    using C = TMCfg<T, R, NW, S, NSPT>;
    constexpr int SPX = C::SPX, C0 = C::C0, PLANE = C::PLANE, PLANE_AL = C::PLANE_AL, NT = C::NT, PUB = C::PUB,
                  CX = C::CX, OY = C::OY, ACOLS = C::ACOLS;
    constexpr int PD = S - 1;  // stage prefetch distance
    constexpr int NSPR = T - NSPT;

    extern __shared__ __align__(128) double sm[];
    double *stage = sm;
    double *lev = sm + S * PLANE_AL;
    uint64_t *bar = reinterpret_cast<uint64_t *>(lev + C::NLEV * PUB);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + S);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int i0 = 2 * lane, j0 = warp * R;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        tma_prefetch_desc(&tmap);
#pragma unroll
        for (int si = 0; si < S; ++si) mbar_init(&bar[si], 1);
        fence_mbar_init();
    }
    // sentinel rows: ghost cells, read but never feeding a kept cell
    for (int q = tid; q < C::NLEV * 2 * CX; q += NT) {
        const int pl = q / (2 * CX), w = q % (2 * CX);
        lev[pl * PUB + (w >= CX ? (C::PUBR - 1) * CX + (w - CX) : w)] = 0.0;
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    // this thread's TMEM scratch: lane quadrant warp % 4 (the hardware's
    // rule), column slot warp / 4
    // (through a shuffle: provably warp-uniform, so the tcgen05 addresses are
    // formed on the uniform datapath)
    const uint32_t ta = __shfl_sync(
        0xffffffffu, *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * C::SLOTCOLS), 0);
    auto a_w0 = [&](int q) { return ta + (uint32_t)(q * ACOLS); };
    auto a_p = [&](int ui, int q) { return ta + (uint32_t)((2 + 2 * ui + q) * ACOLS); };
    auto a_sp = [&](int k) { return ta + (uint32_t)((2 * T + k) * ACOLS); };

    // pending sums of the levels above NSPT stay in registers
    double SpR[NSPR > 0 ? NSPR : 1][R][2];
#pragma unroll
    for (int k = 0; k < (NSPR > 0 ? NSPR : 1); ++k)
#pragma unroll
        for (int r = 0; r < R; ++r) SpR[k][r][0] = SpR[k][r][1] = 0.0;

    uint32_t gbase = 0;  // stage loads issued by this CTA so far (one unit per CTA here)
    {
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
            y_out[r] = (jr >= T - 1) && (jr < T - 1 + OY) && (y < p.ny);
        }
        const bool wint = !__any_sync(0xffffffffu, ringb != 0u);

        const int nload = (z1 - z0) + 2 * T;
        const int nsteps = (z1 - z0) + 3 * T - 1;
        const int bxs = rx0 + p.off - C0, bys = ry0 - 1 + p.off;
        const int64_t pz = p.ex * p.ey;
        double *dcol = p.dst + (int64_t)(ry0 + j0 + p.doff) * p.ex + (rx0 + i0 + p.doff);
        const bool pair = x_out[0] && x_out[1] && p.pair_store;

        auto issue = [&](int s) {
            const int si = (int)((gbase + s) % S);
            const int zs = z0 - T + s + p.off;
            mbar_arrive_expect_tx(&bar[si], PLANE * 8);
            tma_load_3d(stage + si * PLANE_AL, &tmap, &bar[si], bxs, bys, zs);
        };
        if (tid == 0)
            for (int s = 0; s < PD; ++s)
                if (s < nload) issue(s);

        // this warp's rows in the compact level planes
        const int prow = (1 + 2 * warp) * CX + i0;

        auto levels = [&](int s, const double *cur, auto Qc, auto Mc) {
            constexpr int Q = decltype(Qc)::value;
            constexpr int MODE = decltype(Mc)::value;
#pragma unroll
            for (int u = T; u >= 1; --u) {
                const int ui = (u > 1) ? u - 2 : 0;
                const int pout = z0 - T + s - 2 * u + 1;
                const bool z_ring = (pout == -1) || (pout == p.nz);
                double A[R][2], wl[R][2], sp[R][2];
                double2 cm, cp;
                if (u == 1) {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double2 a = lds2(cur + (j0 + r + 1) * SPX + C0 + i0);
                        A[r][0] = a.x;
                        A[r][1] = a.y;
                    }
                    tm_load<R>(a_w0(Q ^ 1), wl);
                    if constexpr (NSPT >= 1) tm_load<R>(a_sp(0), sp);
                    tm_store<R>(a_w0(Q), A);
                    cm = lds2(cur + j0 * SPX + C0 + i0);
                    cp = lds2(cur + (j0 + R + 1) * SPX + C0 + i0);
                } else {
                    tm_load<R>(a_p(ui, Q ^ 1), A);
                    tm_load<R>(a_p(ui, Q), wl);
                    if (u <= NSPT) tm_load<R>(a_sp(u - 1), sp);
                    const double *B = lev + (ui * 2 + (Q ^ 1)) * PUB + prow;
                    cm = lds2(B - CX);
                    cp = lds2(B + 2 * CX);
                }
                if (u > NSPT) {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        sp[r][0] = SpR[u > NSPT ? u - 1 - NSPT : 0][r][0];
                        sp[r][1] = SpR[u > NSPT ? u - 1 - NSPT : 0][r][1];
                    }
                }
                tm_wait_ld();

                double xl[R], xr[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (u == 1) {
                        xl[r] = cur[(j0 + r + 1) * SPX + C0 + i0 - 1];
                        xr[r] = cur[(j0 + r + 1) * SPX + C0 + i0 + 2];
                    } else {
                        xl[r] = __shfl_up_sync(0xffffffffu, A[r][1], 1);
                        xr[r] = __shfl_down_sync(0xffffffffu, A[r][0], 1);
                    }
                }
                double n[R][2], v[R][2];
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int c = 0; c < 2; ++c) v[r][c] = dadd(sp[r][c], A[r][c]);
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
                        n[r][c] = dadd(n[r][c], wl[r][c]);
                    }
                // the new pending sum and (levels below T) the new plane
                if (u <= NSPT) {
                    tm_store<R>(a_sp(u - 1), n);
                } else {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        SpR[u > NSPT ? u - 1 - NSPT : 0][r][0] = n[r][0];
                        SpR[u > NSPT ? u - 1 - NSPT : 0][r][1] = n[r][1];
                    }
                }
                if (u < T) {
                    tm_store<R>(a_p(u - 1, Q), v);
                    double *pub = lev + ((u - 1) * 2 + Q) * PUB + prow;
                    sts2(pub, v[0][0], v[0][1]);
                    sts2(pub + CX, v[R - 1][0], v[R - 1][1]);
                } else if (pout >= z0 && pout < z1) {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        if (!y_out[r]) continue;
                        double *g = dcol + (int64_t)(pout + p.doff) * pz + (int64_t)r * p.ex;
                        if (pair) {
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
        };

        auto one_step = [&](int s, auto Qc) {
            const int si = (int)((gbase + s) % S);
            if (s < nload) mbar_wait(&bar[si], (uint32_t)(((gbase + s) / S) & 1));
            // the previous step's TMEM stores are loaded in this step
            tm_wait_st();
            __syncthreads();
            if (tid == 0 && s + PD < nload) issue(s + PD);
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
        gbase += (uint32_t)nload;
    }
    tm_wait_st();
    tm_fence_before();
    __syncthreads();
    if (warp == 0) {
        tm_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tslot) : "memory");
    }
}

}  // namespace sp200
