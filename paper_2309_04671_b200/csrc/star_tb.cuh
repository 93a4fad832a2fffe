// Two time steps per d0 sweep (temporal blocking) for the Jacobi ping-pong
// `v = S(u); swap(u, v)` with a star S of radius R (written for R <= VEC; built and
// routed for R = 1, where it wins: DESIGN.md §3.1b).
//
// The single-step kernel (star_kernels.cuh) moves 8 B (fp32) per point and step
// through HBM; at radius 1 the arithmetic and shared-memory work per point are
// small, so the step is HBM-bound.  This kernel streams u once and produces
// u(t+2) = S(S(u(t))): every plane of v(t+1) is computed in registers and
// consumed in registers, halving the HBM bytes per step.  Same semantics and the
// same per-step arithmetic (identical FMA order) as two launches of the
// single-step kernel (the fast path's numbers; tests compare the two bit for bit).
//
//  * one producer warp: TMA box per u plane, (32 VEC + 2 RA) x (BY + 4R) with the
//    2R-deep halo both stages need, STAGES-deep mbarrier ring (as star_kernels.cuh);
//  * consumer warp w owns output rows [w TY2, (w+1) TY2) of a 30 VEC x NW TY2 tile
//    and computes v on its rows +- R over 32 lanes x VEC columns (the tile +- one
//    vector): stage 1 is the single-step kernel's STAR plane update on TY1 = TY2 + 2R
//    rows; stage 2 takes v's x-neighbours from the adjacent lanes (shuffles), its
//    y-neighbours from the warp's own rows and its d0 taps through a second register
//    ring, so v never touches shared or global memory;
//  * v outside the map's region box is the v buffer's own (frozen) content, read
//    from global memory on the edge tiles only; u(t+2) goes to a scratch buffer
//    (the host rotates u / scratch; the v buffer is not written by this kernel).
// Reference semantics followed: executor.py:267-286 (maps run in order, swaps
// exchange the name binding), executor.py:108-124 (only the region is written).
#pragma once

#include "star_kernels.cuh"

// 1 (measured slower, not the default): each warp computes v on its own output rows only (plus the tile's halo rows on the first /
// last warp) and takes the neighbouring rows its stage 2 needs from the adjacent warps through
// shared memory (one consumer barrier per plane); 0: every warp recomputes its R halo rows
#ifndef STKB_TB_XCH
#define STKB_TB_XCH 0
#endif

namespace stkb {

__device__ __forceinline__ void sts16(float* p, const float* v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]) : "memory");
}
__device__ __forceinline__ void sts16(double* p, const double* v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_u32(p)), "d"(v[0]), "d"(v[1]) : "memory");
}

template <typename T, int R, int TY2, int NW>
struct TbCfg {
    static constexpr int VEC = 16 / sizeof(T);
    static_assert(R <= VEC, "the x-halo of both stages is one vector");
    static constexpr int RA = VEC;              // u x-halo of the stage-1 columns (one vector each side)
    static constexpr int TY1 = TY2 + 2 * R;     // v rows per warp
    static constexpr int BX = 30 * VEC;         // output columns: lanes 1..30
    static constexpr int BY = NW * TY2;         // output rows
    static constexpr int SW = 32 * VEC + 2 * RA;  // u columns [x0 - VEC - RA, x0 + 31 VEC + RA)
    static constexpr int SH = BY + 4 * R;         // u rows [y0 - 2R, y0 + BY + 2R)
    static constexpr int VW = 32 * VEC;         // v tile (edge items only): [x0 - VEC, x0 + 31 VEC)
    static constexpr int VH = BY + 2 * R;       //   x [y0 - R, y0 + BY + R), the frozen v values
    static constexpr int U_ELEMS = ((SW * SH * int(sizeof(T)) + 127) / 128) * 128 / int(sizeof(T));
    static constexpr int STAGE_ELEMS = U_ELEMS + VW * VH;
    static constexpr uint32_t HALO_BYTES = SW * SH * sizeof(T);
    static constexpr uint32_t V_BYTES = VW * VH * sizeof(T);
    static constexpr uint32_t STAGE_BYTES = STAGE_ELEMS * sizeof(T);
    // v-row exchange (STKB_TB_XCH): each warp publishes its first and last R v rows per
    // plane, double-buffered by plane parity
    static constexpr int XROW = 32 * VEC;  // one v row of the tile
    static constexpr uint32_t XBUF_BYTES = STKB_TB_XCH ? 2u * NW * 2 * R * XROW * sizeof(T) : 0u;
    static constexpr int STAGES_RAW = (200 * 1024 - int(XBUF_BYTES)) / STAGE_BYTES;
    // a power of two: the stage index and phase of plane `it` are a mask and a shift
    static constexpr int STAGES = STAGES_RAW >= 8 ? 8 : (STAGES_RAW >= 4 ? 4 : 2);
    static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t) +
                                   STAGES * sizeof(int32_t) + 16 + XBUF_BYTES;
    static constexpr int THREADS = (NW + 1) * 32;
    static_assert(SW <= 256 && SH <= 256, "TMA box dims are limited to 256");
    static_assert(!STKB_TB_XCH || TY2 >= R, "the exchange needs R own rows per warp");
};

template <typename T, int R, int TY2, int NW, bool DIV>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
star_tb2_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ CUtensorMap tm_v,
                const __grid_constant__ CUtensorMap tm_int, const __grid_constant__ StarArgs<T> a,
                const int32_t* __restrict__ frozen_nz) {
    using C = TbCfg<T, R, TY2, NW>;
    constexpr int VEC = C::VEC, RA = C::RA, BX = C::BX, BY = C::BY, SW = C::SW, TY1 = C::TY1;
    constexpr int STAGES = C::STAGES;
    constexpr int NS = 2 * R + 1;

    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    T* tiles = reinterpret_cast<T*>(base);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(STAGES) * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    volatile int32_t* stage_item = reinterpret_cast<int32_t*>(empty + STAGES);
    T* xbuf = reinterpret_cast<T*>((reinterpret_cast<uintptr_t>(stage_item + STAGES) + 15) & ~uintptr_t(15));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NW) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            // u's halo all zero: read through the interior-only map (TMA zero-fills the halo)
            const bool interior = a.halo_nz && *reinterpret_cast<const volatile int32_t*>(a.halo_nz) == 0;
            const CUtensorMap* um = interior ? &tm_int : &tm_src;
            const int ix = interior ? int(a.g.lead) : 0, iy = interior ? int(a.g.order) : 0,
                      iz = interior ? int(a.g.order0) : 0;
            prefetch_tmap(um);
            prefetch_tmap(&tm_v);
            // v's frozen values around the box are all zero (the usual zero halo): no v tiles
            const bool need_v = *reinterpret_cast<const volatile int32_t*>(frozen_nz) != 0;
            uint32_t it = 0;
            // at most one item per CTA: static assignment, no scheduler atomic (star_kernels.cuh)
            const bool fixed = a.n_items <= int(gridDim.x);
            for (int k = 0;; ++k) {
                const int item = fixed ? int(blockIdx.x) + k * int(gridDim.x) : atomicAdd(a.work_counter, 1);
                if (item >= a.n_items) {
                    const uint32_t s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1u) ^ 1u);
                    stage_item[s] = -1;
                    mbar_arrive(&full[s]);
                    break;
                }
                int tx, ty, tz;
                decode_item(a, item, tx, ty, tz);
                const int x0 = a.x0base + tx * BX;
                const int y0 = a.box.lo1 + ty * BY;
                const int z0 = a.zs[2 * tz];
                const int z1 = a.zs[2 * tz + 1];
                const int c0 = int(a.g.lead) + x0 - VEC - RA;
                const int c1 = y0 + int(a.g.order) - 2 * R;
                // v tiles leaving the region box in (d1, d2) take frozen values from the v buffer
                const bool edge_xy = x0 - VEC < a.box.lo2 || x0 + 31 * VEC > a.box.hi2 || y0 - R < a.box.lo1 ||
                                     y0 + BY + R > a.box.hi1;
                for (int q = z0 - 2 * R; q < z1 + 2 * R; ++q, ++it) {
                    const uint32_t s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1u) ^ 1u);
                    stage_item[s] = item;
                    const int qv = q - R;  // v plane completed with this stage
                    const bool vload = need_v && qv >= z0 - R && qv < z1 + R &&
                                       (edge_xy || qv < a.box.lo0 || qv >= a.box.hi0);
                    T* st = tiles + size_t(s) * C::STAGE_ELEMS;
                    mbar_arrive_expect_tx(&full[s], C::HALO_BYTES + (vload ? C::V_BYTES : 0u));
                    // planes beyond the allocation (q < -order0 or q >= n0 + order0) are
                    // zero-filled by the TMA unit; stage 1 never uses them inside the region
                    tma_load_3d(st, um, &full[s], c0 - ix, c1 - iy, q + int(a.g.order0) - iz);
                    if (vload)
                        tma_load_3d(st + C::U_ELEMS, &tm_v, &full[s], int(a.g.lead) + x0 - VEC,
                                    y0 + int(a.g.order) - R, qv + int(a.g.order0));
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    using K = Pk<T>;
    using P = typename K::P;
    constexpr int W = K::W;
    constexpr int NPK = VEC / W;
    const int xl = lane * VEC;  // stage-1 columns of this lane inside the tile (tile column 0 = x0 - VEC)
    const int jr0 = warp * TY2; // first output row of this warp; its v rows are jr0 - R + i, i < TY1
    P acc1[NS][TY1][NPK];        // v(t+1) ring
    P acc2[NS][TY2][NPK];        // u(t+2) ring
#pragma unroll
    for (int k = 0; k < NS; ++k) {
#pragma unroll
        for (int j = 0; j < TY1; ++j)
#pragma unroll
            for (int i = 0; i < NPK; ++i) acc1[k][j][i] = K::mul(T(0), P{});
#pragma unroll
        for (int j = 0; j < TY2; ++j)
#pragma unroll
            for (int i = 0; i < NPK; ++i) acc2[k][j][i] = K::mul(T(0), P{});
    }
    P chk = K::mul(T(0), P{});
    T chk1 = T(0);
    uint32_t it = 0;
    const int64_t pitch = a.g.pitch, plane = a.g.plane;
    const bool need_v = *reinterpret_cast<const volatile int32_t*>(frozen_nz) != 0;
    // v row i (= tile row jr0 - R + i) is computed by this warp: its own rows, and the R halo
    // rows above / below only on the first / last warp (with the exchange; warp-uniform)
    const bool top = warp == 0, bot = warp == NW - 1;
    auto row_on = [&](int i) -> bool {
        return !STKB_TB_XCH || (i >= R && i < R + TY2) || (i < R && top) || (i >= R + TY2 && bot);
    };
    // u tile rows (relative to jr0) the active v rows read: [first, last]
    const int rr_first = STKB_TB_XCH && !top ? R : 0;
    const int rr_last = STKB_TB_XCH && !bot ? TY2 + 3 * R - 1 : TY1 + 2 * R - 1;

    while (true) {
        mbar_wait(&full[it % STAGES], (it / STAGES) & 1u);
        const int item = __shfl_sync(0xffffffffu, stage_item[it % STAGES], 0);  // warp-uniform
        if (item < 0) break;
        int tx, ty, tz;
        decode_item(a, item, tx, ty, tz);
        const int x0 = a.x0base + tx * BX;
        const int y0 = a.box.lo1 + ty * BY;
        const int z0 = a.zs[2 * tz];
        const int z1 = a.zs[2 * tz + 1];
        const int xv = x0 - VEC + xl;  // first v column of this lane
        const int yv = y0 + jr0 - R;   // first v row of this warp
        // v of this warp's rows x lanes lies inside the region box in (d1, d2)?
        const bool xy_in = __all_sync(0xffffffffu, xv >= a.box.lo2 && xv + VEC <= a.box.hi2) &&
                           yv >= a.box.lo1 && yv + TY1 <= a.box.hi1;
        const int x = x0 + xl - VEC;  // output columns of this lane (lanes 1..30)
        const bool out_lane = lane >= 1 && lane <= 30;
        const bool full_tile = x0 >= a.box.lo2 && x0 + BX <= a.box.hi2 && y0 >= a.box.lo1 && y0 + BY <= a.box.hi1;
        const bool x_any = out_lane && (x + VEC > a.box.lo2) && (x < a.box.hi2);
        T* const dst0 = a.dst + (int64_t(y0 + jr0) + a.g.order) * pitch + a.g.lead + x;
        const int nq = (z1 - z0) + 4 * R;

        for (int qb = 0; qb < nq; qb += NS) {
#pragma unroll
            for (int p = 0; p < NS; ++p) {
                const int qi = qb + p;
                if (qi < nq) {
                    const int q = z0 - 2 * R + qi;  // u plane in the stage
                    const uint32_t s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1u);
                    const T* t = tiles + size_t(s) * C::STAGE_ELEMS;

                    // -------- stage 1: u plane q -> v (the single-step STAR update on TY1 rows)
                    T cvs[TY1][VEC];
#pragma unroll
                    for (int j = 0; j < TY1; ++j) lds16(t + (jr0 + j + R) * SW + xl + RA, cvs[j]);
                    P cv[TY1][NPK];
#pragma unroll
                    for (int j = 0; j < TY1; ++j)
#pragma unroll
                        for (int k = 0; k < NPK; ++k) cv[j][k] = K::make(&cvs[j][k * W]);
                    if (q >= z0 - R && q < z1 + R) {
#pragma unroll
                        for (int j = 0; j < TY1; ++j) {
                            if (!row_on(j)) continue;
                            T xr[VEC + 2 * RA];
                            const T* row = t + (jr0 + j + R) * SW + xl;
                            lds16(row, &xr[0]);
                            lds16(row + RA + VEC, &xr[RA + VEC]);
#pragma unroll
                            for (int i = 0; i < VEC; ++i) xr[RA + i] = cvs[j][i];
#pragma unroll
                            for (int k = 0; k < NPK; ++k) {
                                P s_ = K::fma(a.c0, cv[j][k], acc1[p][j][k]);
#pragma unroll
                                for (int m = 1; m <= R; ++m) {
                                    if (W == 1 || (m % 2) == 0) {
                                        s_ = K::fma(a.cm[2][m - 1], K::make(&xr[RA + k * W - m]), s_);
                                        s_ = K::fma(a.cp[2][m - 1], K::make(&xr[RA + k * W + m]), s_);
                                    } else {
                                        T l[W];
                                        K::put(l, s_);
#pragma unroll
                                        for (int w = 0; w < W; ++w) {
                                            l[w] = fma_t(a.cm[2][m - 1], xr[RA + k * W + w - m], l[w]);
                                            l[w] = fma_t(a.cp[2][m - 1], xr[RA + k * W + w + m], l[w]);
                                        }
                                        s_ = K::make(l);
                                    }
                                }
                                acc1[p][j][k] = s_;
                            }
                        }
#pragma unroll
                        for (int rr = 0; rr < TY1 + 2 * R; ++rr) {
                            if (rr >= R && rr < R + TY1) {
#pragma unroll
                                for (int j = 0; j < TY1; ++j) {
                                    const int m = rr - (j + R);
                                    if (m != 0 && m >= -R && m <= R && row_on(j)) {
                                        const T c = m < 0 ? a.cm[1][-m - 1] : a.cp[1][m - 1];
#pragma unroll
                                        for (int k = 0; k < NPK; ++k)
                                            acc1[p][j][k] = K::fma(c, cv[rr - R][k], acc1[p][j][k]);
                                    }
                                }
                            } else if (rr >= rr_first && rr <= rr_last) {
                                T yv_[VEC];
                                lds16(t + (jr0 + rr) * SW + xl + RA, yv_);
#pragma unroll
                                for (int j = 0; j < TY1; ++j) {
                                    const int m = rr - (j + R);
                                    if (m >= -R && m <= R && row_on(j)) {
                                        const T c = m < 0 ? a.cm[1][-m - 1] : a.cp[1][m - 1];
#pragma unroll
                                        for (int k = 0; k < NPK; ++k)
                                            acc1[p][j][k] = K::fma(c, K::make(&yv_[k * W]), acc1[p][j][k]);
                                    }
                                }
                            }
                        }
                    }
                    if (q < z1 + R) {
#pragma unroll
                        for (int j = 0; j < TY1; ++j)
                            if (row_on(j))
#pragma unroll
                            for (int k = 0; k < NPK; ++k) {
                                acc1[(p + R) % NS][j][k] = K::mul(a.cm[0][R - 1], cv[j][k]);
#pragma unroll
                                for (int m = 1; m < R; ++m)
                                    acc1[(p + m) % NS][j][k] = K::fma(a.cm[0][m - 1], cv[j][k], acc1[(p + m) % NS][j][k]);
                            }
                    }
#pragma unroll
                    for (int j = 0; j < TY1; ++j)
                        if (row_on(j))
#pragma unroll
                        for (int k = 0; k < NPK; ++k)
#pragma unroll
                            for (int m = 1; m <= R; ++m)
                                acc1[(p - m + NS) % NS][j][k] =
                                    K::fma(a.cp[0][m - 1], cv[j][k], acc1[(p - m + NS) % NS][j][k]);

                    // -------- v plane qv = q - R is complete
                    constexpr int ks = (NS - R) % NS;
                    const int qv = q - R;
                    if (qv >= z0 - R && qv < z1 + R) {
                        T vv[TY1][VEC];
#pragma unroll
                        for (int j = 0; j < TY1; ++j)
#pragma unroll
                            for (int k = 0; k < NPK; ++k) {
                                P v = acc1[(p + ks) % NS][j][k];
                                if constexpr (DIV) v = K::mul(a.divisor, v);
                                K::put(&vv[j][k * W], v);
                            }
                        const bool z_in = qv >= a.box.lo0 && qv < a.box.hi0;
                        if (z_in && xy_in) {
#pragma unroll
                            for (int j = 0; j < TY1; ++j)
#pragma unroll
                                for (int k = 0; k < NPK; ++k) chk = K::check(K::make(&vv[j][k * W]), chk);
                        } else {
                            // outside the region box v keeps the v buffer's content (its halo,
                            // or the interior a smaller region leaves alone): the stage's v tile
                            const T* vt = t + C::U_ELEMS + jr0 * C::VW + xl;
#pragma unroll
                            for (int j = 0; j < TY1; ++j) {
                                if (!row_on(j)) continue;
                                const int y = yv + j;
                                const bool row_in = z_in && y >= a.box.lo1 && y < a.box.hi1;
                                T fz[VEC] = {};
                                if (need_v) lds16(vt + j * C::VW, fz);
#pragma unroll
                                for (int e = 0; e < VEC; ++e) {
                                    const int xx = xv + e;
                                    if (row_in && xx >= a.box.lo2 && xx < a.box.hi2) chk1 = fma_t(T(0), vv[j][e], chk1);
                                    else vv[j][e] = fz[e];
                                }
                            }
                        }

                        if constexpr (STKB_TB_XCH) {
                            // publish this warp's first / last R v rows, take the neighbours'
                            T* xb = xbuf + (qv & 1) * (NW * 2 * R * C::XROW);
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                sts16(xb + ((warp * 2 + 0) * R + r) * C::XROW + xl, vv[R + r]);
                                sts16(xb + ((warp * 2 + 1) * R + r) * C::XROW + xl, vv[TY2 + r]);
                            }
                            asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
                            if (!top)
#pragma unroll
                                for (int r = 0; r < R; ++r)
                                    lds16(xb + (((warp - 1) * 2 + 1) * R + r) * C::XROW + xl, vv[r]);
                            if (!bot)
#pragma unroll
                                for (int r = 0; r < R; ++r)
                                    lds16(xb + (((warp + 1) * 2 + 0) * R + r) * C::XROW + xl, vv[R + TY2 + r]);
                        }
                        // -------- stage 2: v plane qv -> u(t+2)
                        P cw[TY2][NPK];
#pragma unroll
                        for (int j = 0; j < TY2; ++j)
#pragma unroll
                            for (int k = 0; k < NPK; ++k) cw[j][k] = K::make(&vv[j + R][k * W]);
                        if (qv >= z0 && qv < z1) {
#pragma unroll
                            for (int j = 0; j < TY2; ++j) {
                                // x-neighbours from the adjacent lanes; the centre sits at an even
                                // offset so the pairs of even shifts stay register pairs
                                constexpr int XO = 2;
                                T xr[VEC + 2 * XO];
#pragma unroll
                                for (int i = 0; i < VEC; ++i) xr[XO + i] = vv[j + R][i];
#pragma unroll
                                for (int e = 0; e < R; ++e) {
                                    xr[XO - 1 - e] = __shfl_up_sync(0xffffffffu, vv[j + R][VEC - 1 - e], 1);
                                    xr[XO + VEC + e] = __shfl_down_sync(0xffffffffu, vv[j + R][e], 1);
                                }
#pragma unroll
                                for (int k = 0; k < NPK; ++k) {
                                    P s_ = K::fma(a.c0, cw[j][k], acc2[p][j][k]);
#pragma unroll
                                    for (int m = 1; m <= R; ++m) {
                                        if (W == 1 || (m % 2) == 0) {
                                            s_ = K::fma(a.cm[2][m - 1], K::make(&xr[XO + k * W - m]), s_);
                                            s_ = K::fma(a.cp[2][m - 1], K::make(&xr[XO + k * W + m]), s_);
                                        } else {
                                            T l[W];
                                            K::put(l, s_);
#pragma unroll
                                            for (int w = 0; w < W; ++w) {
                                                l[w] = fma_t(a.cm[2][m - 1], xr[XO + k * W + w - m], l[w]);
                                                l[w] = fma_t(a.cp[2][m - 1], xr[XO + k * W + w + m], l[w]);
                                            }
                                            s_ = K::make(l);
                                        }
                                    }
                                    acc2[p][j][k] = s_;
                                }
                            }
                            // y-neighbours: the warp's own v rows, in the single-step order
#pragma unroll
                            for (int rr = 0; rr < TY2 + 2 * R; ++rr) {
#pragma unroll
                                for (int j = 0; j < TY2; ++j) {
                                    const int m = rr - (j + R);
                                    if (m != 0 && m >= -R && m <= R) {
                                        const T c = m < 0 ? a.cm[1][-m - 1] : a.cp[1][m - 1];
#pragma unroll
                                        for (int k = 0; k < NPK; ++k)
                                            acc2[p][j][k] = K::fma(c, K::make(&vv[rr][k * W]), acc2[p][j][k]);
                                    }
                                }
                            }
                        }
                        if (qv < z1) {
#pragma unroll
                            for (int j = 0; j < TY2; ++j)
#pragma unroll
                                for (int k = 0; k < NPK; ++k) {
                                    acc2[(p + R) % NS][j][k] = K::mul(a.cm[0][R - 1], cw[j][k]);
#pragma unroll
                                    for (int m = 1; m < R; ++m)
                                        acc2[(p + m) % NS][j][k] =
                                            K::fma(a.cm[0][m - 1], cw[j][k], acc2[(p + m) % NS][j][k]);
                                }
                        }
#pragma unroll
                        for (int j = 0; j < TY2; ++j)
#pragma unroll
                            for (int k = 0; k < NPK; ++k)
#pragma unroll
                                for (int m = 1; m <= R; ++m)
                                    acc2[(p - m + NS) % NS][j][k] =
                                        K::fma(a.cp[0][m - 1], cw[j][k], acc2[(p - m + NS) % NS][j][k]);

                        // -------- u(t+2) plane z = qv - R is complete
                        const int z = qv - R;
                        __syncwarp();
                        mbar_arrive_lane0(&empty[s], lane);
                        if (z >= z0 && z < z1) {
                            T outv[TY2][VEC];
#pragma unroll
                            for (int j = 0; j < TY2; ++j)
#pragma unroll
                                for (int k = 0; k < NPK; ++k) {
                                    P v = acc2[(p + ks) % NS][j][k];
                                    if constexpr (DIV) v = K::mul(a.divisor, v);
                                    K::put(&outv[j][k * W], v);
                                    if (out_lane) chk = K::check(v, chk);
                                }
                            T* const dz = dst0 + (int64_t(z) + a.g.order0) * plane;
                            if (full_tile) {
                                if (out_lane) {
#pragma unroll
                                    for (int j = 0; j < TY2; ++j) stg16(dz + j * pitch, outv[j]);
                                }
                            } else if (x_any) {
#pragma unroll
                                for (int j = 0; j < TY2; ++j) {
                                    const int y = y0 + jr0 + j;
                                    if (y >= a.box.lo1 && y < a.box.hi1)
                                        store_row_masked<T>(dz + j * pitch, outv[j][0], outv[j][1 % VEC],
                                                            outv[j][2 % VEC], outv[j][3 % VEC], x, a.box.lo2,
                                                            a.box.hi2);
                                }
                            }
                        }
                    } else {
                        __syncwarp();
                        mbar_arrive_lane0(&empty[s], lane);
                    }
                    ++it;
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, !K::clean(chk) || chk1 != T(0)) && lane == 0) atomicOr(a.nonfinite, 1);
}

// tile of the fused kernel per dtype (radius 1), coded 100 * (output rows per warp) +
// consumer warps: measured best of 2..5 rows x 7..12 warps, spill-free (ptxas -v)
#ifndef STKB_TB_F32R1
#define STKB_TB_F32R1 311
#endif
#ifndef STKB_TB_F64R1
#define STKB_TB_F64R1 311
#endif
template <typename T, int R>
struct TbTile {
    static_assert(R == 1, "fused sweeps are tuned and routed for radius 1 (stkb200.cu tb_map)");
    static constexpr int CODE = sizeof(T) == 4 ? STKB_TB_F32R1 : STKB_TB_F64R1;
    static constexpr int TY2 = CODE / 100;
    static constexpr int NW = CODE % 100;
};

// *flag |= 1 when a cell of `buf` within R of the box (along any axis, outside it) is not
// bit-for-bit +0: the fused sweep then stages v's frozen values through TMA.  zmask bit 0 / 1:
// check the d0 face below / above the box (a z-slab side whose planes come from a neighbour
// is left out)
template <typename T>
__global__ void frozen_ring_kernel(const T* __restrict__ buf, Geometry g, Box b, int R, int32_t* flag, int zmask) {
    const int64_t X = int64_t(b.hi2 - b.lo2) + 2 * R, Y = int64_t(b.hi1 - b.lo1) + 2 * R;
    const int64_t nz = int64_t(b.hi0 - b.lo0), ny = int64_t(b.hi1 - b.lo1), nx = int64_t(b.hi2 - b.lo2);
    const int64_t nA = 2 * R * Y * X, nB = nz * 2 * R * X, nC = nz * ny * 2 * R;
    bool nonzero = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nA + nB + nC;
         i += int64_t(gridDim.x) * blockDim.x) {
        int64_t z, y, x;
        if (i < nA) {  // planes below / above the box
            const int64_t k = i / (Y * X), r = i - k * Y * X;
            if (!(zmask & (k < R ? 1 : 2))) continue;
            z = k < R ? b.lo0 - R + k : b.hi0 + (k - R);
            y = b.lo1 - R + r / X;
            x = b.lo2 - R + r % X;
        } else if (i < nA + nB) {  // rows before / after, inside the box's planes
            const int64_t j = i - nA, zz = j / (2 * R * X), r = j - zz * 2 * R * X, k = r / X;
            z = b.lo0 + zz;
            y = k < R ? b.lo1 - R + k : b.hi1 + (k - R);
            x = b.lo2 - R + r % X;
        } else {  // columns left / right, inside the box's rows
            const int64_t j = i - nA - nB, row = j / (2 * R), k = j - row * 2 * R;
            z = b.lo0 + row / ny;
            y = b.lo1 + row % ny;
            x = k < R ? b.lo2 - R + k : b.hi2 + (k - R);
        }
        const T v = buf[g.at(z, y, x)];
        if constexpr (sizeof(T) == 4) nonzero |= __float_as_uint(v) != 0u;
        else nonzero |= __double_as_longlong(v) != 0ll;
    }
    (void)nx;
    if (__any_sync(0xffffffffu, nonzero) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T, int R, bool DIV>
cudaError_t launch_tb2_cfg(const StarLaunch& L, StarArgs<T> a, const CUtensorMap* map, cudaStream_t stream) {
    constexpr int TY2 = TbTile<T, R>::TY2, NW = TbTile<T, R>::NW;
    using C = TbCfg<T, R, TY2, NW>;
    auto kern = star_tb2_kernel<T, R, TY2, NW, DIV>;
    if (L.box_w != C::SW || L.box_h != C::SH) return cudaErrorInvalidConfiguration;
    static uint64_t attr_devices = 0;  // per instantiation, per device
    if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_devices)) return e;
    a.n_tx = (a.box.hi2 - a.x0base + C::BX - 1) / C::BX;
    a.n_ty = (a.box.hi1 - a.box.lo1 + C::BY - 1) / C::BY;
    const int n0 = a.box.hi0 - a.box.lo0;
    const int tiles = a.n_tx * a.n_ty;
    const int ctas = L.max_ctas > 0 ? L.max_ctas : L.num_sms;
    if (L.lz > 0) {
        a.lz = L.lz;
    } else {
        int ntz;
        a.lz = choose_lz(n0, tiles, ctas, 2 * R, &ntz);  // each chunk re-streams 4R planes
        if (ntz > kMaxChunks / 2) a.lz = (n0 + kMaxChunks / 2 - 1) / (kMaxChunks / 2);
    }
    a.n_tz = chunk_range(a.box.lo0, n0, a.lz, tiles, ctas, L.taper, a.zs, 0);
    a.n_signal = 0;
    a.order_y_fast = 0;
    a.band_rows = 0;  // item order: tile-row bands of ~one wave (as star_kernels.cuh launch_star_cfg)
    if (L.band_pct > 0 && a.n_tx > 0) {
        const int rows = std::max(1, (ctas * L.band_pct / 100) / a.n_tx);
        if (rows < a.n_ty) a.band_rows = rows;
    }
    a.n_items = tiles * a.n_tz;
    if (a.n_items <= 0) return cudaSuccess;
    const int grid = a.n_items < ctas ? a.n_items : ctas;
    cudaError_t e = cudaMemsetAsync(a.work_counter, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return e;
    kern<<<grid, C::THREADS, C::SMEM, stream>>>(map[0], map[1], map[2], a, L.frozen_nz);
    return cudaGetLastError();
}

template <typename T, int R>
cudaError_t launch_tb2_r(const StarLaunch& L, const StarArgs<T>& a, cudaStream_t s) {
    if (L.has_divisor) return launch_tb2_cfg<T, R, true>(L, a, L.maps, s);
    return launch_tb2_cfg<T, R, false>(L, a, L.maps, s);
}

// host: the TMA boxes of the fused tile (u with its 2R halo; the frozen v tile)
template <typename T>
inline int tb2_tile_t(int R, int* box_w, int* box_h, int* v_w, int* v_h) {
    if (R != 1) return 1;
    using C = TbCfg<T, 1, TbTile<T, 1>::TY2, TbTile<T, 1>::NW>;
    *box_w = C::SW; *box_h = C::SH; *v_w = C::VW; *v_h = C::VH;
    return 0;
}

}  // namespace stkb
