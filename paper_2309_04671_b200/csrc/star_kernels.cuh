// 2.5D d0-streaming star-stencil kernels for sm_100a (STAR and WAVE forms).
//
// Algorithmic spec followed: the reference's streaming plan emulation
// (executor.py:368-488, _PlaneWindow/_streaming_runner/_compute_plane) and the
// emitted `shift`/`unroll`/`semi` templates (codegen/gpu.py:200-421): each
// thread owns (d1,d2) columns and walks the streaming axis d0.  Re-designed
// for B200 rather than translated:
//
//  * one producer warp issues a 3-D TMA box load (cp.async.bulk.tensor) per
//    d0-plane — the (BY+2R) x (BX+2RA) in-plane tile with its halo — into a
//    STAGES-deep shared-memory ring guarded by full/empty mbarriers;
//  * 8 consumer warps: lane -> VEC (=16 B) consecutive d2 outputs, warp -> TY
//    consecutive d1 rows, so every shared read and every global store is a
//    128-bit, conflict-free, coalesced access;
//  * d0 taps never touch shared memory: every loaded plane q adds its centre
//    value into a (2R+1)-deep ring of register accumulators (outputs q-R..q+R),
//    the semi-stencil forward/backward split of executor.py:149-215 applied to
//    the stream axis.  The plane loop is unrolled by 2R+1 so ring slots are
//    static registers (no queue rotation moves);
//  * persistent CTAs (one per SM) walk (x-tile, y-tile, z-chunk) work items;
//    the producer runs ahead across item boundaries;
//  * WAVE: u_prev, kappa and the u centre of output plane q-R ride in the same
//    stage as extra TMA centre boxes, so the epilogue never waits on HBM.
#pragma once

#include "common.cuh"

namespace stkb {

enum { FORM_STAR = 0, FORM_STAR_DIV = 1, FORM_WAVE = 2 };

template <typename T, int R, int FORM, int TY, int NWY>
struct StarCfg {
    static constexpr int VEC = 16 / sizeof(T);
    static constexpr int RA = ((R + VEC - 1) / VEC) * VEC;  // x-halo rounded to a vector
    static constexpr int BX = 32 * VEC;
    static constexpr int BY = NWY * TY;
    static constexpr int SW = BX + 2 * RA;  // shared row width (elements)
    static constexpr int SH = BY + 2 * R;   // shared rows
    static constexpr int HALO_ELEMS_RAW = SW * SH;
    // TMA shared destinations stay 128-byte aligned: round the halo box up
    static constexpr int HALO_ELEMS = ((HALO_ELEMS_RAW * int(sizeof(T)) + 127) / 128) * 128 / int(sizeof(T));
    static constexpr int CTR_ELEMS = BX * BY;
    static constexpr int STAGE_ELEMS = HALO_ELEMS + (FORM == FORM_WAVE ? 3 * CTR_ELEMS : 0);
    static constexpr uint32_t HALO_BYTES = HALO_ELEMS_RAW * sizeof(T);  // bytes the TMA delivers
    static constexpr uint32_t CTR_BYTES = CTR_ELEMS * sizeof(T);
    static constexpr uint32_t STAGE_BYTES = STAGE_ELEMS * sizeof(T);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
    static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t);
    static constexpr int THREADS = (NWY + 1) * 32;
    static_assert(STAGE_BYTES % 128 == 0, "stage must keep 128-B alignment");
    static_assert(SW <= 256 && SH <= 256, "TMA box dims are limited to 256");
};

template <typename T>
__device__ __forceinline__ void lds16(const T* p, T* v) {
    using V = typename Vec16<T>::type;
    V t = *reinterpret_cast<const V*>(p);
    if constexpr (sizeof(T) == 4) { v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
    else { v[0] = t.x; v[1] = t.y; }
}

template <typename T, int R, int FORM, int TY, int NWY>
__global__ void __launch_bounds__((NWY + 1) * 32, 1)
star_stream_kernel(const __grid_constant__ CUtensorMap tm_src,
                   const __grid_constant__ CUtensorMap tm_ctr,
                   const __grid_constant__ CUtensorMap tm_prev,
                   const __grid_constant__ CUtensorMap tm_vel,
                   const __grid_constant__ StarArgs<T> a) {
    using C = StarCfg<T, R, FORM, TY, NWY>;
    constexpr int VEC = C::VEC, RA = C::RA, BX = C::BX, BY = C::BY, SW = C::SW;
    constexpr int STAGES = C::STAGES;
    constexpr int NS = 2 * R + 1;

    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    T* tiles = reinterpret_cast<T*>(base);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(STAGES) * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWY);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NWY) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            prefetch_tmap(&tm_src);
            if constexpr (FORM == FORM_WAVE) {
                prefetch_tmap(&tm_ctr);
                prefetch_tmap(&tm_prev);
                prefetch_tmap(&tm_vel);
            }
            uint32_t it = 0;
            for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
                const int tx = item % a.n_tx;
                const int rest = item / a.n_tx;
                const int ty = rest % a.n_ty;
                const int tz = rest / a.n_ty;
                const int x0 = a.x0base + tx * BX;
                const int y0 = a.box.lo1 + ty * BY;
                const int z0 = a.box.lo0 + tz * a.lz;
                const int z1 = min(z0 + a.lz, a.box.hi0);
                const int c0 = int(a.g.lead) + x0 - RA;
                const int c1 = y0 + int(a.g.order) - R;
                for (int q = z0 - R; q < z1 + R; ++q, ++it) {
                    const uint32_t s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    T* st = tiles + size_t(s) * C::STAGE_ELEMS;
                    if constexpr (FORM == FORM_WAVE) {
                        const int z = q - R;  // output plane completed at this step
                        const bool out = (z >= z0);
                        mbar_arrive_expect_tx(&full[s], C::HALO_BYTES + (out ? 3 * C::CTR_BYTES : 0));
                        tma_load_3d(st, &tm_src, &full[s], c0, c1, q + int(a.g.order0));
                        if (out) {
                            const int cx = int(a.g.lead) + x0;
                            const int cy = y0 + int(a.g.order);
                            const int cz = z + int(a.g.order0);
                            tma_load_3d(st + C::HALO_ELEMS, &tm_ctr, &full[s], cx, cy, cz);
                            tma_load_3d(st + C::HALO_ELEMS + C::CTR_ELEMS, &tm_prev, &full[s], cx, cy, cz);
                            tma_load_3d(st + C::HALO_ELEMS + 2 * C::CTR_ELEMS, &tm_vel, &full[s], cx, cy, cz);
                        }
                    } else {
                        mbar_arrive_expect_tx(&full[s], C::HALO_BYTES);
                        tma_load_3d(st, &tm_src, &full[s], c0, c1, q + int(a.g.order0));
                    }
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int xl = lane * VEC;  // d2 offset inside the tile
    const int jr0 = warp * TY;  // first d1 row of this warp inside the tile
    T acc[NS][TY][VEC];
#pragma unroll
    for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int j = 0; j < TY; ++j)
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc[k][j][i] = T(0);
    bool bad = false;
    uint32_t it = 0;

    for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        const int tx = item % a.n_tx;
        const int rest = item / a.n_tx;
        const int ty = rest % a.n_ty;
        const int tz = rest / a.n_ty;
        const int x0 = a.x0base + tx * BX;
        const int y0 = a.box.lo1 + ty * BY;
        const int z0 = a.box.lo0 + tz * a.lz;
        const int z1 = min(z0 + a.lz, a.box.hi0);
        const int x = x0 + xl;
        const int nq = (z1 - z0) + 2 * R;
        const bool x_full = (x >= a.box.lo2) && (x + VEC <= a.box.hi2);
        const bool x_any = (x + VEC > a.box.lo2) && (x < a.box.hi2);

        for (int qb = 0; qb < nq; qb += NS) {
#pragma unroll
            for (int p = 0; p < NS; ++p) {
                const int qi = qb + p;
                if (qi < nq) {
                    const int q = z0 - R + qi;
                    const uint32_t s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    mbar_wait(&full[s], ph);
                    const T* t = tiles + size_t(s) * C::STAGE_ELEMS;

                    // centre values of this thread's rows in plane q
                    T cv[TY][VEC];
#pragma unroll
                    for (int j = 0; j < TY; ++j) lds16(t + (jr0 + j + R) * SW + xl + RA, cv[j]);

                    const bool main_plane = (q >= z0) && (q < z1);
                    if (main_plane) {
                        T ip[TY][VEC];
                        // d2 (x) taps: left/right vectors of each centre row
#pragma unroll
                        for (int j = 0; j < TY; ++j) {
                            T xr[VEC + 2 * RA];
                            const T* row = t + (jr0 + j + R) * SW + xl;
#pragma unroll
                            for (int k = 0; k < RA / VEC; ++k) {
                                lds16(row + k * VEC, &xr[k * VEC]);
                                lds16(row + RA + VEC + k * VEC, &xr[RA + VEC + k * VEC]);
                            }
#pragma unroll
                            for (int i = 0; i < VEC; ++i) xr[RA + i] = cv[j][i];
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                T s_ = a.c0 * cv[j][i];
#pragma unroll
                                for (int m = 1; m <= R; ++m) {
                                    s_ = fma_t(a.cm[2][m - 1], xr[RA + i - m], s_);
                                    s_ = fma_t(a.cp[2][m - 1], xr[RA + i + m], s_);
                                }
                                ip[j][i] = s_;
                            }
                        }
                        // d1 (y) taps: stream the TY+2R rows of this warp's column
#pragma unroll
                        for (int rr = 0; rr < TY + 2 * R; ++rr) {
                            T yv[VEC];
                            if (rr >= R && rr < R + TY) {
#pragma unroll
                                for (int i = 0; i < VEC; ++i) yv[i] = cv[rr - R][i];
                            } else {
                                lds16(t + (jr0 + rr) * SW + xl + RA, yv);
                            }
#pragma unroll
                            for (int j = 0; j < TY; ++j) {
                                const int m = rr - (j + R);
                                if (m != 0 && m >= -R && m <= R) {
#pragma unroll
                                    for (int i = 0; i < VEC; ++i) {
                                        const T c = m < 0 ? a.cm[1][-m - 1] : a.cp[1][m - 1];
                                        ip[j][i] = fma_t(c, yv[i], ip[j][i]);
                                    }
                                }
                            }
                        }
                        // output q: its accumulator already holds the d0 taps of planes < q
#pragma unroll
                        for (int j = 0; j < TY; ++j)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc[p][j][i] += ip[j][i];
                    }
                    if (q < z1) {
                        // plane q feeds future outputs q+m with the -m coefficient
#pragma unroll
                        for (int j = 0; j < TY; ++j)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                acc[(p + R) % NS][j][i] = a.cm[0][R - 1] * cv[j][i];
#pragma unroll
                                for (int m = 1; m < R; ++m)
                                    acc[(p + m) % NS][j][i] =
                                        fma_t(a.cm[0][m - 1], cv[j][i], acc[(p + m) % NS][j][i]);
                            }
                    }
                    // plane q feeds past outputs q-m with the +m coefficient
#pragma unroll
                    for (int j = 0; j < TY; ++j)
#pragma unroll
                        for (int i = 0; i < VEC; ++i)
#pragma unroll
                            for (int m = 1; m <= R; ++m)
                                acc[(p - m + NS) % NS][j][i] =
                                    fma_t(a.cp[0][m - 1], cv[j][i], acc[(p - m + NS) % NS][j][i]);

                    // output plane z = q - R is complete
                    const int z = q - R;
                    const bool z_out = (z >= z0) && (z < z1);
                    constexpr int ks = (NS - R) % NS;  // slot offset of q - R relative to p
                    T outv[TY][VEC];
                    if (z_out) {
#pragma unroll
                        for (int j = 0; j < TY; ++j)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) {
                                T v = acc[(p + ks) % NS][j][i];
                                if constexpr (FORM == FORM_STAR_DIV) v = v / a.divisor;
                                outv[j][i] = v;
                            }
                        if constexpr (FORM == FORM_WAVE) {
                            const T* cu = t + C::HALO_ELEMS;
                            const T* cpv = cu + C::CTR_ELEMS;
                            const T* cvl = cpv + C::CTR_ELEMS;
#pragma unroll
                            for (int j = 0; j < TY; ++j) {
                                T uu[VEC], pp[VEC], kk[VEC];
                                const int o = (jr0 + j) * BX + xl;
                                lds16(cu + o, uu);
                                lds16(cpv + o, pp);
                                lds16(cvl + o, kk);
#pragma unroll
                                for (int i = 0; i < VEC; ++i)
                                    outv[j][i] = fma_t(kk[i], outv[j][i], fma_t(a.wave_b, pp[i], a.wave_a * uu[i]));
                            }
                        }
                    }
                    // every shared read of stage s is done: hand it back to the producer
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                    ++it;

                    if (z_out && x_any) {
#pragma unroll
                        for (int j = 0; j < TY; ++j) {
                            const int y = y0 + jr0 + j;
                            if (y >= a.box.lo1 && y < a.box.hi1) {
                                T* dp = a.dst + a.g.at(z, y, x);
                                if (x_full) {
                                    stg16(dp, outv[j]);
#pragma unroll
                                    for (int i = 0; i < VEC; ++i) bad |= !isfinite(outv[j][i]);
                                } else {
#pragma unroll
                                    for (int i = 0; i < VEC; ++i)
                                        if (x + i >= a.box.lo2 && x + i < a.box.hi2) {
                                            dp[i] = outv[j][i];
                                            bad |= !isfinite(outv[j][i]);
                                        }
                                }
                            }
                        }
                    }
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
}

// pick the z-chunk length: minimise the per-CTA critical path in plane steps
inline int choose_lz(int n0, int tiles, int ctas, int R, int* n_tz) {
    long best_cost = -1;
    int best = n0;
    for (int lz = 1; lz <= n0; ++lz) {
        const int tz = (n0 + lz - 1) / lz;
        const long items = long(tiles) * tz;
        const long waves = (items + ctas - 1) / ctas;
        const long cost = waves * (lz + 2 * R);
        if (best_cost < 0 || cost < best_cost || (cost == best_cost && lz > best)) {
            best_cost = cost;
            best = lz;
        }
    }
    *n_tz = (n0 + best - 1) / best;
    return best;
}

template <typename T, int R, int FORM, int TY>
cudaError_t launch_star_cfg(const StarLaunch& L, StarArgs<T> a, const CUtensorMap* maps,
                            cudaStream_t stream) {
    constexpr int NWY = 7;  // 7 consumer warps + 1 TMA producer warp: 2 warps per SMSP -> 255 regs/thread
    using C = StarCfg<T, R, FORM, TY, NWY>;
    auto kern = star_stream_kernel<T, R, FORM, TY, NWY>;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int w2 = a.box.hi2 - a.x0base;
    a.n_tx = (w2 + C::BX - 1) / C::BX;
    a.n_ty = (a.box.hi1 - a.box.lo1 + C::BY - 1) / C::BY;
    const int n0 = a.box.hi0 - a.box.lo0;
    const int tiles = a.n_tx * a.n_ty;
    int ctas = L.max_ctas > 0 ? L.max_ctas : L.num_sms;
    if (L.lz > 0) {
        a.lz = L.lz;
        a.n_tz = (n0 + L.lz - 1) / L.lz;
    } else {
        a.lz = choose_lz(n0, tiles, ctas, R, &a.n_tz);
    }
    a.n_items = tiles * a.n_tz;
    if (a.n_items <= 0) return cudaSuccess;
    const int grid = a.n_items < ctas ? a.n_items : ctas;
    kern<<<grid, C::THREADS, C::SMEM, stream>>>(maps[0], maps[1], maps[2], maps[3], a);
    return cudaGetLastError();
}

template <typename T>
constexpr int star_ty(int R) {
    return sizeof(T) == 4 ? (R == 1 ? 8 : (R == 2 ? 6 : 4)) : (R == 1 ? 8 : 4);
}

template <typename T, int R>
cudaError_t launch_star_r(const StarLaunch& L, const StarArgs<T>& a, const CUtensorMap* maps,
                          cudaStream_t s) {
    constexpr int TY = star_ty<T>(R);
    if (L.kind == 2) return launch_star_cfg<T, R, FORM_WAVE, TY>(L, a, maps, s);
    if (L.has_divisor) return launch_star_cfg<T, R, FORM_STAR_DIV, TY>(L, a, maps, s);
    return launch_star_cfg<T, R, FORM_STAR, TY>(L, a, maps, s);
}

template <typename T>
cudaError_t launch_star_t(const StarLaunch& L, const StarArgs<T>& a, const CUtensorMap* maps,
                          cudaStream_t s) {
    switch (L.radius) {
        case 1: return launch_star_r<T, 1>(L, a, maps, s);
        case 2: return launch_star_r<T, 2>(L, a, maps, s);
        case 3: return launch_star_r<T, 3>(L, a, maps, s);
        case 4: return launch_star_r<T, 4>(L, a, maps, s);
        default: return cudaErrorInvalidValue;
    }
}

// tile geometry used to build the tensor-map boxes on the host
template <typename T>
inline void star_tile_t(int R, int* bx, int* by, int* halo_x) {
    constexpr int VEC = 16 / sizeof(T);
    const int ty = R == 1 ? star_ty<T>(1) : R == 2 ? star_ty<T>(2) : R == 3 ? star_ty<T>(3) : star_ty<T>(4);
    *bx = 32 * VEC;
    *by = 7 * ty;
    *halo_x = ((R + VEC - 1) / VEC) * VEC;
}

}  // namespace stkb
