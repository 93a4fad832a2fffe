// Exact 2.5D d0-streaming star kernel: the reference's own arithmetic at streaming speed.
//
// The reference oracle (run_target, executor.py:56-138, :222-286) evaluates a map in
// float64, node by node in parse order, and rounds once to the grid dtype.  For the
// canonical star kernels — the corpus form (corpus.py:77-120)
//     v.at(0..).set(c0*u.at(0..) + c1*u.at(o1) + ... + cn*u.at(on))    [/ D]
// with the offsets in sorted order after the centre (corpus.py:77-90) — that is
//     acc = c0*u0;  acc = acc + c_k*u_k  (k = 1..n, each product and sum rounded in f64);
//     acc = acc / D;  v = (T)acc.
// This kernel performs exactly those IEEE operations (DMUL, DADD, DDIV with explicit
// rounding, no contraction), in exactly that order, so its results are bit-identical to
// run_target — not just within tolerance — while keeping the streaming structure of
// star_kernels.cuh: TMA plane boxes into an mbarrier ring, persistent CTAs, the dynamic
// work-item scheduler.
//
// Sorted star offsets put the d0 taps around the in-plane ones:
//     centre, (-R..-1, 0, 0), (0, -R..-1, 0), (0, 0, -R..-1), (0, 0, 1..R), (0, 1..R, 0),
//     (1..R, 0, 0)
// so an output plane o can start only when its own plane arrives (the centre product comes
// first): the d0-negative taps are taken from a ring of the previous R planes' centre
// values (held in registers, converted to f64 once), the in-plane taps from the staged
// tile, and the d0-positive taps are added one per arriving plane o+1..o+R to a ring of R
// partial sums (f64).  One output row per warp keeps the f64 rings in registers.
#pragma once

#include "star_kernels.cuh"

namespace stkb {

template <typename T, int R>
struct XstarCfg {
    static constexpr int VEC = 16 / sizeof(T);
    static constexpr int RA = ((R + VEC - 1) / VEC) * VEC;
    static constexpr int NWY = 15;  // consumer warps, one output row each
    static constexpr int BX = 32 * VEC;
    static constexpr int BY = NWY;
    static constexpr int SW = BX + 2 * RA;
    static constexpr int SH = BY + 2 * R;
    static constexpr int HALO_ELEMS = ((SW * SH * int(sizeof(T)) + 127) / 128) * 128 / int(sizeof(T));
    static constexpr uint32_t HALO_BYTES = SW * SH * sizeof(T);
    static constexpr uint32_t STAGE_BYTES = HALO_ELEMS * sizeof(T);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
    static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t) +
                                   STAGES * sizeof(int32_t);
    static constexpr int THREADS = (NWY + 1) * 32;
};

__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }

// a / d correctly rounded (what numpy's division gives), from y = RN(1/d) computed on the
// host: q0 = RN(a y) is within one ulp of a/d, the remainder a - d q0 is exact in one FMA,
// and RN(q0 + r y) is then the correctly rounded quotient (Markstein's theorem for a
// correctly rounded reciprocal) — three FP64 operations instead of __ddiv_rn's iteration.
// The theorem needs every intermediate normal: |a| in (2^-900, 2^900) with |d| in
// [2^-64, 2^64] (host-checked; y = 0 otherwise) guarantees it.  Zeros, infinities, NaNs
// and extreme magnitudes take __ddiv_rn.
template <int N>
__device__ __forceinline__ void xdiv(const double (&a)[N], double d, double y, double (&q)[N]) {
    bool fast = y != 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) fast &= fabs(a[i]) > 0x1p-900 && fabs(a[i]) < 0x1p900;
    if (__all_sync(0xffffffffu, fast)) {  // warp-uniform: the rare slow path stays out of line
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const double q0 = __dmul_rn(a[i], y);
            const double r = __fma_rn(-d, q0, a[i]);
            q[i] = __fma_rn(r, y, q0);
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) q[i] = __ddiv_rn(a[i], d);
    }
}

// D0 = false: a 2-D star (the grid lifted to one plane, no d0 halo): no d0 taps, each plane's
// outputs complete when it lands (the corpus 2-D order — centre, d0-, d1-, d1+, d0+ of the 2-D
// grid — is this kernel's d1/d2 order)
template <typename T, int R, bool DIV, bool D0 = true>
__global__ void __launch_bounds__((XstarCfg<T, R>::NWY + 1) * 32, 1)
star_exact_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ CUtensorMap tm_int,
                  const __grid_constant__ CUtensorMap tm_alt, const __grid_constant__ CUtensorMap tm_alt_int,
                  const __grid_constant__ StarArgs<T> a, const __grid_constant__ XstarCoef xc) {
    constexpr int RZ = D0 ? R : 0;  // d0 radius
    using C = XstarCfg<T, R>;
    constexpr int VEC = C::VEC, RA = C::RA, BX = C::BX, BY = C::BY, SW = C::SW, NWY = C::NWY;
    constexpr int STAGES = C::STAGES;

    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    T* tiles = reinterpret_cast<T*>(base);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(STAGES) * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    volatile int32_t* stage_item = reinterpret_cast<int32_t*>(empty + STAGES);

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
        // ------------------------------------------------------------ producer (star_kernels.cuh)
        if (lane == 0) {
            // multi-step launches (small grids, star_kernels.cuh): odd steps read the dst buffer
            // through the alternate maps; a grid barrier separates the steps
            const int nsteps = a.n_steps > 1 ? a.n_steps : 1;
            const bool int0 = a.halo_nz && *reinterpret_cast<const volatile int32_t*>(a.halo_nz) == 0;
            const bool int1 = nsteps > 1 && a.halo_nz_alt && *reinterpret_cast<const volatile int32_t*>(a.halo_nz_alt) == 0;
            uint32_t it = 0;
            // at most one item per CTA (always in multi-step launches): static assignment
            const bool fixed = nsteps > 1 || a.n_items <= int(gridDim.x);
            for (int step = 0; step < nsteps; ++step) {
                const bool odd = (step & 1) != 0;
                const bool interior = odd ? int1 : int0;
                const int ix = interior ? int(a.g.lead) : 0, iy = interior ? int(a.g.order) : 0,
                          iz = interior ? int(a.g.order0) : 0;
                const CUtensorMap* own = odd ? (interior ? &tm_alt_int : &tm_alt) : (interior ? &tm_int : &tm_src);
                if (step == 0) prefetch_tmap(own);
                if (step > 0) {
                    const int32_t target = int32_t(gridDim.x) * step;
                    while (ld_acquire_gpu(a.step_arrive) < target) {
                    }
                    fence_proxy_async_global();
                }
                for (int k = 0;; ++k) {
                    const int item = fixed ? int(blockIdx.x) + k * int(gridDim.x) : atomicAdd(a.work_counter, 1);
                    if (item >= a.n_items) break;
                    int tx, ty, tz;
                    decode_item(a, item, tx, ty, tz);
                    const int x0 = a.x0base + tx * BX;
                    const int y0 = a.box.lo1 + ty * BY;
                    const int z0 = a.zs[2 * tz];
                    const int z1 = a.zs[2 * tz + 1];
                    const int c0 = int(a.g.lead) + x0 - RA - ix;
                    const int c1 = y0 + int(a.g.order) - R - iy;
                    const int tag = item + step * a.n_items;  // the consumers recover the step
                    for (int q = z0 - RZ; q < z1 + RZ; ++q, ++it) {
                        const uint32_t s = it % STAGES;
                        mbar_wait(&empty[s], ((it / STAGES) & 1u) ^ 1u);
                        stage_item[s] = tag;
                        mbar_arrive_expect_tx(&full[s], C::HALO_BYTES);
                        tma_load_3d(tiles + size_t(s) * C::HALO_ELEMS, own, &full[s], c0, c1, q + int(a.g.order0) - iz);
                    }
                }
                // end of a step (-2) or of the launch (-1): a stage without data
                const uint32_t s = it % STAGES;
                mbar_wait(&empty[s], ((it / STAGES) & 1u) ^ 1u);
                stage_item[s] = step + 1 < nsteps ? -2 : -1;
                mbar_arrive(&full[s]);
                ++it;
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int xl = lane * VEC;
    const int jr = warp;  // this warp's output row inside the tile
    if constexpr (!D0) {
        T chk2 = T(0);
        uint32_t it2 = 0;
        const int64_t pitch = a.g.pitch, plane = a.g.plane;
        while (true) {
            const uint32_t s = it2 % STAGES;
            mbar_wait(&full[s], (it2 / STAGES) & 1u);
            const int tag = __shfl_sync(0xffffffffu, stage_item[s], 0);
            if (tag == -1) break;
            if (tag == -2) {  // multi-step: publish this CTA's outputs of the step
                fence_proxy_async_global();
                asm volatile("bar.sync 1, %0;" ::"r"(NWY * 32) : "memory");
                if (threadIdx.x == 0) {
                    __threadfence();
                    atomicAdd(a.step_arrive, 1);
                }
                __syncwarp();
                mbar_arrive_lane0(&empty[s], lane);
                ++it2;
                continue;
            }
            const int step = a.n_steps > 1 ? tag / a.n_items : 0;
            const int item = tag - step * a.n_items;
            T* const dstep = (step & 1) ? a.dst_alt : a.dst;
            int tx, ty, tz;
            decode_item(a, item, tx, ty, tz);
            const int x = a.x0base + tx * BX + xl;
            const int y = a.box.lo1 + ty * BY + jr;
            const int z0 = a.zs[2 * tz], z1 = a.zs[2 * tz + 1];
            const bool y_in = y >= a.box.lo1 && y < a.box.hi1;
            const bool x_full = x >= a.box.lo2 && x + VEC <= a.box.hi2;
            const bool x_any = x + VEC > a.box.lo2 && x < a.box.hi2;
            for (int z = z0; z < z1; ++z) {
                const uint32_t sz = it2 % STAGES;
                mbar_wait(&full[sz], (it2 / STAGES) & 1u);
                const T* t = tiles + size_t(sz) * C::HALO_ELEMS;
                double xr[VEC + 2 * RA];
                {
                    T raw[VEC + 2 * RA];
                    const T* row = t + (jr + R) * SW + xl;
#pragma unroll
                    for (int k = 0; k < (VEC + 2 * RA) / VEC; ++k) lds16(row + k * VEC, &raw[k * VEC]);
#pragma unroll
                    for (int k = 0; k < VEC + 2 * RA; ++k) xr[k] = double(raw[k]);
                }
                double acc[VEC];
#pragma unroll
                for (int i = 0; i < VEC; ++i) acc[i] = xmul(xc.c0, xr[RA + i]);
#pragma unroll
                for (int m = R; m >= 1; --m) {  // (0, -m, 0)
                    T yv[VEC];
                    lds16(t + (jr + R - m) * SW + xl + RA, yv);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cm[1][m - 1], double(yv[i])));
                }
#pragma unroll
                for (int m = R; m >= 1; --m)  // (0, 0, -m)
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cm[2][m - 1], xr[RA + i - m]));
#pragma unroll
                for (int m = 1; m <= R; ++m)  // (0, 0, +m)
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cp[2][m - 1], xr[RA + i + m]));
#pragma unroll
                for (int m = 1; m <= R; ++m) {  // (0, +m, 0)
                    T yv[VEC];
                    lds16(t + (jr + R + m) * SW + xl + RA, yv);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cp[1][m - 1], double(yv[i])));
                }
                __syncwarp();
                mbar_arrive_lane0(&empty[sz], lane);
                ++it2;
                T outv[VEC];
                double qv[VEC];
                if constexpr (DIV) xdiv<VEC>(acc, xc.divisor, xc.recip, qv);
#pragma unroll
                for (int i = 0; i < VEC; ++i) {
                    outv[i] = T(DIV ? qv[i] : acc[i]);
                    chk2 = fma_t(T(0), outv[i], chk2);
                }
                T* const dz = dstep + (int64_t(z) + a.g.order0) * plane + (int64_t(y) + a.g.order) * pitch + a.g.lead + x;
                if (y_in && x_full) stg16(dz, outv);
                else if (y_in && x_any)
                    store_row_masked<T>(dz, outv[0], outv[1 % VEC], outv[2 % VEC], outv[3 % VEC], x, a.box.lo2,
                                        a.box.hi2);
            }
        }
        if (__any_sync(0xffffffffu, chk2 != T(0)) && lane == 0) atomicOr(a.nonfinite, 1);
        return;
    }
    double zneg[R][VEC];  // centre values of the previous R planes (f64), ring by plane
    double part[R][VEC];  // partial sums of the last R outputs, waiting for their d0+ taps
    T chk = T(0);
    uint32_t it = 0;
    const int64_t pitch = a.g.pitch, plane = a.g.plane;

    while (true) {
        mbar_wait(&full[it % STAGES], (it / STAGES) & 1u);
        const int tag = __shfl_sync(0xffffffffu, stage_item[it % STAGES], 0);
        if (tag == -1) break;
        if (tag == -2) {
            // multi-step launch: this CTA's outputs of the step are stored; publish them
            // (star_kernels.cuh: one gpu-scope fence per CTA after the consumer barrier)
            fence_proxy_async_global();
            asm volatile("bar.sync 1, %0;" ::"r"(NWY * 32) : "memory");
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(a.step_arrive, 1);
            }
            __syncwarp();
            mbar_arrive_lane0(&empty[it % STAGES], lane);
            ++it;
            continue;
        }
        const int step = a.n_steps > 1 ? tag / a.n_items : 0;
        const int item = tag - step * a.n_items;
        int tx, ty, tz;
        decode_item(a, item, tx, ty, tz);
        const int x0 = a.x0base + tx * BX;
        const int y0 = a.box.lo1 + ty * BY;
        const int z0 = a.zs[2 * tz];
        const int z1 = a.zs[2 * tz + 1];
        const int x = x0 + xl;
        const int y = y0 + jr;
        const int nq = (z1 - z0) + 2 * R;
        const bool y_in = y >= a.box.lo1 && y < a.box.hi1;
        const bool x_full = x >= a.box.lo2 && x + VEC <= a.box.hi2;
        const bool x_any = x + VEC > a.box.lo2 && x < a.box.hi2;
        T* const dst0 = ((step & 1) ? a.dst_alt : a.dst) + (int64_t(y) + a.g.order) * pitch + a.g.lead + x;

        // plane qi = q - (z0 - R) lives in ring slot qi mod R: unrolled by R, slots are static
        for (int qb = 0; qb < nq; qb += R) {
#pragma unroll
            for (int p = 0; p < R; ++p) {
                const int qi = qb + p;
                if (qi < nq) {
                    const int q = z0 - R + qi;
                    const uint32_t s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1u);
                    const T* t = tiles + size_t(s) * C::HALO_ELEMS;
                    // the centre row of this warp with its x-halo, in f64
                    double xr[VEC + 2 * RA];
                    {
                        T raw[VEC + 2 * RA];
                        const T* row = t + (jr + R) * SW + xl;
#pragma unroll
                        for (int k = 0; k < (VEC + 2 * RA) / VEC; ++k) lds16(row + k * VEC, &raw[k * VEC]);
#pragma unroll
                        for (int k = 0; k < VEC + 2 * RA; ++k) xr[k] = double(raw[k]);
                    }
                    double acc[VEC];
                    const bool q_out = q >= z0 && q < z1;
                    if (q_out) {
#pragma unroll
                        for (int i = 0; i < VEC; ++i) acc[i] = xmul(xc.c0, xr[RA + i]);
#pragma unroll
                        for (int m = R; m >= 1; --m)  // (-m, 0, 0): plane q - m, slot (p - m) mod R
#pragma unroll
                            for (int i = 0; i < VEC; ++i)
                                acc[i] = xadd(acc[i], xmul(xc.cm[0][m - 1], zneg[(p - m + R) % R][i]));
#pragma unroll
                        for (int m = R; m >= 1; --m) {  // (0, -m, 0)
                            T yv[VEC];
                            lds16(t + (jr + R - m) * SW + xl + RA, yv);
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cm[1][m - 1], double(yv[i])));
                        }
#pragma unroll
                        for (int m = R; m >= 1; --m)  // (0, 0, -m)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cm[2][m - 1], xr[RA + i - m]));
#pragma unroll
                        for (int m = 1; m <= R; ++m)  // (0, 0, +m)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cp[2][m - 1], xr[RA + i + m]));
#pragma unroll
                        for (int m = 1; m <= R; ++m) {  // (0, +m, 0)
                            T yv[VEC];
                            lds16(t + (jr + R + m) * SW + xl + RA, yv);
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc[i] = xadd(acc[i], xmul(xc.cp[1][m - 1], double(yv[i])));
                        }
                    }
                    __syncwarp();
                    mbar_arrive_lane0(&empty[s], lane);  // every shared read of stage s is done
                    ++it;
                    // (+m, 0, 0): this plane is the +m tap of output q - m
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        const int o = q - m;
                        if (o >= z0 && o < z1)
#pragma unroll
                            for (int i = 0; i < VEC; ++i)
                                part[(p - m + R) % R][i] =
                                    xadd(part[(p - m + R) % R][i], xmul(xc.cp[0][m - 1], xr[RA + i]));
                    }
                    // output q - R is complete (it shares slot p with output q)
                    const int z = q - R;
                    if (z >= z0 && z < z1) {
                        T outv[VEC];
                        double qv[VEC];
                        if constexpr (DIV) xdiv<VEC>(part[p], xc.divisor, xc.recip, qv);
#pragma unroll
                        for (int i = 0; i < VEC; ++i) {
                            const double v = DIV ? qv[i] : part[p][i];
                            outv[i] = T(v);  // one rounding to the grid dtype (round to nearest even)
                            chk = fma_t(T(0), outv[i], chk);
                        }
                        T* const dz = dst0 + (int64_t(z) + a.g.order0) * plane;
                        if (y_in && x_full) stg16(dz, outv);
                        else if (y_in && x_any)
                            store_row_masked<T>(dz, outv[0], outv[1 % VEC], outv[2 % VEC], outv[3 % VEC], x, a.box.lo2,
                                                a.box.hi2);
                    }
                    if (q_out)
#pragma unroll
                        for (int i = 0; i < VEC; ++i) part[p][i] = acc[i];
#pragma unroll
                    for (int i = 0; i < VEC; ++i) zneg[p][i] = xr[RA + i];
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, chk != T(0)) && lane == 0) atomicOr(a.nonfinite, 1);
}

// ---------------------------------------------------------------------------
// Exact acoustic wave: the c3 program of SURVEY.md §8(d) as the reference parses it,
//     up.at(0,0,0).set(A*u.at(0,0,0) - up.at(0,0,0) + kap.at(0,0,0) * (C0*u.at(0,0,0)
//                      + L1*(S_1) + ... + LR*(S_R)))
//     S_m = u(-m,0,0) + u(m,0,0) + u(0,-m,0) + u(0,m,0) + u(0,0,-m) + u(0,0,m)  (left to right)
// evaluated node by node in float64 (executor.py:81-106) and rounded once.  Each ring sum
// starts with BOTH d0 taps, so output o can only be evaluated once plane o+R has arrived and
// every in-plane tap is still needed: the 2R+1 planes o-R..o+R stay in the shared ring (a
// plane is released after the last output that reads it), and output o is computed from
// shared memory alone when plane o+R lands.  u_prev and kappa are read from global memory.
template <typename T, int R>
struct XwaveCfg {
    static constexpr int VEC = 16 / sizeof(T);
    static constexpr int RA = ((R + VEC - 1) / VEC) * VEC;
    // one output row per warp; fp32 radius >= 3 keeps a 2R+1-plane f64 ring of 4 values per
    // lane: 11 warps (170 registers) instead of 15 (128)
    static constexpr int NWY = (sizeof(T) == 4 && R >= 3) ? 11 : 15;
    static constexpr int BX = 32 * VEC;
    static constexpr int BY = NWY;
    static constexpr int SW = BX + 2 * RA;
    static constexpr int SH = BY + 2 * R;
    static constexpr int HALO_ELEMS = ((SW * SH * int(sizeof(T)) + 127) / 128) * 128 / int(sizeof(T));
    static constexpr uint32_t HALO_BYTES = SW * SH * sizeof(T);
    static constexpr uint32_t STAGE_BYTES = HALO_ELEMS * sizeof(T);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 2 * R + 4 ? 2 * R + 4 : STAGES_RAW;
    static_assert(STAGES >= 2 * R + 2, "the exact wave keeps 2R+1 planes resident plus one in flight");
    static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t) +
                                   STAGES * sizeof(int32_t);
    static constexpr int THREADS = (NWY + 1) * 32;
};

template <typename T, int R>
__global__ void __launch_bounds__((XwaveCfg<T, R>::NWY + 1) * 32, 1)
wave_exact_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ CUtensorMap tm_int,
                  const __grid_constant__ CUtensorMap tm_alt, const __grid_constant__ CUtensorMap tm_alt_int,
                  const __grid_constant__ StarArgs<T> a, const __grid_constant__ XwaveCoef xc) {
    using C = XwaveCfg<T, R>;
    constexpr int VEC = C::VEC, RA = C::RA, BX = C::BX, BY = C::BY, SW = C::SW, NWY = C::NWY;
    constexpr int STAGES = C::STAGES;

    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    T* tiles = reinterpret_cast<T*>(base);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(STAGES) * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    volatile int32_t* stage_item = reinterpret_cast<int32_t*>(empty + STAGES);

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
            // multi-step launches (small grids; the in-place wave ping-pong): as star_exact_kernel
            const int nsteps = a.n_steps > 1 ? a.n_steps : 1;
            const bool int0 = a.halo_nz && *reinterpret_cast<const volatile int32_t*>(a.halo_nz) == 0;
            const bool int1 = nsteps > 1 && a.halo_nz_alt && *reinterpret_cast<const volatile int32_t*>(a.halo_nz_alt) == 0;
            uint32_t it = 0;
            const bool fixed = nsteps > 1 || a.n_items <= int(gridDim.x);
            for (int step = 0; step < nsteps; ++step) {
                const bool odd = (step & 1) != 0;
                const bool interior = odd ? int1 : int0;
                const int ix = interior ? int(a.g.lead) : 0, iy = interior ? int(a.g.order) : 0,
                          iz = interior ? int(a.g.order0) : 0;
                const CUtensorMap* own = odd ? (interior ? &tm_alt_int : &tm_alt) : (interior ? &tm_int : &tm_src);
                if (step == 0) prefetch_tmap(own);
                if (step > 0) {
                    const int32_t target = int32_t(gridDim.x) * step;
                    while (ld_acquire_gpu(a.step_arrive) < target) {
                    }
                    fence_proxy_async_global();
                }
                for (int k = 0;; ++k) {
                    const int item = fixed ? int(blockIdx.x) + k * int(gridDim.x) : atomicAdd(a.work_counter, 1);
                    if (item >= a.n_items) break;
                    int tx, ty, tz;
                    decode_item(a, item, tx, ty, tz);
                    const int x0 = a.x0base + tx * BX;
                    const int y0 = a.box.lo1 + ty * BY;
                    const int z0 = a.zs[2 * tz];
                    const int z1 = a.zs[2 * tz + 1];
                    const int c0 = int(a.g.lead) + x0 - RA - ix;
                    const int c1 = y0 + int(a.g.order) - R - iy;
                    const int tag = item + step * a.n_items;
                    for (int q = z0 - R; q < z1 + R; ++q, ++it) {
                        const uint32_t s = it % STAGES;
                        mbar_wait(&empty[s], ((it / STAGES) & 1u) ^ 1u);
                        stage_item[s] = tag;
                        mbar_arrive_expect_tx(&full[s], C::HALO_BYTES);
                        tma_load_3d(tiles + size_t(s) * C::HALO_ELEMS, own, &full[s], c0, c1, q + int(a.g.order0) - iz);
                    }
                }
                const uint32_t s = it % STAGES;
                mbar_wait(&empty[s], ((it / STAGES) & 1u) ^ 1u);
                stage_item[s] = step + 1 < nsteps ? -2 : -1;
                mbar_arrive(&full[s]);
                ++it;
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int xl = lane * VEC;
    const int jr = warp;
    T chk = T(0);
    uint32_t it = 0;
    const int64_t pitch = a.g.pitch, plane = a.g.plane;

    while (true) {
        mbar_wait(&full[it % STAGES], (it / STAGES) & 1u);
        const int tag = __shfl_sync(0xffffffffu, stage_item[it % STAGES], 0);
        if (tag == -1) break;
        if (tag == -2) {  // multi-step: publish this CTA's outputs of the step (star_exact_kernel)
            fence_proxy_async_global();
            asm volatile("bar.sync 1, %0;" ::"r"(NWY * 32) : "memory");
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(a.step_arrive, 1);
            }
            __syncwarp();
            mbar_arrive_lane0(&empty[it % STAGES], lane);
            ++it;
            continue;
        }
        const int step = a.n_steps > 1 ? tag / a.n_items : 0;
        const int item = tag - step * a.n_items;
        // in-place ping-pong (multi-step launches): odd steps write (and read u_prev from) the
        // even steps' src buffer
        T* const dst = (step & 1) ? a.dst_alt : a.dst;
        const T* const prev = (step & 1) ? a.dst_alt : a.prev;
        int tx, ty, tz;
        decode_item(a, item, tx, ty, tz);
        const int x0 = a.x0base + tx * BX;
        const int y0 = a.box.lo1 + ty * BY;
        const int z0 = a.zs[2 * tz];
        const int z1 = a.zs[2 * tz + 1];
        const int x = x0 + xl;
        const int y = y0 + jr;
        const int nq = (z1 - z0) + 2 * R;
        const bool y_in = y >= a.box.lo1 && y < a.box.hi1;
        const bool x_full = x >= a.box.lo2 && x + VEC <= a.box.hi2;
        const bool x_any = x + VEC > a.box.lo2 && x < a.box.hi2;
        const int64_t row_off = (int64_t(y) + a.g.order) * pitch + a.g.lead + x;
        const uint32_t it0 = it;
        // centre values of the last 2R+1 planes in f64 (ring slot = plane index mod 2R+1; the
        // loop is unrolled by 2R+1 so slots are static registers): the d0 taps of every output
        // come from here, converted once per plane instead of once per use
        constexpr int NS = 2 * R + 1;
        double zr[NS][VEC];
        for (int qb = 0; qb < nq; qb += NS) {
#pragma unroll
            for (int p = 0; p < NS; ++p) {
                const int qi = qb + p;
                if (qi >= nq) break;
                const uint32_t cur = it0 + qi;  // plane q = z0 - R + qi
                mbar_wait(&full[cur % STAGES], (cur / STAGES) & 1u);
                {
                    T c[VEC];
                    lds16(tiles + size_t(cur % STAGES) * C::HALO_ELEMS + (jr + R) * SW + xl + RA, c);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) zr[p][i] = double(c[i]);
                }
                if (qi >= 2 * R) {
                    // output o = z0 + qi - 2R (plane slot p - R): planes o-R .. o+R are resident
                    const int o = z0 + qi - 2 * R;
                    const int64_t off = (int64_t(o) + a.g.order0) * plane + row_off;
                    T pv[VEC] = {}, kv[VEC] = {};
                    if (y_in && x_any) {  // read early: the shared-memory work hides the latency
                        load16(prev + off, pv);  // plain load: u_prev may be the destination (in place)
                        ldg16(a.vel + off, kv);
                    }
                    const T* to = tiles + size_t((cur - R) % STAGES) * C::HALO_ELEMS;
                    const int po = (p - R + NS) % NS;  // slot of plane o (static after unrolling)
                    double xr[VEC + 2 * RA];
                    {
                        T raw[VEC + 2 * RA];
                        const T* row = to + (jr + R) * SW + xl;
#pragma unroll
                        for (int k = 0; k < RA / VEC; ++k) {
                            lds16(row + k * VEC, &raw[k * VEC]);
                            lds16(row + RA + VEC + k * VEC, &raw[RA + VEC + k * VEC]);
                        }
#pragma unroll
                        for (int k = 0; k < RA; ++k) {
                            xr[k] = double(raw[k]);
                            xr[RA + VEC + k] = double(raw[RA + VEC + k]);
                        }
#pragma unroll
                        for (int i = 0; i < VEC; ++i) xr[RA + i] = zr[po][i];
                    }
                    double lap[VEC];
#pragma unroll
                    for (int i = 0; i < VEC; ++i) lap[i] = xmul(xc.c0, xr[RA + i]);
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        T ym[VEC], yp[VEC];
                        lds16(to + (jr + R - m) * SW + xl + RA, ym);
                        lds16(to + (jr + R + m) * SW + xl + RA, yp);
#pragma unroll
                        for (int i = 0; i < VEC; ++i) {
                            double sm = xadd(zr[(po - m + NS) % NS][i], zr[(po + m) % NS][i]);
                            sm = xadd(sm, double(ym[i]));
                            sm = xadd(sm, double(yp[i]));
                            sm = xadd(sm, xr[RA + i - m]);
                            sm = xadd(sm, xr[RA + i + m]);
                            lap[i] = xadd(lap[i], xmul(xc.l[m - 1], sm));
                        }
                    }
                    T outv[VEC];
#pragma unroll
                    for (int i = 0; i < VEC; ++i) {
                        const double head = __dsub_rn(xmul(xc.a, xr[RA + i]), double(pv[i]));
                        outv[i] = T(xadd(head, xmul(double(kv[i]), lap[i])));
                        chk = fma_t(T(0), outv[i], chk);
                    }
                    __syncwarp();
                    // plane o - R is read by no later output of this item
                    mbar_arrive_lane0(&empty[(cur - 2 * R) % STAGES], lane);
                    T* const dz = dst + off;
                    if (y_in && x_full) stg16(dz, outv);
                    else if (y_in && x_any)
                        store_row_masked<T>(dz, outv[0], outv[1 % VEC], outv[2 % VEC], outv[3 % VEC], x, a.box.lo2,
                                            a.box.hi2);
                }
            }
        }
        // the item's last 2R planes
        __syncwarp();
        for (int qi = nq - 2 * R; qi < nq; ++qi) mbar_arrive_lane0(&empty[(it0 + qi) % STAGES], lane);
        it = it0 + nq;
    }
    if (__any_sync(0xffffffffu, chk != T(0)) && lane == 0) atomicOr(a.nonfinite, 1);
}

template <typename T, int R>
cudaError_t launch_xwave_cfg(const StarLaunch& L, StarArgs<T> a, const XwaveCoef& xc, const CUtensorMap* maps,
                             cudaStream_t stream) {
    using C = XwaveCfg<T, R>;
    auto kern = wave_exact_kernel<T, R>;
    if (L.box_w != C::SW || L.box_h != C::SH) return cudaErrorInvalidConfiguration;
    static uint64_t attr_devices = 0;
    if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_devices)) return e;
    a.n_tx = (a.box.hi2 - a.x0base + C::BX - 1) / C::BX;
    a.n_ty = (a.box.hi1 - a.box.lo1 + C::BY - 1) / C::BY;
    const int n0 = a.box.hi0 - a.box.lo0;
    const int tiles = a.n_tx * a.n_ty;
    const int ctas = L.max_ctas > 0 ? L.max_ctas : L.num_sms;
    const bool multi = L.n_steps > 1;
    int ntz;
    if (L.lz > 0) {
        a.lz = L.lz;
    } else if (multi && tiles < ctas) {
        const int per_tile = std::max(1, ctas / tiles);
        a.lz = (n0 + per_tile - 1) / per_tile;
    } else {
        a.lz = choose_lz(n0, tiles, ctas, R, &ntz);
        if (ntz > kMaxChunks / 2) a.lz = (n0 + kMaxChunks / 2 - 1) / (kMaxChunks / 2);
    }
    a.n_tz = chunk_range(a.box.lo0, n0, a.lz, tiles, ctas, L.taper && !multi, a.zs, 0);
    a.n_signal = 0;
    a.band_rows = 0;
    if (L.band_pct > 0 && a.n_tx > 0) {
        const int rows = std::max(1, (ctas * L.band_pct / 100) / a.n_tx);
        if (rows < a.n_ty) a.band_rows = rows;
    }
    a.n_items = tiles * a.n_tz;
    if (a.n_items <= 0) return cudaSuccess;
    const int grid = a.n_items < ctas ? a.n_items : ctas;
    if (multi) {
        a.n_steps = L.n_steps;
        a.step_arrive = L.step_counters + L.n_steps;
        cudaError_t e = cudaMemsetAsync(L.step_counters, 0, (L.n_steps + 1) * sizeof(int32_t), stream);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[6], maps[4], maps[5], a, xc);
    }
    a.n_steps = 1;
    cudaError_t e = cudaMemsetAsync(a.work_counter, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return e;
    kern<<<grid, C::THREADS, C::SMEM, stream>>>(maps[0], maps[6], maps[0], maps[6], a, xc);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_xwave_t(const StarLaunch& L, const StarArgs<T>& a, const XwaveCoef& xc, const CUtensorMap* maps,
                           cudaStream_t s) {
    switch (L.radius) {
        case 1: return launch_xwave_cfg<T, 1>(L, a, xc, maps, s);
        case 2: return launch_xwave_cfg<T, 2>(L, a, xc, maps, s);
        case 3: return launch_xwave_cfg<T, 3>(L, a, xc, maps, s);
        case 4: return launch_xwave_cfg<T, 4>(L, a, xc, maps, s);
        default: return cudaErrorInvalidValue;
    }
}

template <typename T, int R, bool DIV, bool D0 = true>
cudaError_t launch_exact_cfg(const StarLaunch& L, StarArgs<T> a, const XstarCoef& xc, const CUtensorMap* maps,
                             cudaStream_t stream) {
    using C = XstarCfg<T, R>;
    auto kern = star_exact_kernel<T, R, DIV, D0>;
    if (L.box_w != C::SW || L.box_h != C::SH) return cudaErrorInvalidConfiguration;
    static uint64_t attr_devices = 0;
    if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_devices)) return e;
    a.n_tx = (a.box.hi2 - a.x0base + C::BX - 1) / C::BX;
    a.n_ty = (a.box.hi1 - a.box.lo1 + C::BY - 1) / C::BY;
    const int n0 = a.box.hi0 - a.box.lo0;
    const int tiles = a.n_tx * a.n_ty;
    const int ctas = L.max_ctas > 0 ? L.max_ctas : L.num_sms;
    const bool multi = L.n_steps > 1;
    int ntz;
    if (L.lz > 0) {
        a.lz = L.lz;
    } else if (multi && tiles < ctas) {
        // one item per CTA and step, the shortest chunks that fit one wave (star_kernels.cuh)
        const int per_tile = std::max(1, ctas / tiles);
        a.lz = (n0 + per_tile - 1) / per_tile;
    } else {
        a.lz = choose_lz(n0, tiles, ctas, R, &ntz);
        if (ntz > kMaxChunks / 2) a.lz = (n0 + kMaxChunks / 2 - 1) / (kMaxChunks / 2);
    }
    a.n_tz = chunk_range(a.box.lo0, n0, a.lz, tiles, ctas, L.taper && !multi, a.zs, 0);
    a.n_signal = 0;
    a.band_rows = 0;
    if (L.band_pct > 0 && a.n_tx > 0) {
        const int rows = std::max(1, (ctas * L.band_pct / 100) / a.n_tx);
        if (rows < a.n_ty) a.band_rows = rows;
    }
    a.n_items = tiles * a.n_tz;
    if (a.n_items <= 0) return cudaSuccess;
    const int grid = a.n_items < ctas ? a.n_items : ctas;
    if (multi) {
        // several steps, a grid barrier between them: a cooperative launch (every CTA resident)
        a.n_steps = L.n_steps;
        a.step_arrive = L.step_counters + L.n_steps;
        cudaError_t e = cudaMemsetAsync(L.step_counters, 0, (L.n_steps + 1) * sizeof(int32_t), stream);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[6], maps[4], maps[5], a, xc);
    }
    a.n_steps = 1;
    cudaError_t e = cudaMemsetAsync(a.work_counter, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return e;
    kern<<<grid, C::THREADS, C::SMEM, stream>>>(maps[0], maps[6], maps[0], maps[6], a, xc);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_exact_t(const StarLaunch& L, const StarArgs<T>& a, const XstarCoef& xc, const CUtensorMap* maps,
                           cudaStream_t s) {
    const bool div = xc.divisor != 0.0;
    if (L.two_d) switch (L.radius) {  // a 2-D grid lifted to one plane: no d0 taps
        case 1: return div ? launch_exact_cfg<T, 1, true, false>(L, a, xc, maps, s) : launch_exact_cfg<T, 1, false, false>(L, a, xc, maps, s);
        case 2: return div ? launch_exact_cfg<T, 2, true, false>(L, a, xc, maps, s) : launch_exact_cfg<T, 2, false, false>(L, a, xc, maps, s);
        case 3: return div ? launch_exact_cfg<T, 3, true, false>(L, a, xc, maps, s) : launch_exact_cfg<T, 3, false, false>(L, a, xc, maps, s);
        case 4: return div ? launch_exact_cfg<T, 4, true, false>(L, a, xc, maps, s) : launch_exact_cfg<T, 4, false, false>(L, a, xc, maps, s);
        default: return cudaErrorInvalidValue;
    }
    switch (L.radius) {
        case 1: return div ? launch_exact_cfg<T, 1, true>(L, a, xc, maps, s) : launch_exact_cfg<T, 1, false>(L, a, xc, maps, s);
        case 2: return div ? launch_exact_cfg<T, 2, true>(L, a, xc, maps, s) : launch_exact_cfg<T, 2, false>(L, a, xc, maps, s);
        case 3: return div ? launch_exact_cfg<T, 3, true>(L, a, xc, maps, s) : launch_exact_cfg<T, 3, false>(L, a, xc, maps, s);
        case 4: return div ? launch_exact_cfg<T, 4, true>(L, a, xc, maps, s) : launch_exact_cfg<T, 4, false>(L, a, xc, maps, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace stkb
