// Exact 2.5D d0-streaming dense-box kernel (XBOX): the reference's own arithmetic for the
// corpus box stencils (box3d1r..box3d4r, j3d27pt; box2d*, j2d9pt_gol on 2-D grids) at
// streaming speed.
//
// The corpus box form (corpus.py:77-120) is
//     v.at(0,0,0).set(c0*u.at(0,0,0) + c(-R,-R,-R)*u.at(-R,-R,-R) + ... + c(R,R,R)*u.at(R,R,R))  [/ D]
// with every offset of the (2R+1)^3 cube after the centre in sorted (d0, d1, d2) order; the
// oracle (executor.py:81-106) evaluates it left to right in float64 and rounds once.  This
// kernel performs exactly those operations (DMUL, DADD, the division; no contraction) in
// exactly that order, so its results are bit-identical to run_target.
//
// Sorted order runs plane by plane in d0.  Output o starts with its centre (plane o), then
// needs planes o-R .. o-1, then its own plane, then o+1 .. o+R.  So when plane q arrives:
//   * output q starts: acc = c0 u_q, then the taps of planes q-R .. q-1 (still resident in
//     the TMA ring), then those of plane q;
//   * outputs q-1 .. q-R add plane q's taps (their d0 = +1 .. +R layer) to a ring of R
//     partial sums in registers — plane by plane, so each output's order is kept;
//   * output q-R is complete and stored; plane q-R is read by no later output (released).
// The rows of plane q are loaded (and converted to f64) once and feed output q's d0 = 0
// layer and the R continuing outputs.  Same producer, ring and scheduler as star_exact.cuh.
#include "star_exact.cuh"

namespace stkb {

template <typename T, int R, bool D0 = true>
struct XboxCfg {
    static constexpr int VEC = 16 / sizeof(T);
    static constexpr int RA = ((R + VEC - 1) / VEC) * VEC;
    // consumer warps, one output row each; fp32 radius 2 needs more than the 128 registers of
    // 16 warps (the x-windows of 5 rows in f64): 11 warps (168)
    static constexpr int NWY = (D0 && sizeof(T) == 4 && R == 2) ? 11 : 15;
    static constexpr int BX = 32 * VEC;
    static constexpr int BY = NWY;
    static constexpr int SW = BX + 2 * RA;
    static constexpr int SH = BY + 2 * R;
    static constexpr int HALO_ELEMS = ((SW * SH * int(sizeof(T)) + 127) / 128) * 128 / int(sizeof(T));
    static constexpr uint32_t HALO_BYTES = SW * SH * sizeof(T);
    static constexpr uint32_t STAGE_BYTES = HALO_ELEMS * sizeof(T);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static_assert(!D0 || STAGES >= R + 2, "the exact box keeps R+1 planes resident plus one in flight");
    static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t) +
                                   STAGES * sizeof(int32_t);
    static constexpr int THREADS = (NWY + 1) * 32;
};

template <int R>
__device__ __forceinline__ constexpr int xbox_index(int dz, int dy, int dx) {
    return ((dz + R) * (2 * R + 1) + (dy + R)) * (2 * R + 1) + (dx + R);
}

// one row of this lane's x-window (VEC outputs and RA halo values each side), in f64
template <typename T, int VEC, int RA>
__device__ __forceinline__ void xbox_row(const T* row, double* xr) {
    T raw[VEC + 2 * RA];
#pragma unroll
    for (int k = 0; k < (VEC + 2 * RA) / VEC; ++k) lds16(row + k * VEC, &raw[k * VEC]);
#pragma unroll
    for (int k = 0; k < VEC + 2 * RA; ++k) xr[k] = double(raw[k]);
}

// D0 = false: a 2-D box (the grid lifted to one plane, no d0 halo; radius up to 4): the
// centre, then the (2R+1)^2 square row by row, each plane's outputs complete when it lands
template <typename T, int R, bool DIV, bool D0 = true>
__global__ void __launch_bounds__((XboxCfg<T, R, D0>::NWY + 1) * 32, 1)
box_exact_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ CUtensorMap tm_int,
                 const __grid_constant__ CUtensorMap tm_alt, const __grid_constant__ CUtensorMap tm_alt_int,
                 const __grid_constant__ StarArgs<T> a, const __grid_constant__ XboxCoef xc) {
    using C = XboxCfg<T, R, D0>;
    constexpr int RZ = D0 ? R : 0;  // d0 radius
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
            // multi-step launches (small 3-D grids): as star_exact_kernel
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
                    for (int q = z0 - RZ; q < z1 + RZ; ++q, ++it) {
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
    const int jr = warp;  // this warp's output row inside the tile
    if constexpr (!D0) {
        constexpr int W = 2 * R + 1;
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
                double acc[VEC];
                {
                    T cv[VEC];
                    lds16(t + (jr + R) * SW + xl + RA, cv);
#pragma unroll
                    for (int i = 0; i < VEC; ++i) acc[i] = xmul(xc.c[R * W + R], double(cv[i]));
                }
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) {
                    double xr[VEC + 2 * RA];
                    xbox_row<T, VEC, RA>(t + (jr + R + dy) * SW + xl, xr);
#pragma unroll
                    for (int dx = -R; dx <= R; ++dx) {
                        if (dy == 0 && dx == 0) continue;  // the centre came first
#pragma unroll
                        for (int i = 0; i < VEC; ++i)
                            acc[i] = xadd(acc[i], xmul(xc.c[(dy + R) * W + (dx + R)], xr[RA + i + dx]));
                    }
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
    // radius 3..4 (343 / 729 taps): the d0 and d1 loops stay loops (code size); d2 is unrolled
    constexpr int UZ = R <= 2 ? R : 1, UY = R <= 2 ? 2 * R + 1 : 1;
    double part[R][VEC];  // partial sums of the last R outputs, waiting for their d0 > 0 layers
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
        const uint32_t it0 = it;

        // plane qi = q - (z0 - R) lives in ring slot qi mod R: unrolled by R, slots are static
        for (int qb = 0; qb < nq; qb += R) {
#pragma unroll
            for (int p = 0; p < R; ++p) {
                const int qi = qb + p;
                if (qi < nq) {
                    const int q = z0 - R + qi;
                    const uint32_t cur = it0 + qi;
                    mbar_wait(&full[cur % STAGES], (cur / STAGES) & 1u);
                    const T* t = tiles + size_t(cur % STAGES) * C::HALO_ELEMS;
                    const bool start = q >= z0 && q < z1;  // output q begins (warp-uniform)
                    double acc[VEC];
                    if (start) {
                        // centre first, then the d0 = -R .. -1 layers from the resident planes
                        T cv[VEC];
                        lds16(t + (jr + R) * SW + xl + RA, cv);
#pragma unroll
                        for (int i = 0; i < VEC; ++i) acc[i] = xmul(xc.c[xbox_index<R>(0, 0, 0)], double(cv[i]));
#pragma unroll(UZ)
                        for (int dz = -R; dz < 0; ++dz) {
                            const T* tp = tiles + size_t((cur + dz) % STAGES) * C::HALO_ELEMS;
#pragma unroll(UY)
                            for (int dy = -R; dy <= R; ++dy) {
                                double xr[VEC + 2 * RA];
                                xbox_row<T, VEC, RA>(tp + (jr + R + dy) * SW + xl, xr);
#pragma unroll
                                for (int dx = -R; dx <= R; ++dx)
#pragma unroll
                                    for (int i = 0; i < VEC; ++i)
                                        acc[i] = xadd(acc[i], xmul(xc.c[xbox_index<R>(dz, dy, dx)], xr[RA + i + dx]));
                            }
                        }
                    }
                    // plane q, row by row: output q's d0 = 0 layer and outputs q-m's d0 = +m layer
#pragma unroll(UY)
                    for (int dy = -R; dy <= R; ++dy) {
                        double xr[VEC + 2 * RA];
                        xbox_row<T, VEC, RA>(t + (jr + R + dy) * SW + xl, xr);
                        if (start)
#pragma unroll
                            for (int dx = -R; dx <= R; ++dx) {
                                if (dy == 0 && dx == 0) continue;  // the centre came first
#pragma unroll
                                for (int i = 0; i < VEC; ++i)
                                    acc[i] = xadd(acc[i], xmul(xc.c[xbox_index<R>(0, dy, dx)], xr[RA + i + dx]));
                            }
#pragma unroll
                        for (int m = 1; m <= R; ++m) {
                            const int o = q - m;
                            if (o >= z0 && o < z1)
#pragma unroll
                                for (int dx = -R; dx <= R; ++dx)
#pragma unroll
                                    for (int i = 0; i < VEC; ++i)
                                        part[(p - m + R) % R][i] = xadd(part[(p - m + R) % R][i],
                                                                        xmul(xc.c[xbox_index<R>(m, dy, dx)], xr[RA + i + dx]));
                        }
                    }
                    // plane q - R is read by no later output of this item
                    __syncwarp();
                    if (qi >= R) mbar_arrive_lane0(&empty[(cur - R) % STAGES], lane);
                    // output q - R is complete (it shares slot p with output q)
                    const int z = q - R;
                    if (z >= z0 && z < z1) {
                        T outv[VEC];
                        double qv[VEC];
                        if constexpr (DIV) xdiv<VEC>(part[p], xc.divisor, xc.recip, qv);
#pragma unroll
                        for (int i = 0; i < VEC; ++i) {
                            outv[i] = T(DIV ? qv[i] : part[p][i]);  // one rounding (nearest even)
                            chk = fma_t(T(0), outv[i], chk);
                        }
                        T* const dz = dst0 + (int64_t(z) + a.g.order0) * plane;
                        if (y_in && x_full) stg16(dz, outv);
                        else if (y_in && x_any)
                            store_row_masked<T>(dz, outv[0], outv[1 % VEC], outv[2 % VEC], outv[3 % VEC], x, a.box.lo2,
                                                a.box.hi2);
                    }
                    if (start)
#pragma unroll
                        for (int i = 0; i < VEC; ++i) part[p][i] = acc[i];
                }
            }
        }
        // the item's last R planes
        __syncwarp();
        for (int qi = nq - R; qi < nq; ++qi) mbar_arrive_lane0(&empty[(it0 + qi) % STAGES], lane);
        it = it0 + nq;
    }
    if (__any_sync(0xffffffffu, chk != T(0)) && lane == 0) atomicOr(a.nonfinite, 1);
}

template <typename T, int R, bool DIV, bool D0 = true>
cudaError_t launch_xbox_cfg(const StarLaunch& L, StarArgs<T> a, const XboxCoef& xc, const CUtensorMap* maps,
                            cudaStream_t stream) {
    using C = XboxCfg<T, R, D0>;
    auto kern = box_exact_kernel<T, R, DIV, D0>;
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
cudaError_t launch_xbox_t(const StarLaunch& L, const StarArgs<T>& a, const XboxCoef& xc, cudaStream_t s) {
    const bool d = xc.divisor != 0.0;
    if (L.two_d) switch (L.radius) {  // a 2-D grid lifted to one plane: the square only
        case 1: return d ? launch_xbox_cfg<T, 1, true, false>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 1, false, false>(L, a, xc, L.maps, s);
        case 2: return d ? launch_xbox_cfg<T, 2, true, false>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 2, false, false>(L, a, xc, L.maps, s);
        case 3: return d ? launch_xbox_cfg<T, 3, true, false>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 3, false, false>(L, a, xc, L.maps, s);
        case 4: return d ? launch_xbox_cfg<T, 4, true, false>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 4, false, false>(L, a, xc, L.maps, s);
        default: return cudaErrorInvalidValue;
    }
    switch (L.radius) {
        case 1: return d ? launch_xbox_cfg<T, 1, true>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 1, false>(L, a, xc, L.maps, s);
        case 2: return d ? launch_xbox_cfg<T, 2, true>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 2, false>(L, a, xc, L.maps, s);
        case 3: return d ? launch_xbox_cfg<T, 3, true>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 3, false>(L, a, xc, L.maps, s);
        case 4: return d ? launch_xbox_cfg<T, 4, true>(L, a, xc, L.maps, s) : launch_xbox_cfg<T, 4, false>(L, a, xc, L.maps, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_xbox_f32(const StarLaunch& L, const StarArgs<float>& a, const XboxCoef& xc, cudaStream_t s) {
    return launch_xbox_t<float>(L, a, xc, s);
}

cudaError_t launch_xbox_f64(const StarLaunch& L, const StarArgs<double>& a, const XboxCoef& xc, cudaStream_t s) {
    return launch_xbox_t<double>(L, a, xc, s);
}

// the exact box kernel's tile, for the host's tensor-map boxes
int xbox_tile(int dtype, int radius, bool two_d, int* bx, int* by, int* halo_x) {
    auto set = [&](auto cfg) {
        using C = decltype(cfg);
        *bx = C::BX;
        *by = C::BY;
        *halo_x = C::RA;
        return 0;
    };
    if (two_d) {
        if (dtype == 1) {
            if (radius == 1) return set(XboxCfg<float, 1, false>{});
            if (radius == 2) return set(XboxCfg<float, 2, false>{});
            if (radius == 3) return set(XboxCfg<float, 3, false>{});
            if (radius == 4) return set(XboxCfg<float, 4, false>{});
        } else {
            if (radius == 1) return set(XboxCfg<double, 1, false>{});
            if (radius == 2) return set(XboxCfg<double, 2, false>{});
            if (radius == 3) return set(XboxCfg<double, 3, false>{});
            if (radius == 4) return set(XboxCfg<double, 4, false>{});
        }
        return 1;
    }
    if (dtype == 1) {
        if (radius == 1) return set(XboxCfg<float, 1>{});
        if (radius == 2) return set(XboxCfg<float, 2>{});
        if (radius == 3) return set(XboxCfg<float, 3>{});
        if (radius == 4) return set(XboxCfg<float, 4>{});
    } else {
        if (radius == 1) return set(XboxCfg<double, 1>{});
        if (radius == 2) return set(XboxCfg<double, 2>{});
        if (radius == 3) return set(XboxCfg<double, 3>{});
        if (radius == 4) return set(XboxCfg<double, 4>{});
    }
    return 1;
}
}  // namespace stkb
