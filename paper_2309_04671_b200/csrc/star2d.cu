// 1.5D d0-streaming star kernels for 2-D grids (the reference's 2-D streaming
// plan, planning.py:78-86 `streaming_1_5d`: d0 is streamed, d1 is the lane axis).
//
// Each warp owns 32 x VEC consecutive d1 points and a chunk of d0 rows.  Rows
// arrive through a per-warp shared-memory ring filled with asynchronous 16-byte
// copies (cp.async.cg, L2 only): D rows are in flight per warp without holding
// registers, which is what a bandwidth-bound 2-D sweep needs (a register
// prefetch of one row per warp left HBM half idle).  The edge lanes also fetch
// the d1 halo chunks, so every lane reads its row segment + halo from shared
// memory with 128-bit loads; the d0 taps go through the same (2R+1)-deep
// register accumulator ring (loop unrolled by 2R+1) and packed FFMA2 math as
// the 3-D kernel.
#include "star_kernels.cuh"

namespace stkb {

// Star2DArgs: common.cuh (shared with the host side of stkb200.cu)

// the same coefficients in the grid dtype, read straight from the parameter bank
template <typename T>
struct Coef2D {
    T c0, cm0[4], cp0[4], cm1[4], cp1[4], rdiv;
    T cb[81];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    // src-size 0 zero-fills the 16 bytes without reading global memory
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#ifndef STKB_2D_DEPTH
#define STKB_2D_DEPTH 8
#endif
#ifndef STKB_2D_WARPS
#define STKB_2D_WARPS 4
#endif

template <typename T, int R>
struct Ring2D {
    static constexpr int VEC = 16 / sizeof(T);
    static constexpr int RA = ((R + VEC - 1) / VEC) * VEC;
    static constexpr int NS = 2 * R + 1;
    static constexpr int D = NS * ((STKB_2D_DEPTH + NS - 1) / NS);  // rows in flight per warp
    static constexpr int SWR = 32 * VEC + 2 * RA;       // one ring row: left halo | 32 lanes | right halo
    static constexpr int WARPS = STKB_2D_WARPS;
    static constexpr size_t SMEM = size_t(WARPS) * D * SWR * sizeof(T);
};

template <typename T, int R, bool DIV, bool BOX>
__global__ void __launch_bounds__(32 * STKB_2D_WARPS) star2d_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                     const __grid_constant__ Star2DArgs a,
                                                     const __grid_constant__ Coef2D<T> cf) {
    using K = Pk<T>;
    using P = typename K::P;
    using G = Ring2D<T, R>;
    constexpr int VEC = G::VEC, RA = G::RA, NS = G::NS, D = G::D, SWR = G::SWR;
    constexpr int W = K::W;
    constexpr int NPK = VEC / W;
    constexpr int NH = RA / VEC;  // 16-byte halo chunks per side
    extern __shared__ __align__(16) unsigned char smem2d[];
    const int lane = threadIdx.x & 31;
    T* const ring = reinterpret_cast<T*>(smem2d) + size_t(threadIdx.x >> 5) * D * SWR;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= a.n_tx * a.n_tz) return;  // whole warps only
    const int tx = wid % a.n_tx, tz = wid / a.n_tx;
    const int xw = a.x0base + tx * 32 * VEC;  // warp's first column
    const int x = xw + lane * VEC;
    const int z0 = a.lo0 + tz * a.lz;
    const int z1 = min(z0 + a.lz, a.hi0);
    const int nq = (z1 - z0) + 2 * R;
    const bool x_full = x >= a.lo1 && x + VEC <= a.hi1;
    const bool x_any = x + VEC > a.lo1 && x < a.hi1;
    const T c0 = cf.c0;
    const T* cmz = cf.cm0;
    const T* cpz = cf.cp0;
    const T* cmx = cf.cm1;
    const T* cpx = cf.cp1;
    const T rdiv = cf.rdiv;
    const T* wrow = src + a.lead + xw;  // + (q + order) * pitch
    T* out0 = dst + a.lead + x;
    // column chunks past the padded row are zero-filled instead of read
    const int64_t row_end = a.pitch - a.lead - xw;  // elements left in the row from xw
    const bool c_ok = lane * VEC + VEC <= row_end;
    const bool r_ok = lane >= 32 - NH && (32 * VEC + (lane - (32 - NH)) * VEC + VEC <= row_end);

    auto issue = [&](int qi) {
        if (qi < nq) {
            const int q = z0 - R + qi;
            const T* g = wrow + int64_t(q + a.order) * a.pitch;
            T* r = ring + (qi % D) * SWR;
            cp_async16(r + RA + lane * VEC, g + lane * VEC, c_ok);
            if (BOX || (q >= z0 && q < z1)) {  // star: only output rows need the d1 halo
                if (lane < NH) cp_async16(r + lane * VEC, g - RA + lane * VEC, true);
                else if (lane >= 32 - NH) {
                    const int k = lane - (32 - NH);
                    cp_async16(r + RA + 32 * VEC + k * VEC, g + 32 * VEC + k * VEC, r_ok);
                }
            }
        }
        cp_async_commit();  // empty groups keep the wait count uniform
    };

    P acc[NS][NPK];
#pragma unroll
    for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int i = 0; i < NPK; ++i) acc[k][i] = K::mul(T(0), P{});
    P chk = K::mul(T(0), P{});
#pragma unroll
    for (int d = 0; d < D - 1; ++d) issue(d);

    for (int qb = 0; qb < nq; qb += NS) {
#pragma unroll
        for (int p = 0; p < NS; ++p) {
            const int qi = qb + p;
            if (qi >= nq) break;
            const int q = z0 - R + qi;
            __syncwarp();  // the slot refilled next was read by every lane last iteration
            issue(qi + D - 1);
            cp_async_wait<D - 1>();
            __syncwarp();  // row qi of every lane has landed
            const T* r = ring + (qi % D) * SWR + lane * VEC;
            T xr[VEC + 2 * RA];
#pragma unroll
            for (int k = 0; k < (VEC + 2 * RA) / VEC; ++k) lds16(r + k * VEC, &xr[k * VEC]);
            P cv[NPK];
#pragma unroll
            for (int k = 0; k < NPK; ++k) cv[k] = K::make(&xr[RA + k * W]);
            if constexpr (BOX) {
                // row q adds its layer dy of the (2R+1)^2 square to output row q - dy; the
                // dy = -R layer is the first one output q + R receives (it initialises the slot)
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) {
                    constexpr int NW = 2 * R + 1;
                    const int slot = (p - dy + 2 * NS) % NS;
#pragma unroll
                    for (int k = 0; k < NPK; ++k) {
                        P s_ = dy == -R ? K::mul(cf.cb[(dy + R) * NW], K::make(&xr[RA + k * W - R]))
                                        : K::fma(cf.cb[(dy + R) * NW], K::make(&xr[RA + k * W - R]), acc[slot][k]);
#pragma unroll
                        for (int dx = -R + 1; dx <= R; ++dx)
                            s_ = K::fma(cf.cb[(dy + R) * NW + dx + R], K::make(&xr[RA + k * W + dx]), s_);
                        acc[slot][k] = s_;
                    }
                }
            } else {
            if (q >= z0 && q < z1) {
#pragma unroll
                for (int k = 0; k < NPK; ++k) {
                    P s_ = K::fma(c0, cv[k], acc[p][k]);
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        if (W == 1 || (m % 2) == 0) {
                            s_ = K::fma(cmx[m - 1], K::make(&xr[RA + k * W - m]), s_);
                            s_ = K::fma(cpx[m - 1], K::make(&xr[RA + k * W + m]), s_);
                        } else {
                            T l[W];
                            K::put(l, s_);
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                l[w] = fma_t(cmx[m - 1], xr[RA + k * W + w - m], l[w]);
                                l[w] = fma_t(cpx[m - 1], xr[RA + k * W + w + m], l[w]);
                            }
                            s_ = K::make(l);
                        }
                    }
                    acc[p][k] = s_;
                }
            }
            if (q < z1) {
#pragma unroll
                for (int k = 0; k < NPK; ++k) {
                    acc[(p + R) % NS][k] = K::mul(cmz[R - 1], cv[k]);
#pragma unroll
                    for (int m = 1; m < R; ++m) acc[(p + m) % NS][k] = K::fma(cmz[m - 1], cv[k], acc[(p + m) % NS][k]);
                }
            }
#pragma unroll
            for (int k = 0; k < NPK; ++k)
#pragma unroll
                for (int m = 1; m <= R; ++m)
                    acc[(p - m + NS) % NS][k] = K::fma(cpz[m - 1], cv[k], acc[(p - m + NS) % NS][k]);
            }  // star
            const int z = q - R;
            if (z >= z0 && z < z1 && x_any) {
                T v[VEC];
#pragma unroll
                for (int k = 0; k < NPK; ++k) {
                    P o = acc[(p + NS - R) % NS][k];
                    if constexpr (DIV) o = K::mul(rdiv, o);
                    K::put(&v[k * W], o);
                }
                T* dp = out0 + int64_t(z + a.order) * a.pitch;
                if (x_full) {
#pragma unroll
                    for (int k = 0; k < NPK; ++k) chk = K::check(K::make(&v[k * W]), chk);
                    stg16(dp, v);
                } else {
#pragma unroll
                    for (int i = 0; i < VEC; ++i)
                        if (x + i >= a.lo1 && x + i < a.hi1) {
                            dp[i] = v[i];
                            chk = K::check(K::make(&v[i - i % W]), chk);
                        }
                }
            }
        }
    }
    cp_async_wait<0>();
    if (__any_sync(0xffffffffu, !K::clean(chk)) && lane == 0) atomicOr(a.nonfinite, 1);
}

template <typename T, int R, bool BOX>
cudaError_t launch2d_rb(const Star2DArgs& a, const Coef2D<T>& cf, const void* src, void* dst, bool div, cudaStream_t s) {
    const int warps = a.n_tx * a.n_tz;
    const int blocks = (warps + Ring2D<T, R>::WARPS - 1) / Ring2D<T, R>::WARPS;
    constexpr size_t smem = Ring2D<T, R>::SMEM;
    auto kern = div ? star2d_kernel<T, R, true, BOX> : star2d_kernel<T, R, false, BOX>;
    static uint64_t attr_devices[2] = {0, 0};  // per instantiation pair, per device
    if (cudaError_t e = ensure_smem_attr(kern, int(smem), attr_devices[div])) return e;
    kern<<<blocks, 32 * Ring2D<T, R>::WARPS, smem, s>>>(static_cast<const T*>(src), static_cast<T*>(dst), a, cf);
    return cudaGetLastError();
}

template <typename T, int R>
cudaError_t launch2d_r(const Star2DArgs& a, const void* src, void* dst, bool div, cudaStream_t s) {
    Coef2D<T> cf;
    cf.c0 = T(a.c0);
    for (int m = 0; m < 4; ++m) {
        cf.cm0[m] = T(a.cm0[m]); cf.cp0[m] = T(a.cp0[m]); cf.cm1[m] = T(a.cm1[m]); cf.cp1[m] = T(a.cp1[m]);
    }
    cf.rdiv = T(a.rdiv);
    for (int i = 0; i < 81; ++i) cf.cb[i] = T(a.cb[i]);
    if (a.box) return launch2d_rb<T, R, true>(a, cf, src, dst, div, s);
    return launch2d_rb<T, R, false>(a, cf, src, dst, div, s);
}

template <typename T>
cudaError_t launch2d_t(Star2DArgs a, int R, const void* src, void* dst, bool div, int num_sms, cudaStream_t s) {
    constexpr int VEC = 16 / sizeof(T);
    a.x0base = a.lo1 - (a.lo1 % VEC);
    a.n_tx = (a.hi1 - a.x0base + 32 * VEC - 1) / (32 * VEC);
    const int n0 = a.hi0 - a.lo0;
    // warps per SM to aim for (measured, 16384^2): short radii want many short chunks
    // (balance), long radii fewer (each chunk re-streams 2R rows)
    const int per_sm = R <= 2 ? 128 : (sizeof(T) == 8 || R == 3 ? 64 : 32);
    const int target = num_sms * per_sm;
    int tz = (target + a.n_tx - 1) / a.n_tx;
    int lz = (n0 + tz - 1) / tz;
    if (lz < 2 * R) lz = 2 * R;
    // mid-size grids: chunks of at least 4R rows (each chunk re-streams 2R rows) while a dozen
    // warps per SM remain (2048^2 radius 4: +16 %; small grids keep the short chunks)
    if (lz < 4 * R && int64_t(a.n_tx) * ((n0 + 4 * R - 1) / (4 * R)) >= int64_t(num_sms) * 12) lz = 4 * R;
    if (lz > n0) lz = n0;
    a.lz = lz;
    a.n_tz = (n0 + lz - 1) / lz;
    if (n0 <= 0 || a.hi1 <= a.lo1) return cudaSuccess;
    switch (R) {
        case 1: return launch2d_r<T, 1>(a, src, dst, div, s);
        case 2: return launch2d_r<T, 2>(a, src, dst, div, s);
        case 3: return launch2d_r<T, 3>(a, src, dst, div, s);
        case 4: return launch2d_r<T, 4>(a, src, dst, div, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_star2d(int dtype, const Star2DArgs& a, int R, const void* src, void* dst, bool div, int num_sms,
                          cudaStream_t s) {
    if (dtype == 1) return launch2d_t<float>(a, R, src, dst, div, num_sms, s);
    return launch2d_t<double>(a, R, src, dst, div, num_sms, s);
}

}  // namespace stkb
