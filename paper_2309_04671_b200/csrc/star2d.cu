// 1.5D d0-streaming star kernels for 2-D grids (the reference's 2-D streaming
// plan, planning.py:78-86 `streaming_1_5d`: d0 is streamed, d1 is the lane axis).
//
// A 2-D grid of the paper's size (Listing 1: 1000^2, 4 MB fp32) lives in L2, so
// the design drops the TMA/shared-memory staging of the 3-D kernel: each warp
// owns 32 x VEC consecutive d1 points and a chunk of d0 rows; every lane
// fetches its row segment plus the d1 halo with 128-bit loads (neighbouring
// lanes share L1 lines), and the d0 taps go through the same (2R+1)-deep
// register accumulator ring (static slots, loop unrolled by 2R+1) and packed
// FFMA2 math as the 3-D kernel.
#include "star_kernels.cuh"

namespace stkb {

struct Star2DArgs {
    int64_t pitch;   // elements between consecutive d0 rows
    int64_t lead;    // column of interior d1 = 0
    int32_t order;   // halo (rows and columns)
    int32_t lo0, hi0, lo1, hi1;  // output box (interior coordinates)
    int32_t x0base;  // lo1 rounded down to the vector width
    int32_t n_tx, lz, n_tz;
    int32_t* nonfinite;
    double c0, cm0[4], cp0[4], cm1[4], cp1[4];  // d0 / d1 coefficients (offset -m / +m)
    double rdiv;     // 1/divisor or 0
};

// the same coefficients in the grid dtype, read straight from the parameter bank
template <typename T>
struct Coef2D {
    T c0, cm0[4], cp0[4], cm1[4], cp1[4], rdiv;
};

template <typename T, int R, bool DIV>
__global__ void __launch_bounds__(128) star2d_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                     const __grid_constant__ Star2DArgs a,
                                                     const __grid_constant__ Coef2D<T> cf) {
    using K = Pk<T>;
    using P = typename K::P;
    constexpr int VEC = 16 / sizeof(T);
    constexpr int W = K::W;
    constexpr int NPK = VEC / W;
    constexpr int RA = ((R + VEC - 1) / VEC) * VEC;
    constexpr int NS = 2 * R + 1;
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= a.n_tx * a.n_tz) return;
    const int tx = wid % a.n_tx, tz = wid / a.n_tx;
    const int x = a.x0base + (tx * 32 + lane) * VEC;
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
    const T* row0 = src + a.lead + x;  // + (q + order) * pitch
    T* out0 = dst + a.lead + x;
    P acc[NS][NPK];
#pragma unroll
    for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int i = 0; i < NPK; ++i) acc[k][i] = K::mul(T(0), P{});
    P chk = K::mul(T(0), P{});
    // rows in flight: a ring of D prefetched rows (left halo | centre | right halo);
    // D divides the unroll factor NS so ring slots stay static registers
    constexpr int D = 1;  // deeper rings (D = 3) cost occupancy and measured slower
    T nx[D][VEC + 2 * RA];
    auto fetch = [&](int qi_, T* dst) {
        const int q_ = z0 - R + qi_;
        const T* nrow = row0 + int64_t(q_ + a.order) * a.pitch;
        ldg16(nrow, *reinterpret_cast<T(*)[VEC]>(&dst[RA]));
        if (q_ >= z0 && q_ < z1) {
#pragma unroll
            for (int k = 0; k < RA / VEC; ++k) {
                ldg16(nrow - RA + k * VEC, *reinterpret_cast<T(*)[VEC]>(&dst[k * VEC]));
                ldg16(nrow + VEC + k * VEC, *reinterpret_cast<T(*)[VEC]>(&dst[RA + VEC + k * VEC]));
            }
        }
    };
#pragma unroll
    for (int d = 0; d < D; ++d)
        if (d < nq) fetch(d, nx[d]);

    for (int qb = 0; qb < nq; qb += NS) {
#pragma unroll
        for (int p = 0; p < NS; ++p) {
            const int qi = qb + p;
            if (qi >= nq) break;
            const int q = z0 - R + qi;
            // this row was fetched D steps ahead; refill its ring slot with row qi + D
            T xr[VEC + 2 * RA];
#pragma unroll
            for (int i = 0; i < VEC + 2 * RA; ++i) xr[i] = nx[p % D][i];
            if (qi + D < nq) fetch(qi + D, nx[p % D]);
            P cv[NPK];
#pragma unroll
            for (int k = 0; k < NPK; ++k) cv[k] = K::make(&xr[RA + k * W]);
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
            const int z = q - R;
            if (z >= z0 && z < z1 && x_any) {
                T v[VEC];
#pragma unroll
                for (int k = 0; k < NPK; ++k) {
                    P o = acc[(p + NS - R) % NS][k];
                    if constexpr (DIV) o = K::mul(rdiv, o);
                    K::put(&v[k * W], o);
                    chk = K::check(o, chk);
                }
                T* dp = out0 + int64_t(z + a.order) * a.pitch;
                if (x_full) {
                    stg16(dp, v);
                } else {
#pragma unroll
                    for (int i = 0; i < VEC; ++i)
                        if (x + i >= a.lo1 && x + i < a.hi1) dp[i] = v[i];
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, !K::clean(chk)) && lane == 0) atomicOr(a.nonfinite, 1);
}

template <typename T, int R>
cudaError_t launch2d_r(const Star2DArgs& a, const void* src, void* dst, bool div, cudaStream_t s) {
    const int warps = a.n_tx * a.n_tz;
    const int blocks = (warps + 3) / 4;
    Coef2D<T> cf;
    cf.c0 = T(a.c0);
    for (int m = 0; m < 4; ++m) {
        cf.cm0[m] = T(a.cm0[m]); cf.cp0[m] = T(a.cp0[m]); cf.cm1[m] = T(a.cm1[m]); cf.cp1[m] = T(a.cp1[m]);
    }
    cf.rdiv = T(a.rdiv);
    if (div)
        star2d_kernel<T, R, true><<<blocks, 128, 0, s>>>(static_cast<const T*>(src), static_cast<T*>(dst), a, cf);
    else
        star2d_kernel<T, R, false><<<blocks, 128, 0, s>>>(static_cast<const T*>(src), static_cast<T*>(dst), a, cf);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch2d_t(Star2DArgs a, int R, const void* src, void* dst, bool div, int num_sms, cudaStream_t s) {
    constexpr int VEC = 16 / sizeof(T);
    a.x0base = a.lo1 - (a.lo1 % VEC);
    a.n_tx = (a.hi1 - a.x0base + 32 * VEC - 1) / (32 * VEC);
    const int n0 = a.hi0 - a.lo0;
    // enough warps to cover every SM several times; chunks no shorter than the halo
    const int target = num_sms * 32;
    int tz = (target + a.n_tx - 1) / a.n_tx;
    int lz = (n0 + tz - 1) / tz;
    if (lz < 2 * R) lz = 2 * R;
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
