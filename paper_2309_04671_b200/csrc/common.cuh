// Shared device helpers and launch descriptors for the sm_100a stencil kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current device only:
// `mask` (one static per kernel instantiation) records the devices it was set on
template <typename K>
inline cudaError_t ensure_smem_attr(K kern, int smem, uint64_t& mask) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (mask & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) mask |= bit;
    return e;
}

namespace stkb {

// ---------------------------------------------------------------------------
// geometry of a domain's pitched device layout (generalises the reference's
// IndexScheme, codegen/common.py:14-76: flat(i) = lead_pad + sum (i_d+order)*stride_d
// with a per-row lead pad and a 128-byte row pitch instead of lead_pad = 0).
struct Geometry {
    int64_t n0, n1, n2;   // interior extents
    int64_t order;        // halo width of d1 and d2
    int64_t order0;       // halo width of d0 (== order for 3-D grids; 0 for 2-D grids lifted to 3-D)
    int64_t pitch;        // elements per padded row (multiple of 128 B)
    int64_t plane;        // elements per padded plane = pitch * (n1 + 2*order)
    int64_t lead;         // column of interior x = 0 within a row (128 B)
    // flat element index of interior coordinate (z, y, x)
    __host__ __device__ __forceinline__ int64_t at(int64_t z, int64_t y, int64_t x) const {
        return (z + order0) * plane + (y + order) * pitch + lead + x;
    }
};

constexpr int kMaxChunks = 96;

struct Box {
    int32_t lo0, hi0, lo1, hi1, lo2, hi2;
};

// Arguments of the 2.5D streaming star kernel (STAR and WAVE forms).
template <typename T>
struct StarArgs {
    Geometry g;
    Box box;
    int32_t x0base;            // lo2 rounded down to the vector width
    int32_t n_tx, n_ty, n_tz;  // work-item grid: x tiles, y tiles, z chunks
    int32_t lz;                // nominal z-chunk length
    int32_t zs[2 * kMaxChunks];  // z-chunk t = [zs[2t], zs[2t+1]) (interior d0 coordinates)
    int32_t n_signal;          // items of chunks t < n_signal bump *signal when stored
    int32_t* signal;
    int32_t n_items;
    T* dst;
    const T* src;              // centre re-read (WAVE)
    const T* prev;             // WAVE
    const T* vel;              // WAVE
    int32_t* nonfinite;        // sticky flag
    int32_t* work_counter;     // dynamic tile scheduler (reset before each launch)
    T c0;                      // centre
    T cm[3][4];                // [axis][m-1] coefficient of offset -m
    T cp[3][4];                // [axis][m-1] coefficient of offset +m
    T divisor;
    T wave_a, wave_b;
    int32_t store_hint;        // 1: streaming (evict-first) output stores
    int32_t order_y_fast;      // work items walk y tiles fastest
    int32_t band_rows;         // > 0: items walk bands of this many tile rows, every chunk of a band
                               // before the next band (a band is about one wave of CTAs)
    const int32_t* halo_nz;    // src buffer's halo flag: 0 = its halo is all +0, so the producer reads
                               // through the interior-only tensor map (TMA zero-fills the halo, no DRAM)
    // fused halo exchange (multi-GPU z-slabs): src planes q < 0 are read by TMA
    // straight from the lower neighbour's buffer (its plane pull_lo_n0 + q) when
    // bit 0 of `pull` is set, planes q >= n0 from the upper neighbour's (plane q - n0)
    // when bit 1 is — over NVLink, in place of this slab's own halo planes
    int32_t pull;
    int32_t pull_lo_n0;
    // several time steps in one launch (small grids, Jacobi ping-pong): step s reads
    // src (even s) / dst (odd s) and writes the other; a grid barrier (step_arrive)
    // separates the steps; work_counter then holds one counter per step
    int32_t n_steps;
    T* dst_alt;                  // odd steps write here (the even steps' src buffer)
    const int32_t* halo_nz_alt;  // halo flag of dst (the src of odd steps)
    int32_t* step_arrive;        // CTAs that stored all their items of a step (cumulative)
    T cb[729];                 // BOX: dense (2R+1)^3 coefficients, [dz][dy][dx], R <= 4 (last: the
                               // other fields keep their parameter-bank offsets)
};

// coefficients of the exact star kernel (star_exact.cuh): the reference's float64 constants
struct XstarCoef {
    double c0;
    double cm[3][4];  // [axis][m-1] coefficient of offset -m
    double cp[3][4];  // [axis][m-1] coefficient of offset +m
    double divisor;   // 0: none, else the sum is divided by it (IEEE division, as numpy does)
    double recip;     // RN(1 / divisor) when the divisor is in [2^-64, 2^64] (xdiv), else 0
};

// arguments of the 1.5-D kernel for 2-D grids (star2d.cu)
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
    int32_t box;     // dense (2R+1)^2 coefficient square instead of the star
    double cb[81];   // box: cb[(dy+R)*(2R+1) + (dx+R)]
};

// coefficients of the exact box kernel (box_exact.cu): c[((dz+R)(2R+1) + (dy+R))(2R+1) + (dx+R)]
struct XboxCoef {
    double c[729];  // 3-D radius <= 4; 2-D: c[(dy+R)(2R+1) + (dx+R)], radius <= 4
    double divisor;  // 0: none
    double recip;    // RN(1 / divisor) when usable (star_exact.cuh xdiv), else 0
};

// coefficients of the exact wave kernel (star_exact.cuh): a*u - p + k*(c0*u + sum_m l[m-1]*S_m)
struct XwaveCoef {
    double a;
    double c0;
    double l[4];
};

// ---------------------------------------------------------------------------
// mbarrier / TMA PTX wrappers (sm_90+ ISA, used here for sm_100a)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// one arrival per warp, from lane 0, as a predicated instruction (no divergent branch)
__device__ __forceinline__ void mbar_arrive_lane0(uint64_t* bar, int lane) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, 0;\n\t"
                 "@p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n\t}"
                 ::"r"(smem_u32(bar)), "r"(lane) : "memory");
}

// STKB_MBAR_SUSPEND_NS > 0: each try_wait may suspend the warp up to that long (woken when the
// phase completes) instead of returning at once and spinning (experiment switch)
#ifndef STKB_MBAR_SUSPEND_NS
#define STKB_MBAR_SUSPEND_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if STKB_MBAR_SUSPEND_NS > 0
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}" ::"r"(smem_u32(bar)), "r"(parity), "r"(uint32_t(STKB_MBAR_SUSPEND_NS)) : "memory");
#else
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
#endif
}

// 3-D tiled TMA load global -> shared, completion counted on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)),
          "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// make this thread's generic-proxy global writes visible to later async-proxy (TMA)
// reads, and order an acquire before this thread's own TMA reads
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// vector types: 16 bytes per access
template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

template <typename T>
__device__ __forceinline__ void load16(const T* p, T (&v)[16 / sizeof(T)]) {
    using V = typename Vec16<T>::type;
    V t = *reinterpret_cast<const V*>(p);
    if constexpr (sizeof(T) == 4) { v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
    else { v[0] = t.x; v[1] = t.y; }
}

// streaming global loads of read-once centre values (WAVE: prev, vel)
template <typename T>
__device__ __forceinline__ void ldg_stream16(const T* p, T (&v)[16 / sizeof(T)]) {
    if constexpr (sizeof(T) == 4) {
        float4 t = __ldcs(reinterpret_cast<const float4*>(p));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
        double2 t = __ldcs(reinterpret_cast<const double2*>(p));
        v[0] = t.x; v[1] = t.y;
    }
}

template <typename T>
__device__ __forceinline__ void ldg16(const T* p, T (&v)[16 / sizeof(T)]) {
    if constexpr (sizeof(T) == 4) {
        float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
        double2 t = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = t.x; v[1] = t.y;
    }
}

template <typename T>
__device__ __forceinline__ void stg16_cs(T* p, const T (&v)[16 / sizeof(T)]) {
    if constexpr (sizeof(T) == 4) __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
    else __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
}

template <typename T>
__device__ __forceinline__ void stg16(T* p, const T (&v)[16 / sizeof(T)]) {
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    }
}

__device__ __forceinline__ float fma_t(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_t(double a, double b, double c) { return __fma_rn(a, b, c); }

}  // namespace stkb

// host-side launchers implemented per dtype (star_f32.cu / star_f64.cu)
namespace stkb {
struct StarLaunch {
    int kind;          // 1 = STAR, 2 = WAVE, 4 = BOX
    int radius;
    bool has_divisor;
    const CUtensorMap* maps;  // [7]: src halo box, src/prev/vel centre boxes, lower/upper neighbour halo boxes,
                              // src halo box over the interior only
    int box_w, box_h;  // halo box the tensor maps were encoded with (must equal the kernel's tile)
    int num_sms;
    int max_ctas;      // 0 = auto (one per SM)
    int lz;            // 0 = auto
    bool taper;        // shorten the last z-chunks
    int n_ranges;      // 0: one range = the map box; else disjoint d0 ranges, launched as one grid
    const int32_t* rlo;
    const int32_t* rhi;
    int n_signal_ranges;   // the first ranges are "signal" ranges (one chunk each)
    int32_t* signal;       // counter bumped once per stored signal item
    int* signal_items;     // out: number of signal items of this launch
    const int32_t* frozen_nz;  // fused sweeps: != 0 when v's frozen values next to the box are not all zero
    int band_pct = 0;      // item order: tile-row bands of band_pct % of a wave (0 = z-major)
    int n_steps = 1;       // > 1: a multi-step launch (StarArgs::n_steps); counters = n_steps work
    int32_t* step_counters = nullptr;  // counters followed by the step-arrive counter (zeroed here)
    bool two_d = false;    // exact kernels: a 2-D grid lifted to one plane (no d0 taps, no d0 halo)
    bool small_tile = false;  // star/wave on a small grid: the 16-row tile (star_kernels.cuh)
};
int star_tile(int dtype, int radius, int kind, bool small, int* bx, int* by, int* halo_x);
cudaError_t launch_star_f32(const StarLaunch& L, const StarArgs<float>& a, cudaStream_t s);
cudaError_t launch_star_f64(const StarLaunch& L, const StarArgs<double>& a, cudaStream_t s);
cudaError_t launch_exact_f32(const StarLaunch& L, const StarArgs<float>& a, const XstarCoef& xc, cudaStream_t s);
cudaError_t launch_exact_f64(const StarLaunch& L, const StarArgs<double>& a, const XstarCoef& xc, cudaStream_t s);
int exact_tile(int dtype, int radius, bool wave, int* bx, int* by, int* halo_x);
cudaError_t launch_xbox_f32(const StarLaunch& L, const StarArgs<float>& a, const XboxCoef& xc, cudaStream_t s);
cudaError_t launch_xbox_f64(const StarLaunch& L, const StarArgs<double>& a, const XboxCoef& xc, cudaStream_t s);
int xbox_tile(int dtype, int radius, bool two_d, int* bx, int* by, int* halo_x);
cudaError_t launch_xwave_f32(const StarLaunch& L, const StarArgs<float>& a, const XwaveCoef& xc, cudaStream_t s);
cudaError_t launch_xwave_f64(const StarLaunch& L, const StarArgs<double>& a, const XwaveCoef& xc, cudaStream_t s);
}  // namespace stkb
