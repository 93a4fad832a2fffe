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

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace stkb {

enum { FORM_STAR = 0, FORM_STAR_DIV = 1, FORM_WAVE = 2, FORM_BOX = 3, FORM_BOX_DIV = 4 };

template <typename T, int R, int FORM, int TY, int NWY, int LW = 0>
struct StarCfg {
    // elements per lane: one 16-byte vector by default, LW (a multiple of it) when given
    static constexpr int VEC = LW > 0 ? LW : int(16 / sizeof(T));
    static_assert((VEC * sizeof(T)) % 16 == 0, "a lane holds whole 16-byte vectors");
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
#ifdef STKB_EXP_NOYHALO
    static constexpr uint32_t HALO_BYTES = SW * BY * sizeof(T);  // experiment: no y-halo rows loaded
#elif defined(STKB_EXP_NOXHALO)
    static constexpr uint32_t HALO_BYTES = BX * SH * sizeof(T);  // experiment: no x-halo columns loaded
#else
    static constexpr uint32_t HALO_BYTES = HALO_ELEMS_RAW * sizeof(T);  // bytes the TMA delivers
#endif
    static constexpr uint32_t CTR_BYTES = CTR_ELEMS * sizeof(T);
    static constexpr uint32_t STAGE_BYTES = STAGE_ELEMS * sizeof(T);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
#ifndef STKB_MAX_STAGES
#define STKB_MAX_STAGES 8
#endif
    static constexpr int STAGES = STAGES_RAW > STKB_MAX_STAGES ? STKB_MAX_STAGES : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
    static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t) +
                                   STAGES * sizeof(int32_t);
    static constexpr int THREADS = (NWY + 1) * 32;
    static_assert(STAGE_BYTES % 128 == 0, "stage must keep 128-B alignment");
    static_assert(SW <= 256 && SH <= 256, "TMA box dims are limited to 256");
};

// 128-bit shared loads through an explicit shared-window address (LDS.128;
// a generic pointer here would compile to LD.E.128 through the generic path)
__device__ __forceinline__ void lds16(const float* p, float* v) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void lds16(const double* p, double* v) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(smem_u32(p)));
}

// N consecutive elements (whole 16-byte vectors): shared loads / global stores
template <typename T, int N>
__device__ __forceinline__ void ldsv(const T* p, T* v) {
    constexpr int E = 16 / sizeof(T);
#pragma unroll
    for (int k = 0; k < N / E; ++k) lds16(p + k * E, v + k * E);
}
template <typename T, int N>
__device__ __forceinline__ void stgv(T* p, const T (&v)[N], bool streaming) {
    constexpr int E = 16 / sizeof(T);
#pragma unroll
    for (int k = 0; k < N / E; ++k) {
        T w[E];
#pragma unroll
        for (int i = 0; i < E; ++i) w[i] = v[k * E + i];
        if (streaming) stg16_cs(p + k * E, w);
        else stg16(p + k * E, w);
    }
}

// ---------------------------------------------------------------------------
// lane packs: fp32 runs two points per instruction (FFMA2 / FMUL2, sm_100),
// fp64 one.  `Pk<T>::P` holds W consecutive d2 points of one row.
template <typename T> struct Pk;
template <> struct Pk<float> {
    static constexpr int W = 2;
    struct P { float x, y; };
    static __device__ __forceinline__ P make(const float* v) { return P{v[0], v[1]}; }
    static __device__ __forceinline__ void put(float* v, P p) { v[0] = p.x; v[1] = p.y; }
    static __device__ __forceinline__ P fma(float c, P b, P acc) {  // c*b + acc, c broadcast
        P d;
        asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
            "mov.b64 rc, {%5, %6};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
            : "=f"(d.x), "=f"(d.y) : "f"(c), "f"(b.x), "f"(b.y), "f"(acc.x), "f"(acc.y));
        return d;
    }
    static __device__ __forceinline__ P fmav(P a, P b, P acc) {  // a*b + acc, lane-wise
        P d;
        asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
            "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
            : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(acc.x), "f"(acc.y));
        return d;
    }
    static __device__ __forceinline__ P mul(float c, P b) {
        P d;
        asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
            "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
            : "=f"(d.x), "=f"(d.y) : "f"(c), "f"(b.x), "f"(b.y));
        return d;
    }
    // 0 stays 0 for finite lanes; an inf/nan lane turns the check into nan
    static __device__ __forceinline__ P check(P v, P chk) { return fma(0.0f, v, chk); }
    static __device__ __forceinline__ bool clean(P chk) { return chk.x == 0.0f && chk.y == 0.0f; }
};
template <> struct Pk<double> {
    static constexpr int W = 1;
    struct P { double x; };
    static __device__ __forceinline__ P make(const double* v) { return P{v[0]}; }
    static __device__ __forceinline__ void put(double* v, P p) { v[0] = p.x; }
    static __device__ __forceinline__ P fma(double c, P b, P acc) { return P{__fma_rn(c, b.x, acc.x)}; }
    static __device__ __forceinline__ P fmav(P a, P b, P acc) { return P{__fma_rn(a.x, b.x, acc.x)}; }
    static __device__ __forceinline__ P mul(double c, P b) { return P{__dmul_rn(c, b.x)}; }
    static __device__ __forceinline__ P check(P v, P chk) { return P{__fma_rn(0.0, v.x, chk.x)}; }
    static __device__ __forceinline__ bool clean(P chk) { return chk.x == 0.0; }
};

// work item -> (x tile, y tile, z chunk); z-major so concurrent items are
// neighbours.  order_y_fast walks y tiles fastest (experiment switch).
template <typename A>
__device__ __forceinline__ void decode_item(const A& a, int item, int& tx, int& ty, int& tz) {
    if (a.band_rows > 0) {
        // bands of about one wave of tiles, each band's chunks in order: chunk k+1 of a
        // tile is handed out while chunk k still runs, so the 2R planes both read are
        // one DRAM read; y-neighbours inside a band stay n_tx items apart
        const int per_band = a.band_rows * a.n_tx * a.n_tz;
        const int band = item / per_band;
        const int rem = item - band * per_band;
        const int rows = min(a.band_rows, a.n_ty - band * a.band_rows);
        const int tiles = rows * a.n_tx;
        tz = rem / tiles;
        const int r = rem - tz * tiles;
        ty = band * a.band_rows + r / a.n_tx;
        tx = r - (r / a.n_tx) * a.n_tx;
        return;
    }
    const int per = a.n_tx * a.n_ty;
    tz = item / per;
    const int r = item - tz * per;
    if (a.order_y_fast == 1) {
        ty = r % a.n_ty;
        tx = r / a.n_ty;
    } else if (a.order_y_fast >= 2) {
        // bands of G tile rows: y fastest inside a band, then x, then the next band
        const int G = a.order_y_fast;
        const int band = r / (G * a.n_tx);
        const int rb = r - band * G * a.n_tx;
        const int rows = min(G, a.n_ty - band * G);
        ty = band * G + rb % rows;
        tx = rb / rows;
    } else {
        tx = r % a.n_tx;
        ty = r / a.n_tx;
    }
}

// streaming (evict-first) output stores: a compile-time experiment switch (measured ±1 %)
#ifndef STKB_STORE_STREAMING
#define STKB_STORE_STREAMING false
#endif

// cold path: one output row of a tile that straddles the region box
template <typename T>
__device__ __noinline__ void store_row_masked(T* dz, T v0, T v1, T v2, T v3, int x, int lo2, int hi2) {
    constexpr int VEC = 16 / sizeof(T);
    const T v[4] = {v0, v1, v2, v3};
#pragma unroll
    for (int i = 0; i < VEC; ++i)
        if (x + i >= lo2 && x + i < hi2) dz[i] = v[i];
}

// the same for N <= 4 values per lane, passed by value (an array argument would push the
// caller's output row through local memory on every plane)
template <typename T, int N>
__device__ __noinline__ void store_row_masked_n(T* dz, T v0, T v1, T v2, T v3, int x, int lo2, int hi2) {
    static_assert(N <= 4, "at most 4 values per lane");
    const T v[4] = {v0, v1, v2, v3};
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (x + i >= lo2 && x + i < hi2) dz[i] = v[i];
}

template <typename T, int R, int FORM, int TY, int NWY, bool ODD_SCALAR, bool PULL, int LW = 0>
__global__ void __launch_bounds__((NWY + 1) * 32, 1)
star_stream_kernel(const __grid_constant__ CUtensorMap tm_src,
                   const __grid_constant__ CUtensorMap tm_ctr,
                   const __grid_constant__ CUtensorMap tm_prev,
                   const __grid_constant__ CUtensorMap tm_vel,
                   const __grid_constant__ CUtensorMap tm_lo,   // lower neighbour's src (a.pull & 1)
                   const __grid_constant__ CUtensorMap tm_hi,   // upper neighbour's src (a.pull & 2)
                   const __grid_constant__ CUtensorMap tm_int,  // src interior only (a.halo_nz)
                   const __grid_constant__ StarArgs<T> a) {
    using C = StarCfg<T, R, FORM, TY, NWY, LW>;
    constexpr int VEC = C::VEC, RA = C::RA, BX = C::BX, BY = C::BY, SW = C::SW;
    constexpr int STAGES = C::STAGES;
    constexpr int NS = 2 * R + 1;

    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    T* tiles = reinterpret_cast<T*>(base);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(STAGES) * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    volatile int32_t* stage_item = reinterpret_cast<int32_t*>(empty + STAGES);  // work item of each stage

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
            // a src whose halo is all zero is read through the interior-only map: the TMA
            // zero-fills the halo instead of fetching it (the padded grid's own halo is ~1.5 %
            // of a 1024^3 step's reads)
            const int nsteps = PULL ? 1 : a.n_steps;
            const bool interior0 = a.halo_nz && *reinterpret_cast<const volatile int32_t*>(a.halo_nz) == 0;
            // multi-step launches (never PULL): odd steps read the dst buffer through tm_lo (full)
            // or tm_hi (interior only)
            const bool interior1 = nsteps > 1 && a.halo_nz_alt &&
                                   *reinterpret_cast<const volatile int32_t*>(a.halo_nz_alt) == 0;
            prefetch_tmap(interior0 ? &tm_int : &tm_src);
            if constexpr (PULL) {
                if (a.pull & 1) prefetch_tmap(&tm_lo);
                if (a.pull & 2) prefetch_tmap(&tm_hi);
            } else if (nsteps > 1) {
                prefetch_tmap(interior1 ? &tm_hi : &tm_lo);
            }
            if constexpr (FORM == FORM_WAVE) {
                prefetch_tmap(&tm_ctr);
                prefetch_tmap(&tm_prev);
                prefetch_tmap(&tm_vel);
            }
            uint32_t it = 0;
            for (int step = 0; step < nsteps; ++step) {
                const bool odd = (step & 1) != 0;
                const bool interior = odd ? interior1 : interior0;
                const int ix = interior ? int(a.g.lead) : 0, iy = interior ? int(a.g.order) : 0,
                          iz = interior ? int(a.g.order0) : 0;
                const CUtensorMap* own = odd ? (interior ? &tm_hi : &tm_lo) : (interior ? &tm_int : &tm_src);
                if (step > 0) {
                    // grid barrier: every CTA has stored its items of the previous step (they
                    // published them with a release after a proxy fence); then order this
                    // thread's TMA reads after the acquire
                    const int32_t target = int32_t(gridDim.x) * step;
                    while (ld_acquire_gpu(a.step_arrive) < target) {
                    }
                    fence_proxy_async_global();
                }
                // dynamic tile scheduler: items are handed out in (z-chunk, y-tile, x-tile)
                // order, so CTAs working at the same time stream neighbouring tiles and
                // share their halo rows through L2
                // (multi-step launches — every CTA is resident and has about one item per step —
                // and launches with at most one item per CTA assign items statically: no
                // scheduler atomic after a grid barrier or at the kernel start)
                const bool fixed = nsteps > 1 || a.n_items <= int(gridDim.x);
                for (int k = 0;; ++k) {
                    const int item = fixed ? int(blockIdx.x) + k * int(gridDim.x)
                                           : atomicAdd(a.work_counter + step, 1);
                    if (item >= a.n_items) break;
                    int tx, ty, tz;
                    decode_item(a, item, tx, ty, tz);
                    const int x0 = a.x0base + tx * BX;
                    const int y0 = a.box.lo1 + ty * BY;
                    const int z0 = a.zs[2 * tz];
                    const int z1 = a.zs[2 * tz + 1];
                    const int c0 = int(a.g.lead) + x0 - RA;
                    const int c1 = y0 + int(a.g.order) - R;
                    const int tag = item + step * a.n_items;  // the consumers recover the step
                    for (int q = z0 - R; q < z1 + R; ++q, ++it) {
                        const uint32_t s = it % STAGES;
                        const uint32_t ph = (it / STAGES) & 1u;
                        mbar_wait(&empty[s], ph ^ 1u);
                        stage_item[s] = tag;
                        T* st = tiles + size_t(s) * C::STAGE_ELEMS;
                        // src plane q: this slab's own (incl. its halo), or a neighbour's over NVLink
                        const CUtensorMap* hm = own;
#ifdef STKB_EXP_L2SRC
                        // experiment: every plane read from a window of STKB_EXP_L2SRC planes (an
                        // L2-resident source: the kernel's rate with HBM writes only)
                        int hz = ((q % STKB_EXP_L2SRC) + STKB_EXP_L2SRC) % STKB_EXP_L2SRC + int(a.g.order0) - iz;
#else
                        int hz = q + int(a.g.order0) - iz;
#endif
                        int hx = c0 - ix, hy = c1 - iy;
                        if constexpr (PULL) {
                            if (q < 0 && (a.pull & 1)) {
                                hm = &tm_lo;
                                hz = q + a.pull_lo_n0 + int(a.g.order0);
                                hx = c0;
                                hy = c1;
                            } else if (q >= int(a.g.n0) && (a.pull & 2)) {
                                hm = &tm_hi;
                                hz = q - int(a.g.n0) + int(a.g.order0);
                                hx = c0;
                                hy = c1;
                            }
                        }
                        if constexpr (FORM == FORM_WAVE) {
                            const int z = q - R;  // output plane completed at this step
                            const bool out = (z >= z0);
                            mbar_arrive_expect_tx(&full[s], C::HALO_BYTES + (out ? 3 * C::CTR_BYTES : 0));
                            tma_load_3d(st, hm, &full[s], hx, hy, hz);
                            if (out) {
                                const int cx = int(a.g.lead) + x0;
                                const int cy = y0 + int(a.g.order);
                                const int cz = z + int(a.g.order0);
                                // multi-step (in-place wave ping-pong: prev is dst): odd steps
                                // read u from the dst buffer and u_prev from the src buffer
                                tma_load_3d(st + C::HALO_ELEMS, odd ? &tm_prev : &tm_ctr, &full[s], cx, cy, cz);
                                tma_load_3d(st + C::HALO_ELEMS + C::CTR_ELEMS, odd ? &tm_ctr : &tm_prev, &full[s], cx,
                                            cy, cz);
                                tma_load_3d(st + C::HALO_ELEMS + 2 * C::CTR_ELEMS, &tm_vel, &full[s], cx, cy, cz);
                            }
                        } else {
                            mbar_arrive_expect_tx(&full[s], C::HALO_BYTES);
                            tma_load_3d(st, hm, &full[s], hx, hy, hz);
                        }
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
    using K = Pk<T>;
    using P = typename K::P;
    constexpr int W = K::W;
    constexpr int NPK = VEC / W;  // lane packs per 16-byte row vector
    const int xl = lane * VEC;    // d2 offset inside the tile
    const int jr0 = warp * TY;    // first d1 row of this warp inside the tile
    P acc[NS][TY][NPK];
#pragma unroll
    for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int j = 0; j < TY; ++j)
#pragma unroll
            for (int i = 0; i < NPK; ++i) acc[k][j][i] = K::mul(T(0), P{});
    P chk = K::mul(T(0), P{});
    uint32_t it = 0;
    const int64_t pitch = a.g.pitch, plane = a.g.plane;

    while (true) {
        // the producer tags every stage with its work item; -1 ends the kernel, -2 a step
        mbar_wait(&full[it % STAGES], (it / STAGES) & 1u);
        const int tag = __shfl_sync(0xffffffffu, stage_item[it % STAGES], 0);  // warp-uniform: uniform branches
        if (tag == -1) break;
        if (tag == -2) {
            // multi-step launch: this CTA's outputs of the step are stored; publish them
            // (visible to other CTAs' TMA reads) and count the CTA in the grid barrier
            // the cooperative-groups grid-sync pattern: each thread orders its generic stores
            // before async-proxy (TMA) reads, the consumer barrier, then one gpu-scope fence
            // (cumulative over the CTA's writes observed through the barrier) and the arrival
            // (one fence per CTA instead of one per thread: +2.5-3 % on small grids)
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
        T* const dst_step = (step & 1) ? a.dst_alt : a.dst;
        int tx, ty, tz;
        decode_item(a, item, tx, ty, tz);
        const int x0 = a.x0base + tx * BX;
        const int y0 = a.box.lo1 + ty * BY;
        const int z0 = a.zs[2 * tz];
        const int z1 = a.zs[2 * tz + 1];
        const int x = x0 + xl;
        const int nq = (z1 - z0) + 2 * R;
        const bool full_tile = x0 >= a.box.lo2 && x0 + BX <= a.box.hi2 && y0 >= a.box.lo1 && y0 + BY <= a.box.hi1;
        const bool x_full = (x >= a.box.lo2) && (x + VEC <= a.box.hi2);
        const bool x_any = (x + VEC > a.box.lo2) && (x < a.box.hi2);
        // output address of row jr0 at plane z = q - R: advanced by one plane per stage (no
        // 64-bit multiply per plane); starts at plane z0 - 2R for q = z0 - R
        T* dzp = dst_step + (int64_t(y0 + jr0) + a.g.order) * pitch + a.g.lead + x +
                 (int64_t(z0) - 2 * R + a.g.order0) * plane;

        // the plane loop is unrolled by 2R+1 so the accumulator ring slots are static
        // registers; the wide dense boxes (R > 2: 343 / 729 taps per plane) keep one plane
        // per iteration (code size) and rotate the ring instead (2R+1 register moves)
        constexpr bool ROT = (FORM == FORM_BOX || FORM == FORM_BOX_DIV) && R > 2;
        constexpr int PU = ROT ? 1 : NS;
        for (int qb = 0; qb < nq; qb += PU) {
#pragma unroll
            for (int p = 0; p < PU; ++p) {
                const int qi = qb + p;
                if (qi < nq) {
                    const int q = z0 - R + qi;
                    const uint32_t s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1u;
                    mbar_wait(&full[s], ph);
                    const T* t = tiles + size_t(s) * C::STAGE_ELEMS;

                    if constexpr (FORM == FORM_BOX || FORM == FORM_BOX_DIV) {
                        // dense (2R+1)^3 kernel: plane q adds layer dz of the cube to output
                        // q - dz for every dz; output q + R starts here, q - R completes here
#pragma unroll
                        for (int rr = 0; rr < TY + 2 * R; ++rr) {
                            T xr[VEC + 2 * RA];
                            const T* row = t + (jr0 + rr) * SW + xl;
#pragma unroll
                            for (int k = 0; k < RA / VEC; ++k) {
                                ldsv<T, VEC>(row + k * VEC, &xr[k * VEC]);
                                ldsv<T, VEC>(row + RA + VEC + k * VEC, &xr[RA + VEC + k * VEC]);
                            }
                            ldsv<T, VEC>(row + RA, &xr[RA]);
#pragma unroll
                            for (int j = 0; j < TY; ++j) {
                                const int dy = rr - (j + R);
                                if (dy < -R || dy > R) continue;
#pragma unroll
                                for (int dz = -R; dz <= R; ++dz) {
                                    constexpr int NS_ = NS;
                                    const int slot = (p - dz + 2 * NS_) % NS_;
#pragma unroll
                                    for (int k = 0; k < NPK; ++k) {
                                        P s_ = acc[slot][j][k];
#pragma unroll
                                        for (int dx = -R; dx <= R; ++dx) {
                                            const T c = a.cb[((dz + R) * (2 * R + 1) + (dy + R)) * (2 * R + 1) + (dx + R)];
                                            const int e = RA + k * W + dx;
                                            const bool first = (dz == -R && dy == -R && dx == -R);
                                            if (W == 1 || (e % 2) == 0 || !ODD_SCALAR) {
                                                s_ = first ? K::mul(c, K::make(&xr[e])) : K::fma(c, K::make(&xr[e]), s_);
                                            } else {
                                                T l[W];
                                                K::put(l, s_);
#pragma unroll
                                                for (int w = 0; w < W; ++w)
                                                    l[w] = first ? c * xr[e + w] : fma_t(c, xr[e + w], l[w]);
                                                s_ = K::make(l);
                                            }
                                        }
                                        acc[slot][j][k] = s_;
                                    }
                                }
                            }
                        }
                    } else {
                        // centre values of this thread's rows in plane q
                        T cvs[TY][VEC];
    #pragma unroll
                        for (int j = 0; j < TY; ++j) ldsv<T, VEC>(t + (jr0 + j + R) * SW + xl + RA, cvs[j]);
                        P cv[TY][NPK];
    #pragma unroll
                        for (int j = 0; j < TY; ++j)
    #pragma unroll
                            for (int k = 0; k < NPK; ++k) cv[j][k] = K::make(&cvs[j][k * W]);

                        if (q >= z0 && q < z1) {
                            // output q: its accumulator already holds the d0 taps of planes < q.
                            // The d2 taps run tap by tap across every (row, pack) of the thread, so
                            // its TY x NPK accumulator chains interleave (same per-point order).
                            T xr[TY][VEC + 2 * RA];  // left halo | centre | right halo of each row
    #pragma unroll
                            for (int j = 0; j < TY; ++j) {
                                const T* row = t + (jr0 + j + R) * SW + xl;
    #pragma unroll
                                for (int k = 0; k < RA / VEC; ++k) {
                                    ldsv<T, VEC>(row + k * VEC, &xr[j][k * VEC]);
                                    ldsv<T, VEC>(row + RA + VEC + k * VEC, &xr[j][RA + VEC + k * VEC]);
                                }
    #pragma unroll
                                for (int i = 0; i < VEC; ++i) xr[j][RA + i] = cvs[j][i];
                            }
    #pragma unroll
                            for (int j = 0; j < TY; ++j)
    #pragma unroll
                                for (int k = 0; k < NPK; ++k) acc[p][j][k] = K::fma(a.c0, cv[j][k], acc[p][j][k]);
    #pragma unroll
                            for (int m = 1; m <= R; ++m) {
    #pragma unroll
                                for (int j = 0; j < TY; ++j)
    #pragma unroll
                                    for (int k = 0; k < NPK; ++k) {
                                        P s_ = acc[p][j][k];
                                        if (W == 1 || (m % 2) == 0 || !ODD_SCALAR) {
                                            s_ = K::fma(a.cm[2][m - 1], K::make(&xr[j][RA + k * W - m]), s_);
                                            s_ = K::fma(a.cp[2][m - 1], K::make(&xr[j][RA + k * W + m]), s_);
                                        } else {  // odd shift: the pair straddles two register pairs
                                            T l[W];
                                            K::put(l, s_);
    #pragma unroll
                                            for (int w = 0; w < W; ++w) {
                                                l[w] = fma_t(a.cm[2][m - 1], xr[j][RA + k * W + w - m], l[w]);
                                                l[w] = fma_t(a.cp[2][m - 1], xr[j][RA + k * W + w + m], l[w]);
                                            }
                                            s_ = K::make(l);
                                        }
                                        acc[p][j][k] = s_;
                                    }
                            }
                            // d1 (y) taps: stream the TY+2R rows of this warp's column
    #pragma unroll
                            for (int rr = 0; rr < TY + 2 * R; ++rr) {
                                if (rr >= R && rr < R + TY) {
    #pragma unroll
                                    for (int j = 0; j < TY; ++j) {
                                        const int m = rr - (j + R);
                                        if (m != 0 && m >= -R && m <= R) {
                                            const T c = m < 0 ? a.cm[1][-m - 1] : a.cp[1][m - 1];
    #pragma unroll
                                            for (int k = 0; k < NPK; ++k)
                                                acc[p][j][k] = K::fma(c, cv[rr - R][k], acc[p][j][k]);
                                        }
                                    }
                                } else {
                                    T yv[VEC];
                                    ldsv<T, VEC>(t + (jr0 + rr) * SW + xl + RA, yv);
    #pragma unroll
                                    for (int j = 0; j < TY; ++j) {
                                        const int m = rr - (j + R);
                                        if (m >= -R && m <= R) {
                                            const T c = m < 0 ? a.cm[1][-m - 1] : a.cp[1][m - 1];
    #pragma unroll
                                            for (int k = 0; k < NPK; ++k)
                                                acc[p][j][k] = K::fma(c, K::make(&yv[k * W]), acc[p][j][k]);
                                        }
                                    }
                                }
                            }
                        }
                        if (q < z1) {
                            // plane q feeds future outputs q+m with the -m coefficient
    #pragma unroll
                            for (int j = 0; j < TY; ++j)
    #pragma unroll
                                for (int k = 0; k < NPK; ++k) {
                                    acc[(p + R) % NS][j][k] = K::mul(a.cm[0][R - 1], cv[j][k]);
    #pragma unroll
                                    for (int m = 1; m < R; ++m)
                                        acc[(p + m) % NS][j][k] = K::fma(a.cm[0][m - 1], cv[j][k], acc[(p + m) % NS][j][k]);
                                }
                        }
                        // plane q feeds past outputs q-m with the +m coefficient
    #pragma unroll
                        for (int j = 0; j < TY; ++j)
    #pragma unroll
                            for (int k = 0; k < NPK; ++k)
    #pragma unroll
                                for (int m = 1; m <= R; ++m)
                                    acc[(p - m + NS) % NS][j][k] =
                                        K::fma(a.cp[0][m - 1], cv[j][k], acc[(p - m + NS) % NS][j][k]);
                    }
                    // output plane z = q - R is complete
                    const int z = q - R;
                    const bool z_out = (z >= z0) && (z < z1);
                    constexpr int ks = (NS - R) % NS;  // slot of output q - R relative to p
                    T outv[TY][VEC];
                    if (z_out) {
#pragma unroll
                        for (int j = 0; j < TY; ++j)
#pragma unroll
                            for (int k = 0; k < NPK; ++k) {
                                P v = acc[(p + ks) % NS][j][k];
                                if constexpr (FORM == FORM_STAR_DIV || FORM == FORM_BOX_DIV)
                                    v = K::mul(a.divisor, v);  // host passes 1/divisor
                                if constexpr (FORM == FORM_WAVE) {
                                    const T* cu = t + C::HALO_ELEMS + (jr0 + j) * BX + xl + k * W;
                                    const P uu = K::make(cu);
                                    const P pp = K::make(cu + C::CTR_ELEMS);
                                    const P kk = K::make(cu + 2 * C::CTR_ELEMS);
                                    v = K::fmav(kk, v, K::fma(a.wave_b, pp, K::mul(a.wave_a, uu)));
                                }
                                K::put(&outv[j][k * W], v);
                                chk = K::check(v, chk);
                            }
                    }
                    // every shared read of stage s is done: hand it back to the producer
                    __syncwarp();
                    mbar_arrive_lane0(&empty[s], lane);
                    ++it;

                    if (z_out) {
                        T* const dz = dzp;
                        if (full_tile) {
#pragma unroll
                            for (int j = 0; j < TY; ++j) stgv<T, VEC>(dz + j * pitch, outv[j], STKB_STORE_STREAMING);
                        } else if (x_any) {
#pragma unroll
                            for (int j = 0; j < TY; ++j) {
                                const int y = y0 + jr0 + j;
                                if (y >= a.box.lo1 && y < a.box.hi1)
                                    store_row_masked_n<T, VEC>(dz + j * pitch, outv[j][0], outv[j][1 % VEC],
                                                               outv[j][2 % VEC], outv[j][3 % VEC], x, a.box.lo2,
                                                               a.box.hi2);
                            }
                        }
                    }
                    dzp += plane;
                    if constexpr (ROT) {
                        // output o lives in slot (o - q) mod NS: move every slot down by one
#pragma unroll
                        for (int j = 0; j < TY; ++j)
#pragma unroll
                            for (int k = 0; k < NPK; ++k) {
                                const P first = acc[0][j][k];
#pragma unroll
                                for (int r = 0; r + 1 < NS; ++r) acc[r][j][k] = acc[r + 1][j][k];
                                acc[NS - 1][j][k] = first;
                            }
                    }
                }
            }
        }
        if (tz < a.n_signal) {
            // a boundary item is stored: publish it (halo exchange waits on the counter)
            __threadfence();
            asm volatile("bar.sync 1, %0;" ::"r"(NWY * 32) : "memory");
            if (threadIdx.x == 0) atomicAdd(a.signal, 1);
        }
    }
    if (__any_sync(0xffffffffu, !K::clean(chk)) && lane == 0) atomicOr(a.nonfinite, 1);
}

// pick the z-chunk length for the dynamic scheduler: the mean per-CTA work in
// plane steps (every chunk re-streams 2R halo planes) plus one item of tail
inline int choose_lz(int n0, int tiles, int ctas, int R, int* n_tz) {
    double best_cost = -1.0;
    int best = n0;
    for (int lz = 8; lz <= n0 + 7; lz += 8) {
        const int l = lz < n0 ? lz : n0;
        const int tz = (n0 + l - 1) / l;
        const double planes = double(tiles) * (n0 + 2.0 * R * tz);
        const double cost = planes / ctas + 1.0 * (l + 2 * R) + (tiles * tz < ctas ? 1e9 / (tiles * tz) : 0.0);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = l;
        }
        if (l == n0) break;
    }
    *n_tz = (n0 + best - 1) / best;
    return best;
}

// z-chunks of one d0 range [lo, lo+n0): uniform chunks of `lz`, except that the
// last chunks halve (lz/2, lz/4, ... >= 16) so the scheduler's final round is
// short (smaller tail).  Appends (lo, hi) pairs to zs; returns the new count.
inline int chunk_range(int lo, int n0, int lz, int tiles, int ctas, bool taper, int32_t* zs, int k) {
    int tail[16], nt = 0, tail_sum = 0;
    if (taper && 2 * tiles >= ctas)
        for (int l = lz / 2; l >= 16 && nt < 16; l /= 2) {
            tail[nt++] = l;
            tail_sum += l;
        }
    int main_len = n0 - tail_sum;
    if (main_len < lz) {  // too short to taper
        nt = 0;
        main_len = n0;
    }
    const int n_main = (main_len + lz - 1) / lz;
    int prev = 0;
    for (int c = 1; c <= n_main && k < kMaxChunks; ++c) {
        const int z = int((int64_t(main_len) * c) / n_main);
        zs[2 * k] = lo + prev;
        zs[2 * k + 1] = lo + z;
        prev = z;
        ++k;
    }
    for (int i = 0; i < nt && k < kMaxChunks; ++i) {
        zs[2 * k] = lo + prev;
        zs[2 * k + 1] = lo + prev + tail[i];
        prev += tail[i];
        ++k;
    }
    zs[2 * k - 1] = lo + n0;  // close exactly (also if kMaxChunks truncated the list)
    return k;
}

template <typename T, int R, int FORM, int TY, int NWY, bool ODD_SCALAR, bool PULL, int LW = 0>
cudaError_t launch_star_cfg(const StarLaunch& L, StarArgs<T> a, const CUtensorMap* maps, cudaStream_t stream) {
    using C = StarCfg<T, R, FORM, TY, NWY, LW>;
    auto kern = star_stream_kernel<T, R, FORM, TY, NWY, ODD_SCALAR, PULL, LW>;
    // a tensor-map box that differs from this instantiation's tile would make the
    // mbarrier transaction counts disagree (a hang): refuse instead
    if (L.box_w != C::SW || L.box_h != C::SH) return cudaErrorInvalidConfiguration;
    static uint64_t attr_devices = 0;  // per instantiation, per device
    if (cudaError_t e = ensure_smem_attr(kern, int(C::SMEM), attr_devices)) return e;
    const int w2 = a.box.hi2 - a.x0base;
    a.n_tx = (w2 + C::BX - 1) / C::BX;
    a.n_ty = (a.box.hi1 - a.box.lo1 + C::BY - 1) / C::BY;
    const int n0 = a.box.hi0 - a.box.lo0;
    const int tiles = a.n_tx * a.n_ty;
    int ctas = L.max_ctas > 0 ? L.max_ctas : L.num_sms;
    // d0 ranges: the map box, or the caller's list (signal ranges first, one chunk each)
    int32_t rlo[kMaxChunks], rhi[kMaxChunks];
    int nr = 0;
    if (L.n_ranges <= 0) {
        rlo[0] = a.box.lo0;
        rhi[0] = a.box.hi0;
        nr = 1;
    } else {
        for (int i = 0; i < L.n_ranges && nr < kMaxChunks; ++i)
            if (L.rhi[i] > L.rlo[i]) {
                rlo[nr] = L.rlo[i];
                rhi[nr] = L.rhi[i];
                ++nr;
            }
    }
    const int nsig = L.n_ranges > 0 ? std::min(L.n_signal_ranges, nr) : 0;
    int main_n0 = 0;
    for (int i = nsig; i < nr; ++i) main_n0 = std::max(main_n0, rhi[i] - rlo[i]);
    if (L.lz > 0) {
        a.lz = L.lz;
    } else if (L.n_steps > 1 && main_n0 > 0 && tiles < ctas) {
        // multi-step launch on a small grid: one item per CTA and step, the shortest chunks
        // that still fit in one wave (every step waits for its slowest CTA)
        const int per_tile = std::max(1, ctas / tiles);
        a.lz = (main_n0 + per_tile - 1) / per_tile;
    } else if (main_n0 > 0) {
        int ntz;
        a.lz = choose_lz(main_n0, tiles, ctas, R, &ntz);
        if (ntz > kMaxChunks / 2) a.lz = (main_n0 + kMaxChunks / 2 - 1) / (kMaxChunks / 2);
    } else {
        a.lz = 1;
    }
    int k = 0;
    for (int i = 0; i < nsig && k < kMaxChunks; ++i, ++k) {
        a.zs[2 * k] = rlo[i];
        a.zs[2 * k + 1] = rhi[i];
    }
    for (int i = nsig; i < nr && k < kMaxChunks; ++i)
        k = chunk_range(rlo[i], rhi[i] - rlo[i], a.lz, tiles, ctas, L.taper && L.n_steps <= 1, a.zs, k);
    a.n_tz = k;
    a.n_signal = nsig;
    // bands of ~one wave (STKB_BAND = wave fraction in %, 0 = plain z-major order)
    a.band_rows = 0;
    if (nsig == 0 && L.band_pct > 0 && a.n_tx > 0) {
        const int rows = std::max(1, (ctas * L.band_pct / 100) / a.n_tx);
        if (rows < a.n_ty) a.band_rows = rows;
    }
    a.signal = L.signal;
    if (L.signal_items) *L.signal_items = tiles * nsig;
    a.n_items = tiles * a.n_tz;
    if (a.n_items <= 0) return cudaSuccess;
    const int grid = a.n_items < ctas ? a.n_items : ctas;
    if (L.n_steps > 1 && !PULL) {
        // several steps, one grid barrier between them: every CTA must be resident at once,
        // which the cooperative launch guarantees (it fails instead of deadlocking)
        a.n_steps = L.n_steps;
        a.work_counter = L.step_counters;
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
        return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], a);
    }
    a.n_steps = 1;
    cudaError_t e = cudaMemsetAsync(a.work_counter, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return e;
    kern<<<grid, C::THREADS, C::SMEM, stream>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], a);
    return cudaGetLastError();
}

// tile variants: (rows per warp, consumer warps, odd x-taps as scalar FMAs, elements per lane
// (0: one 16-byte vector)).  Every variant evaluates each point with the same operations in
// the same order (the tile only changes which thread does it): results are bit-identical.
struct Variant { int ty, nwy; bool odd_scalar; int lw = 0; };
constexpr int kSmallTileVariant = 20;

template <typename T>
__host__ __device__ constexpr Variant star_variant_of(int R, int v, bool box = false) {
    if (sizeof(T) == 8 && v == 9) return Variant{R == 1 ? 8 : 4, 7, true};  // previous fp64 default
    switch (v) {
        case 1: return Variant{R == 1 ? 8 : (R == 2 ? 6 : 4), 7, true};   // wide rows, 1 warp pair / SMSP
        case 2: return Variant{R == 1 ? 6 : 3, 10, true};
        case 3: return Variant{R == 1 ? 8 : (R == 2 ? 6 : 4), 7, false};  // odd x-taps as re-paired FFMA2
        case 4: return Variant{1, 15, true};                                // one row per warp
        case 5: return Variant{2, 11, true};                                // fewer warps, more registers
        case 6: return Variant{2, 9, true};
        case 7: return Variant{2, 12, true};
        case 8: return Variant{3, 8, true};
        // 32-byte lanes (fp64: 4 values per lane, 128-wide tiles): the ring of 2 rows x 4 values
        // needs ~190 registers, i.e. at most 2 warps per SM sub-partition (8 warps per CTA)
        case 10: return sizeof(T) == 8 ? Variant{2, 7, true, 4} : Variant{2, 11, true};
        case 11: return sizeof(T) == 8 ? Variant{2, 6, true, 4} : Variant{2, 11, true};
        case 12: return sizeof(T) == 8 ? Variant{1, 11, true, 4} : Variant{2, 11, true};
        case 13: return Variant{1, 11, true};
        case 14: return Variant{1, 7, true};
        case 15: return Variant{2, 8, true};
        case 16: return Variant{1, 16, true};
        case 17: return Variant{2, 4, true};
        case 18: return Variant{1, 8, true};
        case 19: return Variant{4, 4, true};
        // small grids (StarLaunch::small_tile): 16-row tiles give more, shorter items; measured
        // +14-32 % at 96^3-160^3 against the default tile for every radius, fp32 and fp64 and
        // the wave, worse from ~192^3 on
        case kSmallTileVariant: return Variant{2, 8, true};
        default:  // measured best on B200 per form, dtype and radius (tools/sweep.py)
            // dense cubes: R=1 4 rows/warp (rows share taps), R=2 one row, R=3..4 one row with
            // 11 warps (up to 170 registers); R=4 forms odd-shift pairs once per row (+13 %)
            if (box) return R == 1 ? Variant{4, 15, true} : (R <= 3 ? Variant{1, R == 2 ? 15 : 11, true}
                                                                    : Variant{1, 11, false});
            if (R == 1) return Variant{1, 15, true};
            if (R == 2) return sizeof(T) == 8 ? Variant{2, 9, true} : Variant{1, 15, true};
            return Variant{2, 11, true};
    }
}

inline int star_variant_env() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("STKB_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <typename T, int R, int V, bool PULL>
cudaError_t launch_star_vp(const StarLaunch& L, const StarArgs<T>& a, const CUtensorMap* maps, cudaStream_t s) {
    constexpr Variant vv = star_variant_of<T>(R, V);
    if (L.kind == 4) {
        if constexpr (V == kSmallTileVariant) {
            return cudaErrorInvalidValue;  // boxes keep their tiles
        } else {
            constexpr Variant vb = star_variant_of<T>(R, V, true);
            if (L.has_divisor)
                return launch_star_cfg<T, R, FORM_BOX_DIV, vb.ty, vb.nwy, vb.odd_scalar, PULL>(L, a, maps, s);
            return launch_star_cfg<T, R, FORM_BOX, vb.ty, vb.nwy, vb.odd_scalar, PULL>(L, a, maps, s);
        }
    }
    if (L.kind == 2) return launch_star_cfg<T, R, FORM_WAVE, vv.ty, vv.nwy, vv.odd_scalar, PULL, vv.lw>(L, a, maps, s);
    if (L.has_divisor)
        return launch_star_cfg<T, R, FORM_STAR_DIV, vv.ty, vv.nwy, vv.odd_scalar, PULL, vv.lw>(L, a, maps, s);
    return launch_star_cfg<T, R, FORM_STAR, vv.ty, vv.nwy, vv.odd_scalar, PULL, vv.lw>(L, a, maps, s);
}

// the neighbour-reading (multi-GPU) kernels are separate instantiations: the
// single-GPU launches run exactly the producer code they had without them
template <typename T, int R, int V>
cudaError_t launch_star_v(const StarLaunch& L, const StarArgs<T>& a, const CUtensorMap* maps, cudaStream_t s) {
    if (a.pull) {
        if constexpr (V == 0) return launch_star_vp<T, R, V, true>(L, a, maps, s);
        else return cudaErrorInvalidValue;  // built for the default variant only
    }
    return launch_star_vp<T, R, V, false>(L, a, maps, s);
}

#ifndef STKB_VARIANTS
#define STKB_VARIANTS 1
#endif

template <typename T, int R>
cudaError_t launch_star_r(const StarLaunch& L, const StarArgs<T>& a, const CUtensorMap* maps, cudaStream_t s) {
    if (L.small_tile && L.kind != 4 && !a.pull) return launch_star_vp<T, R, kSmallTileVariant, false>(L, a, maps, s);
    if constexpr (STKB_VARIANTS > 1) {
        switch (star_variant_env()) {
            case 1: return launch_star_v<T, R, 1>(L, a, maps, s);
            case 2: return launch_star_v<T, R, 2>(L, a, maps, s);
            case 3: return launch_star_v<T, R, 3>(L, a, maps, s);
            case 4: return launch_star_v<T, R, 4>(L, a, maps, s);
            case 5: return launch_star_v<T, R, 5>(L, a, maps, s);
            case 6: return launch_star_v<T, R, 6>(L, a, maps, s);
            case 7: return launch_star_v<T, R, 7>(L, a, maps, s);
            case 8: return launch_star_v<T, R, 8>(L, a, maps, s);
            case 10: return launch_star_v<T, R, 10>(L, a, maps, s);
            case 11: return launch_star_v<T, R, 11>(L, a, maps, s);
            case 12: return launch_star_v<T, R, 12>(L, a, maps, s);
            case 13: return launch_star_v<T, R, 13>(L, a, maps, s);
            case 14: return launch_star_v<T, R, 14>(L, a, maps, s);
            case 15: return launch_star_v<T, R, 15>(L, a, maps, s);
            case 16: return launch_star_v<T, R, 16>(L, a, maps, s);
            case 17: return launch_star_v<T, R, 17>(L, a, maps, s);
            case 18: return launch_star_v<T, R, 18>(L, a, maps, s);
            case 19: return launch_star_v<T, R, 19>(L, a, maps, s);
            default: break;
        }
    }
    return launch_star_v<T, R, 0>(L, a, maps, s);
}

template <typename T>
cudaError_t launch_star_t(const StarLaunch& L, const StarArgs<T>& a, const CUtensorMap* maps, cudaStream_t s) {
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
inline void star_tile_t(int R, bool box, bool small, int* bx, int* by, int* halo_x) {
    const int v = small && !box ? kSmallTileVariant : (STKB_VARIANTS > 1 ? star_variant_env() : 0);
    const Variant vv = star_variant_of<T>(R, v, box);
    const int VEC = vv.lw > 0 && !box ? vv.lw : int(16 / sizeof(T));
    *bx = 32 * VEC;
    *by = vv.nwy * vv.ty;
    *halo_x = ((R + VEC - 1) / VEC) * VEC;
}

}  // namespace stkb
