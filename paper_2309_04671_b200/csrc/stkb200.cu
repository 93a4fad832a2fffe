// libstkb200: the C-ABI (include/stkb200.h) over the sm_100a kernels.
//
// A domain owns the pitched device copies of one target's grids, a stream, the
// TMA tensor maps of every buffer, and a step program (maps + swaps) that it
// replays through a CUDA graph.  The name -> buffer binding follows the
// reference's swap semantics (executor.py:229-230): a swap is free, it only
// exchanges which device buffer a grid name denotes.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/stkb200.h"
#include "common.cuh"

namespace stkb {
cudaError_t launch_expr(int dtype, const Geometry& g, const Box& box, const int32_t* code,
                        const double* consts, int n_code, int n_args, const void* const* rd,
                        void* const* wr, int32_t* flag, int num_sms, cudaStream_t s);
cudaError_t launch_compare(int dtype, const Geometry& g, const void* ref, const void* got, void* partials,
                           int blocks, cudaStream_t s);
size_t compare_partial_bytes();
cudaError_t launch_signal_add(int32_t* p, int32_t v, cudaStream_t s);
cudaError_t launch_repitch(void* stage, void* dev, int64_t r0, int64_t nrows, int64_t rows_per_plane,
                           int64_t row_bytes, int64_t row_pitch_bytes, int64_t plane_pitch_bytes, bool to_device,
                           int num_sms, cudaStream_t s);
// Star2DArgs: common.cuh
cudaError_t launch_tb2_f32(const StarLaunch& L, const StarArgs<float>& a, cudaStream_t s);
cudaError_t launch_tb2_f64(const StarLaunch& L, const StarArgs<double>& a, cudaStream_t s);
int tb2_tile(int dtype, int radius, int* box_w, int* box_h, int* v_w, int* v_h);
cudaError_t launch_frozen_ring(int dtype, const Geometry& g, const Box& b, int R, const void* buf, int32_t* flag,
                               int num_sms, cudaStream_t s, int zmask = 3);
cudaError_t launch_copy_halo(const void* src, void* dst, const Geometry& g, int esz, int num_sms, cudaStream_t s);
cudaError_t launch_star2d(int dtype, const Star2DArgs& a, int R, const void* src, void* dst, bool div, int num_sms,
                          cudaStream_t s);
}  // namespace stkb

using namespace stkb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    // a failed runtime call (e.g. cudaMalloc out of memory) also sets the thread's last error;
    // it is reported here, so clear it (non-sticky errors) lest a later launch check see it
    if (code == STKB_ERR_CUDA) (void)cudaGetLastError();
    return code;
}

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(STKB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr int kMaxTags = 64;
constexpr int kMaxMaps = 256;
constexpr int kMaxMultiSteps = 64;  // time steps per multi-step launch
constexpr int kFrozenFlag = kMaxTags + 2 * kMaxMaps;  // d_flags slot: v's frozen ring is not all zero
constexpr int kHaloFlag = kFrozenFlag + 4;            // per buffer: its halo may hold non-zero values
constexpr int kNumFlags = kHaloFlag + 40;

struct MapOp {
    stkb_map_desc d;
    int slot = 0;  // index of this map's scheduler counter
    std::vector<int32_t> code;
    std::vector<double> consts;
    int32_t* d_code = nullptr;
    double* d_consts = nullptr;
    bool snapshot[STKB_EXPR_MAX_ARGS] = {};  // EXPR: arg written and read -> read a copy
    std::vector<double> cube;                // BOX: the (2R+1)^3 coefficients (any R)
};

struct ProgOp {
    int kind;  // 0 = map, 1 = swap
    int map;
    int a, b;
};

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encoder() {
    if (g_encode) return STKB_OK;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
        return fail(STKB_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return STKB_OK;
}

}  // namespace

struct stkb_domain {
    stkb_domain_desc desc{};
    Geometry g{};
    size_t elem = 4;
    int num_sms = 148;
    std::vector<void*> bufs;
    std::vector<void*> snap;  // snapshot buffers for EXPR maps (lazily)
    std::vector<int32_t> binding;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<MapOp> maps;
    std::vector<ProgOp> prog;
    std::map<std::tuple<int, int, int>, CUtensorMap> tmaps;  // (buffer, box w, box h)
    // graph cache: start binding -> (exec of `period` steps, kernels per replay)
    std::map<std::vector<int32_t>, std::pair<cudaGraphExec_t, int64_t>> graphs;
    int gperiod = 0;
    bool warmed = false;  // one direct step ran since the program changed
    // timing
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool timed = false;
    int64_t last_launches = 0;
    int32_t last_mode = 0;  // how the last stkb_run executed: 0 single steps, 1 fused sweeps, 2 multi-step
    int32_t* d_flags = nullptr;
    void* d_partials = nullptr;
    void* d_stage = nullptr;  // H2D staging: contiguous PCIe copies, then a repitch kernel
    // z-slab neighbours for the fused halo exchange: [0] lower (rank-1), [1] upper (rank+1)
    struct Peer {
        bool set = false;
        std::vector<void*> bufs;  // the neighbour's buffer i (same binding history on every rank)
        std::map<std::tuple<int, int, int>, CUtensorMap> tmaps;  // (buffer, box w, box h) over bufs
        int32_t* flags = nullptr; // the neighbour's step flags ([0] from its lower, [1] from its upper)
        int64_t n0 = 0;           // the neighbour's slab thickness
    } peer[2];
    int32_t* d_peer_flags = nullptr;  // my step flags: [0] written by my lower, [1] by my upper neighbour
    size_t stage_bytes = 0;
    int lz_override = 0;
    int ctas_override = 0;
    int l2promo = 2;      // tensor-map L2 promotion (STKB_L2PROMO: 0 none, 1 64B, 2 128B (measured best), 3 256B)
    int store_hint = 0;   // STKB_STORE_HINT: 0 default, 1 streaming (.cs) stores
    bool taper = true;    // STKB_TAPER=0 disables the shortened final z-chunks
    int order_y_fast = 0; // STKB_ORDER_Y=1: work items walk y tiles fastest
    bool prescale = false; // STKB_PRESCALE=1: fold a Jacobi divisor into the coefficients (fill_coefs)
    int band_pct = 100;   // STKB_BAND: item order in tile-row bands of this % of a wave (0: z-major; StarArgs::band_rows)
    // two time steps per sweep (star_tb.cuh) for the Jacobi ping-pong of a radius <= 2 star:
    // u(t+2) goes to a scratch buffer bufs[scratch] and u's binding rotates with it
    bool tb = true;                // STKB_TB=0 disables
    int scratch = -1;              // index of the scratch buffer in bufs (allocated on first use)
    bool tb_warmed = false;
    int64_t ext_writes = 0;        // bumped by every API that hands out or writes buffer memory
    int64_t tb_pair_epoch = -1;    // ext_writes when bufs[tb_pair[0]] / [1] last had equal frozen parts
    int tb_pair[2] = {-1, -1};
    std::map<std::pair<int, int>, cudaGraphExec_t> tb_graphs;  // (u buffer, scratch) -> 2 fused passes
    // halo flags (d_flags[kHaloFlag + buffer]): 0 = that buffer's halo is all +0, so its stencil
    // reads go through an interior-only tensor map; recomputed when ext_writes moved
    int64_t halo_epoch = 0;
    // several ping-pong steps per launch for small grids (star_kernels.cuh, StarArgs::n_steps)
    int32_t* d_multi = nullptr;    // per-step work counters + the step-arrive counter
    cudaError_t last_launch_error = cudaSuccess;
    int64_t small_tile_points = int64_t(1) << 22;  // STKB_SMALL_TILE_POINTS: the small-grid tile up to here
    int64_t multi_max_points = int64_t(1) << 25;  // STKB_MULTI_POINTS: grids up to this many points
    bool multi = true;             // STKB_MULTI=0 disables
    bool halo_external = false;  // z-slab machinery writes halo planes (exchange, peers): full maps only
    std::map<std::tuple<int, int, int>, CUtensorMap> tmaps_int;  // (buffer, box w, box h), interior only
};

namespace {

// Step flags carry "launch v completed" as the bit pair {v mod 3, (v-1) mod 3}.  A
// neighbour's completed count k stays within [c-2, c] while I wait to start launch c
// (each launch waits for both neighbours' previous one), so the bit (c-1) mod 3 is set
// exactly when k >= c-1.  The values a stream writes and waits for then repeat every
// three launches, which lets a captured CUDA graph of the slab step be replayed.
int32_t peer_mask(int32_t v) {
    const int a = ((v % 3) + 3) % 3, b = (a + 2) % 3;
    return (1 << a) | (1 << b);
}

// a 3-D tiled tensor map over one pitched grid buffer of `n0` interior planes
int encode_tmap(stkb_domain* dom, void* base, int64_t n0, int bw, int bh, CUtensorMap* m) {
    int rc = get_encoder();
    if (rc) return rc;
    const Geometry& g = dom->g;
    cuuint64_t dims[3] = {cuuint64_t(g.pitch), cuuint64_t(g.n1 + 2 * g.order), cuuint64_t(n0 + 2 * g.order0)};
    cuuint64_t strides[2] = {cuuint64_t(g.pitch * dom->elem), cuuint64_t(g.plane * dom->elem)};
    cuuint32_t box[3] = {cuuint32_t(bw), cuuint32_t(bh), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    static const CUtensorMapL2promotion promo[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    CUresult r = g_encode(m, dom->elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                          3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, promo[dom->l2promo & 3],
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(STKB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return STKB_OK;
}

// the same box over the interior only (origin at interior (0,0,0), extents n2 x n1 x n0):
// the TMA zero-fills every coordinate in the halo instead of reading it
int encode_map_int(stkb_domain* dom, int buffer, int bw, int bh, const CUtensorMap** out) {
    auto key = std::make_tuple(buffer, bw, bh);
    auto it = dom->tmaps_int.find(key);
    if (it != dom->tmaps_int.end()) {
        *out = &it->second;
        return STKB_OK;
    }
    int rc = get_encoder();
    if (rc) return rc;
    const Geometry& g = dom->g;
    char* base = static_cast<char*>(dom->bufs[buffer]) + size_t(g.at(0, 0, 0)) * dom->elem;  // 128-B aligned
    cuuint64_t dims[3] = {cuuint64_t(g.n2), cuuint64_t(g.n1), cuuint64_t(g.n0)};
    cuuint64_t strides[2] = {cuuint64_t(g.pitch * dom->elem), cuuint64_t(g.plane * dom->elem)};
    cuuint32_t box[3] = {cuuint32_t(bw), cuuint32_t(bh), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    static const CUtensorMapL2promotion promo[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    CUtensorMap m;
    CUresult r = g_encode(&m, dom->elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                          3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, promo[dom->l2promo & 3], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(STKB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    auto res = dom->tmaps_int.emplace(key, m);
    *out = &res.first->second;
    return STKB_OK;
}

int encode_map(stkb_domain* dom, int buffer, int bw, int bh, const CUtensorMap** out) {
    auto key = std::make_tuple(buffer, bw, bh);
    auto it = dom->tmaps.find(key);
    if (it != dom->tmaps.end()) {
        *out = &it->second;
        return STKB_OK;
    }
    CUtensorMap m;
    int rc = encode_tmap(dom, dom->bufs[buffer], dom->g.n0, bw, bh, &m);
    if (rc) return rc;
    auto res = dom->tmaps.emplace(key, m);
    *out = &res.first->second;
    return STKB_OK;
}

// the same box over a z-neighbour's buffer (peer memory: TMA reads it over NVLink)
int encode_peer_map(stkb_domain* dom, int side, int buffer, int bw, int bh, const CUtensorMap** out) {
    auto& p = dom->peer[side];
    auto key = std::make_tuple(buffer, bw, bh);
    auto it = p.tmaps.find(key);
    if (it != p.tmaps.end()) {
        *out = &it->second;
        return STKB_OK;
    }
    CUtensorMap m;
    int rc = encode_tmap(dom, p.bufs[buffer], p.n0, bw, bh, &m);
    if (rc) return rc;
    auto res = p.tmaps.emplace(key, m);
    *out = &res.first->second;
    return STKB_OK;
}

// a buffer's halo flag := "may be non-zero" (its memory was handed out or written from
// outside); the next ensure_halo_flags recomputes it
void mark_halo_dirty(stkb_domain* dom, int buffer) {
    ++dom->ext_writes;
    const int n = int(dom->bufs.size());
    for (int b = buffer < 0 ? 0 : buffer; b < (buffer < 0 ? n : buffer + 1); ++b)
        cudaMemsetAsync(dom->d_flags + kHaloFlag + b, 0x01, sizeof(int32_t), dom->stream);
}

// recompute every buffer's halo flag after outside writes (not while the stream is being
// captured: the flags then stay conservative, "may be non-zero")
int ensure_halo_flags(stkb_domain* dom) {
    if (dom->desc.ndim != 3 || dom->halo_external || dom->halo_epoch == dom->ext_writes) return STKB_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(dom->stream, &cs));
    if (cs != cudaStreamCaptureStatusNone) return STKB_OK;
    const Geometry& g = dom->g;
    const Box inner{0, int32_t(g.n0), 0, int32_t(g.n1), 0, int32_t(g.n2)};
    // a z-slab side with a fused-exchange neighbour never reads its own halo planes (the
    // pulling kernels fetch those planes from the neighbour): leave that face out
    const int zmask = (dom->peer[0].set ? 0 : 1) | (dom->peer[1].set ? 0 : 2);
    for (size_t b = 0; b < dom->bufs.size(); ++b)
        CUDA_TRY(launch_frozen_ring(dom->desc.dtype, g, inner, int(g.order), dom->bufs[b],
                                    dom->d_flags + kHaloFlag + b, dom->num_sms, dom->stream, zmask));
    dom->halo_epoch = dom->ext_writes;
    return STKB_OK;
}

// star coefficients into the kernel arguments.  A divisor (Jacobi `/d`) is either applied
// by the kernel as a multiply by 1/d after the sum (returns true), or — `prescale` — folded
// into the coefficients on the host in float64 (returns false: one multiply less per point;
// same tolerance, different rounding)
template <typename T>
bool fill_coefs(StarArgs<T>& a, const stkb_map_desc& d, bool prescale) {
    const int R = d.radius;
    const bool fold = prescale && d.divisor != 0.0;
    const double sc = fold ? 1.0 / d.divisor : 1.0;
    a.c0 = T(d.coef[0] * sc);
    for (int ax = 0; ax < 3; ++ax)
        for (int m = 1; m <= 4; ++m) {
            a.cm[ax][m - 1] = m <= R ? T(d.coef[1 + ax * 2 * R + 2 * (m - 1)] * sc) : T(0);
            a.cp[ax][m - 1] = m <= R ? T(d.coef[1 + ax * 2 * R + 2 * (m - 1) + 1] * sc) : T(0);
        }
    a.divisor = d.divisor != 0.0 && !fold ? T(1.0 / d.divisor) : T(0);  // the kernel multiplies by it
    return d.divisor != 0.0 && !fold;
}

Box box_of(const stkb_map_desc& d) {
    Box b;
    b.lo0 = int32_t(d.lo[0]); b.hi0 = int32_t(d.hi[0]);
    b.lo1 = int32_t(d.lo[1]); b.hi1 = int32_t(d.hi[1]);
    b.lo2 = int32_t(d.lo[2]); b.hi2 = int32_t(d.hi[2]);
    return b;
}

// 2-D star maps: the 1.5-D streaming kernel (d0 streamed, d1 on lanes)
int launch_star2d_map(stkb_domain* dom, const MapOp& op, const std::vector<int32_t>& bind) {
    const stkb_map_desc& d = op.d;
    Star2DArgs a{};
    a.pitch = dom->g.pitch;
    a.lead = dom->g.lead;
    a.order = int32_t(dom->g.order);
    a.lo0 = int32_t(d.lo[1]); a.hi0 = int32_t(d.hi[1]);  // lifted: d0 of the 2-D grid is the row axis
    a.lo1 = int32_t(d.lo[2]); a.hi1 = int32_t(d.hi[2]);
    a.nonfinite = dom->d_flags + (d.tag & (kMaxTags - 1));
    const int R = d.radius;
    a.c0 = d.coef[0];
    for (int m = 1; m <= 4; ++m) {
        a.cm0[m - 1] = m <= R ? d.coef[1 + 2 * (m - 1)] : 0.0;
        a.cp0[m - 1] = m <= R ? d.coef[1 + 2 * (m - 1) + 1] : 0.0;
        a.cm1[m - 1] = m <= R ? d.coef[1 + 2 * R + 2 * (m - 1)] : 0.0;
        a.cp1[m - 1] = m <= R ? d.coef[1 + 2 * R + 2 * (m - 1) + 1] : 0.0;
    }
    a.rdiv = d.divisor != 0.0 ? 1.0 / d.divisor : 0.0;
    if (d.kind == STKB_MAP_BOX) {
        a.box = 1;
        for (int i = 0; i < (2 * R + 1) * (2 * R + 1); ++i) a.cb[i] = d.box_coef[i];
    }
    cudaError_t e = launch_star2d(dom->desc.dtype, a, R, dom->bufs[bind[d.src]], dom->bufs[bind[d.dst]],
                                  d.divisor != 0.0, dom->num_sms, dom->stream);
    if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("2-D star kernel launch: ") + cudaGetErrorString(e));
    return STKB_OK;
}

struct RangeSpec {
    int n = 0;
    const int32_t* lo = nullptr;
    const int32_t* hi = nullptr;
    int n_signal = 0;
    int* signal_items = nullptr;
};

template <typename T>
int launch_star_map(stkb_domain* dom, const MapOp& op, const std::vector<int32_t>& bind,
                    const RangeSpec& rs = RangeSpec(), bool pull = false, int n_steps = 1) {
    const stkb_map_desc& d = op.d;
    const bool exact2d = dom->desc.ndim == 2 && (d.kind == STKB_MAP_XSTAR || d.kind == STKB_MAP_XBOX);
    if (dom->desc.ndim == 2 && !exact2d) return launch_star2d_map(dom, op, bind);
    if (int rc = ensure_halo_flags(dom)) return rc;
    StarArgs<T> a{};
    a.g = dom->g;
    a.box = box_of(d);
    constexpr int VEC = 16 / sizeof(T);
    a.x0base = a.box.lo2 - (a.box.lo2 % VEC);
    const int sb = bind[d.src];
    a.dst = static_cast<T*>(dom->bufs[bind[d.dst]]);
    a.src = static_cast<const T*>(dom->bufs[sb]);
    a.prev = d.prev >= 0 ? static_cast<const T*>(dom->bufs[bind[d.prev]]) : nullptr;
    a.vel = d.vel >= 0 ? static_cast<const T*>(dom->bufs[bind[d.vel]]) : nullptr;
    a.nonfinite = dom->d_flags + (d.tag & (kMaxTags - 1));
    a.work_counter = dom->d_flags + kMaxTags + op.slot;
    const int R = d.radius;
    const bool div = fill_coefs(a, d, dom->prescale);
    a.wave_a = T(d.wave_a);
    a.wave_b = T(d.wave_b);
    a.store_hint = dom->store_hint;
    a.order_y_fast = dom->order_y_fast;
    if (d.kind == STKB_MAP_BOX) {
        const double sc = div || d.divisor == 0.0 ? 1.0 : 1.0 / d.divisor;  // prescaled: fold 1/d in
        for (size_t i = 0; i < op.cube.size(); ++i) a.cb[i] = T(op.cube[i] * sc);
    }

    // small grids take the 16-row tile (more, shorter work items); the neighbour-pulling and
    // range launches of the slab engine keep the default tile
    const bool small = !pull && rs.n == 0 && (d.kind == STKB_MAP_STAR || d.kind == STKB_MAP_WAVE) &&
                       dom->g.n0 * dom->g.n1 * dom->g.n2 <= dom->small_tile_points;
    int bx, by, hx;
    if (d.kind == STKB_MAP_XBOX)
        xbox_tile(dom->desc.dtype, R, exact2d, &bx, &by, &hx);
    else if (d.kind == STKB_MAP_XSTAR || d.kind == STKB_MAP_XWAVE)
        exact_tile(dom->desc.dtype, R, d.kind == STKB_MAP_XWAVE, &bx, &by, &hx);
    else star_tile(dom->desc.dtype, R, d.kind, small, &bx, &by, &hx);
    const CUtensorMap* m_halo = nullptr;
#ifdef STKB_EXP_NOYHALO
    const int lw = bx + 2 * hx, lh = by;
#elif defined(STKB_EXP_NOXHALO)
    const int lw = bx, lh = by + 2 * R;
#else
    const int lw = bx + 2 * hx, lh = by + 2 * R;
#endif
    int rc = encode_map(dom, sb, lw, lh, &m_halo);
    if (rc) return rc;
    CUtensorMap maps[7];
    for (int i = 0; i < 6; ++i) maps[i] = *m_halo;
    if (dom->desc.ndim == 3) {
        const CUtensorMap* m_int = nullptr;
        if ((rc = encode_map_int(dom, sb, lw, lh, &m_int))) return rc;
        maps[6] = *m_int;
        a.halo_nz = dom->halo_external ? nullptr : dom->d_flags + kHaloFlag + sb;
    } else {
        maps[6] = *m_halo;
    }
    if (pull) {
        // src planes beyond this slab come straight from the neighbours' buffers
        for (int side = 0; side < 2; ++side) {
            if (!dom->peer[side].set) continue;
            const CUtensorMap* pm;
            if ((rc = encode_peer_map(dom, side, sb, bx + 2 * hx, by + 2 * R, &pm))) return rc;
            maps[4 + side] = *pm;
            a.pull |= 1 << side;
        }
        a.pull_lo_n0 = int32_t(dom->peer[0].n0);
    }
    if (n_steps > 1) {
        // multi-step ping-pong: odd steps read the dst buffer (maps 4 / 5) and write src's
        const int db = bind[d.dst];
        const CUtensorMap *m_alt = nullptr, *m_alt_int = nullptr;
        if ((rc = encode_map(dom, db, lw, lh, &m_alt))) return rc;
        maps[4] = *m_alt;
        a.dst_alt = static_cast<T*>(dom->bufs[sb]);
        if (dom->desc.ndim == 3) {
            if ((rc = encode_map_int(dom, db, lw, lh, &m_alt_int))) return rc;
            maps[5] = *m_alt_int;
            a.halo_nz_alt = dom->halo_external ? nullptr : dom->d_flags + kHaloFlag + db;
        } else {  // 2-D (exact one-plane mode): halo flags are 3-D only; always the full map
            maps[5] = *m_alt;
            a.halo_nz_alt = nullptr;
        }
    }
    if (d.kind == STKB_MAP_WAVE) {
        const CUtensorMap *mc, *mp, *mv;
        if ((rc = encode_map(dom, sb, bx, by, &mc))) return rc;
        if ((rc = encode_map(dom, bind[d.prev], bx, by, &mp))) return rc;
        if ((rc = encode_map(dom, bind[d.vel], bx, by, &mv))) return rc;
        maps[1] = *mc;
        maps[2] = *mp;
        maps[3] = *mv;
    }
    StarLaunch L{};
    L.kind = d.kind;
    L.radius = R;
    L.has_divisor = div;
    L.maps = maps;
    L.box_w = bx + 2 * hx;
    L.box_h = by + 2 * R;  // (STKB_EXP_NOYHALO loads fewer rows; the stage keeps this shape)
    L.num_sms = dom->num_sms;
    L.two_d = exact2d;
    L.small_tile = small;
    L.max_ctas = dom->ctas_override;
    L.lz = dom->lz_override;
    L.taper = dom->taper;
    L.band_pct = dom->band_pct;
    L.n_ranges = rs.n;
    L.rlo = rs.lo;
    L.rhi = rs.hi;
    L.n_signal_ranges = rs.n_signal;
    L.signal = dom->d_flags + kMaxTags + kMaxMaps + op.slot;
    L.signal_items = rs.signal_items;
    if (n_steps > 1) {
        if (!dom->d_multi && cudaMalloc(&dom->d_multi, (kMaxMultiSteps + 1) * sizeof(int32_t)) != cudaSuccess)
            return fail(STKB_ERR_CUDA, "multi-step counters");
        L.n_steps = n_steps;
        L.step_counters = dom->d_multi;
    }
    cudaError_t e;
    if (d.kind == STKB_MAP_XWAVE) {
        if (rs.n > 0 || pull || (n_steps > 1 && d.prev != d.dst))
            return fail(STKB_ERR_UNSUPPORTED, "exact wave maps launch over their box");
        XwaveCoef xc{};
        xc.a = d.wave_a;
        xc.c0 = d.coef[0];
        for (int m = 1; m <= R; ++m) xc.l[m - 1] = d.coef[m];
        if constexpr (sizeof(T) == 4) e = launch_xwave_f32(L, a, xc, dom->stream);
        else e = launch_xwave_f64(L, a, xc, dom->stream);
    } else if (d.kind == STKB_MAP_XBOX) {
        if (rs.n > 0 || pull) return fail(STKB_ERR_UNSUPPORTED, "exact box maps launch over their box");
        XboxCoef xc{};
        for (size_t i = 0; i < op.cube.size() && i < 729; ++i) xc.c[i] = op.cube[i];
        xc.divisor = d.divisor;
        const double ad = std::fabs(d.divisor);
        xc.recip = ad >= 0x1p-64 && ad <= 0x1p64 ? 1.0 / d.divisor : 0.0;
        if constexpr (sizeof(T) == 4) e = launch_xbox_f32(L, a, xc, dom->stream);
        else e = launch_xbox_f64(L, a, xc, dom->stream);
    } else if (d.kind == STKB_MAP_XSTAR) {
        if (rs.n > 0 || pull) return fail(STKB_ERR_UNSUPPORTED, "exact star maps launch over their box");
        XstarCoef xc{};
        xc.c0 = d.coef[0];
        // a 2-D star's axes (d0, d1 of the grid) are the lifted plane's d1, d2
        const int nax = exact2d ? 2 : 3, ax0 = exact2d ? 1 : 0;
        for (int ax = 0; ax < nax; ++ax)
            for (int m = 1; m <= R; ++m) {
                xc.cm[ax0 + ax][m - 1] = d.coef[1 + ax * 2 * R + 2 * (m - 1)];
                xc.cp[ax0 + ax][m - 1] = d.coef[1 + ax * 2 * R + 2 * (m - 1) + 1];
            }
        xc.divisor = d.divisor;
        const double ad = std::fabs(d.divisor);
        xc.recip = ad >= 0x1p-64 && ad <= 0x1p64 ? 1.0 / d.divisor : 0.0;  // correctly rounded (host IEEE)
        if constexpr (sizeof(T) == 4) e = launch_exact_f32(L, a, xc, dom->stream);
        else e = launch_exact_f64(L, a, xc, dom->stream);
    } else if constexpr (sizeof(T) == 4) {
        e = launch_star_f32(L, a, dom->stream);
    } else {
        e = launch_star_f64(L, a, dom->stream);
    }
    dom->last_launch_error = e;
    if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("star kernel launch: ") + cudaGetErrorString(e));
    return STKB_OK;
}

int launch_expr_map(stkb_domain* dom, MapOp& op, const std::vector<int32_t>& bind) {
    const stkb_map_desc& d = op.d;
    const void* rd[STKB_EXPR_MAX_ARGS];
    void* wr[STKB_EXPR_MAX_ARGS];
    const size_t bytes = size_t(dom->g.plane) * size_t(dom->g.n0 + 2 * dom->g.order0) * dom->elem;
    for (int i = 0; i < d.n_args; ++i) {
        void* b = dom->bufs[bind[d.args[i]]];
        wr[i] = b;
        rd[i] = b;
        if (op.snapshot[i]) {
            // the oracle snapshots every grid before a map (executor.py:66-69)
            CUDA_TRY(cudaMemcpyAsync(dom->snap[i], b, bytes, cudaMemcpyDeviceToDevice, dom->stream));
            rd[i] = dom->snap[i];
        }
    }
    cudaError_t e = launch_expr(dom->desc.dtype, dom->g, box_of(d), op.d_code, op.d_consts, int(op.code.size() / 5),
                                d.n_args, rd, wr, dom->d_flags + (d.tag & (kMaxTags - 1)), dom->num_sms,
                                dom->stream);
    if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("expr kernel launch: ") + cudaGetErrorString(e));
    return STKB_OK;
}

// enqueue one step of the program starting from `bind`; updates `bind`
int enqueue_step(stkb_domain* dom, std::vector<int32_t>& bind, int64_t* launches) {
    for (const ProgOp& p : dom->prog) {
        if (p.kind == 1) {
            std::swap(bind[p.a], bind[p.b]);
            continue;
        }
        MapOp& op = dom->maps[p.map];
        int rc;
        if (op.d.kind == STKB_MAP_EXPR) rc = launch_expr_map(dom, op, bind);
        else if (dom->desc.dtype == STKB_F32) rc = launch_star_map<float>(dom, op, bind);
        else rc = launch_star_map<double>(dom, op, bind);
        if (rc) return rc;
        ++*launches;
    }
    return STKB_OK;
}

void invalidate_graph(stkb_domain* dom) {
    for (auto& kv : dom->graphs) cudaGraphExecDestroy(kv.second.first);
    dom->graphs.clear();
    for (auto& kv : dom->tb_graphs) cudaGraphExecDestroy(kv.second);
    dom->tb_graphs.clear();
    dom->tb_warmed = false;
    // a new program may write u or the scratch outside the fused map's box: the pair no
    // longer agrees there
    dom->tb_pair_epoch = -1;
    dom->gperiod = 0;
    dom->warmed = false;
}

// period of the binding permutation induced by one step
int binding_period(const stkb_domain* dom) {
    std::vector<int32_t> b(dom->binding.size());
    for (size_t i = 0; i < b.size(); ++i) b[i] = int32_t(i);
    std::vector<int32_t> cur = b;
    for (int k = 1; k <= 16; ++k) {
        for (const ProgOp& p : dom->prog)
            if (p.kind == 1) std::swap(cur[p.a], cur[p.b]);
        if (cur == b) return k;
    }
    return 0;
}

// The step program is `v = S(u); swap(u, v)` (either swap order) with S a fast 3-D
// STAR map of radius <= 2: two steps can run as one fused sweep.  Returns the map.
const MapOp* tb_map(const stkb_domain* dom) {
    if (!dom->tb || dom->desc.ndim != 3 || dom->prog.size() != 2) return nullptr;
    const ProgOp& m = dom->prog[0];
    const ProgOp& w = dom->prog[1];
    if (m.kind != 0 || w.kind != 1) return nullptr;
    const MapOp& op = dom->maps[m.map];
    const stkb_map_desc& d = op.d;
    // radius 1 only: at radius 2 the v rows each warp recomputes (TY2 + 4 for TY2 outputs
    // within the register budget) cost more than the halved HBM traffic saves (measured)
    if (d.kind != STKB_MAP_STAR || d.radius != 1 || d.precision != STKB_PREC_FAST) return nullptr;
    if (!((w.a == d.src && w.b == d.dst) || (w.a == d.dst && w.b == d.src))) return nullptr;
    if (d.lo[0] >= d.hi[0] || d.lo[1] >= d.hi[1] || d.lo[2] >= d.hi[2]) return nullptr;
    return &op;
}

// The step program is `v = S(u); swap(u, v)` with S a fast 3-D STAR map on a small grid
// (at most multi_max_points interior points: a step is a few microseconds, so launch
// and pipeline start-up dominate): several steps run per launch, separated by a grid
// barrier inside the kernel (StarArgs::n_steps).  Per point the arithmetic is the
// single-step kernel's, so every grid ends bit-identical to single steps.
const MapOp* multi_map(const stkb_domain* dom) {
    if (!dom->multi || dom->desc.ndim == 1 || dom->prog.size() != 2 || dom->halo_external) return nullptr;
    if (dom->g.n0 * dom->g.n1 * dom->g.n2 > dom->multi_max_points) return nullptr;
    const ProgOp& m = dom->prog[0];
    const ProgOp& w = dom->prog[1];
    if (m.kind != 0 || w.kind != 1) return nullptr;
    const MapOp& op = dom->maps[m.map];
    const stkb_map_desc& d = op.d;
    // fast stars, boxes and the in-place wave, and the exact star (the same streaming structure
    // and multi-step protocol; the wave's odd steps swap its u / u_prev centre maps)
    const bool wave_ok = (d.kind == STKB_MAP_WAVE || d.kind == STKB_MAP_XWAVE) && d.prev == d.dst;
    // 2-D grids: the exact kernels' one-plane mode (the fast 2-D kernel keeps single steps)
    if (dom->desc.ndim == 2 && d.kind != STKB_MAP_XSTAR && d.kind != STKB_MAP_XBOX) return nullptr;
    if ((d.kind != STKB_MAP_STAR && d.kind != STKB_MAP_BOX && d.kind != STKB_MAP_XSTAR && d.kind != STKB_MAP_XBOX &&
         !wave_ok) ||
        d.precision != STKB_PREC_FAST)
        return nullptr;
    if (!((w.a == d.src && w.b == d.dst) || (w.a == d.dst && w.b == d.src))) return nullptr;
    if (d.lo[0] >= d.hi[0] || d.lo[1] >= d.hi[1] || d.lo[2] >= d.hi[2]) return nullptr;
    return &op;
}

// one fused sweep: u(t+2) = S(S(u(t))) from bufs[binding[u]] into bufs[scratch]; v's buffer
// supplies the values outside the region box; then u's binding and the scratch swap
template <typename T>
int launch_tb2_map(stkb_domain* dom, const MapOp& op) {
    const stkb_map_desc& d = op.d;
    const int ub = dom->binding[d.src], vb = dom->binding[d.dst];
    StarArgs<T> a{};
    a.g = dom->g;
    a.box = box_of(d);
    constexpr int VEC = 16 / sizeof(T);
    a.x0base = a.box.lo2 - (a.box.lo2 % VEC);
    a.dst = static_cast<T*>(dom->bufs[dom->scratch]);
    a.src = static_cast<const T*>(dom->bufs[ub]);
    a.prev = static_cast<const T*>(dom->bufs[vb]);
    a.nonfinite = dom->d_flags + (d.tag & (kMaxTags - 1));
    a.work_counter = dom->d_flags + kMaxTags + op.slot;
    const int R = d.radius;
    const bool div = fill_coefs(a, d, dom->prescale);
    int bw, bh, vw, vh;
    if (tb2_tile(dom->desc.dtype, R, &bw, &bh, &vw, &vh)) return fail(STKB_ERR_UNSUPPORTED, "fused sweep radius");
    const CUtensorMap *m_halo = nullptr, *m_v = nullptr;
    if (int rc = encode_map(dom, ub, bw, bh, &m_halo)) return rc;
    if (int rc = encode_map(dom, vb, vw, vh, &m_v)) return rc;
    const CUtensorMap* m_int = nullptr;
    if (int rc = encode_map_int(dom, ub, bw, bh, &m_int)) return rc;
    a.halo_nz = dom->halo_external ? nullptr : dom->d_flags + kHaloFlag + ub;
    CUtensorMap maps[3] = {*m_halo, *m_v, *m_int};
    StarLaunch L{};
    L.kind = d.kind;
    L.radius = R;
    L.has_divisor = div;
    L.maps = maps;
    L.band_pct = dom->band_pct;
    L.frozen_nz = dom->d_flags + kFrozenFlag;
    L.box_w = bw;
    L.box_h = bh;
    L.num_sms = dom->num_sms;
    L.max_ctas = dom->ctas_override;
    L.lz = dom->lz_override;
    L.taper = dom->taper;
    cudaError_t e;
    if constexpr (sizeof(T) == 4) e = launch_tb2_f32(L, a, dom->stream);
    else e = launch_tb2_f64(L, a, dom->stream);
    if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("fused star kernel launch: ") + cudaGetErrorString(e));
    std::swap(dom->binding[d.src], dom->scratch);
    return STKB_OK;
}

int enqueue_tb2(stkb_domain* dom, const MapOp& op) {
    return dom->desc.dtype == STKB_F32 ? launch_tb2_map<float>(dom, op) : launch_tb2_map<double>(dom, op);
}

int check_name(const stkb_domain* dom, int32_t n, const char* what) {
    if (n < 0 || n >= dom->desc.n_grids) return fail(STKB_ERR_ARG, std::string(what) + ": grid name index out of range");
    return STKB_OK;
}

}  // namespace

extern "C" {

int stkb_abi_version(void) { return STKB_ABI_VERSION; }

const char* stkb_last_error(void) { return g_err.c_str(); }

int stkb_device_count(int32_t* count) {
    int n = 0;
    CUDA_TRY(cudaGetDeviceCount(&n));
    *count = n;
    return STKB_OK;
}

int stkb_domain_create(const stkb_domain_desc* desc, stkb_domain** out) {
    if (!desc || !out) return fail(STKB_ERR_ARG, "null argument");
    if (desc->dtype != STKB_F32 && desc->dtype != STKB_F64) return fail(STKB_ERR_ARG, "dtype must be STKB_F32 or STKB_F64");
    if (desc->ndim < 1 || desc->ndim > 3) return fail(STKB_ERR_UNSUPPORTED, "grids have 1 to 3 dimensions");
    if (desc->n_grids < 1 || desc->n_grids > 32) return fail(STKB_ERR_ARG, "n_grids must be in 1..32");
    if (desc->order < 0 || desc->order > 16) return fail(STKB_ERR_ARG, "order must be in 0..16");
    for (int d = 0; d < desc->ndim; ++d)
        if (desc->shape[d] < 1 || desc->shape[d] > (1 << 24)) return fail(STKB_ERR_ARG, "extent out of range");
    CUDA_TRY(cudaSetDevice(desc->device));
    auto* dom = new stkb_domain();
    dom->desc = *desc;
    dom->elem = desc->dtype == STKB_F32 ? 4 : 8;
    const int64_t per128 = 128 / int64_t(dom->elem);
    Geometry& g = dom->g;
    if (desc->ndim == 3) {
        g.n0 = desc->shape[0]; g.n1 = desc->shape[1]; g.n2 = desc->shape[2];
        g.order0 = desc->order;
    } else if (desc->ndim == 2) {  // 2-D grids are lifted to a single d0 plane without d0 halo
        g.n0 = 1; g.n1 = desc->shape[0]; g.n2 = desc->shape[1];
        g.order0 = 0;
    } else {  // 1-D grids: one row of one plane (the d1 halo rows stay zero and unread)
        g.n0 = 1; g.n1 = 1; g.n2 = desc->shape[0];
        g.order0 = 0;
    }
    g.order = desc->order;
    g.lead = std::max<int64_t>(per128, ((desc->order + per128 - 1) / per128) * per128);
    g.pitch = ((g.lead + g.n2 + g.order + per128 - 1) / per128) * per128;
    g.plane = g.pitch * (g.n1 + 2 * g.order);
    const size_t bytes = size_t(g.plane) * size_t(g.n0 + 2 * g.order0) * dom->elem;
    int dev = desc->device;
    cudaDeviceGetAttribute(&dom->num_sms, cudaDevAttrMultiProcessorCount, dev);
    dom->bufs.assign(desc->n_grids, nullptr);
    dom->snap.assign(STKB_EXPR_MAX_ARGS, nullptr);
    dom->binding.resize(desc->n_grids);
    for (int i = 0; i < desc->n_grids; ++i) dom->binding[i] = i;
    auto cleanup = [&](const std::string& msg) {
        stkb_domain_destroy(dom);
        return fail(STKB_ERR_CUDA, msg);
    };
    for (int i = 0; i < desc->n_grids; ++i) {
        cudaError_t e = cudaMalloc(&dom->bufs[i], bytes);
        if (e != cudaSuccess) return cleanup(std::string("cudaMalloc grid buffer: ") + cudaGetErrorString(e));
        e = cudaMemset(dom->bufs[i], 0, bytes);
        if (e != cudaSuccess) return cleanup(std::string("cudaMemset: ") + cudaGetErrorString(e));
    }
    if (cudaStreamCreateWithFlags(&dom->own_stream, cudaStreamNonBlocking) != cudaSuccess) return cleanup("stream");
    dom->stream = dom->own_stream;
    if (cudaEventCreate(&dom->ev0) != cudaSuccess || cudaEventCreate(&dom->ev1) != cudaSuccess) return cleanup("event");
    // [0, kMaxTags): sticky non-finite flags per map tag; then one scheduler counter
    // per map; then one boundary-signal counter per map (slab halo exchange)
    if (cudaMalloc(&dom->d_flags, kNumFlags * sizeof(int32_t)) != cudaSuccess) return cleanup("flags");
    cudaMemset(dom->d_flags, 0, kNumFlags * sizeof(int32_t));
    if (cudaMalloc(&dom->d_peer_flags, 2 * sizeof(int32_t)) != cudaSuccess) return cleanup("peer flags");
    {
        const int32_t done0[2] = {peer_mask(0), peer_mask(0)};  // "launch 0 completed"
        cudaMemcpy(dom->d_peer_flags, done0, sizeof(done0), cudaMemcpyHostToDevice);
    }
    if (const char* s = getenv("STKB_LZ")) dom->lz_override = atoi(s);
    if (const char* s = getenv("STKB_CTAS")) dom->ctas_override = atoi(s);
    if (const char* s = getenv("STKB_L2PROMO")) dom->l2promo = atoi(s);
    if (const char* s = getenv("STKB_STORE_HINT")) dom->store_hint = atoi(s);
    if (const char* s = getenv("STKB_TAPER")) dom->taper = atoi(s) != 0;
    if (const char* s = getenv("STKB_ORDER_Y")) dom->order_y_fast = atoi(s);
    if (const char* s = getenv("STKB_BAND")) dom->band_pct = atoi(s);
    if (const char* s = getenv("STKB_PRESCALE")) dom->prescale = atoi(s) != 0;
    if (const char* s = getenv("STKB_TB")) dom->tb = atoi(s) != 0;
    if (const char* s = getenv("STKB_MULTI")) dom->multi = atoi(s) != 0;
    if (const char* s = getenv("STKB_MULTI_POINTS")) dom->multi_max_points = atoll(s);
    if (const char* s = getenv("STKB_SMALL_TILE_POINTS")) dom->small_tile_points = atoll(s);
    *out = dom;
    return STKB_OK;
}

int stkb_domain_destroy(stkb_domain* dom) {
    if (!dom) return STKB_OK;
    cudaSetDevice(dom->desc.device);
    if (dom->stream) cudaStreamSynchronize(dom->stream);
    invalidate_graph(dom);
    for (auto& m : dom->maps) {
        if (m.d_code) cudaFree(m.d_code);
        if (m.d_consts) cudaFree(m.d_consts);
    }
    for (void* b : dom->bufs) if (b) cudaFree(b);
    for (void* b : dom->snap) if (b) cudaFree(b);
    if (dom->d_flags) cudaFree(dom->d_flags);
    if (dom->d_partials) cudaFree(dom->d_partials);
    if (dom->d_stage) cudaFree(dom->d_stage);
    if (dom->d_peer_flags) cudaFree(dom->d_peer_flags);
    if (dom->d_multi) cudaFree(dom->d_multi);
    if (dom->ev0) cudaEventDestroy(dom->ev0);
    if (dom->ev1) cudaEventDestroy(dom->ev1);
    if (dom->own_stream) cudaStreamDestroy(dom->own_stream);
    delete dom;
    return STKB_OK;
}

int stkb_layout(const stkb_domain* dom, int64_t* pitch, int64_t* plane, int64_t* lead, int64_t* elems) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (pitch) *pitch = dom->g.pitch;
    if (plane) *plane = dom->g.plane;
    if (lead) *lead = dom->g.lead;
    if (elems) *elems = dom->g.plane * (dom->g.n0 + 2 * dom->g.order0);
    return STKB_OK;
}

int stkb_device_ptr(stkb_domain* dom, int32_t name, void** dptr) {
    if (!dom || !dptr) return fail(STKB_ERR_ARG, "null argument");
    if (int rc = check_name(dom, name, "stkb_device_ptr")) return rc;
    cudaSetDevice(dom->desc.device);
    mark_halo_dirty(dom, dom->binding[name]);  // the caller may write through the pointer
    *dptr = dom->bufs[dom->binding[name]];
    return STKB_OK;
}

int stkb_mark_dirty(stkb_domain* dom, int32_t name) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (int rc = check_name(dom, name, "stkb_mark_dirty")) return rc;
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    mark_halo_dirty(dom, dom->binding[name]);
    return STKB_OK;
}

int stkb_zero(stkb_domain* dom, int32_t name) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (int rc = check_name(dom, name, "stkb_zero")) return rc;
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    const size_t bytes = size_t(dom->g.plane) * size_t(dom->g.n0 + 2 * dom->g.order0) * dom->elem;
    ++dom->ext_writes;
    CUDA_TRY(cudaMemsetAsync(dom->bufs[dom->binding[name]], 0, bytes, dom->stream));
    CUDA_TRY(cudaMemsetAsync(dom->d_flags + kHaloFlag + dom->binding[name], 0, sizeof(int32_t), dom->stream));
    return STKB_OK;
}

int stkb_set_stream(stkb_domain* dom, void* stream) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    dom->stream = stream ? static_cast<cudaStream_t>(stream) : dom->own_stream;
    return STKB_OK;
}

// A pitched cudaMemcpy2D runs at ~60 % of PCIe speed on B200 hosts; transfers go
// through a device staging buffer in contiguous chunks, repitched on the device.
static bool ensure_stage(stkb_domain* dom, size_t want) {
    constexpr size_t kStage = size_t(256) << 20;
    if (!dom->d_stage) {
        dom->stage_bytes = std::min(kStage, want);
        if (cudaMalloc(&dom->d_stage, dom->stage_bytes) != cudaSuccess) {
            cudaGetLastError();
            dom->d_stage = nullptr;
        }
    }
    return dom->d_stage != nullptr;
}

// A host grid's C-order padded box in lifted 3-D terms: interior extents s and halo widths
// h per axis (a 2-D grid is one plane without d0 halo, a 1-D grid one row of one plane).
struct HostBox {
    int64_t s[3];
    int64_t h[3];
    int64_t planes() const { return s[0] + 2 * h[0]; }
    int64_t rows_per_plane() const { return s[1] + 2 * h[1]; }
    int64_t row_elems() const { return s[2] + 2 * h[2]; }
};

static HostBox domain_box(const stkb_domain* dom) {
    const Geometry& g = dom->g;
    HostBox b{{g.n0, g.n1, g.n2}, {g.order0, dom->desc.ndim >= 2 ? g.order : 0, g.order}};
    return b;
}

// the layout of a grid of `shape` (ndim axes, as the domain) and halo `order`
static int grid_box(const stkb_domain* dom, const int64_t* shape, int32_t order, HostBox* out) {
    const int nd = dom->desc.ndim;
    const Geometry& g = dom->g;
    if (!shape) return fail(STKB_ERR_ARG, "null shape");
    if (order < 0 || order > g.order) return fail(STKB_ERR_ARG, "grid order exceeds the domain's halo order");
    HostBox b{{1, 1, 1}, {0, 0, 0}};
    for (int d = 0; d < nd; ++d) {
        b.s[3 - nd + d] = shape[d];
        b.h[3 - nd + d] = order;
    }
    const int64_t ext[3] = {g.n0, g.n1, g.n2};
    for (int d = 0; d < 3; ++d)
        if (b.s[d] < 1 || b.s[d] > ext[d]) return fail(STKB_ERR_ARG, "grid extent exceeds the domain's");
    *out = b;
    return STKB_OK;
}

static bool same_box(const HostBox& a, const HostBox& b) {
    for (int d = 0; d < 3; ++d)
        if (a.s[d] != b.s[d] || a.h[d] != b.h[d]) return false;
    return true;
}

// host box <-> pitched device buffer through the staging buffer: contiguous PCIe copies
// of whole host rows, scattered/gathered on the device by the repitch kernel
static int copy_box(stkb_domain* dom, int32_t name, const HostBox& hb, void* host, bool to_device) {
    const Geometry& g = dom->g;
    const size_t e = dom->elem;
    const size_t row = size_t(hb.row_elems()) * e;
    const int64_t rpp = hb.rows_per_plane();
    const int64_t rows = hb.planes() * rpp;
    char* base = static_cast<char*>(dom->bufs[dom->binding[name]]) + size_t(g.at(-hb.h[0], -hb.h[1], -hb.h[2])) * e;
    const int64_t rp = g.pitch * int64_t(e), pp = g.plane * int64_t(e);
    char* h = static_cast<char*>(host);
    if (!ensure_stage(dom, size_t(rows) * row)) {  // no memory for staging: pitched copies, plane by plane
        for (int64_t p = 0; p < hb.planes(); ++p) {
            char* d = base + p * pp;
            char* hp = h + size_t(p * rpp) * row;
            if (to_device)
                CUDA_TRY(cudaMemcpy2DAsync(d, size_t(rp), hp, row, row, size_t(rpp), cudaMemcpyHostToDevice, dom->stream));
            else
                CUDA_TRY(cudaMemcpy2DAsync(hp, row, d, size_t(rp), row, size_t(rpp), cudaMemcpyDeviceToHost, dom->stream));
        }
        return STKB_OK;
    }
    const int64_t chunk = std::max<int64_t>(1, int64_t(dom->stage_bytes / row));
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
        const int64_t nr = std::min(chunk, rows - r0);
        if (to_device) {
            CUDA_TRY(cudaMemcpyAsync(dom->d_stage, h + size_t(r0) * row, size_t(nr) * row, cudaMemcpyHostToDevice,
                                     dom->stream));
            CUDA_TRY(launch_repitch(dom->d_stage, base, r0, nr, rpp, int64_t(row), rp, pp, true, dom->num_sms,
                                    dom->stream));
        } else {
            CUDA_TRY(launch_repitch(dom->d_stage, base, r0, nr, rpp, int64_t(row), rp, pp, false, dom->num_sms,
                                    dom->stream));
            CUDA_TRY(cudaMemcpyAsync(h + size_t(r0) * row, dom->d_stage, size_t(nr) * row, cudaMemcpyDeviceToHost,
                                     dom->stream));
        }
    }
    return STKB_OK;
}

static int copy_h2d(stkb_domain* dom, int32_t name, const void* host, const HostBox* hb = nullptr) {
    if (!dom || !host) return fail(STKB_ERR_ARG, "null argument");
    if (int rc = check_name(dom, name, "stkb_upload")) return rc;
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    mark_halo_dirty(dom, dom->binding[name]);
    const HostBox own = domain_box(dom);
    if (hb && !same_box(*hb, own)) {  // a smaller box: every cell it does not cover is zero
        const size_t bytes = size_t(dom->g.plane) * size_t(dom->g.n0 + 2 * dom->g.order0) * dom->elem;
        CUDA_TRY(cudaMemsetAsync(dom->bufs[dom->binding[name]], 0, bytes, dom->stream));
    }
    return copy_box(dom, name, hb ? *hb : own, const_cast<void*>(host), true);
}

static int copy_d2h(stkb_domain* dom, int32_t name, void* host, const HostBox* hb = nullptr) {
    if (!dom || !host) return fail(STKB_ERR_ARG, "null argument");
    if (int rc = check_name(dom, name, "stkb_download")) return rc;
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    return copy_box(dom, name, hb ? *hb : domain_box(dom), host, false);
}

int stkb_upload_grid(stkb_domain* dom, int32_t name, const void* host, const int64_t* shape, int32_t order,
                     int32_t sync) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    HostBox hb;
    if (int rc = grid_box(dom, shape, order, &hb)) return rc;
    if (int rc = copy_h2d(dom, name, host, &hb)) return rc;
    if (sync) CUDA_TRY(cudaStreamSynchronize(dom->stream));
    return STKB_OK;
}

int stkb_download_grid(stkb_domain* dom, int32_t name, void* host, const int64_t* shape, int32_t order,
                       int32_t sync) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    HostBox hb;
    if (int rc = grid_box(dom, shape, order, &hb)) return rc;
    if (int rc = copy_d2h(dom, name, host, &hb)) return rc;
    if (sync) CUDA_TRY(cudaStreamSynchronize(dom->stream));
    return STKB_OK;
}

int stkb_upload_async(stkb_domain* dom, int32_t name, const void* host) { return copy_h2d(dom, name, host); }
int stkb_download_async(stkb_domain* dom, int32_t name, void* host) { return copy_d2h(dom, name, host); }

int stkb_upload(stkb_domain* dom, int32_t name, const void* host) {
    if (int rc = copy_h2d(dom, name, host)) return rc;
    CUDA_TRY(cudaStreamSynchronize(dom->stream));
    return STKB_OK;
}

int stkb_download(stkb_domain* dom, int32_t name, void* host) {
    if (int rc = copy_d2h(dom, name, host)) return rc;
    CUDA_TRY(cudaStreamSynchronize(dom->stream));
    return STKB_OK;
}

int stkb_program_reset(stkb_domain* dom) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    cudaSetDevice(dom->desc.device);
    cudaStreamSynchronize(dom->stream);
    invalidate_graph(dom);
    for (auto& m : dom->maps) {
        if (m.d_code) cudaFree(m.d_code);
        if (m.d_consts) cudaFree(m.d_consts);
    }
    dom->maps.clear();
    dom->prog.clear();
    return STKB_OK;
}

int stkb_program_add_map(stkb_domain* dom, const stkb_map_desc* md) {
    if (!dom || !md) return fail(STKB_ERR_ARG, "null argument");
    const stkb_map_desc& d = *md;
    const Geometry& g = dom->g;
    const int nd = dom->desc.ndim;
    // region box in lifted 3-D interior coordinates
    int64_t lo[3], hi[3];
    if (nd == 3) {
        for (int i = 0; i < 3; ++i) { lo[i] = d.lo[i]; hi[i] = d.hi[i]; }
    } else if (nd == 2) {
        lo[0] = 0; hi[0] = 1;
        lo[1] = d.lo[0]; hi[1] = d.hi[0];
        lo[2] = d.lo[1]; hi[2] = d.hi[1];
    } else {
        lo[0] = 0; hi[0] = 1;
        lo[1] = 0; hi[1] = 1;
        lo[2] = d.lo[0]; hi[2] = d.hi[0];
    }
    const int64_t ext[3] = {g.n0, g.n1, g.n2};
    for (int i = 0; i < 3; ++i)
        if (lo[i] < 0 || hi[i] > ext[i] || lo[i] > hi[i])
            return fail(STKB_ERR_ARG, "map region outside the interior");
    MapOp op;
    op.d = d;
    for (int i = 0; i < 3; ++i) { op.d.lo[i] = lo[i]; op.d.hi[i] = hi[i]; }
    if (d.kind == STKB_MAP_STAR || d.kind == STKB_MAP_WAVE || d.kind == STKB_MAP_BOX || d.kind == STKB_MAP_XSTAR ||
        d.kind == STKB_MAP_XWAVE || d.kind == STKB_MAP_XBOX) {
        if ((d.kind == STKB_MAP_XWAVE && nd != 3) || ((d.kind == STKB_MAP_XSTAR || d.kind == STKB_MAP_XBOX) && nd == 1))
            return fail(STKB_ERR_UNSUPPORTED, "exact streaming maps are 3-D (stars and boxes also 2-D)");
        if (nd != 3 && !(nd == 2 && d.kind != STKB_MAP_WAVE))
            return fail(STKB_ERR_UNSUPPORTED, nd == 1 ? "1-D maps run as EXPR maps" : "2-D grids stream star and box maps only");
        if (d.radius < 1 || d.radius > 4) return fail(STKB_ERR_UNSUPPORTED, "streaming star kernels cover radius 1..4");
        if ((d.kind == STKB_MAP_BOX || d.kind == STKB_MAP_XBOX) && nd == 3) {
            const int n = 2 * d.radius + 1;
            if (d.radius > 2 && !d.box_coef_ext)
                return fail(STKB_ERR_ARG, "a 3-D box map of radius > 2 passes its coefficients in box_coef_ext");
            const double* src = d.radius > 2 ? d.box_coef_ext : d.box_coef;
            op.cube.assign(src, src + size_t(n) * n * n);
        }
        if (d.kind == STKB_MAP_XBOX && nd == 2) {
            const int n = 2 * d.radius + 1;
            op.cube.assign(d.box_coef, d.box_coef + size_t(n) * n);
        }
        op.d.box_coef_ext = nullptr;  // copied: the caller's array need not outlive this call
        if (d.radius > g.order) return fail(STKB_ERR_ARG, "stencil radius exceeds the grid halo order");
        if (int rc = check_name(dom, d.src, "src")) return rc;
        if (int rc = check_name(dom, d.dst, "dst")) return rc;
        if (d.src == d.dst) return fail(STKB_ERR_ARG, "star map reads and writes the same grid (needs a snapshot: use EXPR)");
        if (d.kind == STKB_MAP_WAVE || d.kind == STKB_MAP_XWAVE) {
            if (int rc = check_name(dom, d.prev, "prev")) return rc;
            if (int rc = check_name(dom, d.vel, "vel")) return rc;
            if (d.vel == d.dst) return fail(STKB_ERR_ARG, "wave map writes its velocity grid");
        }
        if (d.precision != STKB_PREC_FAST) return fail(STKB_ERR_UNSUPPORTED, "unknown precision");
    } else if (d.kind == STKB_MAP_EXPR) {
        if (d.n_args < 1 || d.n_args > STKB_EXPR_MAX_ARGS) return fail(STKB_ERR_ARG, "EXPR map: n_args out of range");
        if (d.n_code < 1 || !d.code) return fail(STKB_ERR_ARG, "EXPR map: empty code");
        for (int i = 0; i < d.n_args; ++i)
            if (int rc = check_name(dom, d.args[i], "EXPR arg")) return rc;
        op.code.assign(d.code, d.code + 5 * size_t(d.n_code));
        op.consts.assign(d.consts, d.consts + std::max(0, d.n_consts));
        // static checks: stack discipline, argument indices, halo-safe offsets
        bool written[STKB_EXPR_MAX_ARGS] = {}, read[STKB_EXPR_MAX_ARGS] = {};
        int sp = 0, maxsp = 0;
        const int64_t o0 = g.order0, o = g.order;
        for (int pc = 0; pc < d.n_code; ++pc) {
            const int32_t* ins = &op.code[5 * pc];
            int32_t oz = ins[2], oy = ins[3], ox = ins[4];
            if (nd == 2 && (ins[0] == STKB_OP_READ || ins[0] == STKB_OP_STORE)) { ox = ins[3]; oy = ins[2]; oz = 0; }
            if (nd == 1 && (ins[0] == STKB_OP_READ || ins[0] == STKB_OP_STORE)) { ox = ins[2]; oy = 0; oz = 0; }
            switch (ins[0]) {
                case STKB_OP_CONST:
                    if (ins[1] < 0 || ins[1] >= d.n_consts) return fail(STKB_ERR_ARG, "EXPR: const index");
                    ++sp; break;
                case STKB_OP_READ:
                case STKB_OP_STORE:
                    if (ins[1] < 0 || ins[1] >= d.n_args) return fail(STKB_ERR_ARG, "EXPR: arg index");
                    if (lo[0] + oz < -o0 || hi[0] - 1 + oz >= g.n0 + o0 || lo[1] + oy < -o ||
                        hi[1] - 1 + oy >= g.n1 + o || lo[2] + ox < -o || hi[2] - 1 + ox >= g.n2 + o)
                        return fail(STKB_ERR_ARG, "EXPR: offset reaches beyond the halo");
                    if (ins[0] == STKB_OP_READ) { read[ins[1]] = true; ++sp; }
                    else {
                        if (lo[0] + oz < 0 || hi[0] - 1 + oz >= g.n0 || lo[1] + oy < 0 || hi[1] - 1 + oy >= g.n1 ||
                            lo[2] + ox < 0 || hi[2] - 1 + ox >= g.n2)
                            return fail(STKB_ERR_ARG, "update destination offset writes outside the interior");
                        written[ins[1]] = true; --sp;
                    }
                    // lift 2-D offsets into the 3-D lane layout the kernel reads
                    op.code[5 * pc + 2] = oz; op.code[5 * pc + 3] = oy; op.code[5 * pc + 4] = ox;
                    break;
                case STKB_OP_LOCAL:
                    if (ins[1] < 0 || ins[1] >= STKB_EXPR_MAX_LOCALS) return fail(STKB_ERR_ARG, "EXPR: local index");
                    ++sp; break;
                case STKB_OP_SETLOCAL:
                    if (ins[1] < 0 || ins[1] >= STKB_EXPR_MAX_LOCALS) return fail(STKB_ERR_ARG, "EXPR: local index");
                    --sp; break;
                case STKB_OP_ADD: case STKB_OP_SUB: case STKB_OP_MUL: case STKB_OP_DIV: --sp; break;
                case STKB_OP_NEG: break;
                default: return fail(STKB_ERR_ARG, "EXPR: unknown opcode");
            }
            if (sp < 0) return fail(STKB_ERR_ARG, "EXPR: stack underflow");
            maxsp = std::max(maxsp, sp);
        }
        if (sp != 0) return fail(STKB_ERR_ARG, "EXPR: unbalanced stack");
        if (maxsp > STKB_EXPR_MAX_STACK) return fail(STKB_ERR_UNSUPPORTED, "EXPR: expression too deep");
        // a grid that is both read and written is read from a pre-map copy,
        // and aliases (the same name bound to several params) share one
        for (int i = 0; i < d.n_args; ++i) {
            bool w = false, r = false;
            for (int j = 0; j < d.n_args; ++j)
                if (d.args[j] == d.args[i]) { w |= written[j]; r |= read[j]; }
            op.snapshot[i] = w && r;
        }
        CUDA_TRY(cudaSetDevice(dom->desc.device));
        const size_t gbytes = size_t(g.plane) * size_t(g.n0 + 2 * g.order0) * dom->elem;
        for (int i = 0; i < d.n_args; ++i)
            if (op.snapshot[i] && !dom->snap[i]) CUDA_TRY(cudaMalloc(&dom->snap[i], gbytes));
        CUDA_TRY(cudaMalloc(&op.d_code, op.code.size() * sizeof(int32_t)));
        CUDA_TRY(cudaMemcpy(op.d_code, op.code.data(), op.code.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        const size_t nc = std::max<size_t>(1, op.consts.size());
        CUDA_TRY(cudaMalloc(&op.d_consts, nc * sizeof(double)));
        if (!op.consts.empty())
            CUDA_TRY(cudaMemcpy(op.d_consts, op.consts.data(), op.consts.size() * sizeof(double), cudaMemcpyHostToDevice));
        op.d.code = nullptr;
        op.d.consts = nullptr;
    } else {
        return fail(STKB_ERR_ARG, "unknown map kind");
    }
    if (dom->maps.size() >= size_t(kMaxMaps)) return fail(STKB_ERR_ARG, "too many maps in one step program");
    op.slot = int(dom->maps.size());
    invalidate_graph(dom);
    dom->maps.push_back(std::move(op));
    dom->prog.push_back(ProgOp{0, int(dom->maps.size()) - 1, 0, 0});
    return STKB_OK;
}

int stkb_program_add_swap(stkb_domain* dom, int32_t a, int32_t b) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (int rc = check_name(dom, a, "swap")) return rc;
    if (int rc = check_name(dom, b, "swap")) return rc;
    invalidate_graph(dom);
    dom->prog.push_back(ProgOp{1, -1, a, b});
    return STKB_OK;
}

// CUDA graph of two fused sweeps from the current (u buffer, scratch) pair; capturing
// runs nothing
int tb_graph(stkb_domain* dom, const MapOp& tb, cudaGraphExec_t* out) {
    const std::pair<int, int> key(dom->binding[tb.d.src], dom->scratch);
    auto it = dom->tb_graphs.find(key);
    if (it == dom->tb_graphs.end()) {
        CUDA_TRY(cudaStreamBeginCapture(dom->stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_tb2(dom, tb);
        if (rc == STKB_OK) rc = enqueue_tb2(dom, tb);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(dom->stream, &graph);
        dom->binding[tb.d.src] = key.first;  // capturing did not run the sweeps
        dom->scratch = key.second;
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        cudaGraphExec_t ex = nullptr;
        e = cudaGraphInstantiate(&ex, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        it = dom->tb_graphs.emplace(key, ex).first;
    }
    *out = it->second;
    return STKB_OK;
}

int stkb_run(stkb_domain* dom, int64_t steps) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (steps < 0) return fail(STKB_ERR_ARG, "negative step count");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    int64_t launches = 0;
    int64_t done = 0;
    const int period = binding_period(dom);
    const bool graphs_ok = period > 0 && getenv("STKB_NO_GRAPH") == nullptr;
    if (int rc = ensure_halo_flags(dom)) return rc;  // before the timed events
    if (const MapOp* mm = steps >= 2 ? multi_map(dom) : nullptr) {
        CUDA_TRY(cudaEventRecord(dom->ev0, dom->stream));
        while (done < steps) {
            const int n = int(std::min<int64_t>(kMaxMultiSteps, steps - done));
            const int rc = dom->desc.dtype == STKB_F32
                               ? launch_star_map<float>(dom, *mm, dom->binding, RangeSpec(), false, n)
                               : launch_star_map<double>(dom, *mm, dom->binding, RangeSpec(), false, n);
            if (rc && done == 0 && dom->last_launch_error == cudaErrorCooperativeLaunchTooLarge) {
                cudaGetLastError();  // not sticky: clear it
                // not every CTA could be resident (the device is shared): single steps instead
                dom->multi = false;
                return stkb_run(dom, steps);
            }
            if (rc) return rc;
            ++launches;
            if (n & 1) std::swap(dom->binding[mm->d.src], dom->binding[mm->d.dst]);
            done += n;
        }
        CUDA_TRY(cudaEventRecord(dom->ev1, dom->stream));
        dom->timed = true;
        dom->last_launches = launches;
        dom->last_mode = 2;
        return STKB_OK;
    }
    if (const MapOp* tb = steps >= 4 ? tb_map(dom) : nullptr) {
        // fused sweeps for all but the last 2..3 steps, which run as single steps so
        // that v ends up holding its own final value
        const int64_t n_tb = (steps - 2) / 2;
        const size_t bytes = size_t(dom->g.plane) * size_t(dom->g.n0 + 2 * dom->g.order0) * dom->elem;
        if (dom->scratch < 0) {  // host-side setup stays outside the timed events
            void* b = nullptr;
            CUDA_TRY(cudaMalloc(&b, bytes));
            dom->bufs.push_back(b);
            dom->scratch = int(dom->bufs.size()) - 1;
            // zero pitch padding, as in every grid buffer (kernels never write it)
            CUDA_TRY(cudaMemsetAsync(b, 0, bytes, dom->stream));
            dom->tb_pair_epoch = -1;
        }
        cudaGraphExec_t gx = nullptr;
        if (graphs_ok && dom->tb_warmed && n_tb >= 2)
            if (int rc = tb_graph(dom, *tb, &gx)) return rc;
        CUDA_TRY(cudaEventRecord(dom->ev0, dom->stream));
        // the scratch takes over u's halo and whatever interior the region leaves alone
        // (the fused kernel writes only the region); skipped while both still match
        const int ub = dom->binding[tb->d.src];
        const bool paired = dom->tb_pair_epoch == dom->ext_writes &&
                            ((dom->tb_pair[0] == ub && dom->tb_pair[1] == dom->scratch) ||
                             (dom->tb_pair[1] == ub && dom->tb_pair[0] == dom->scratch));
        if (!paired) {
            const stkb_map_desc& d = tb->d;
            const bool whole = d.lo[0] == 0 && d.lo[1] == 0 && d.lo[2] == 0 && d.hi[0] == dom->g.n0 &&
                               d.hi[1] == dom->g.n1 && d.hi[2] == dom->g.n2;
            if (whole) {  // only the halo shell is u's own: the sweeps write the whole interior
                CUDA_TRY(launch_copy_halo(dom->bufs[ub], dom->bufs[dom->scratch], dom->g, int(dom->elem),
                                          dom->num_sms, dom->stream));
                ++launches;
            } else {
                CUDA_TRY(cudaMemcpyAsync(dom->bufs[dom->scratch], dom->bufs[ub], bytes, cudaMemcpyDeviceToDevice,
                                         dom->stream));
            }
            CUDA_TRY(cudaMemcpyAsync(dom->d_flags + kHaloFlag + dom->scratch, dom->d_flags + kHaloFlag + ub,
                                     sizeof(int32_t), cudaMemcpyDeviceToDevice, dom->stream));  // same halo
            dom->tb_pair[0] = ub;
            dom->tb_pair[1] = dom->scratch;
            dom->tb_pair_epoch = dom->ext_writes;
        }
        // are v's values next to the box (its halo, for a full-interior map) all zero?
        CUDA_TRY(launch_frozen_ring(dom->desc.dtype, dom->g, box_of(tb->d), tb->d.radius,
                                    dom->bufs[dom->binding[tb->d.dst]], dom->d_flags + kFrozenFlag, dom->num_sms,
                                    dom->stream));
        ++launches;
        int64_t k = 0;
        if (!dom->tb_warmed || !graphs_ok) {  // attributes and tensor maps outside any capture
            if (int rc = enqueue_tb2(dom, *tb)) return rc;
            ++launches;
            dom->tb_warmed = true;
            k = 1;
        }
        if (graphs_ok && n_tb - k >= 2) {
            if (k > 0)  // after the warm-up sweep (captured while it runs)
                if (int rc = tb_graph(dom, *tb, &gx)) return rc;
            const int64_t reps = (n_tb - k) / 2;
            for (int64_t r = 0; r < reps; ++r) CUDA_TRY(cudaGraphLaunch(gx, dom->stream));
            launches += 2 * reps;
            k += 2 * reps;  // two rotations: u and the scratch are back where they started
        }
        for (; k < n_tb; ++k) {
            if (int rc = enqueue_tb2(dom, *tb)) return rc;
            ++launches;
        }
        // the binding of 2 n_tb single steps (a ping-pong swap twice per pair: unchanged)
        done = 2 * n_tb;
        for (; done < steps; ++done)
            if (int rc = enqueue_step(dom, dom->binding, &launches)) return rc;
        CUDA_TRY(cudaEventRecord(dom->ev1, dom->stream));
        dom->timed = true;
        dom->last_launches = launches;
        dom->last_mode = 1;
        return STKB_OK;
    }
    CUDA_TRY(cudaEventRecord(dom->ev0, dom->stream));
    // the first step after a program change runs uncaptured: it sets kernel
    // attributes and encodes tensor maps outside any capture
    if (graphs_ok && !dom->warmed && steps > 0) {
        if (int rc = enqueue_step(dom, dom->binding, &launches)) return rc;
        dom->warmed = true;
        done = 1;
    }
    if (graphs_ok && steps - done >= period) {
        auto it = dom->graphs.find(dom->binding);
        if (it == dom->graphs.end()) {
            cudaStream_t cap = dom->stream;
            CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            std::vector<int32_t> b = dom->binding;
            int64_t n = 0;
            int rc = STKB_OK;
            for (int k = 0; k < period && rc == STKB_OK; ++k) rc = enqueue_step(dom, b, &n);
            cudaGraph_t graph = nullptr;
            cudaError_t e = cudaStreamEndCapture(cap, &graph);
            if (rc) {
                if (graph) cudaGraphDestroy(graph);
                return rc;
            }
            if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
            cudaGraphExec_t ex = nullptr;
            e = cudaGraphInstantiate(&ex, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) return fail(STKB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
            it = dom->graphs.emplace(dom->binding, std::make_pair(ex, n)).first;
            dom->gperiod = period;
        }
        const int64_t reps = (steps - done) / period;
        for (int64_t r = 0; r < reps; ++r) CUDA_TRY(cudaGraphLaunch(it->second.first, dom->stream));
        launches += reps * it->second.second;
        done += reps * period;  // the binding is back where it started
    }
    for (; done < steps; ++done)
        if (int rc = enqueue_step(dom, dom->binding, &launches)) return rc;
    CUDA_TRY(cudaEventRecord(dom->ev1, dom->stream));
    dom->timed = true;
    dom->last_launches = launches;
    dom->last_mode = 0;
    return STKB_OK;
}

int stkb_run_once(stkb_domain* dom) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    dom->tb_pair_epoch = -1;  // writes outside the fused-sweep loop (buffer pair state unknown)
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    int64_t launches = 0;
    CUDA_TRY(cudaEventRecord(dom->ev0, dom->stream));
    if (int rc = enqueue_step(dom, dom->binding, &launches)) return rc;
    CUDA_TRY(cudaEventRecord(dom->ev1, dom->stream));
    dom->timed = true;
    dom->last_launches = launches;
    dom->last_mode = 0;
    return STKB_OK;
}

int stkb_sync(stkb_domain* dom) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    CUDA_TRY(cudaStreamSynchronize(dom->stream));
    return STKB_OK;
}

int stkb_elapsed_ms(stkb_domain* dom, double* ms) {
    if (!dom || !ms) return fail(STKB_ERR_ARG, "null argument");
    if (!dom->timed) return fail(STKB_ERR_STATE, "no run recorded");
    CUDA_TRY(cudaEventSynchronize(dom->ev1));
    float f = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&f, dom->ev0, dom->ev1));
    *ms = f;
    return STKB_OK;
}

int stkb_run_mode(const stkb_domain* dom, int32_t* mode) {
    if (!dom || !mode) return fail(STKB_ERR_ARG, "null argument");
    *mode = dom->last_mode;
    return STKB_OK;
}

int stkb_launches(stkb_domain* dom, int64_t* count) {
    if (!dom || !count) return fail(STKB_ERR_ARG, "null argument");
    *count = dom->last_launches;
    return STKB_OK;
}

int stkb_binding(const stkb_domain* dom, int32_t name, int32_t* buffer) {
    if (!dom || !buffer) return fail(STKB_ERR_ARG, "null argument");
    if (int rc = check_name(dom, name, "stkb_binding")) return rc;
    *buffer = dom->binding[name];
    return STKB_OK;
}

int stkb_nonfinite(stkb_domain* dom, int32_t tag, int32_t* flag) {
    if (!dom || !flag) return fail(STKB_ERR_ARG, "null argument");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    int32_t* p = dom->d_flags + (tag & (kMaxTags - 1));
    CUDA_TRY(cudaMemcpyAsync(flag, p, sizeof(int32_t), cudaMemcpyDeviceToHost, dom->stream));
    CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(int32_t), dom->stream));
    CUDA_TRY(cudaStreamSynchronize(dom->stream));
    return STKB_OK;
}

int stkb_launch_map(stkb_domain* dom, int32_t map_index, int64_t lo0, int64_t hi0) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    dom->tb_pair_epoch = -1;  // writes outside the fused-sweep loop (buffer pair state unknown)
    if (map_index < 0 || map_index >= int32_t(dom->maps.size())) return fail(STKB_ERR_ARG, "map index out of range");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    MapOp& op = dom->maps[map_index];
    const stkb_map_desc saved = op.d;
    op.d.lo[0] = std::max<int64_t>(saved.lo[0], lo0);
    op.d.hi[0] = std::min<int64_t>(saved.hi[0], hi0);
    int rc = STKB_OK;
    if (op.d.hi[0] > op.d.lo[0]) {
        if (op.d.kind == STKB_MAP_EXPR) rc = launch_expr_map(dom, op, dom->binding);
        else if (dom->desc.dtype == STKB_F32) rc = launch_star_map<float>(dom, op, dom->binding);
        else rc = launch_star_map<double>(dom, op, dom->binding);
    }
    op.d = saved;
    return rc;
}

int stkb_launch_map_ranges(stkb_domain* dom, int32_t map_index, int32_t n_ranges, const int64_t* lo0,
                           const int64_t* hi0, int32_t n_signal, int32_t* signal_items) {
    if (!dom || (n_ranges > 0 && (!lo0 || !hi0))) return fail(STKB_ERR_ARG, "null argument");
    dom->tb_pair_epoch = -1;  // writes outside the fused-sweep loop (buffer pair state unknown)
    if (map_index < 0 || map_index >= int32_t(dom->maps.size())) return fail(STKB_ERR_ARG, "map index out of range");
    if (n_ranges < 0 || n_ranges > 64 || n_signal < 0 || n_signal > n_ranges)
        return fail(STKB_ERR_ARG, "bad range list");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    MapOp& op = dom->maps[map_index];
    const stkb_map_desc saved = op.d;
    int32_t lo[64], hi[64];
    for (int i = 0; i < n_ranges; ++i) {  // clip to the map's own d0 box
        lo[i] = int32_t(std::max<int64_t>(saved.lo[0], lo0[i]));
        hi[i] = int32_t(std::min<int64_t>(saved.hi[0], hi0[i]));
    }
    int items = 0;
    int rc = STKB_OK;
    const bool streaming = op.d.kind != STKB_MAP_EXPR && op.d.kind != STKB_MAP_XSTAR && op.d.kind != STKB_MAP_XWAVE &&
                           op.d.kind != STKB_MAP_XBOX &&
                           dom->desc.ndim == 3;
    if (streaming) {
        RangeSpec rs;
        rs.n = n_ranges;
        rs.lo = lo;
        rs.hi = hi;
        rs.n_signal = n_signal;
        rs.signal_items = &items;
        rc = dom->desc.dtype == STKB_F32 ? launch_star_map<float>(dom, op, dom->binding, rs)
                                         : launch_star_map<double>(dom, op, dom->binding, rs);
    } else {
        // one launch per range; a stream-ordered marker after the signal ranges
        int32_t* sig = dom->d_flags + kMaxTags + kMaxMaps + op.slot;
        for (int i = 0; i < n_ranges && rc == STKB_OK; ++i) {
            if (hi[i] > lo[i]) {
                op.d.lo[0] = lo[i];
                op.d.hi[0] = hi[i];
                if (op.d.kind == STKB_MAP_EXPR) rc = launch_expr_map(dom, op, dom->binding);
                else if (dom->desc.dtype == STKB_F32) rc = launch_star_map<float>(dom, op, dom->binding);
                else rc = launch_star_map<double>(dom, op, dom->binding);
            }
            if (rc == STKB_OK && n_signal > 0 && i == n_signal - 1) {
                cudaError_t e = launch_signal_add(sig, 1, dom->stream);
                if (e != cudaSuccess) rc = fail(STKB_ERR_CUDA, cudaGetErrorString(e));
                items = 1;
            }
        }
        op.d = saved;
    }
    if (signal_items) *signal_items = items;
    return rc;
}

int stkb_launch_map_pull(stkb_domain* dom, int32_t map_index) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    dom->tb_pair_epoch = -1;  // writes outside the fused-sweep loop (buffer pair state unknown)
    if (map_index < 0 || map_index >= int32_t(dom->maps.size())) return fail(STKB_ERR_ARG, "map index out of range");
    MapOp& op = dom->maps[map_index];
    if (op.d.kind == STKB_MAP_EXPR || op.d.kind == STKB_MAP_XSTAR || op.d.kind == STKB_MAP_XWAVE ||
        op.d.kind == STKB_MAP_XBOX || dom->desc.ndim != 3)
        return fail(STKB_ERR_UNSUPPORTED, "the fused halo exchange needs a 3-D streaming map");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    return dom->desc.dtype == STKB_F32 ? launch_star_map<float>(dom, op, dom->binding, RangeSpec(), true)
                                       : launch_star_map<double>(dom, op, dom->binding, RangeSpec(), true);
}

int stkb_peer_fetch_halo(stkb_domain* dom, void* stream, int32_t planes) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (planes < 0 || planes > dom->g.order0) return fail(STKB_ERR_ARG, "planes must be in 0..order");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : dom->stream;
    ++dom->ext_writes;
    dom->halo_external = true;
    for (int b = 0; b < dom->desc.n_grids; ++b)  // my halo planes now hold the neighbours' data
        CUDA_TRY(cudaMemsetAsync(dom->d_flags + kHaloFlag + b, 0x01, sizeof(int32_t), s));
    const size_t pb = size_t(dom->g.plane) * dom->elem;
    for (int side = 0; side < 2; ++side) {
        const auto& p = dom->peer[side];
        if (!p.set) continue;
        const int64_t np = std::min<int64_t>(planes, p.n0);
        if (np <= 0) continue;
        // lower: my planes [order0 - np, order0) <- its [order0 + n0' - np, order0 + n0')
        // upper: my planes [order0 + n0, order0 + n0 + np) <- its [order0, order0 + np)
        const int64_t mine = side == 0 ? dom->g.order0 - np : dom->g.order0 + dom->g.n0;
        const int64_t theirs = side == 0 ? dom->g.order0 + p.n0 - np : dom->g.order0;
        for (int b = 0; b < dom->desc.n_grids; ++b)
            CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dom->bufs[b]) + mine * pb,
                                     static_cast<const char*>(p.bufs[b]) + theirs * pb, size_t(np) * pb,
                                     cudaMemcpyDefault, s));
    }
    return STKB_OK;
}

int stkb_buffer_ipc_handle(stkb_domain* dom, int32_t buffer, void* handle) {
    if (!dom || !handle) return fail(STKB_ERR_ARG, "null argument");
    if (buffer < 0 || buffer >= dom->desc.n_grids) return fail(STKB_ERR_ARG, "buffer index out of range");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, dom->bufs[buffer]));
    memcpy(handle, &h, sizeof(h));
    return STKB_OK;
}

int stkb_flags_ipc_handle(stkb_domain* dom, void* handle) {
    if (!dom || !handle) return fail(STKB_ERR_ARG, "null argument");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, dom->d_peer_flags));
    memcpy(handle, &h, sizeof(h));
    return STKB_OK;
}

int stkb_flags_ptr(stkb_domain* dom, void** dptr) {
    if (!dom || !dptr) return fail(STKB_ERR_ARG, "null argument");
    *dptr = dom->d_peer_flags;
    return STKB_OK;
}

int stkb_buffer_ptr(stkb_domain* dom, int32_t buffer, void** dptr) {
    if (!dom || !dptr) return fail(STKB_ERR_ARG, "null argument");
    if (buffer < 0 || buffer >= dom->desc.n_grids) return fail(STKB_ERR_ARG, "buffer index out of range");
    *dptr = dom->bufs[buffer];
    return STKB_OK;
}

int stkb_ipc_open(int32_t device, const void* handle, void** dptr) {
    if (!handle || !dptr) return fail(STKB_ERR_ARG, "null argument");
    CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    return STKB_OK;
}

int stkb_ipc_close(int32_t device, void* dptr) {
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaIpcCloseMemHandle(dptr));
    return STKB_OK;
}

int stkb_set_peer(stkb_domain* dom, int32_t side, int32_t n_bufs, void* const* bufs, void* flags, int64_t peer_n0) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (side < 0 || side > 1) return fail(STKB_ERR_ARG, "side is 0 (lower) or 1 (upper)");
    auto& p = dom->peer[side];
    if (!bufs) {  // detach
        p = stkb_domain::Peer();
        ++dom->ext_writes;
        return STKB_OK;
    }
    if (n_bufs != dom->desc.n_grids || !flags) return fail(STKB_ERR_ARG, "peer needs one pointer per buffer and its flags");
    if (peer_n0 < dom->g.order0) return fail(STKB_ERR_ARG, "a neighbour slab must hold at least `order` planes");
    p.bufs.assign(bufs, bufs + n_bufs);
    p.tmaps.clear();
    ++dom->ext_writes;  // halo flags: this side's z face no longer counts
    p.flags = static_cast<int32_t*>(flags);
    p.n0 = peer_n0;
    p.set = true;
    return STKB_OK;
}

static PFN_cuStreamWaitValue32_v2 get_wait_fn() {
    static PFN_cuStreamWaitValue32_v2 fn_ = nullptr;
    if (!fn_) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess && fn)
            fn_ = reinterpret_cast<PFN_cuStreamWaitValue32_v2>(fn);
    }
    return fn_;
}

int stkb_peer_signal(stkb_domain* dom, void* stream, int32_t value) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    static PFN_cuStreamWriteValue32_v2 write_fn = nullptr;
    if (!write_fn) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail(STKB_ERR_CUDA, "cuStreamWriteValue32 entry point unavailable");
        write_fn = reinterpret_cast<PFN_cuStreamWriteValue32_v2>(fn);
    }
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    CUstream st = static_cast<CUstream>(stream ? stream : dom->stream);
    for (int side = 0; side < 2; ++side) {
        const auto& p = dom->peer[side];
        if (!p.set) continue;
        // I am my lower neighbour's upper neighbour (its slot 1) and vice versa;
        // the default flags fence this write after every prior store of the stream
        int32_t* slot = p.flags + (side == 0 ? 1 : 0);
        CUresult r = write_fn(st, reinterpret_cast<CUdeviceptr>(slot), cuuint32_t(peer_mask(value)),
                              CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) return fail(STKB_ERR_CUDA, "cuStreamWriteValue32 failed: " + std::to_string(int(r)));
    }
    return STKB_OK;
}

int stkb_peer_wait(stkb_domain* dom, void* stream, int32_t value) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    PFN_cuStreamWaitValue32_v2 wait_fn = get_wait_fn();
    if (!wait_fn) return fail(STKB_ERR_CUDA, "cuStreamWaitValue32 entry point unavailable");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    CUstream st = static_cast<CUstream>(stream ? stream : dom->stream);
    for (int side = 0; side < 2; ++side) {
        if (!dom->peer[side].set) continue;
        CUresult r = wait_fn(st, reinterpret_cast<CUdeviceptr>(dom->d_peer_flags + side),
                             cuuint32_t(1u << (((value % 3) + 3) % 3)), CU_STREAM_WAIT_VALUE_AND);
        if (r != CUDA_SUCCESS) return fail(STKB_ERR_CUDA, "cuStreamWaitValue32 failed: " + std::to_string(int(r)));
    }
    return STKB_OK;
}

int stkb_stream_wait_signal(stkb_domain* dom, void* stream, int32_t map_index, int32_t value) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (map_index < 0 || map_index >= int32_t(dom->maps.size())) return fail(STKB_ERR_ARG, "map index out of range");
    PFN_cuStreamWaitValue32_v2 wait_fn = get_wait_fn();
    if (!wait_fn) return fail(STKB_ERR_CUDA, "cuStreamWaitValue32 entry point unavailable");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    int32_t* sig = dom->d_flags + kMaxTags + kMaxMaps + dom->maps[map_index].slot;
    CUresult r = wait_fn(static_cast<CUstream>(stream ? stream : dom->stream), reinterpret_cast<CUdeviceptr>(sig),
                         cuuint32_t(value), CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(STKB_ERR_CUDA, "cuStreamWaitValue32 failed: " + std::to_string(int(r)));
    return STKB_OK;
}

int stkb_reset_signal(stkb_domain* dom, int32_t map_index, void* stream) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (map_index < 0 || map_index >= int32_t(dom->maps.size())) return fail(STKB_ERR_ARG, "map index out of range");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    int32_t* sig = dom->d_flags + kMaxTags + kMaxMaps + dom->maps[map_index].slot;
    CUDA_TRY(cudaMemsetAsync(sig, 0, sizeof(int32_t), stream ? static_cast<cudaStream_t>(stream) : dom->stream));
    return STKB_OK;
}

int stkb_prepare(stkb_domain* dom) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    return ensure_halo_flags(dom);
}

int stkb_enable_peer(int32_t device, int32_t peer) {
    if (device == peer) return STKB_OK;
    int ok = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&ok, device, peer));
    if (!ok) return fail(STKB_ERR_UNSUPPORTED, "no peer access between these GPUs");
    CUDA_TRY(cudaSetDevice(device));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();  // clear the non-sticky error
        e = cudaSuccess;
    }
    CUDA_TRY(e);
    return STKB_OK;
}

int stkb_set_fused_steps(stkb_domain* dom, int32_t enable) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    dom->tb = enable != 0;
    return STKB_OK;
}

int stkb_set_multi_steps(stkb_domain* dom, int32_t enable, int64_t max_points) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (max_points < 0) return fail(STKB_ERR_ARG, "max_points must be >= 0");
    dom->multi = enable != 0;
    if (max_points > 0) dom->multi_max_points = max_points;
    return STKB_OK;
}

int stkb_set_max_ctas(stkb_domain* dom, int32_t ctas) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    dom->ctas_override = std::max<int32_t>(0, ctas);
    return STKB_OK;
}

int stkb_apply_swap(stkb_domain* dom, int32_t a, int32_t b) {
    if (!dom) return fail(STKB_ERR_ARG, "null domain");
    if (int rc = check_name(dom, a, "swap")) return rc;
    if (int rc = check_name(dom, b, "swap")) return rc;
    std::swap(dom->binding[a], dom->binding[b]);
    return STKB_OK;
}

int stkb_plane_span(stkb_domain* dom, int32_t name, int64_t z0, int64_t nplanes, void** dptr, int64_t* bytes) {
    if (!dom || !dptr || !bytes) return fail(STKB_ERR_ARG, "null argument");
    if (int rc = check_name(dom, name, "stkb_plane_span")) return rc;
    cudaSetDevice(dom->desc.device);
    mark_halo_dirty(dom, dom->binding[name]);
    dom->halo_external = true;  // views for the halo exchange
    const Geometry& g = dom->g;
    if (nplanes < 0 || z0 < -g.order0 || z0 + nplanes > g.n0 + g.order0)
        return fail(STKB_ERR_ARG, "plane span outside the padded grid");
    *dptr = static_cast<char*>(dom->bufs[dom->binding[name]]) + size_t(z0 + g.order0) * size_t(g.plane) * dom->elem;
    *bytes = nplanes * g.plane * int64_t(dom->elem);
    return STKB_OK;
}

int stkb_run_target(stkb_domain* dom, void* const* host, int64_t iters) {
    if (!dom || !host) return fail(STKB_ERR_ARG, "null argument");
    for (int i = 0; i < dom->desc.n_grids; ++i)
        if (int rc = copy_h2d(dom, i, host[i])) return rc;
    if (int rc = stkb_run(dom, iters)) return rc;
    for (int i = 0; i < dom->desc.n_grids; ++i)
        if (int rc = copy_d2h(dom, i, host[i])) return rc;
    CUDA_TRY(cudaStreamSynchronize(dom->stream));
    return STKB_OK;
}

int stkb_compare(stkb_domain* dom, int32_t a, int32_t b, double* max_err, double* sum_sq, int64_t* worst,
                 double* scale) {
    if (!dom || !max_err || !sum_sq || !worst || !scale) return fail(STKB_ERR_ARG, "null argument");
    if (int rc = check_name(dom, a, "compare")) return rc;
    if (int rc = check_name(dom, b, "compare")) return rc;
    CUDA_TRY(cudaSetDevice(dom->desc.device));
    const int blocks = dom->num_sms * 4;
    const size_t pb = compare_partial_bytes();
    if (!dom->d_partials) CUDA_TRY(cudaMalloc(&dom->d_partials, blocks * pb));
    CUDA_TRY(launch_compare(dom->desc.dtype, dom->g, dom->bufs[dom->binding[a]], dom->bufs[dom->binding[b]],
                            dom->d_partials, blocks, dom->stream));
    std::vector<unsigned char> host(blocks * pb);
    CUDA_TRY(cudaMemcpyAsync(host.data(), dom->d_partials, blocks * pb, cudaMemcpyDeviceToHost, dom->stream));
    CUDA_TRY(cudaStreamSynchronize(dom->stream));
    struct P { double max_err, sum_sq, scale; long long worst; };
    double me = 0, ss = 0, sc = 0;
    long long w = -1;
    for (int i = 0; i < blocks; ++i) {
        P p;
        memcpy(&p, host.data() + i * pb, sizeof(P));
        if (p.worst >= 0 && (w < 0 || p.max_err > me || (p.max_err == me && p.worst < w))) { me = p.max_err; w = p.worst; }
        ss += p.sum_sq;
        sc = std::max(sc, p.scale);
    }
    *max_err = me;
    *sum_sq = ss;
    *worst = w;
    *scale = sc;
    return STKB_OK;
}

}  // extern "C"
