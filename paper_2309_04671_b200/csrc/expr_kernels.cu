// Exact-evaluation and utility kernels.
//
// expr_kernel: evaluates a kernel's expression bytecode per point in float64,
// in parse order, with one rounding per store — the oracle's arithmetic rule
// (executor.py:1-10, _MapContext.eval executor.py:81-106, store :108-124) and
// the emitted templates' double-literal rule (codegen/common.py:88-113).  The
// IEEE double ops are explicit (__dadd_rn, __dmul_rn, ...) so no FMA
// contraction can change a rounding: results are bit-identical to run_target.
// Any kernel the reference accepts (star, box, "other", locals, scalars,
// several updates, 2-D) runs here; the tuned streaming kernels cover the star
// forms at HBM speed.
#include <algorithm>

#include "common.cuh"
#include "../../include/stkb200.h"

namespace stkb {

template <typename T>
struct ExprArgs {
    Geometry g;
    Box box;
    const int32_t* code;
    const double* consts;
    int32_t n_code;
    int32_t n_args;
    const T* rd[STKB_EXPR_MAX_ARGS];
    T* wr[STKB_EXPR_MAX_ARGS];
    int32_t* nonfinite;
};

template <typename T>
__global__ void __launch_bounds__(256) expr_kernel(const __grid_constant__ ExprArgs<T> a) {
    const int64_t e2 = a.box.hi2 - a.box.lo2;
    const int64_t e1 = a.box.hi1 - a.box.lo1;
    const int64_t e0 = a.box.hi0 - a.box.lo0;
    const int64_t n = e0 * e1 * e2;
    bool bad = false;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = a.box.lo2 + idx % e2;
        const int64_t y = a.box.lo1 + (idx / e2) % e1;
        const int64_t z = a.box.lo0 + idx / (e2 * e1);
        double stack[STKB_EXPR_MAX_STACK];
        double loc[STKB_EXPR_MAX_LOCALS];
        int sp = 0;
        for (int pc = 0; pc < a.n_code; ++pc) {
            const int32_t* ins = a.code + 5 * pc;
            const int op = __ldg(ins);
            const int i1 = __ldg(ins + 1);
            switch (op) {
                case STKB_OP_CONST: stack[sp++] = __ldg(a.consts + i1); break;
                case STKB_OP_READ: {
                    const int64_t off = a.g.at(z + __ldg(ins + 2), y + __ldg(ins + 3), x + __ldg(ins + 4));
                    stack[sp++] = double(a.rd[i1][off]);
                    break;
                }
                case STKB_OP_LOCAL: stack[sp++] = loc[i1]; break;
                case STKB_OP_ADD: --sp; stack[sp - 1] = __dadd_rn(stack[sp - 1], stack[sp]); break;
                case STKB_OP_SUB: --sp; stack[sp - 1] = __dsub_rn(stack[sp - 1], stack[sp]); break;
                case STKB_OP_MUL: --sp; stack[sp - 1] = __dmul_rn(stack[sp - 1], stack[sp]); break;
                case STKB_OP_DIV: --sp; stack[sp - 1] = __ddiv_rn(stack[sp - 1], stack[sp]); break;
                case STKB_OP_NEG: stack[sp - 1] = -stack[sp - 1]; break;
                case STKB_OP_SETLOCAL: loc[i1] = stack[--sp]; break;
                case STKB_OP_STORE: {
                    const int64_t off = a.g.at(z + __ldg(ins + 2), y + __ldg(ins + 3), x + __ldg(ins + 4));
                    const T v = T(stack[--sp]);
                    a.wr[i1][off] = v;
                    bad |= !isfinite(v);
                    break;
                }
                default: break;
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.nonfinite, 1);
}

template <typename T>
cudaError_t launch_expr_t(const Geometry& g, const Box& box, const int32_t* code, const double* consts,
                          int n_code, int n_args, const void* const* rd, void* const* wr, int32_t* flag,
                          int num_sms, cudaStream_t s) {
    ExprArgs<T> a{};
    a.g = g;
    a.box = box;
    a.code = code;
    a.consts = consts;
    a.n_code = n_code;
    a.n_args = n_args;
    for (int i = 0; i < n_args; ++i) {
        a.rd[i] = static_cast<const T*>(rd[i]);
        a.wr[i] = static_cast<T*>(wr[i]);
    }
    a.nonfinite = flag;
    const int64_t n = int64_t(box.hi0 - box.lo0) * (box.hi1 - box.lo1) * (box.hi2 - box.lo2);
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = int64_t(num_sms) * 8;
    if (blocks > cap) blocks = cap;
    expr_kernel<T><<<int(blocks), 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_expr(int dtype, const Geometry& g, const Box& box, const int32_t* code,
                        const double* consts, int n_code, int n_args, const void* const* rd,
                        void* const* wr, int32_t* flag, int num_sms, cudaStream_t s) {
    if (dtype == STKB_F32)
        return launch_expr_t<float>(g, box, code, consts, n_code, n_args, rd, wr, flag, num_sms, s);
    return launch_expr_t<double>(g, box, code, consts, n_code, n_args, rd, wr, flag, num_sms, s);
}

// ---------------------------------------------------------------------------
// compare (grids.py:163-174) over the interior: per-block partials, host finish

struct ComparePartial {
    double max_err;
    double sum_sq;
    double scale;
    long long worst;  // flat interior index, first occurrence of the max
};

template <typename T>
__global__ void __launch_bounds__(256) compare_kernel(Geometry g, const T* ref, const T* got,
                                                      ComparePartial* out) {
    __shared__ ComparePartial sh[256];
    const int64_t n = g.n0 * g.n1 * g.n2;
    ComparePartial p{0.0, 0.0, 0.0, -1};
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = idx % g.n2;
        const int64_t y = (idx / g.n2) % g.n1;
        const int64_t z = idx / (g.n2 * g.n1);
        const int64_t off = g.at(z, y, x);
        const double a = double(ref[off]);
        const double b = double(got[off]);
        const double d = fabs(a - b);
        if (p.worst < 0 || d > p.max_err) { p.max_err = d; p.worst = idx; }
        p.sum_sq += d * d;
        p.scale = fmax(p.scale, fabs(a));
    }
    sh[threadIdx.x] = p;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            ComparePartial o = sh[threadIdx.x + w];
            ComparePartial& m = sh[threadIdx.x];
            if (o.worst >= 0 && (m.worst < 0 || o.max_err > m.max_err ||
                                 (o.max_err == m.max_err && o.worst < m.worst))) {
                m.max_err = o.max_err;
                m.worst = o.worst;
            }
            m.sum_sq += o.sum_sq;
            m.scale = fmax(m.scale, o.scale);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

cudaError_t launch_compare(int dtype, const Geometry& g, const void* ref, const void* got, void* partials,
                           int blocks, cudaStream_t s) {
    if (dtype == STKB_F32)
        compare_kernel<float><<<blocks, 256, 0, s>>>(g, static_cast<const float*>(ref),
                                                      static_cast<const float*>(got),
                                                      static_cast<ComparePartial*>(partials));
    else
        compare_kernel<double><<<blocks, 256, 0, s>>>(g, static_cast<const double*>(ref),
                                                       static_cast<const double*>(got),
                                                       static_cast<ComparePartial*>(partials));
    return cudaGetLastError();
}

size_t compare_partial_bytes() { return sizeof(ComparePartial); }

// copy `nrows` rows of `row_words` 32-bit words between two row pitches
// (the unpitched GridBuffer layout <-> the 128-byte pitched device layout)
// rows [r0, r0 + nrows) of a host-layout box: row r is row r % rows_per_plane of plane
// r / rows_per_plane; one side is the contiguous staging buffer (row r - r0 at
// (r - r0) * row_words), the other the pitched device buffer (plane / row pitches)
__global__ void __launch_bounds__(256) repitch_kernel(uint32_t* __restrict__ stage, uint32_t* __restrict__ dev,
                                                      int64_t r0, int64_t nrows, int64_t rows_per_plane,
                                                      int64_t row_words, int64_t row_pitch, int64_t plane_pitch,
                                                      bool to_device) {
    for (int64_t k = blockIdx.x; k < nrows; k += gridDim.x) {
        const int64_t r = r0 + k;
        uint32_t* s = stage + k * row_words;
        uint32_t* d = dev + (r / rows_per_plane) * plane_pitch + (r % rows_per_plane) * row_pitch;
        if (to_device)
            for (int64_t i = threadIdx.x; i < row_words; i += blockDim.x) d[i] = s[i];
        else
            for (int64_t i = threadIdx.x; i < row_words; i += blockDim.x) s[i] = d[i];
    }
}

cudaError_t launch_repitch(void* stage, void* dev, int64_t r0, int64_t nrows, int64_t rows_per_plane,
                           int64_t row_bytes, int64_t row_pitch_bytes, int64_t plane_pitch_bytes, bool to_device,
                           int num_sms, cudaStream_t s) {
    if (nrows <= 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>(nrows, int64_t(num_sms) * 16);
    repitch_kernel<<<int(blocks), 256, 0, s>>>(static_cast<uint32_t*>(stage), static_cast<uint32_t*>(dev), r0, nrows,
                                               rows_per_plane, row_bytes / 4, row_pitch_bytes / 4,
                                               plane_pitch_bytes / 4, to_device);
    return cudaGetLastError();
}

__global__ void signal_add_kernel(int32_t* p, int32_t v) {
    __threadfence();
    atomicAdd(p, v);
}

// stream-ordered "these launches are done" marker for maps without an in-kernel
// signal; like the in-kernel one it only ever adds (the waiter tracks the sum)
cudaError_t launch_signal_add(int32_t* p, int32_t v, cudaStream_t s) {
    signal_add_kernel<<<1, 1, 0, s>>>(p, v);
    return cudaGetLastError();
}

}  // namespace stkb
