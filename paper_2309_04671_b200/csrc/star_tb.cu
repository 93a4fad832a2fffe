// Instantiations of the two-steps-per-sweep kernel (star_tb.cuh): fp32 / fp64, radius 1 (the
// host routes radius 1 only: see tb_map in stkb200.cu).
#include "star_tb.cuh"

namespace stkb {
cudaError_t launch_tb2_f32(const StarLaunch& L, const StarArgs<float>& a, cudaStream_t s) {
    switch (L.radius) {
        case 1: return launch_tb2_r<float, 1>(L, a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tb2_f64(const StarLaunch& L, const StarArgs<double>& a, cudaStream_t s) {
    switch (L.radius) {
        case 1: return launch_tb2_r<double, 1>(L, a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_frozen_ring(int dtype, const Geometry& g, const Box& b, int R, const void* buf, int32_t* flag,
                               int num_sms, cudaStream_t s, int zmask) {
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    if (dtype == 1) frozen_ring_kernel<float><<<2 * num_sms, 256, 0, s>>>(static_cast<const float*>(buf), g, b, R, flag, zmask);
    else frozen_ring_kernel<double><<<2 * num_sms, 256, 0, s>>>(static_cast<const double*>(buf), g, b, R, flag, zmask);
    return cudaGetLastError();
}

// dst's halo shell (every cell outside the interior, up to `order` away) := src's,
// one warp per padded row: whole rows in the d0/d1 halo, the 2*order d2 halo cells
// of interior rows.  The fused sweeps' scratch takes over u's halo this way when the
// map covers the whole interior (else the host copies the whole buffer).
__global__ void copy_halo_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, Geometry g,
                                 int esz) {
    const int64_t rows_per_plane = g.n1 + 2 * g.order, rows = (g.n0 + 2 * g.order0) * rows_per_plane;
    const int lane = threadIdx.x & 31;
    const int64_t row_bytes = g.pitch * esz;
    const int64_t lo = (g.lead - g.order) * esz, hi = (g.lead + g.n2 + g.order) * esz;
    for (int64_t r = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32; r < rows;
         r += int64_t(gridDim.x) * blockDim.x / 32) {
        const int64_t z = r / rows_per_plane, y = r - z * rows_per_plane;
        const unsigned char* s = src + r * row_bytes;
        unsigned char* d = dst + r * row_bytes;
        if (z < g.order0 || z >= g.order0 + g.n0 || y < g.order || y >= g.order + g.n1) {
            for (int64_t b = lo + lane * 4; b < hi; b += 128)  // 4-byte granules: lo/hi are 4-aligned
                *reinterpret_cast<uint32_t*>(d + b) = *reinterpret_cast<const uint32_t*>(s + b);
        } else {
            const int64_t nb = g.order * esz;  // bytes per side
            for (int64_t b = lane * 4; b < 2 * nb; b += 128) {
                const int64_t off = b < nb ? lo + b : (g.lead + g.n2) * esz + (b - nb);
                *reinterpret_cast<uint32_t*>(d + off) = *reinterpret_cast<const uint32_t*>(s + off);
            }
        }
    }
}

cudaError_t launch_copy_halo(const void* src, void* dst, const Geometry& g, int esz, int num_sms, cudaStream_t s) {
    copy_halo_kernel<<<4 * num_sms, 256, 0, s>>>(static_cast<const unsigned char*>(src),
                                                 static_cast<unsigned char*>(dst), g, esz);
    return cudaGetLastError();
}

int tb2_tile(int dtype, int radius, int* box_w, int* box_h, int* v_w, int* v_h) {
    if (dtype == 1) return tb2_tile_t<float>(radius, box_w, box_h, v_w, v_h);
    return tb2_tile_t<double>(radius, box_w, box_h, v_w, v_h);
}
}  // namespace stkb
