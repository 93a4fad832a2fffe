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
                               int num_sms, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    if (dtype == 1) frozen_ring_kernel<float><<<2 * num_sms, 256, 0, s>>>(static_cast<const float*>(buf), g, b, R, flag);
    else frozen_ring_kernel<double><<<2 * num_sms, 256, 0, s>>>(static_cast<const double*>(buf), g, b, R, flag);
    return cudaGetLastError();
}

int tb2_tile(int dtype, int radius, int* box_w, int* box_h, int* v_w, int* v_h) {
    if (dtype == 1) return tb2_tile_t<float>(radius, box_w, box_h, v_w, v_h);
    return tb2_tile_t<double>(radius, box_w, box_h, v_w, v_h);
}
}  // namespace stkb
