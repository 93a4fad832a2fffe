// Instantiations of the exact streaming star kernel (star_exact.cuh): fp32 / fp64 grids,
// radius 1..4, with or without the Jacobi divisor.
#include "star_exact.cuh"

namespace stkb {
cudaError_t launch_exact_f32(const StarLaunch& L, const StarArgs<float>& a, const XstarCoef& xc, cudaStream_t s) {
    return launch_exact_t<float>(L, a, xc, L.maps, s);
}

cudaError_t launch_exact_f64(const StarLaunch& L, const StarArgs<double>& a, const XstarCoef& xc, cudaStream_t s) {
    return launch_exact_t<double>(L, a, xc, L.maps, s);
}

cudaError_t launch_xwave_f32(const StarLaunch& L, const StarArgs<float>& a, const XwaveCoef& xc, cudaStream_t s) {
    return launch_xwave_t<float>(L, a, xc, L.maps, s);
}

cudaError_t launch_xwave_f64(const StarLaunch& L, const StarArgs<double>& a, const XwaveCoef& xc, cudaStream_t s) {
    return launch_xwave_t<double>(L, a, xc, L.maps, s);
}

// exact star and exact wave share the tile shape (one output row per warp, 15 warps)
int exact_tile(int dtype, int radius, int* bx, int* by, int* halo_x) {
    if (radius < 1 || radius > 4) return 1;
    if (dtype == 1) {
        *bx = XstarCfg<float, 1>::BX;
        *by = XstarCfg<float, 1>::BY;
        *halo_x = ((radius + 3) / 4) * 4;
    } else {
        *bx = XstarCfg<double, 1>::BX;
        *by = XstarCfg<double, 1>::BY;
        *halo_x = ((radius + 1) / 2) * 2;
    }
    return 0;
}
}  // namespace stkb
