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

template <typename T, int R>
static void tile_of(bool wave, int* bx, int* by, int* halo_x) {
    if (wave) {
        *bx = XwaveCfg<T, R>::BX;
        *by = XwaveCfg<T, R>::BY;
        *halo_x = XwaveCfg<T, R>::RA;
    } else {
        *bx = XstarCfg<T, R>::BX;
        *by = XstarCfg<T, R>::BY;
        *halo_x = XstarCfg<T, R>::RA;
    }
}

template <typename T>
static int tile_t(int radius, bool wave, int* bx, int* by, int* halo_x) {
    switch (radius) {
        case 1: tile_of<T, 1>(wave, bx, by, halo_x); return 0;
        case 2: tile_of<T, 2>(wave, bx, by, halo_x); return 0;
        case 3: tile_of<T, 3>(wave, bx, by, halo_x); return 0;
        case 4: tile_of<T, 4>(wave, bx, by, halo_x); return 0;
        default: return 1;
    }
}

// tile of the exact star (wave = false) or exact wave kernel, for the host's tensor-map boxes
int exact_tile(int dtype, int radius, bool wave, int* bx, int* by, int* halo_x) {
    return dtype == 1 ? tile_t<float>(radius, wave, bx, by, halo_x) : tile_t<double>(radius, wave, bx, by, halo_x);
}
}  // namespace stkb
