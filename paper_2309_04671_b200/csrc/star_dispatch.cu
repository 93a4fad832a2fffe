// Radius dispatch of the streaming star kernels and their host-side tile geometry.
#include "star_kernels.cuh"

namespace stkb {
#define DECL(tn, T)                                                                          \
    cudaError_t launch_star_##tn##_r1(const StarLaunch&, const StarArgs<T>&, cudaStream_t);  \
    cudaError_t launch_star_##tn##_r2(const StarLaunch&, const StarArgs<T>&, cudaStream_t);  \
    cudaError_t launch_star_##tn##_r3(const StarLaunch&, const StarArgs<T>&, cudaStream_t);  \
    cudaError_t launch_star_##tn##_r4(const StarLaunch&, const StarArgs<T>&, cudaStream_t);
DECL(f32, float)
DECL(f64, double)
#undef DECL

cudaError_t launch_star_f32(const StarLaunch& L, const StarArgs<float>& a, cudaStream_t s) {
    switch (L.radius) {
        case 1: return launch_star_f32_r1(L, a, s);
        case 2: return launch_star_f32_r2(L, a, s);
        case 3: return launch_star_f32_r3(L, a, s);
        case 4: return launch_star_f32_r4(L, a, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_star_f64(const StarLaunch& L, const StarArgs<double>& a, cudaStream_t s) {
    switch (L.radius) {
        case 1: return launch_star_f64_r1(L, a, s);
        case 2: return launch_star_f64_r2(L, a, s);
        case 3: return launch_star_f64_r3(L, a, s);
        case 4: return launch_star_f64_r4(L, a, s);
        default: return cudaErrorInvalidValue;
    }
}

int star_tile(int dtype, int radius, int kind, bool small, int* bx, int* by, int* halo_x) {
    if (radius < 1 || radius > 4) return 1;
    const bool box = kind == 4;  // STKB_MAP_BOX
    if (dtype == 1) star_tile_t<float>(radius, box, small, bx, by, halo_x);
    else star_tile_t<double>(radius, box, small, bx, by, halo_x);
    return 0;
}
}  // namespace stkb
