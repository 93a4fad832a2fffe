// fp64 instantiations of the streaming star kernels.
#include "star_kernels.cuh"

namespace stkb {
cudaError_t launch_star_f64(const StarLaunch& L, const StarArgs<double>& a, cudaStream_t s) {
    return launch_star_t<double>(L, a, L.maps, s);
}

int star_tile(int dtype, int radius, int kind, int* bx, int* by, int* halo_x) {
    (void)kind;
    if (radius < 1 || radius > 4) return 1;
    if (dtype == 1) star_tile_t<float>(radius, bx, by, halo_x);
    else star_tile_t<double>(radius, bx, by, halo_x);
    return 0;
}
}  // namespace stkb
