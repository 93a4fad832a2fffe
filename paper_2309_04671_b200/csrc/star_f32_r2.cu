// f32 radius-2 instantiations of the streaming star kernels (one TU per radius: parallel builds).
#include "star_kernels.cuh"

namespace stkb {
cudaError_t launch_star_f32_r2(const StarLaunch& L, const StarArgs<float>& a, cudaStream_t s) {
    return launch_star_r<float, 2>(L, a, L.maps, s);
}
}  // namespace stkb
