// f32 radius-1 instantiations of the streaming star kernels (one TU per radius: parallel builds).
#include "star_kernels.cuh"

namespace stkb {
cudaError_t launch_star_f32_r1(const StarLaunch& L, const StarArgs<float>& a, cudaStream_t s) {
    return launch_star_r<float, 1>(L, a, L.maps, s);
}
}  // namespace stkb
