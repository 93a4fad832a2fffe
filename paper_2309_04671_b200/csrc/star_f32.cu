// fp32 instantiations of the streaming star kernels.
#include "star_kernels.cuh"

namespace stkb {
cudaError_t launch_star_f32(const StarLaunch& L, const StarArgs<float>& a, cudaStream_t s) {
    return launch_star_t<float>(L, a, L.maps, s);
}
}  // namespace stkb
