// float instantiation of the fused step kernels (csrc/step_impl.cuh).
#include "step_impl.cuh"

namespace tlbm {
int step_launch_f32(const tlbm_step_args *a, cudaStream_t s) {
    return step_detail::launch_dtype<float>(a, s);
}
}  // namespace tlbm
