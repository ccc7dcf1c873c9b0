// double instantiation of the fused step kernels (csrc/step_impl.cuh).
#include "step_impl.cuh"

namespace tlbm {
int step_launch_f64(const tlbm_step_args *a, cudaStream_t s) {
    return step_detail::launch_dtype<double>(a, s);
}
}  // namespace tlbm
