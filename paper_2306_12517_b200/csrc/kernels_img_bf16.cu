// K1 instantiations for __nv_bfloat16 output (split per type for a parallel build).
#include "image_kernel.cuh"

namespace bbx {
int launch_img_bf16(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  return launch_img_typed<__nv_bfloat16>(P, A, st, vec);
}
}  // namespace bbx
