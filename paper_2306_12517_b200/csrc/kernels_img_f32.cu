// K1 instantiations for float output (split per type for a parallel build).
#include "image_kernel.cuh"

namespace bbx {
int launch_img_f32(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  return launch_img_typed<float>(P, A, st, vec);
}
}  // namespace bbx
