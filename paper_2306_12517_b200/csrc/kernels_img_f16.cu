// K1 instantiations for __half output (split per type for a parallel build).
#include "image_kernel.cuh"

namespace bbx {
int launch_img_f16(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  return launch_img_typed<__half>(P, A, st, vec);
}
}  // namespace bbx
