// K1 instantiations for uint8_t output (split per type for a parallel build).
#include "image_kernel.cuh"

namespace bbx {
int launch_img_u8(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  return launch_img_typed<uint8_t>(P, A, st, vec);
}
}  // namespace bbx
