// stage_ring_p3_f32.cu -- ring stage kernel, P3, float (one TU for parallel builds)
#include "stage_ring.cuh"
namespace dgl {
cudaError_t launch_ring_p3_f32(bool alpha, const StageArgs &a) {
  return alpha ? dgk::launch_ring<float, 2, 3, true>(a) : dgk::launch_ring<float, 2, 3, false>(a);
}
}  // namespace dgl
