// stage_ring_p1_f32.cu -- ring stage kernel, P1, float (one TU for parallel builds)
#include "stage_ring.cuh"
namespace dgl {
cudaError_t launch_ring_p1_f32(bool alpha, const StageArgs &a) {
  return alpha ? dgk::launch_ring<float, 4, 1, true>(a) : dgk::launch_ring<float, 4, 1, false>(a);
}
}  // namespace dgl
