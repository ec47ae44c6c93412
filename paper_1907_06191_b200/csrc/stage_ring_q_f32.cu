// stage_ring_q_f32.cu -- ring stage kernel, N4 quadrilaterals Q1 / Q2, float (one TU for parallel builds)
#include "stage_ring.cuh"
namespace dgl {
cudaError_t launch_ring_q_f32(int P, bool alpha, const StageArgs &a) {
  if (P == 101) return alpha ? dgk::launch_ring<float, 2, 101, true>(a) : dgk::launch_ring<float, 2, 101, false>(a);
  return alpha ? dgk::launch_ring<float, 2, 102, true>(a) : dgk::launch_ring<float, 2, 102, false>(a);
}
}  // namespace dgl
