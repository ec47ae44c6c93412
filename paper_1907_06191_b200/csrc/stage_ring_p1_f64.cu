// stage_ring_p1_f64.cu -- ring stage kernel, P1, double (one TU for parallel builds)
#include "stage_ring.cuh"
namespace dgl {
cudaError_t launch_ring_p1_f64(bool alpha, const StageArgs &a) {
  return alpha ? dgk::launch_ring<double, 2, 1, true>(a) : dgk::launch_ring<double, 2, 1, false>(a);
}
}  // namespace dgl
