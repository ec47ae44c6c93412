// stage_ring_p3_f64.cu -- ring stage kernel, P3, double (one TU for parallel builds)
#include "stage_ring.cuh"
namespace dgl {
cudaError_t launch_ring_p3_f64(bool alpha, const StageArgs &a) {
  return alpha ? dgk::launch_ring<double, 1, 3, true>(a) : dgk::launch_ring<double, 1, 3, false>(a);
}
}  // namespace dgl
