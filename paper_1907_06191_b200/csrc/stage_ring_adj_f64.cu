// stage_ring_adj_f64.cu -- ring stage kernel with the TRANSPOSED operator L^T
// (adjoint moments, opts.adjoint), fp64 P1 / P2 triangles and Q1 / Q2 (one TU)
#include "stage_ring.cuh"
namespace dgl {
cudaError_t launch_ring_adj_f64(int P, bool alpha, const StageArgs &a) {
  if (P == 1) return alpha ? dgk::launch_ring<double, 2, 1, true, true>(a) : dgk::launch_ring<double, 2, 1, false, true>(a);
  if (P == 2) return alpha ? dgk::launch_ring<double, 1, 2, true, true>(a) : dgk::launch_ring<double, 1, 2, false, true>(a);
  if (P == 101) return alpha ? dgk::launch_ring<double, 1, 101, true, true>(a) : dgk::launch_ring<double, 1, 101, false, true>(a);
  if (P == 102) return alpha ? dgk::launch_ring<double, 1, 102, true, true>(a) : dgk::launch_ring<double, 1, 102, false, true>(a);
  return cudaErrorInvalidValue;
}
}  // namespace dgl
