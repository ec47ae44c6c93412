// stage_pair.cu -- K3d instances (fused SSP-RK3 stages 2 + 3): P1 / P2
// triangles, fp64 / fp32, in the ring kernel's state layout (P1: 16-byte
// lanes, P2: 8-byte lanes)
#include "stage_pair.cuh"
namespace dgl {
cudaError_t launch_pair(int prec, int P, const StageArgs &a) {
  if (P == 1) return prec == 64 ? dgk::launch_pair<double, 2, 1>(a) : dgk::launch_pair<float, 4, 1>(a);
  if (P == 2) return prec == 64 ? dgk::launch_pair<double, 1, 2>(a) : dgk::launch_pair<float, 2, 2>(a);
  return cudaErrorInvalidValue;
}
int pair_width() { return dgk::PairGeom<double, 2, 1>::W; }
}  // namespace dgl
