// stage_v12_f64.cu -- v1/v2 stage kernels, fp64 (one TU for parallel builds)
#include "stage_v12.cuh"
namespace dgl {
cudaError_t launch_v12_f64(int which, int P, bool alpha, const StageArgs &a) {
  return dgk::launch_v12<double, 2>(which, P, alpha, a);
}
}  // namespace dgl
