// stage_v12_f32.cu -- v1/v2 stage kernels, fp32 (one TU for parallel builds)
#include "stage_v12.cuh"
namespace dgl {
cudaError_t launch_v12_f32(int which, int P, bool alpha, const StageArgs &a) {
  return dgk::launch_v12<float, 4>(which, P, alpha, a);
}
}  // namespace dgl
