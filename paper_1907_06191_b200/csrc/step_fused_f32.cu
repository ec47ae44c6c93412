// step_fused_f32.cu -- K3 fused SSP-RK3 step, float (one TU for parallel builds)
#include "step_fused.cuh"
namespace dgl {
cudaError_t launch_fused_f32(const StageArgs &a) { return dgk::launch_fused<float>(a); }
}  // namespace dgl
