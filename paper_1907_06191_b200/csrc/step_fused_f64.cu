// step_fused_f64.cu -- K3 fused SSP-RK3 step, double (one TU for parallel builds)
#include "step_fused.cuh"
namespace dgl {
cudaError_t launch_fused_f64(const StageArgs &a) { return dgk::launch_fused<double>(a); }
}  // namespace dgl
