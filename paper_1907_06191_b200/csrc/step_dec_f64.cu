// step_dec_f64.cu -- K3b decoupled fused step, fp64 P1 (one TU for parallel builds)
#include "step_dec.cuh"
namespace dgl {
cudaError_t launch_dec_f64(const StageArgs &a) { return dgk::launch_step_dec(a); }
}  // namespace dgl
