// step_wave.cu -- K3c wavefront step (P1/P2 triangles, fp64/fp32)
#include "stage_wave.cuh"
namespace dgl {
int wave_band_rows() { return dgk::wave_band_rows(); }
cudaError_t launch_wave(int prec, int P, const StageArgs &a) {
  if (P == 1) return prec == 64 ? dgk::launch_wave<double, 2, 1>(a) : dgk::launch_wave<float, 4, 1>(a);
  return prec == 64 ? dgk::launch_wave<double, 1, 2>(a) : dgk::launch_wave<float, 2, 2>(a);
}
}  // namespace dgl
