// launch.cu -- dispatch of the stage kernels to their translation units
#include "launch.h"
#include "stage_ring.cuh"
#include "step_fused.cuh"

namespace dgl {

int ring_width(int P, bool alpha) {
  using namespace dgk;
  if (P == 1) {
    const int m = ring_mode<1>(alpha);
    return m == RING_PLAIN ? RingCfg<1, 16, RING_PLAIN>::W
           : m == RING_U0_STAGED ? RingCfg<1, 16, RING_U0_STAGED>::W : RingCfg<1, 16, RING_U0_DIRECT>::W;
  }
  if (P == 101 || P == 102) {
    const int m1 = ring_mode<101>(alpha), m2 = ring_mode<102>(alpha);
    if (P == 101)
      return m1 == RING_PLAIN ? RingCfg<101, 8, RING_PLAIN>::W
             : m1 == RING_U0_STAGED ? RingCfg<101, 8, RING_U0_STAGED>::W : RingCfg<101, 8, RING_U0_DIRECT>::W;
    return m2 == RING_PLAIN ? RingCfg<102, 8, RING_PLAIN>::W
           : m2 == RING_U0_STAGED ? RingCfg<102, 8, RING_U0_STAGED>::W : RingCfg<102, 8, RING_U0_DIRECT>::W;
  }
  if (P == 3) {
    const int m = ring_mode<3>(alpha);
    return m == RING_PLAIN ? RingCfg<3, 8, RING_PLAIN>::W
           : m == RING_U0_STAGED ? RingCfg<3, 8, RING_U0_STAGED>::W : RingCfg<3, 8, RING_U0_DIRECT>::W;
  }
  const int m = ring_mode<2>(alpha);
  return m == RING_PLAIN ? RingCfg<2, 8, RING_PLAIN>::W
         : m == RING_U0_STAGED ? RingCfg<2, 8, RING_U0_STAGED>::W : RingCfg<2, 8, RING_U0_DIRECT>::W;
}

cudaError_t launch_stage(int which, int prec, int P, bool alpha, const StageArgs &a) {
  if (which == 0 || which == 1)
    return prec == 64 ? launch_v12_f64(which, P, alpha, a) : launch_v12_f32(which, P, alpha, a);
  if (P == 1) return prec == 64 ? launch_ring_p1_f64(alpha, a) : launch_ring_p1_f32(alpha, a);
  if (P == 3) return prec == 64 ? launch_ring_p3_f64(alpha, a) : launch_ring_p3_f32(alpha, a);
  if (P > 100) return prec == 64 ? launch_ring_q_f64(P, alpha, a) : launch_ring_q_f32(P, alpha, a);
  return prec == 64 ? launch_ring_p2_f64(alpha, a) : launch_ring_p2_f32(alpha, a);
}

int fused_width(int prec) { return prec == 64 ? dgk::FusedCfg<double>::W : dgk::FusedCfg<float>::W; }

cudaError_t launch_step_fused(int prec, const StageArgs &a) {
  return prec == 64 ? launch_fused_f64(a) : launch_fused_f32(a);
}

}  // namespace dgl
