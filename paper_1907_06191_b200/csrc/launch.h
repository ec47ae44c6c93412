// launch.h -- host-side launchers of the stage kernels (one translation unit
// per kernel family / precision / degree, compiled in parallel).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace dgl {

struct StageArgs {
  const void *Uin = nullptr, *U0 = nullptr;  // U0 may alias Uout (stage 3)
  void *Uout = nullptr;
  const int4 *nbr = nullptr;
  const void *A = nullptr;          // v1 only: operator table in global memory
  const void *Aabs = nullptr;       // ring, ABSORB: [16][16][5][2d][2d] boundary-pixel blocks
  const int4 *rowtab = nullptr;     // ring only: [nstrips][ny] {h0, c0, c1, h1}
  const int4 *rowtab_na = nullptr;  // ring, no-alpha stage: its own strip width
  int nstrips_na = 0, n1_use_na = 0;
  int nact = 0, ny = 0, nstrips = 0, ngroups = 0, nsm = 148;
  int px = 32, wpb = 4;             // v1/v2 mapping
  int diag = 0;                     // ring diagnostic (stream without compute)
  int ahead_alpha = 0, ahead_noalpha = 0;  // ring: max rows in flight (0 = default)
  int n1_use = 0, n2_use = 0;       // ring: slots used of rings 1 / 2 (0 = all)
  double alpha = 0, cs = 0;
  // ring, N1 active windows: per source group the bounding box {x0, x1, y0, y1}
  // of its sources; only output rows / strips within the box grown by wr
  // pixels are computed (nullptr = the whole grid)
  const int4 *gbox = nullptr;
  int wr = 0;
  int band_rows = 0;                // ring: max rows per band (0 = heuristic)
  // K3c wavefront step: per-item completion counters, (stage, band) order of a
  // group's items, 1-based step index within the chunk
  unsigned *wave_cnt = nullptr;
  const int2 *wave_tab = nullptr;
  unsigned wave_epoch = 0;
  // K3d: strip-major 16-bit neighbour table of the U2 pixels (see stage_pair.cuh)
  const uint16_t *nbs = nullptr;
  // ring, quads: strip-major copies of the neighbour table (per strip, rows in
  // order, each row's computed pixels) and their offsets [nstrips][ny + 1], for
  // the alpha stages (nbi) and the stage without alpha (nbi_na; its strips may
  // differ)
  const int4 *nbi = nullptr, *nbi_na = nullptr;
  const int *nbi_off = nullptr, *nbi_off_na = nullptr;
  cudaStream_t st = nullptr;
};

// which: 0 = v1 (table in gmem), 1 = v2 (immediates), 2 = v3 ring (bulk TMA)
cudaError_t launch_stage(int which, int prec, int P, bool alpha, const StageArgs &a);
// strip width of the ring kernel for degree code P (1..3 triangles, 101/102
// quads; its row table depends on it)
int ring_width(int P, bool alpha);
// K3: one fused SSP-RK3 step per pass (P1); a.rowtab = rowtab3 [nstrips][ny][2]
cudaError_t launch_step_fused(int prec, const StageArgs &a);
int fused_width(int prec);
cudaError_t launch_fused_f64(const StageArgs &a);
cudaError_t launch_fused_f32(const StageArgs &a);
// K3b: the fused step with decoupled warp roles (fp64 P1, temporal_steps = 3)
cudaError_t launch_dec_f64(const StageArgs &a);

// K3c: one SSP-RK3 step as an L2-resident wavefront of ring items (temporal_steps
// = 4; P1/P2 triangles, REFLECT): a.Uin = u (in place), a.U0 = U1, a.Uout = U2
cudaError_t launch_wave(int prec, int P, const StageArgs &a);
int wave_band_rows();

// K3d: SSP-RK3 stages 2 and 3 fused in one launch (temporal_steps = 5; P1/P2
// triangles, REFLECT): a.Uin = U1, a.U0 = u (read only), a.Uout = u' (must not
// alias u), a.rowtab = the pair row table [nstrips][ny][2] of strips pair_width()
cudaError_t launch_pair(int prec, int P, const StageArgs &a);
int pair_width();

// per-TU entry points
cudaError_t launch_v12_f64(int which, int P, bool alpha, const StageArgs &a);
cudaError_t launch_v12_f32(int which, int P, bool alpha, const StageArgs &a);
cudaError_t launch_ring_p1_f64(bool alpha, const StageArgs &a);
cudaError_t launch_ring_p1_f32(bool alpha, const StageArgs &a);
cudaError_t launch_ring_p2_f64(bool alpha, const StageArgs &a);
cudaError_t launch_ring_p2_f32(bool alpha, const StageArgs &a);
cudaError_t launch_ring_p3_f64(bool alpha, const StageArgs &a);
cudaError_t launch_ring_p3_f32(bool alpha, const StageArgs &a);
cudaError_t launch_ring_q_f64(int P, bool alpha, const StageArgs &a);   // P = 101 (Q1), 102 (Q2)
// the ring kernel with the transposed operator L^T (adjoint moments; fp64 P1/P2)
cudaError_t launch_ring_adj_f64(int P, bool alpha, const StageArgs &a);
cudaError_t launch_ring_q_f32(int P, bool alpha, const StageArgs &a);

}  // namespace dgl
