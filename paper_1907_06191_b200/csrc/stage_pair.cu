// stage_pair.cu -- K3d instances (fused SSP-RK3 stages 2 + 3): P1 / P2
// triangles, fp64 / fp32, in the ring kernel's state layout (P1: 16-byte
// lanes, P2: 8-byte lanes).  Tuning builds (-DDGDIFF_TUNING) also carry other
// warp splits (DGDIFF_PAIR_WARPS=nb,nc) and diagnostics (DGDIFF_PAIR_DIAG);
// the product uses the defaults.
#include <cstdio>
#include "stage_pair.cuh"
namespace dgl {
namespace {
#ifdef DGDIFF_TUNING
int pair_diag() {
  static const int v = [] {
    const char *e = dgk::tune_env("DGDIFF_PAIR_DIAG");
    return e ? atoi(e) : 0;
  }();
  return v;
}
int pair_warps() {
  static const int v = [] {
    int nb = 0, nc = 0;
    if (const char *e = dgk::tune_env("DGDIFF_PAIR_WARPS")) sscanf(e, "%d,%d", &nb, &nc);
    return nb * 100 + nc;
  }();
  return v;
}
template <typename T, int NV, int P>
cudaError_t launch_tuned(const StageArgs &a) {
  switch (pair_warps()) {
    case 806: return dgk::launch_pair<T, NV, P, 8, 6>(a, pair_diag());
    case 804: return dgk::launch_pair<T, NV, P, 8, 4>(a, pair_diag());
    case 605: return dgk::launch_pair<T, NV, P, 6, 5>(a, pair_diag());
    case 704: return dgk::launch_pair<T, NV, P, 7, 4>(a, pair_diag());
    case 705: return dgk::launch_pair<T, NV, P, 7, 5>(a, pair_diag());
    case 706: return dgk::launch_pair<T, NV, P, 7, 6>(a, pair_diag());
    case 907: return dgk::launch_pair<T, NV, P, 9, 7>(a, pair_diag());
    case 1006: return dgk::launch_pair<T, NV, P, 10, 6>(a, pair_diag());
    default: return dgk::launch_pair<T, NV, P>(a, pair_diag());
  }
}
#else
template <typename T, int NV, int P>
cudaError_t launch_tuned(const StageArgs &a) {
  return dgk::launch_pair<T, NV, P>(a);
}
#endif
}  // namespace
cudaError_t launch_pair(int prec, int P, const StageArgs &a) {
  if (P == 1) return prec == 64 ? launch_tuned<double, 2, 1>(a) : launch_tuned<float, 4, 1>(a);
  if (P == 2) return prec == 64 ? launch_tuned<double, 1, 2>(a) : launch_tuned<float, 2, 2>(a);
  return cudaErrorInvalidValue;
}
int pair_width() { return dgk::PairGeom<double, 2, 1>::W; }
}  // namespace dgl
