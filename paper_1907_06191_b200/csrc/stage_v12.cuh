// stage_v12.cuh -- K2 v1 (operator table in global memory) and the launcher
// of v1/v2 (global-load kernels, 16-byte lanes).  Kept as references for the
// ring kernel and for parity/performance comparisons (opts.kernel = 1, 2).
#pragma once
#include "kernels.cuh"
#include "launch.h"
#include "stage_imm.cuh"

namespace dgk {

// ---------------------------------------------------------------------------
// K2 v1: one RK stage,  Uout = Uin + alpha (U0 - Uin) + cs * sum_o A[code][o] Uin[p+o]
// A in units D/h^2 (exact dyadic); cs = beta dt D/h^2 applied after the sum
// (SURVEY F4/F9).  One warp = one pixel x G sources; a CTA = WPB source groups
// of one contiguous range of pixels (pixel index uniform over the CTA).
// U0 may alias Uout (stage 3 writes u in place: same element, same thread).
// ---------------------------------------------------------------------------
template <typename T, int NV, int D2>
__device__ __forceinline__ void block_mv(T (&acc)[D2][NV], const T *__restrict__ Ab, const T (&x)[D2][NV]) {
#pragma unroll
  for (int r = 0; r < D2; r++)
#pragma unroll
    for (int c = 0; c < D2; c++) {
      T a = __ldg(Ab + r * D2 + c);
#pragma unroll
      for (int e = 0; e < NV; e++) acc[r][e] = fma(a, x[c][e], acc[r][e]);
    }
}

template <typename T, int NV, int D2, bool HAS_ALPHA>
__global__ void __launch_bounds__(256) k_stage(const T *__restrict__ Uin, const T *U0, T *Uout,
                                               const int4 *__restrict__ nbr, const T *__restrict__ A,
                                               int nact, int ngroups, int px_per_cta, T alpha, T cs) {
  constexpr int G = 32 * NV;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ngroups) return;
  const size_t gofs = (size_t)g * nact * D2 * G + lane * NV;
  const T *Ug = Uin + gofs;
  const int a0 = blockIdx.x * px_per_cta;
  const int a1 = min(nact, a0 + px_per_cta);
  for (int a = a0; a < a1; a++) {
    const int4 nb = __ldg(&nbr[a]);
    const int code = open_code(nb);
    const T *Ac = A + (size_t)code * 5 * D2 * D2;
    T xs[D2][NV], acc[D2][NV];
#pragma unroll
    for (int k = 0; k < D2; k++) ldv<T, NV>(Ug + ((size_t)a * D2 + k) * G, xs[k]);
#pragma unroll
    for (int k = 0; k < D2; k++)
#pragma unroll
      for (int e = 0; e < NV; e++) acc[k][e] = (T)0;
    block_mv<T, NV, D2>(acc, Ac, xs);
    const int nbi[4] = {nb.x, nb.y, nb.z, nb.w};
#pragma unroll
    for (int o = 0; o < 4; o++) {
      if (nbi[o] < 0) continue;  // closed face: neighbour is axon / outside, u+ = 0
      T xn[D2][NV];
#pragma unroll
      for (int k = 0; k < D2; k++) ldv<T, NV>(Ug + ((size_t)nbi[o] * D2 + k) * G, xn[k]);
      block_mv<T, NV, D2>(acc, Ac + (o + 1) * D2 * D2, xn);
    }
    T *out = Uout + gofs + (size_t)a * D2 * G;
    const T *u0 = U0 + gofs + (size_t)a * D2 * G;
#pragma unroll
    for (int k = 0; k < D2; k++) {
      T y[NV];
      if (HAS_ALPHA) {
        T z[NV];
        ldvc<T, NV>(u0 + (size_t)k * G, z);
#pragma unroll
        for (int e = 0; e < NV; e++) y[e] = xs[k][e] + alpha * (z[e] - xs[k][e]) + cs * acc[k][e];
      } else {
#pragma unroll
        for (int e = 0; e < NV; e++) y[e] = xs[k][e] + cs * acc[k][e];
      }
      stv<T, NV>(out + (size_t)k * G, y);
    }
  }
}


template <typename T, int NV>
cudaError_t launch_v12(int which, int P, bool alpha, const dgl::StageArgs &a) {
  dim3 grid((a.nact + a.px - 1) / a.px, (a.ngroups + a.wpb - 1) / a.wpb);
  const T *Uin = (const T *)a.Uin, *U0 = (const T *)a.U0;
  T *Uout = (T *)a.Uout;
  const T al = (T)a.alpha, cs = (T)a.cs;
  const int th = 32 * a.wpb;
  if (which == 0) {
    const T *A = (const T *)a.A;
    if (P == 1) {
      if (alpha) k_stage<T, NV, 6, true><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, A, a.nact, a.ngroups, a.px, al, cs);
      else k_stage<T, NV, 6, false><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, A, a.nact, a.ngroups, a.px, al, cs);
    } else {
      if (alpha) k_stage<T, NV, 12, true><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, A, a.nact, a.ngroups, a.px, al, cs);
      else k_stage<T, NV, 12, false><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, A, a.nact, a.ngroups, a.px, al, cs);
    }
  } else {
    if (P == 1) {
      if (alpha) k_stage_imm<T, NV, 1, true><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, a.nact, a.ngroups, a.px, al, cs);
      else k_stage_imm<T, NV, 1, false><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, a.nact, a.ngroups, a.px, al, cs);
    } else {
      if (alpha) k_stage_imm<T, NV, 2, true><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, a.nact, a.ngroups, a.px, al, cs);
      else k_stage_imm<T, NV, 2, false><<<grid, th, 0, a.st>>>(Uin, U0, Uout, a.nbr, a.nact, a.ngroups, a.px, al, cs);
    }
  }
  return cudaGetLastError();
}

}  // namespace dgk
