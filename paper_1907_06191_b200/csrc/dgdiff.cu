// dgdiff.cu -- C-ABI (include/dgdiff.h), host driver and sm_100a kernels of the
// hot path of arXiv 1907.06191 (PAPER.md, cited P:<line>).
//
//   K1 k_init      Dirac Cauchy data for a chunk of sources
//   K2 k_stage_ring one SSP-RK3 stage of the DG operator (Eq. (7))
//                  as a 5-point composite stencil over extracellular pixels
//   K3 k_step_fused (temporal blocking, opt-in; step_fused.cuh)
//   K4 k_moments   m00 m10 m01 m20 m11 m02 per source
//   K5 k_finalize  mixture mean and covariance Sigma; preceded by
//                  one ncclAllReduce of the moment table when nranks > 1
//
// No CPU fallback exists: every step of the path runs in these kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dgdiff.h"
#include "kernels.cuh"
#include "operator.h"
#include "launch.h"
#include "mc_walk.cuh"
#include "stage_imm.cuh"  // compile-time operator (tab<P>) for the create-time check

using namespace dgk;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;
static dgdiff_status fail(dgdiff_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? DGDIFF_E_NOMEM : DGDIFF_E_CUDA,        \
                  "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__);       \
  } while (0)

// ---------------------------------------------------------------------------
// device constants
// ---------------------------------------------------------------------------
#define DMAXK 10                   // max dofs per triangle on the GPU path (P3)
// per-handle tables passed by value as kernel parameters (they live in the
// launch's constant bank; a module-wide __constant__ would be shared by every
// handle of the process, whatever its degree / element type)
struct MomW { double w[2 * 6 * DMAXK]; };   // moment weights (unit pixel)
struct CentreW { double v[2 * DMAXK]; };    // basis values at the pixel centre (mixture nodes)

struct InitVals { double v[2 * DMAXK]; };  // projected Dirac / h^2

// ---------------------------------------------------------------------------
// K1: zero the chunk's u and write the projected Dirac at each source pixel
// ---------------------------------------------------------------------------
// N1 windows: per group g only the active range [grange[g].x, grange[g].y)
// (the rows the group's stages can read) is written, and the two work
// registers Za, Zb are zeroed over the same range (blockIdx.y = group)
template <typename T, int NV, int D2>
__global__ void __launch_bounds__(256) k_init_win(T *__restrict__ U, T *__restrict__ Za, T *__restrict__ Zb,
                                                  int nact, const int2 *__restrict__ grange,
                                                  const int *__restrict__ src_a, InitVals iv,
                                                  const double *__restrict__ px, int64_t nvalid) {
  constexpr int G = 32 * NV;
  const int g = blockIdx.y;
  const int2 rg = __ldg(&grange[g]);
  const int64_t base = ((int64_t)g * nact + rg.x) * D2 * 32;
  const int64_t nvec = (int64_t)(rg.y - rg.x) * D2 * 32;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(v & 31);
    const int64_t r = v >> 5;
    const int k = (int)(r % D2);
    const int a = rg.x + (int)(r / D2);
    T x[NV], z[NV];
#pragma unroll
    for (int e = 0; e < NV; e++) {
      const int s = g * G + lane * NV + e;
      const double iv_k = px ? __ldg(&px[min((int64_t)s, nvalid - 1) * (2 + D2) + 2 + k]) : iv.v[k];
      x[e] = (__ldg(&src_a[s]) == a) ? (T)iv_k : (T)0;
      z[e] = (T)0;
    }
    stv<T, NV>(U + (base + v) * NV, x);
    stv<T, NV>(Za + (base + v) * NV, z);
    stv<T, NV>(Zb + (base + v) * NV, z);
  }
}

template <typename T, int NV, int D2>
__global__ void __launch_bounds__(256) k_init(T *__restrict__ U, int64_t nvec, int nact,
                                              const int *__restrict__ src_a, InitVals iv,
                                              const double *__restrict__ px /* nullable: [nvalid][2 + D2] */,
                                              int64_t nvalid) {
  constexpr int G = 32 * NV;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    int lane = (int)(v & 31);
    int64_t r = v >> 5;               // (g, a, k)
    int k = (int)(r % D2);
    int64_t ga = r / D2;
    int a = (int)(ga % nact);
    int64_t g = ga / nact;
    T x[NV];
#pragma unroll
    for (int e = 0; e < NV; e++) {
      int s = (int)(g * G + lane * NV + e);
      const double iv_k = px ? __ldg(&px[min((int64_t)s, nvalid - 1) * (2 + D2) + 2 + k]) : iv.v[k];
      x[e] = (__ldg(&src_a[s]) == a) ? (T)iv_k : (T)0;
    }
    stv<T, NV>(U + v * NV, x);
  }
}

// ---------------------------------------------------------------------------
// K4: per-source moments about the source point (readings R12, R14):
//   m_ab = h^(2+a+b) sum_pixels sum_T sum_j c_j int (xi+X)^a (eta+Y)^b N_j
// with X = i - xs, Y = j - ys, (xs, ys) the source point in pixel units (the
// pixel centre is + 1/2 for pixel sources; N4 sub-pixel points otherwise).  fp64 accumulation.  Each CTA
// reduces a contiguous pixel range; k_mom_reduce then sums the per-CTA
// partials in CTA order (deterministic, independent of chunking and ranks).
// ---------------------------------------------------------------------------
template <typename T, int NV, int D2>
__global__ void __launch_bounds__(256) k_moments(const T *__restrict__ U, const int2 *__restrict__ pix,
                                                 const double2 *__restrict__ src_xy, int nact, int ngroups,
                                                 int px_per_cta, double *__restrict__ partial,
                                                 int64_t chunk, const int2 *__restrict__ grange /* nullable (N1) */,
                                                 MomW mw) {
  constexpr int NT = (D2 == 4 || D2 == 9) ? 1 : 2;   // elements per pixel (quads: 1)
  constexpr int G = 32 * NV, d = D2 / NT;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ngroups) return;
  const T *Ug = U + (size_t)g * nact * D2 * G + lane * NV;
  double is[NV], js[NV], m[6][NV];
#pragma unroll
  for (int e = 0; e < NV; e++) {
    const double2 s = __ldg(&src_xy[g * G + lane * NV + e]);
    is[e] = s.x;
    js[e] = s.y;
#pragma unroll
    for (int q = 0; q < 6; q++) m[q][e] = 0.0;
  }
  int a0 = blockIdx.x * px_per_cta;
  int a1 = min(nact, a0 + px_per_cta);
  if (grange) {   // N1: outside the group's range the state is zero (and not maintained)
    const int2 rg = __ldg(&grange[g]);
    a0 = max(a0, rg.x);
    a1 = min(a1, rg.y);
  }
  for (int a = a0; a < a1; a++) {
    const int2 ij = __ldg(&pix[a]);
    T c[D2][NV];
#pragma unroll
    for (int k = 0; k < D2; k++) ldv<T, NV>(Ug + ((size_t)a * D2 + k) * G, c[k]);
#pragma unroll
    for (int e = 0; e < NV; e++) {
      double P[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int t = 0; t < NT; t++)
#pragma unroll
        for (int q = 0; q < 6; q++)
#pragma unroll
          for (int j = 0; j < d; j++) P[q] = fma(mw.w[(t * 6 + q) * DMAXK + j], (double)c[t * d + j][e], P[q]);
      const double X = ij.x - is[e], Y = ij.y - js[e];
      m[0][e] += P[0];
      m[1][e] += P[1] + X * P[0];
      m[2][e] += P[2] + Y * P[0];
      m[3][e] += P[3] + 2.0 * X * P[1] + X * X * P[0];
      m[4][e] += P[4] + X * P[2] + Y * P[1] + X * Y * P[0];
      m[5][e] += P[5] + 2.0 * Y * P[2] + Y * Y * P[0];
    }
  }
#pragma unroll
  for (int e = 0; e < NV; e++) {
    double *o = partial + ((size_t)blockIdx.x * chunk + g * G + lane * NV + e) * 6;
#pragma unroll
    for (int q = 0; q < 6; q++) o[q] = m[q][e];
  }
}

// sum the partials in a fixed order (deterministic, independent of chunking
// and ranks): one warp per source, lane l sums the CTAs b = l, l + 32, ... in
// increasing order, then a fixed shuffle tree; scale by h powers; write rows
// of the table.  (Round 2: the one-thread-per-source loop over all CTAs took
// 3.6 ms per chunk -- latency-bound with a few hundred threads -- i.e. 9 % of
// a windowed c4 solve.)
__global__ void __launch_bounds__(256) k_mom_reduce(const double *__restrict__ partial, int nblk, int64_t chunk,
                                                    int64_t nvalid, double h, double *__restrict__ mom /* rows of this chunk */,
                                                    const int32_t *__restrict__ dest /* nullable: also scatter row s to */,
                                                    double *__restrict__ mom_all /* row dest[s] (N1 sorted chunks) */) {
  const int lane = threadIdx.x & 31;
  const int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nvalid) return;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int b = lane; b < nblk; b += 32) {
    const double *p = partial + ((size_t)b * chunk + s) * 6;
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] += p[q];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] += __shfl_down_sync(0xffffffffu, acc[q], off);
  if (lane != 0) return;
  const double h2 = h * h, h3 = h2 * h, h4 = h2 * h2;
  double *o = mom + s * 6;
  o[0] = acc[0] * h2;
  o[1] = acc[1] * h3;
  o[2] = acc[2] * h3;
  o[3] = acc[3] * h4;
  o[4] = acc[4] * h4;
  o[5] = acc[5] * h4;
  if (dest) {
    double *a = mom_all + (size_t)dest[s] * 6;
#pragma unroll
    for (int q = 0; q < 6; q++) a[q] = o[q];
  }
}

// ---------------------------------------------------------------------------
// Adjoint moments (opts.adjoint, round 2).  The scheme is linear, so a
// source's moment m = w_s^T P(dt L)^N u0_s equals (P(dt L^T)^N w_s)^T u0_s,
// and the weights w_s of (x - x_s)^a (y - y_s)^b are combinations of the six
// weight fields of 1, x', y', x'^2, x'y', y'^2 (x' = x - x_o about an origin
// o).  k_adj_init writes those fields for AO origins into lanes 6 o + q of one
// source group (the other lanes zero); the stages then run with the
// transposed table; k_adj_eval reads each source's six values at its pixel
// (against the projected Dirac, as K4 integrates a density) and re-centres
// them on the source point.
// ---------------------------------------------------------------------------
constexpr int ADJ_MAXO = 30;                   // origins (6 field lanes each)
template <int G> __host__ __device__ constexpr int adj_per_group() { return G / 6; }
template <int G> __host__ __device__ constexpr int adj_groups() { return (ADJ_MAXO + G / 6 - 1) / (G / 6); }
struct AdjOrigins { double x[ADJ_MAXO], y[ADJ_MAXO]; int n; };

template <int D2, int G, int NT>
__global__ void k_adj_init(double *__restrict__ U, const int2 *__restrict__ pix, int nact, double h, MomW mw,
                           AdjOrigins org) {
  constexpr int d = D2 / NT, OPG = adj_per_group<G>();   // NT elements per pixel (quads: 1)
  const int64_t per_group = (int64_t)nact * D2 * G;
  const int64_t total = per_group * adj_groups<G>();
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx % G);
    const int k = (int)((idx / G) % D2);
    const int a = (int)((idx % per_group) / ((int64_t)G * D2));
    const int gi = (int)(idx / per_group);
    const int o = lane / 6 < OPG ? gi * OPG + lane / 6 : ADJ_MAXO, q = lane % 6;
    double v = 0.0;
    if (o < org.n) {
      const int t = k / d, jl = k % d;
      const int2 ij = __ldg(&pix[a]);
      const double X = ij.x - org.x[o], Y = ij.y - org.y[o];
      const double *w = mw.w + t * 6 * DMAXK + jl;   // unit-pixel integrals of xi^a eta^b N_jl
      const double w00 = w[0], w10 = w[DMAXK], w01 = w[2 * DMAXK], w20 = w[3 * DMAXK], w11 = w[4 * DMAXK],
                   w02 = w[5 * DMAXK];
      const double h2 = h * h, h3 = h2 * h, h4 = h2 * h2;
      v = q == 0 ? h2 * w00
        : q == 1 ? h3 * (w10 + X * w00)
        : q == 2 ? h3 * (w01 + Y * w00)
        : q == 3 ? h4 * (w20 + 2.0 * X * w10 + X * X * w00)
        : q == 4 ? h4 * (w11 + X * w01 + Y * w10 + X * Y * w00)
                 : h4 * (w02 + 2.0 * Y * w01 + Y * Y * w00);
    }
    U[idx] = v;
  }
}

template <int D2, int G>
__global__ void k_adj_eval(const double *__restrict__ U, int nact, const int32_t *__restrict__ src, int64_t b, int64_t nloc,
                           const int *__restrict__ aidx, int nx, double h, InitVals iv, AdjOrigins org,
                           double *__restrict__ mom, const double *__restrict__ px /* nullable: points, shard rows */) {
  constexpr int OPG = adj_per_group<G>();
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nloc) return;
  const int64_t s = b + k;
  const int i = src[2 * s], j = src[2 * s + 1];
  const int a = __ldg(&aidx[(size_t)j * nx + i]);
  // N4 sub-pixel points: the point and its projected-Dirac row (R21)
  const double *row = px ? px + k * (2 + D2) : nullptr;
  const double xs = row ? row[0] : i + 0.5, ys = row ? row[1] : j + 0.5;
  int o = 0;
  double best = 1e300;
  for (int c = 0; c < org.n; c++) {
    const double dx = xs - org.x[c], dy = ys - org.y[c], r = dx * dx + dy * dy;
    if (r < best) { best = r; o = c; }
  }
  double E[6];
#pragma unroll
  for (int q = 0; q < 6; q++) {
    double e = 0.0;
#pragma unroll
    for (int kk = 0; kk < D2; kk++)
      e = fma(U[(size_t)(o / OPG) * nact * D2 * G + ((size_t)a * D2 + kk) * G + 6 * (o % OPG) + q],
              row ? row[2 + kk] : iv.v[kk], e);
    E[q] = e;
  }
  const double dX = h * (xs - org.x[o]), dY = h * (ys - org.y[o]);
  double *m = mom + s * 6;
  m[0] = E[0];
  m[1] = E[1] - dX * E[0];
  m[2] = E[2] - dY * E[0];
  m[3] = E[3] - 2.0 * dX * E[1] + dX * dX * E[0];
  m[4] = E[4] - dX * E[2] - dY * E[1] + dX * dY * E[0];
  m[5] = E[5] - 2.0 * dY * E[2] + dY * dY * E[0];
}

// ---------------------------------------------------------------------------
// K5: mixture and its covariance from the full
// [n][6] table, fixed-order reduction (bitwise identical on every rank).
// out[0..5] = sxx sxy syy mux muy flags (bit0 degenerate, bit1 non-finite)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_finalize(const double *__restrict__ mom, int64_t n, int centering,
                                                  double *__restrict__ out) {
  __shared__ double sh[5][256];
  __shared__ int shf[256];
  const int t = threadIdx.x;
  const int64_t b = n * t / 256, e = n * (t + 1) / 256;
  double s[5] = {0, 0, 0, 0, 0};
  int flag = 0;
  for (int64_t i = b; i < e; i++) {
    const double *m = mom + i * 6;
    if (!(m[0] > 0)) flag |= isfinite(m[0]) ? 1 : 2;
    double ux = m[1] / m[0], uy = m[2] / m[0];  // centring + normalisation
    double xx = m[3] / m[0], xy = m[4] / m[0], yy = m[5] / m[0];
    if (centering == 1) { xx -= ux * ux; xy -= ux * uy; yy -= uy * uy; ux = 0; uy = 0; }
    s[0] += ux; s[1] += uy; s[2] += xx; s[3] += xy; s[4] += yy;
  }
  for (int q = 0; q < 5; q++) sh[q][t] = s[q];
  shf[t] = flag;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) {
      for (int q = 0; q < 5; q++) sh[q][t] += sh[q][t + w];
      shf[t] |= shf[t + w];
    }
    __syncthreads();
  }
  if (t == 0) {
    double inv = 1.0 / (double)n;
    double mx = sh[0][0] * inv, my = sh[1][0] * inv;
    out[0] = sh[2][0] * inv - mx * mx;
    out[1] = sh[3][0] * inv - mx * my;
    out[2] = sh[4][0] * inv - my * my;
    out[3] = mx;
    out[4] = my;
    int f = shf[0];
    for (int q = 0; q < 3; q++)
      if (!isfinite(out[q])) f |= 2;
    out[5] = (double)f;
  }
}

// canonical fp64 copy of one source's state: out[a][k]
// (N1 windows: outside group g's maintained range [grange.x, grange.y) the
// registers are not maintained and the density is exactly zero)
template <typename T, int NV, int D2>
__global__ void k_gather(const T *__restrict__ U, int nact, int g, int slot, double *__restrict__ out,
                         const int2 *__restrict__ grange /* nullable */) {
  constexpr int G = 32 * NV;
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= (int64_t)nact * D2) return;
  if (grange) {
    const int2 rg = grange[g];
    const int64_t a = r / D2;
    if (a < rg.x || a >= rg.y) {
      out[r] = 0.0;
      return;
    }
  }
  out[r] = (double)U[((size_t)g * nact * D2 + r) * G + slot];
}

// source pixel -> active index for a chunk (padding slots repeat the last
// valid source, so they never widen an N1 group box)
// (src_xy = source point in pixel units: the pixel centre, or the N4
// sub-pixel point from px[k][0..1])
__global__ void k_src_prep(const int32_t *__restrict__ src, int64_t nvalid, int64_t chunk,
                           const int *__restrict__ aidx, int nx, int *__restrict__ src_a,
                           int2 *__restrict__ src_ij, double2 *__restrict__ src_xy,
                           const double *__restrict__ px, int pxs) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= chunk) return;
  int64_t k = s < nvalid ? s : nvalid - 1;
  int i = src[2 * k], j = src[2 * k + 1];
  src_a[s] = aidx[(size_t)j * nx + i];
  src_ij[s] = make_int2(i, j);
  src_xy[s] = px ? make_double2(px[k * pxs], px[k * pxs + 1]) : make_double2(i + 0.5, j + 0.5);
}

// ---------------------------------------------------------------------------
// N2: mixture density grid on the displacement lattice [-R, R]^2.
// One thread per node (dx, dy) loops over the chunk's sources in order (fixed
// summation order: deterministic).  Node value of source s: the mean of the L
// and U traces at the centre of pixel (is+dx, js+dy), divided by m00_s.
// ---------------------------------------------------------------------------
template <typename T, int NV, int D2>
__global__ void k_mixture(const T *__restrict__ U, const int *__restrict__ aidx, int nx, int ny, int nact,
                          const int2 *__restrict__ src_ij, const double *__restrict__ mom, int64_t nvalid, int R,
                          double *__restrict__ grid, const int2 *__restrict__ grange /* nullable (N1) */,
                          CentreW cw) {
  constexpr int NT = (D2 == 4 || D2 == 9) ? 1 : 2;
  constexpr int G = 32 * NV, d = D2 / NT;
  const int side = 2 * R + 1;
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= side * side) return;
  const int dx = cell % side - R, dy = cell / side - R;
  double acc = 0.0;
  for (int64_t s = 0; s < nvalid; s++) {
    const int2 ij = __ldg(&src_ij[s]);
    const int i = ij.x + dx, j = ij.y + dy;
    if (i < 0 || j < 0 || i >= nx || j >= ny) continue;
    const int a = __ldg(&aidx[(size_t)j * nx + i]);
    if (a < 0) continue;
    const int64_t g = s / G;
    if (grange) {   // N1: outside the group's maintained range the density is exactly zero
      const int2 rg = __ldg(&grange[g]);
      if (a < rg.x || a >= rg.y) continue;
    }
    const int slot = (int)(s % G);
    const T *p = U + ((size_t)g * nact + a) * D2 * G + slot;
    double vl = 0.0, vu = 0.0;
#pragma unroll
    for (int k = 0; k < d; k++) {
      vl += cw.v[k] * (double)p[(size_t)k * G];
      if (NT == 2) vu += cw.v[DMAXK + k] * (double)p[(size_t)(d + k) * G];
    }
    acc += (NT == 2 ? 0.5 * (vl + vu) : vl) / mom[s * 6];   // quads: one element, its centre value
  }
  grid[cell] += acc;
}

// normalise by the source count and evaluate the Eq. (9) residual against the
// Gaussian N(x; mu, Sigma); one block, fixed-order reduction
__global__ void __launch_bounds__(256) k_mixture_final(const double *__restrict__ gsum, int R, double h, int64_t n,
                                                       double sxx, double sxy, double syy, double mx, double my,
                                                       double *__restrict__ grid_out, double *__restrict__ res_out) {
  __shared__ double sh[256];
  const int side = 2 * R + 1, ncell = side * side, t = threadIdx.x;
  const double det = sxx * syy - sxy * sxy;
  const double ixx = syy / det, ixy = -sxy / det, iyy = sxx / det;
  const double norm = 1.0 / (2.0 * M_PI * sqrt(det));
  const double inv_n = 1.0 / (double)n;
  const int b = (int)((int64_t)ncell * t / 256), e = (int)((int64_t)ncell * (t + 1) / 256);
  double r = 0.0;
  for (int c = b; c < e; c++) {
    const double v = gsum[c] * inv_n;
    grid_out[c] = v;
    const double x = (c % side - R) * h - mx, y = (c / side - R) * h - my;
    const double gauss = norm * exp(-0.5 * (ixx * x * x + 2.0 * ixy * x * y + iyy * y * y));
    r += (gauss - v) * (gauss - v);
  }
  sh[t] = r;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) sh[t] += sh[t + w];
    __syncthreads();
  }
  if (t == 0) *res_out = sh[0];
}

// ---------------------------------------------------------------------------
// NCCL (dlopen'ed: only needed when nranks > 1)
// ---------------------------------------------------------------------------
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char *(*errStr)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return false;
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    return commInitRank && allReduce && commDestroy && errStr;
  }
};
static NcclApi g_nccl;

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
struct dgdiff_s {
  int nx = 0, ny = 0, p = 1, d = 3, D2 = 6;
  double h = 1, D = 1;
  dgdiff_opts o;
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t nact = 0;
  int4 *d_nbr = nullptr;
  int4 *d_rowtab = nullptr;  // [nstrips][ny] {h0, c0, c1, h1} for the ring kernel
  int4 *d_rowtab3 = nullptr; // [nstrips3][ny][2] u/U1/U2/output bounds for the fused step
  int4 *d_rowtab_na = nullptr; // ring row table of the stage without the alpha term
  int4 *d_nbi[2] = {nullptr, nullptr};   // quads: strip-major neighbour tables [stage without / with alpha]
  int *d_nbi_off[2] = {nullptr, nullptr};  // and their (strip, row) offsets [nstrips][ny + 1]
  int4 *d_rowtab_pair = nullptr; // K3d (fused stages 2+3): [nstrips_pair][ny][2]
  int nstrips_pair = 0;
  uint16_t *d_nbs_pair = nullptr;  // K3d strip-major neighbour table
  int nstrips_na = 0;
  int nstrips3 = 0;
  double macs_per_stage = 0; // structural MACs of one stage over all active pixels (per source)
  int nstrips = 0, ring_w = 0, nsm = 148;
  int2 *d_pix = nullptr;
  int *d_aidx = nullptr;
  std::vector<int> h_aidx;
  void *d_A = nullptr;
  void *d_Aabs = nullptr;  // ABSORB boundary-pixel blocks (state precision)
  dgop::Table tab;
  dgop::QuadTable qtab;      // N4 quads (element = 1)
  // chunk buffers
  void *d_U[3] = {nullptr, nullptr, nullptr};
  void *d_Ubase = nullptr;
  int64_t chunk_cap = 0;  // sources the U buffers hold
  bool chunk_cap_fit = false;  // chunk_cap was limited by free device memory
  int *d_src_a = nullptr;
  int2 *d_src_ij = nullptr;
  double2 *d_src_xy = nullptr;   // source points, pixel units (per chunk slot)
  double *d_px = nullptr;        // N4 sub-pixel sources: [nloc][2 + D2] point + init row (chunk order)
  int64_t px_cap = 0;
  bool points = false;           // last solve used sub-pixel points
  const double *cur_px = nullptr;  // rows of the chunk being solved (points mode)
  double *d_partial = nullptr;
  size_t partial_cap = 0;
  unsigned *d_wcnt = nullptr;                      // K3c: per-item completion counters
  size_t wcnt_cap = 0;
  int2 *d_wtab = nullptr;                          // K3c: (stage, band) order of a group's items
  int wtab_nb = 0;
  int32_t *d_src = nullptr;
  int64_t src_cap = 0;
  std::vector<int32_t> h_src_stage;                // pageable staging copy of the sources
  double *d_mom = nullptr;
  int64_t mom_cap = 0;
  double *d_out = nullptr;
  // N1 active windows
  MomW momw;                                       // this handle's moment weights (kernel parameter)
  CentreW centw;                                   // and mixture node weights
  bool windows = false;
  bool win_apx = false;                            // windows = 2: clip the boxes at win_k sigma (F7)
  double win_k = 20.0;                             // (env DGDIFF_WINK overrides; experiments)
  bool quad = false;                               // N4 quadrilateral Q_p elements (opts.element = 1)
  int halo = 1;                                    // composite stencil reach (quads: 2)
  int32_t *d_srcw = nullptr, *d_perm = nullptr;   // sorted local sources [nloc][2], their global indices
  int64_t srcw_cap = 0;
  double *d_momc = nullptr;                        // chunk-ordered moment rows (sorted order)
  int64_t momc_cap = 0;
  int4 *d_gbox = nullptr;                          // per group source box of the current chunk
  int2 *d_grange = nullptr;                        // per group maintained active range [a0, a1)
  int64_t gbox_cap = 0;
  int wband = 32;                                  // ring band rows under windows (env DGDIFF_WBAND; swept 12-256 on c4)
  std::vector<int4> h_gbox;
  std::vector<int64_t> h_spos;                     // N1: global source index -> position in this rank's chunk order (-1: other rank)
  std::vector<int> h_pre;                          // 2-D prefix counts of active pixels [(ny+1)][(nx+1)]
  int64_t last_chunk_pos0 = 0;                     // sorted position of the last chunk's first source
  // mixture grid (N2)
  double *d_mix = nullptr, *d_mix_out = nullptr;
  int mix_R = 0;
  bool mix_reduced = false, have_sigma = false;
  bool mom_reduced = false;                        // the [n][6] table holds every rank's rows
  double last_sigma[3] = {0, 0, 0}, last_mu[2] = {0, 0};
  // last solve
  bool solved = false;
  int64_t last_n = 0, last_nsteps = 0;
  double last_dt = 0;
  int64_t last_chunk_begin = -1, last_chunk_n = 0;  // global source index range kept (keep_density)
  int64_t last_chunk_size = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  bool logical = false;                            // nranks > 1 without a communicator
  // stats
  dgdiff_stats_t st;
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  size_t ev_used = 0;
  int64_t ev_launches_pending = 0;
  // dominant-kernel timing (K3d: the stage-pair launches, one event pair each)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evd;
  size_t evd_used = 0;
  bool stage_detail = false;          // env DGDIFF_STAGE_DETAIL=1: per-stage events
  int ahead_alpha = 0, ahead_noalpha = 0;  // env DGDIFF_AHEAD=a,n (tuning experiments)
  int n1_use = 0, n2_use = 0;              // env DGDIFF_RING=n1,n2 (tuning experiments)
  double mean_tile = 0;                    // mean ring-kernel row tile (pixel tiles)
  cudaEvent_t sev[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
  bool sev_pending[3] = {false, false, false};
  double stage_detail_ms[3] = {0, 0, 0};
};

static size_t tsize(const dgdiff_s *H) { return H->o.precision == 32 ? 4 : 8; }
// lane width of the state layout: 16 B for the global-load kernels (v1, v2),
// 8 B for the row-ring kernel (v3, default) so that four full row tiles fit
// K3 (fused step) is used for P1 when temporal_steps == 2 (or by default, see
// use_fused); its groups are 32 sources (one value per lane)
static bool use_fused(const dgdiff_s *H) {
  if (H->p != 1 || H->o.kernel == 1 || H->o.kernel == 2) return false;
  return H->o.temporal_steps == 2 || H->o.temporal_steps == 3;   // 3: K3b, decoupled warp roles
}
// values per lane of the state layout: v1/v2 16-byte lanes; ring P1 16-byte,
// ring P2 8-byte lanes (tile size); fused step one value per lane
static int lane_nv(const dgdiff_s *H) {
  const int ts = (int)tsize(H);
  if (H->o.kernel == 1 || H->o.kernel == 2) return 16 / ts;
  if (use_fused(H)) return 1;
  if (H->quad) return 8 / ts;
  return (H->p == 1 ? 16 : 8) / ts;
}
static int gsize(const dgdiff_s *H) { return 32 * lane_nv(H); }
static bool use_ring(const dgdiff_s *H) { return !(H->o.kernel == 1 || H->o.kernel == 2); }

extern "C" void dgdiff_opts_default(dgdiff_opts *o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->precision = 64;
  o->outer_bc = 0;
  o->centering = 0;
  o->temporal_steps = 0;
  o->device = -1;
  o->rank = 0;
  o->nranks = 1;
  o->nccl_id = nullptr;
  o->keep_density = 0;
  o->max_chunk = 0;
  o->stream = nullptr;
  o->kernel = 0;
  o->mixture_radius = 0;
}

extern "C" const char *dgdiff_last_error(void) { return g_err.c_str(); }

extern "C" double dgdiff_dt_max(int32_t degree, double h, double D) {
  // SSP-RK3 real-axis stability limit 2.5127453 over the Bloch spectral radius
  // of the composite operator (R8): rho_1 = 60, rho_2 = 192.7953,
  // rho_3 = 462.37
  double rho = degree == 1 ? 60.0 : degree == 2 ? 192.7953 : degree == 3 ? 462.37 : 0.0;
  if (rho == 0.0 || !(h > 0) || !(D > 0)) return 0.0;
  return 2.5127453 / rho * h * h / D;
}

extern "C" void dgdiff_shard(int64_t n, int32_t rank, int32_t nranks, int64_t *begin, int64_t *end) {
  if (nranks < 1) nranks = 1;
  if (rank < 0) rank = 0;
  if (rank >= nranks) rank = nranks - 1;
  if (begin) *begin = n * rank / nranks;
  if (end) *end = n * (rank + 1) / nranks;
}

extern "C" dgdiff_status dgdiff_operator_table(int32_t degree, double *A, double *W, double *init) {
  if (degree < 1 || degree > 3) return fail(DGDIFF_E_ARG, "degree %d not supported (1..3)", degree);
  try {
    dgop::Table T = dgop::build(degree);
    if (A) memcpy(A, T.A.data(), T.A.size() * sizeof(double));
    if (W) memcpy(W, T.W.data(), T.W.size() * sizeof(double));
    if (init) memcpy(init, T.init.data(), T.init.size() * sizeof(double));
  } catch (std::exception &e) {
    return fail(DGDIFF_E_ARG, "operator precompute failed: %s", e.what());
  }
  return DGDIFF_OK;
}

static void release(dgdiff_s *H) {
  if (!H) return;
  for (auto &p : H->ev) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  for (auto &p : H->evd) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  for (int k = 0; k < 3; k++)
    for (int e = 0; e < 2; e++)
      if (H->sev[k][e]) cudaEventDestroy(H->sev[k][e]);
  cudaFree(H->d_Ubase);
  cudaFree(H->d_nbr);
  cudaFree(H->d_rowtab);
  cudaFree(H->d_rowtab3);
  cudaFree(H->d_rowtab_na);
  for (int v = 0; v < 2; v++) {
    cudaFree(H->d_nbi[v]);
    cudaFree(H->d_nbi_off[v]);
  }
  cudaFree(H->d_rowtab_pair);
  cudaFree(H->d_nbs_pair);
  cudaFree(H->d_pix);
  cudaFree(H->d_aidx);
  cudaFree(H->d_A);
  cudaFree(H->d_Aabs);
  cudaFree(H->d_src_a);
  cudaFree(H->d_src_ij);
  cudaFree(H->d_src_xy);
  cudaFree(H->d_px);
  cudaFree(H->d_partial);
  cudaFree(H->d_wcnt);
  cudaFree(H->d_wtab);
  cudaFree(H->d_src);
  cudaFree(H->d_mom);
  cudaFree(H->d_out);
  cudaFree(H->d_mix);
  cudaFree(H->d_mix_out);
  cudaFree(H->d_srcw);
  cudaFree(H->d_perm);
  cudaFree(H->d_momc);
  cudaFree(H->d_gbox);
  cudaFree(H->d_grange);
  if (H->comm && g_nccl.commDestroy) g_nccl.commDestroy(H->comm);
  if (H->own_stream && H->stream) cudaStreamDestroy(H->stream);
  delete H;
}

extern "C" void dgdiff_destroy(dgdiff_t H) {
  if (!H) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(H->dev);
  release(H);
  cudaSetDevice(cur);
}

static dgdiff_status create_impl(dgdiff_s *H, const uint8_t *mask) {
  const int nx = H->nx, ny = H->ny;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(DGDIFF_E_CUDA, "no CUDA device (%s): the GPU path has no CPU fallback",
                e != cudaSuccess ? cudaGetErrorString(e) : "count 0");
  if (H->o.device >= 0) {
    if (H->o.device >= ndev) return fail(DGDIFF_E_ARG, "device %d of %d", H->o.device, ndev);
    CK(cudaSetDevice(H->o.device));
  }
  CK(cudaGetDevice(&H->dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, H->dev));
  if (prop.major < 10)
    return fail(DGDIFF_E_CUDA, "device %s is sm_%d%d; this library is built for sm_100a", prop.name,
                prop.major, prop.minor);
  if (H->o.stream) {
    H->stream = (cudaStream_t)H->o.stream;
  } else {
    CK(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));
    H->own_stream = true;
  }
  // K0 operator tables
  dgop::QuadTable &qt = H->qtab;
  try {
    if (H->quad) qt = dgop::build_quad(H->p);
    else H->tab = dgop::build(H->p);
  } catch (std::exception &ex) {
    return fail(DGDIFF_E_ARG, "operator precompute failed: %s", ex.what());
  }
  if (H->quad) {
    // compiled Q tables == this run's K0; moment weights / init / centre values
    // in the triangle layout with t = 0 only
    const int d = H->D2;
    for (int b = 0; b < 28; b++)
      for (int r = 0; r < d; r++)
        for (int c = 0; c < d; c++) {
          const double v = H->p == 1 ? dgk::tab<101>(b, r, c) : dgk::tab<102>(b, r, c);
          if (v != qt.blocks[((size_t)b * d + r) * d + c]) return fail(DGDIFF_E_ARG, "compiled Q table differs from K0");
        }
    H->tab.p = H->p;
    H->tab.d = d;
    H->tab.W.assign((size_t)2 * 6 * d, 0.0);
    for (int q = 0; q < 6; q++)
      for (int k = 0; k < d; k++) H->tab.W[(size_t)q * d + k] = qt.W[(size_t)q * d + k];
    H->tab.init = qt.init;
    H->tab.cw.assign((size_t)2 * d, 0.0);
    for (int k = 0; k < d; k++) H->tab.cw[k] = qt.cw[k];
  }
  // the kernels carry the operator as compile-time immediates (tables.inc,
  // generated from K0 at build time): check them against this run's K0
  if (!H->quad) {
    const int D2 = H->D2;
    auto A = [&](int code, int o, int r, int c) { return H->tab.A[(((size_t)code * 5 + o) * D2 + r) * D2 + c]; };
    for (int code = 0; code < 16; code++)
      for (int r = 0; r < D2; r++)
        for (int c = 0; c < D2; c++) {
          auto tb = [&](int b) {
            return H->p == 1 ? dgk::tab<1>(b, r, c) : H->p == 2 ? dgk::tab<2>(b, r, c) : dgk::tab<3>(b, r, c);
          };
          if (tb(9 + code) != A(code, 0, r, c)) return fail(DGDIFF_E_ARG, "compiled operator table differs from K0 (self)");
          double self = tb(0);   // V + sum of the open F_f: exact on the dyadic P1/P2 tables
          for (int f = 0; f < 4; f++)
            if ((code >> f) & 1) self += tb(1 + f);
          if (H->p <= 2 && self != A(code, 0, r, c))
            return fail(DGDIFF_E_ARG, "compiled operator table differs from K0 (V + F)");
          for (int f = 0; f < 4; f++)
            if (A(code, 1 + f, r, c) != (((code >> f) & 1) ? tb(5 + f) : 0.0))
              return fail(DGDIFF_E_ARG, "compiled operator table differs from K0 (neighbour)");
        }
  }
  // active pixels in raster order, their open-face neighbours (out of grid
  // counts as axon under REFLECT, reading R9)
  std::vector<int> aidx((size_t)nx * ny, -1);
  std::vector<int2> pix;
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++)
      if (!mask[(size_t)j * nx + i]) {
        aidx[(size_t)j * nx + i] = (int)pix.size();
        pix.push_back(make_int2(i, j));
      }
  H->nact = (int64_t)pix.size();
  H->h_aidx = aidx;
  if (H->nact == 0) return fail(DGDIFF_E_ARG, "substrate has no extracellular pixel");
  std::vector<int4> nbr(H->nact);
  // neighbour index: active index, -1 for an axon pixel (or the outer square
  // under REFLECT, reading R9), -2 for a face on the outer square under ABSORB
  const int outside = H->o.outer_bc == 1 ? -2 : -1;
  auto at = [&](int i, int j) {
    return (i < 0 || j < 0 || i >= nx || j >= ny) ? outside : aidx[(size_t)j * nx + i];
  };
  for (int64_t a = 0; a < H->nact; a++) {
    int i = pix[a].x, j = pix[a].y;
    nbr[a] = make_int4(at(i + 1, j), at(i - 1, j), at(i, j + 1), at(i, j - 1));
  }
  // quads: [a][2] int4 = E W N S, then the pixels two steps away EE WW NN SS
  std::vector<int4> nbr_q;
  if (H->quad) {
    nbr_q.resize((size_t)2 * H->nact);
    for (int64_t a = 0; a < H->nact; a++) {
      int i = pix[a].x, j = pix[a].y;
      nbr_q[2 * a] = nbr[a];
      nbr_q[2 * a + 1] = make_int4(at(i + 2, j), at(i - 2, j), at(i, j + 2), at(i, j - 2));
    }
  }
  // ring kernel row tables (one per strip width: the stage without the alpha
  // term may use wider strips): active-index bounds of every (strip, row) tile
  if (use_ring(H)) {
    std::vector<int> cum((size_t)ny * (nx + 1));
    int run = 0;
    for (int j = 0; j < ny; j++) {
      for (int i = 0; i < nx; i++) {
        cum[(size_t)j * (nx + 1) + i] = run;
        if (!mask[(size_t)j * nx + i]) run++;
      }
      cum[(size_t)j * (nx + 1) + nx] = run;
    }
    for (int va = 0; va < 2; va++) {
      const bool alpha = va == 1;
      const int W = dgl::ring_width(H->quad ? 100 + H->p : H->p, alpha);
      const int ns = (nx + W - 1) / W;
      const int hl = H->halo;
      std::vector<int4> rtab((size_t)ns * ny);
      for (int s = 0; s < ns; s++)
        for (int j = 0; j < ny; j++) {
          const int x0 = s * W;
          auto c = [&](int x) { return cum[(size_t)j * (nx + 1) + std::max(0, std::min(nx, x))]; };
          rtab[(size_t)s * ny + j] = make_int4(c(x0 - hl), c(x0), c(x0 + W), c(x0 + W + hl));
        }
      // mean halo.d row-tile size (pixel tiles): the ring kernel without the
      // alpha term keeps ~8 mean rows in flight (measured optimum on c2/c4:
      // deeper TMA queues delay the row the consumers need next)
      double tiles = 0;
      for (const int4 &t : rtab) tiles += t.w - t.x;
      if (H->quad) {
        // item neighbour buffers (stage_ring.cuh, Gm::NBI): the neighbour
        // entries of every strip's computed pixels, strip by strip, rows in
        // order, so that an item (strip, band of rows) is one contiguous run
        std::vector<int4> nbi;
        std::vector<int> off((size_t)ns * (ny + 1));
        nbi.reserve(nbr_q.size());
        for (int s = 0; s < ns; s++)
          for (int j = 0; j <= ny; j++) {
            off[(size_t)s * (ny + 1) + j] = (int)(nbi.size() / 2);
            if (j == ny) break;
            const int4 t = rtab[(size_t)s * ny + j];
            for (int a = t.y; a < t.z; a++) {
              nbi.push_back(nbr_q[2 * (size_t)a]);
              nbi.push_back(nbr_q[2 * (size_t)a + 1]);
            }
          }
        if ((int64_t)nbi.size() != 2 * H->nact) return fail(DGDIFF_E_ARG, "strip-major neighbour table: pixel count");
        CK(cudaMalloc(&H->d_nbi[va], sizeof(int4) * nbi.size()));
        CK(cudaMemcpy(H->d_nbi[va], nbi.data(), sizeof(int4) * nbi.size(), cudaMemcpyHostToDevice));
        CK(cudaMalloc(&H->d_nbi_off[va], sizeof(int) * off.size()));
        CK(cudaMemcpy(H->d_nbi_off[va], off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
      }
      int4 *d = nullptr;
      CK(cudaMalloc(&d, sizeof(int4) * rtab.size()));
      CK(cudaMemcpy(d, rtab.data(), sizeof(int4) * rtab.size(), cudaMemcpyHostToDevice));
      if (alpha) {
        H->d_rowtab = d;
        H->nstrips = ns;
        H->ring_w = W;
      } else {
        H->d_rowtab_na = d;
        H->nstrips_na = ns;
        H->mean_tile = tiles / (double)std::max<size_t>(1, rtab.size());
      }
    }
  }
  // fused-step row table (P1): bounds of the u (3-column halo), U1 (2), U2 (1)
  // and output ranges of every (strip, row)
  if (H->p == 1 && !H->quad) {
    const int W = dgl::fused_width(H->o.precision);
    H->nstrips3 = (nx + W - 1) / W;
    std::vector<int> cum((size_t)ny * (nx + 1));
    int run = 0;
    for (int j = 0; j < ny; j++) {
      for (int i = 0; i < nx; i++) {
        cum[(size_t)j * (nx + 1) + i] = run;
        if (!mask[(size_t)j * nx + i]) run++;
      }
      cum[(size_t)j * (nx + 1) + nx] = run;
    }
    std::vector<int4> rt3((size_t)H->nstrips3 * ny * 2);
    for (int s = 0; s < H->nstrips3; s++)
      for (int j = 0; j < ny; j++) {
        const int x0 = s * W;
        auto c = [&](int x) { return cum[(size_t)j * (nx + 1) + std::max(0, std::min(nx, x))]; };
        rt3[((size_t)s * ny + j) * 2] = make_int4(c(x0 - 3), c(x0 - 2), c(x0 - 1), c(x0));
        rt3[((size_t)s * ny + j) * 2 + 1] = make_int4(c(x0 + W), c(x0 + W + 1), c(x0 + W + 2), c(x0 + W + 3));
      }
    CK(cudaMalloc(&H->d_rowtab3, sizeof(int4) * rt3.size()));
    CK(cudaMemcpy(H->d_rowtab3, rt3.data(), sizeof(int4) * rt3.size(), cudaMemcpyHostToDevice));
  }
  // K3d row table (P1 / P2 triangles): per (strip of W, row) the active-index
  // bounds of the U1 tile [x0-2, x0+W+2), the U2 pixels [x0-1, x0+W+1) and the
  // output pixels [x0, x0+W)
  if (!H->quad && H->p <= 2) {
    const int W = dgl::pair_width();
    H->nstrips_pair = (nx + W - 1) / W;
    std::vector<int> cum((size_t)ny * (nx + 1));
    int run = 0;
    for (int j = 0; j < ny; j++) {
      for (int i = 0; i < nx; i++) {
        cum[(size_t)j * (nx + 1) + i] = run;
        if (!mask[(size_t)j * nx + i]) run++;
      }
      cum[(size_t)j * (nx + 1) + nx] = run;
    }
    // and the strip-major 16-bit neighbour table of the U2 pixels: open-face
    // code (bits 0-3), the N / S neighbours' positions in the tiles of rows
    // j+1 / j-1 (bits 4-7 / 8-11, counted from column x0-2); rowtab .z of
    // the second int4 = the (strip, row)'s first entry
    std::vector<int4> rp((size_t)H->nstrips_pair * ny * 2);
    std::vector<uint16_t> nbs;
    nbs.reserve((size_t)H->nact * (W + 2) / W + 64);
    auto act = [&](int i, int j) { return i >= 0 && j >= 0 && i < nx && j < ny && !mask[(size_t)j * nx + i]; };
    for (int s = 0; s < H->nstrips_pair; s++)
      for (int j = 0; j < ny; j++) {
        const int x0 = s * W;
        auto cr = [&](int jj, int x) { return cum[(size_t)jj * (nx + 1) + std::max(0, std::min(nx, x))]; };
        auto c = [&](int x) { return cr(j, x); };
        rp[((size_t)s * ny + j) * 2] = make_int4(c(x0 - 2), c(x0 - 1), c(x0 + W + 1), c(x0 + W + 2));
        rp[((size_t)s * ny + j) * 2 + 1] = make_int4(c(x0), c(x0 + W), (int)nbs.size(), 0);
        for (int i = std::max(0, x0 - 1); i < std::min(nx, x0 + W + 1); i++) {
          if (!act(i, j)) continue;
          int e = (act(i + 1, j) ? 1 : 0) | (act(i - 1, j) ? 2 : 0) | (act(i, j + 1) ? 4 : 0) | (act(i, j - 1) ? 8 : 0);
          if (e & 4) e |= (aidx[(size_t)(j + 1) * nx + i] - cr(j + 1, x0 - 2)) << 4;
          if (e & 8) e |= (aidx[(size_t)(j - 1) * nx + i] - cr(j - 1, x0 - 2)) << 8;
          nbs.push_back((uint16_t)e);
        }
      }
    nbs.resize(nbs.size() + 16, 0);   // the bulk copies round the end up to 16 bytes
    CK(cudaMalloc(&H->d_rowtab_pair, sizeof(int4) * rp.size()));
    CK(cudaMemcpy(H->d_rowtab_pair, rp.data(), sizeof(int4) * rp.size(), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&H->d_nbs_pair, sizeof(uint16_t) * nbs.size()));
    CK(cudaMemcpy(H->d_nbs_pair, nbs.data(), sizeof(uint16_t) * nbs.size(), cudaMemcpyHostToDevice));
  }
  H->nsm = prop.multiProcessorCount;
  const std::vector<int4> &nbr_dev = H->quad ? nbr_q : nbr;
  CK(cudaMalloc(&H->d_nbr, sizeof(int4) * nbr_dev.size()));
  CK(cudaMalloc(&H->d_pix, sizeof(int2) * H->nact));
  CK(cudaMalloc(&H->d_aidx, sizeof(int) * (size_t)nx * ny));
  CK(cudaMemcpy(H->d_nbr, nbr_dev.data(), sizeof(int4) * nbr_dev.size(), cudaMemcpyHostToDevice));
  // algorithmic MACs of one stage (per source): structural non-zeros of the
  // pixel's self block plus its open neighbour blocks
  {
    double macs = 0;
    for (int64_t a = 0; a < H->nact; a++) {
      const int4 nb = nbr[a];
      const int code = (nb.x >= 0) | ((nb.y >= 0) << 1) | ((nb.z >= 0) << 2) | ((nb.w >= 0) << 3);
      if (H->quad) {
        const int d = H->D2, opp[4] = {1, 0, 3, 2};
        auto nnz = [&](int b) {
          int k = 0;
          for (int e = 0; e < d * d; e++) k += qt.blocks[(size_t)b * d * d + e] != 0.0;
          return k;
        };
        const int4 n2 = nbr_q[2 * a + 1];
        const int far[4] = {n2.x, n2.y, n2.z, n2.w};
        macs += nnz(code);
        for (int f = 0; f < 4; f++)
          if ((code >> f) & 1) macs += nnz(((code >> opp[f]) & 1) ? 16 + f : 20 + f) + (far[f] >= 0 ? nnz(24 + f) : 0);
        continue;
      }
      macs += H->tab.nnz[code * 5 + 0];
      for (int f = 0; f < 4; f++)
        if ((code >> f) & 1) macs += H->tab.nnz[code * 5 + 1 + f];
    }
    H->macs_per_stage = macs;
  }
  CK(cudaMemcpy(H->d_pix, pix.data(), sizeof(int2) * H->nact, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(H->d_aidx, aidx.data(), sizeof(int) * (size_t)nx * ny, cudaMemcpyHostToDevice));
  // operator table in the state precision (exact: dyadic entries)
  size_t na = H->tab.A.size();
  if (na == 0) {
    // quads: the v1 table kernel does not exist for them
  } else if (H->o.precision == 32) {
    std::vector<float> A32(na);
    for (size_t k = 0; k < na; k++) A32[k] = (float)H->tab.A[k];
    CK(cudaMalloc(&H->d_A, na * sizeof(float)));
    CK(cudaMemcpy(H->d_A, A32.data(), na * sizeof(float), cudaMemcpyHostToDevice));
  } else if (H->o.adjoint) {
    // the transposed composite operator L^T for the adjoint fields: the self
    // block of code c transposed; the block coupling a pixel to its
    // neighbour across open face f is [L_{q,p}]^T = (N_opp(f))^T (the shared
    // face is open from both sides, so q's block for p is the fixed N)
    const int D2 = 2 * H->tab.d;
    std::vector<double> AT(na, 0.0);
    auto Ai = [&](int code, int o, int r, int c) { return ((size_t)(code * 5 + o) * D2 + r) * D2 + c; };
    const int opp[5] = {0, 2, 1, 4, 3};
    for (int code = 0; code < 16; code++)
      for (int r = 0; r < D2; r++)
        for (int c = 0; c < D2; c++) {
          AT[Ai(code, 0, r, c)] = H->tab.A[Ai(code, 0, c, r)];
          for (int f = 1; f <= 4; f++)
            if ((code >> (f - 1)) & 1) AT[Ai(code, f, r, c)] = H->tab.A[Ai(15, opp[f], c, r)];
        }
    CK(cudaMalloc(&H->d_A, na * sizeof(double)));
    CK(cudaMemcpy(H->d_A, AT.data(), na * sizeof(double), cudaMemcpyHostToDevice));
  } else {
    CK(cudaMalloc(&H->d_A, na * sizeof(double)));
    CK(cudaMemcpy(H->d_A, H->tab.A.data(), na * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (H->o.outer_bc == 1) {
    std::vector<double> Ab;
    try {
      Ab = H->quad ? dgop::build_quad_absorb(H->p) : dgop::build_absorb(H->p);
    } catch (std::exception &ex) {
      return fail(DGDIFF_E_ARG, "absorbing operator precompute failed: %s", ex.what());
    }
    if (H->o.precision == 32) {
      std::vector<float> A32(Ab.begin(), Ab.end());
      CK(cudaMalloc(&H->d_Aabs, A32.size() * sizeof(float)));
      CK(cudaMemcpy(H->d_Aabs, A32.data(), A32.size() * sizeof(float), cudaMemcpyHostToDevice));
    } else {
      CK(cudaMalloc(&H->d_Aabs, Ab.size() * sizeof(double)));
      CK(cudaMemcpy(H->d_Aabs, Ab.data(), Ab.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  double W[2 * 6 * DMAXK] = {0};
  for (int t = 0; t < 2; t++)
    for (int q = 0; q < 6; q++)
      for (int j = 0; j < H->d; j++) W[(t * 6 + q) * DMAXK + j] = H->tab.W[(t * 6 + q) * H->d + j];
  // (quads: H->d = D2, t = 1 rows are zero and unused)
  memcpy(H->momw.w, W, sizeof W);
  double CWv[2 * DMAXK] = {0};
  for (int t = 0; t < 2; t++)
    for (int j = 0; j < H->d; j++) CWv[t * DMAXK + j] = H->tab.cw[t * H->d + j];
  memcpy(H->centw.v, CWv, sizeof CWv);
  if (H->o.mixture_radius > 0) {
    H->mix_R = H->o.mixture_radius;
    const size_t nc = (size_t)(2 * H->mix_R + 1) * (2 * H->mix_R + 1);
    CK(cudaMalloc(&H->d_mix, nc * sizeof(double)));
    CK(cudaMalloc(&H->d_mix_out, (nc + 1) * sizeof(double)));
  }
  CK(cudaMalloc(&H->d_out, 8 * sizeof(double)));
  // NCCL
  // NCCL communicator: required when nranks > 1; with nranks == 1 an explicit
  // nccl_id also creates one (a one-rank world: exercises the same path)
  // nranks > 1 without an id: a LOGICAL rank (no communicator): the handle
  // solves its shard only and leaves the other rows of the table zero; the
  // caller combines the ranks' tables (dgdiff_covariance_table)
  H->logical = H->o.nranks > 1 && !H->o.nccl_id;
  if (H->o.nccl_id) {
    if (!g_nccl.load()) return fail(DGDIFF_E_NCCL, "cannot load libnccl.so.2: %s", dlerror());
    ncclUniqueId id;
    memcpy(&id, H->o.nccl_id, sizeof id);
    ncclResult_t r = g_nccl.commInitRank(&H->comm, H->o.nranks, id, H->o.rank);
    if (r != ncclSuccess) return fail(DGDIFF_E_NCCL, "ncclCommInitRank: %s", g_nccl.errStr(r));
  }
  H->st.n_active = H->nact;
  H->windows = H->o.windows == 1 || H->o.windows == 2;
  H->win_apx = H->o.windows == 2;
  // clip factor per element type (reading R23, measured with
  // tools/sweep_wink.py: max relative moment error <= 1e-14 against the
  // whole-grid solve on c3): P1 20, P2 30, P3 45, Q1 25, Q2 40 sigma
  H->win_k = H->quad ? (H->p == 1 ? 25.0 : 40.0) : (H->p == 1 ? 20.0 : H->p == 2 ? 30.0 : 45.0);
  if (const char *wk = tune_env("DGDIFF_WINK")) H->win_k = atof(wk);
  if (H->windows) {
    // 2-D prefix counts of extracellular pixels: algorithmic bytes of windowed stages
    H->h_pre.assign((size_t)(ny + 1) * (nx + 1), 0);
    for (int j = 0; j < ny; j++)
      for (int i = 0; i < nx; i++)
        H->h_pre[(size_t)(j + 1) * (nx + 1) + i + 1] = H->h_pre[(size_t)j * (nx + 1) + i + 1] +
                                                       H->h_pre[(size_t)(j + 1) * (nx + 1) + i] -
                                                       H->h_pre[(size_t)j * (nx + 1) + i] + (mask[(size_t)j * nx + i] ? 0 : 1);
  }
  const char *sd = getenv("DGDIFF_STAGE_DETAIL");
  H->stage_detail = sd && sd[0] == '1';
  if (const char *ah = tune_env("DGDIFF_AHEAD")) sscanf(ah, "%d,%d", &H->ahead_alpha, &H->ahead_noalpha);
  if (const char *rg = tune_env("DGDIFF_RING")) sscanf(rg, "%d,%d", &H->n1_use, &H->n2_use);
  if (const char *wb = tune_env("DGDIFF_WBAND")) H->wband = atoi(wb);
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_create(dgdiff_t *out, const uint8_t *mask, int32_t nx, int32_t ny, double h,
                                       double D, int32_t degree, const dgdiff_opts *opts) {
  if (!out) return fail(DGDIFF_E_ARG, "out is NULL");
  *out = nullptr;
  if (!mask || nx < 1 || ny < 1) return fail(DGDIFF_E_ARG, "mask NULL or empty grid %dx%d", nx, ny);
  if ((int64_t)nx * ny >= (1LL << 31)) return fail(DGDIFF_E_ARG, "grid too large");
  if (!(h > 0) || !(D > 0) || !std::isfinite(h) || !std::isfinite(D))
    return fail(DGDIFF_E_ARG, "h and D must be positive and finite");
  if (degree < 1 || degree > 3) return fail(DGDIFF_E_ARG, "degree %d not supported (1..3)", degree);
  dgdiff_opts o;
  if (opts) o = *opts; else dgdiff_opts_default(&o);
  if (o.precision != 32 && o.precision != 64) return fail(DGDIFF_E_ARG, "precision must be 32 or 64");
  if (o.outer_bc != 0 && o.outer_bc != 1) return fail(DGDIFF_E_ARG, "outer_bc must be 0 (REFLECT) or 1 (ABSORB)");
  if (o.outer_bc == 1 && (o.kernel == 1 || o.kernel == 2 || o.temporal_steps >= 2))
    return fail(DGDIFF_E_ARG, "outer_bc ABSORB runs on the default ring kernel only");
  if (o.windows < 0 || o.windows > 2) return fail(DGDIFF_E_ARG, "windows must be 0, 1 or 2");
  if (degree == 3 && (o.kernel == 1 || o.kernel == 2 || o.temporal_steps >= 2))
    return fail(DGDIFF_E_ARG, "P3 (N4) runs on the default ring kernel only");
  if (o.windows != 0 && (o.kernel == 1 || o.kernel == 2 || o.temporal_steps >= 2))
    return fail(DGDIFF_E_ARG, "windows (N1) run on the default ring kernel only");
  if (o.centering != 0 && o.centering != 1) return fail(DGDIFF_E_ARG, "centering must be 0 or 1");
  if (o.element != 0 && o.element != 1) return fail(DGDIFF_E_ARG, "element must be 0 (triangles) or 1 (quadrilaterals)");
  if (o.element == 1 && (degree > 2 || o.kernel == 1 || o.kernel == 2 || o.temporal_steps >= 2))
    return fail(DGDIFF_E_ARG, "quadrilateral Q_p (N4): degree 1 or 2, default ring kernel only");
  if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks) return fail(DGDIFF_E_ARG, "bad rank/nranks");
  if (o.temporal_steps < 0 || o.temporal_steps > 5) return fail(DGDIFF_E_ARG, "temporal_steps must be 0..5");
  if (o.temporal_steps == 5 && (degree > 2 || o.element != 0 || o.kernel != 0 || o.outer_bc != 0 || o.windows != 0))
    return fail(DGDIFF_E_ARG, "temporal_steps 5 (K3d, fused stages 2+3): P1/P2 triangles, REFLECT, ring kernel, no windows");
  if (o.temporal_steps == 3 && o.precision != 64)
    return fail(DGDIFF_E_ARG, "temporal_steps 3 (K3b) is fp64 only");
  if (o.temporal_steps == 4 && o.kernel != 0)
    return fail(DGDIFF_E_ARG, "temporal_steps 4 (K3c wavefront) runs the ring kernel's items only");
  if (o.kernel < 0 || o.kernel > 3) return fail(DGDIFF_E_ARG, "kernel must be 0..3");
  if (o.max_chunk < 0) return fail(DGDIFF_E_ARG, "max_chunk < 0");
  if (o.mixture_radius < 0 || o.mixture_radius > 2048) return fail(DGDIFF_E_ARG, "mixture_radius must be in [0, 2048]");
  if (o.adjoint != 0 && o.adjoint != 1) return fail(DGDIFF_E_ARG, "adjoint must be 0 or 1");
  if (o.adjoint == 1 && (degree > 2 || o.outer_bc != 0 || o.windows != 0 || o.temporal_steps > 1 || o.kernel == 2 ||
                         o.kernel == 3 || o.mixture_radius != 0 || o.keep_density != 0 ||
                         ((o.precision == 32 || o.element == 1) && o.kernel == 1)))
    return fail(DGDIFF_E_ARG, "adjoint moments: P1/P2 triangles or Q1/Q2, REFLECT, no windows / temporal blocking / "
                              "mixture / densities (fp32 handles and quads: ring kernel)");
  dgdiff_s *H = new dgdiff_s();
  H->nx = nx; H->ny = ny; H->h = h; H->D = D; H->p = degree;
  H->d = (degree + 1) * (degree + 2) / 2;
  H->D2 = 2 * H->d;
  if (o.element == 1) {   // one Q_p element per pixel
    H->quad = true;
    H->halo = 2;
    H->D2 = (degree + 1) * (degree + 1);
    H->d = H->D2;
  }
  H->o = o;
  memset(&H->st, 0, sizeof H->st);
  dgdiff_status s = create_impl(H, mask);
  if (s != DGDIFF_OK) {
    release(H);
    return s;
  }
  *out = H;
  return DGDIFF_OK;
}

// ---------------------------------------------------------------------------
// solve
// ---------------------------------------------------------------------------
// algorithmic flops of one SSP-RK3 step for `chunk` sources: 3 stages of the
// structural MACs (2 flops each) plus the RK combinations per dof (stage 1:
// 1 FMA = 2 flops; stages 2, 3: sub + FMA + FMA = 5 flops)
// N1 window radius (pixels) after `stages` RK stages ending at time t: the
// exact support reach (halo pixels per stage) or, for windows = 2, at most
// K sigma = K sqrt(2 D t) / h (+ one stencil reach), K per element type
// (R23): the DG tails are below rounding there (SURVEY F7 measured ~15 sigma
// for P1; higher degrees have longer tails)
static int64_t win_radius(const dgdiff_s *H, int64_t stages, double t) {
  const int64_t exact = H->halo * stages;
  if (!H->win_apx) return exact;
  const int64_t apx = (int64_t)std::ceil(H->win_k * std::sqrt(2.0 * H->D * t) / H->h) + 2 * H->halo;
  return std::min(exact, apx);
}

static double fused_flops_per_step(const dgdiff_s *H, int64_t chunk) {
  const double dofs = (double)H->nact * H->D2;
  return (double)chunk * (3.0 * 2.0 * H->macs_per_stage + dofs * (2.0 + 5.0 + 5.0));
}

template <typename T, int NV, int D2>
static dgdiff_status run_chunk(dgdiff_s *H, int64_t nvalid, int64_t chunk, double dt, int64_t nsteps,
                               double *mom_rows) {
  constexpr int G = 32 * NV;
  const int ngroups = (int)(chunk / G);
  const int nact = (int)H->nact;
  cudaStream_t st = H->stream;
  T *u = (T *)H->d_U[0], *Ua = (T *)H->d_U[1], *Ub = (T *)H->d_U[2];
  // K1
  InitVals iv;
  const double ih2 = 1.0 / (H->h * H->h);
  for (int k = 0; k < D2; k++) iv.v[k] = H->tab.init[k] * ih2;
  int64_t nvec = (int64_t)ngroups * nact * D2 * 32;
  int blocks = (int)std::min<int64_t>((nvec + 255) / 256, 148 * 64);
  if (H->windows) {
    // N1: the stages touch only the rows each group's growing box can reach;
    // u and the two work registers are (re)initialised over exactly those rows
    dim3 ig((unsigned)std::min<int64_t>(std::max<int64_t>(1, (nvec / std::max(1, ngroups) + 255) / 256), 2048),
            (unsigned)ngroups);
    k_init_win<T, NV, D2><<<ig, 256, 0, st>>>(u, Ua, Ub, nact, H->d_grange, H->d_src_a, iv, H->cur_px, nvalid);
  } else {
    k_init<T, NV, D2><<<blocks, 256, 0, st>>>(u, nvec, nact, H->d_src_a, iv, H->cur_px, nvalid);
  }
  H->st.launches++;
  // K2 x 3 per step (SSP-RK3 increment form, R7)
  const int wpb = std::min(ngroups, 4);
  const int px = 32;
  dim3 grid((nact + px - 1) / px, (ngroups + wpb - 1) / wpb);
  const double c = dt * H->D / (H->h * H->h);
  const T *A = (const T *)H->d_A;
  const double pass = (double)nact * D2 * chunk * sizeof(T);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (H->timing && nsteps > 0) {
    if (H->ev_used == H->ev.size()) {
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      H->ev.push_back({a, b});
    }
    e0 = H->ev[H->ev_used].first;
    e1 = H->ev[H->ev_used].second;
    H->ev_used++;
    CK(cudaEventRecord(e0, st));
  }
  // per-stage breakdown (timing mode, first step of the chunk only)
  auto stage_ev = [&](int k, bool begin) -> dgdiff_status {
    if (!H->timing || !H->stage_detail) return DGDIFF_OK;
    if (!H->sev[k][0]) { CK(cudaEventCreate(&H->sev[k][0])); CK(cudaEventCreate(&H->sev[k][1])); }
    CK(cudaEventRecord(H->sev[k][begin ? 0 : 1], st));
    if (!begin) H->sev_pending[k] = true;
    return DGDIFF_OK;
  };
  constexpr int P = D2 == 6 ? 1 : D2 == 12 ? 2 : D2 == 20 ? 3 : D2 == 4 ? 101 : 102;
  dgl::StageArgs sa;
  sa.nbr = H->d_nbr;
  sa.A = A;
  sa.Aabs = H->d_Aabs;
  sa.rowtab = H->d_rowtab;
  sa.nact = nact;
  sa.ny = H->ny;
  sa.nstrips = H->nstrips;
  sa.ngroups = ngroups;
  sa.nsm = H->nsm;
  sa.px = px;
  sa.wpb = wpb;
  sa.diag = (tune_env("DGDIFF_K2_DIAG") && atoi(tune_env("DGDIFF_K2_DIAG")) == 1) ? 1 : 0;   // tuning builds only
  sa.ahead_alpha = H->ahead_alpha;
  sa.ahead_noalpha = H->ahead_noalpha;
  sa.n1_use = H->n1_use;
  sa.n1_use_na = H->n1_use > 0 ? H->n1_use : (int)(8.0 * H->mean_tile + 0.5);
  sa.rowtab_na = H->d_rowtab_na;
  sa.nbi = H->d_nbi[1];
  sa.nbi_off = H->d_nbi_off[1];
  sa.nbi_na = H->d_nbi[0];
  sa.nbi_off_na = H->d_nbi_off[0];
  sa.nstrips_na = H->nstrips_na;
  sa.n2_use = H->n2_use;
  sa.st = st;
  const int which = H->o.kernel == 1 ? 0 : H->o.kernel == 2 ? 1 : 2;
  const int prec = (int)(8 * sizeof(T));
  // N1: extracellular pixels of group g's box grown by r (algorithmic bytes)
  auto box_px = [&](int g, int r) -> double {
    const int4 b = H->h_gbox[g];
    const int x0 = std::max(0, b.x - r), x1 = std::min(H->nx - 1, b.y + r);
    const int y0 = std::max(0, b.z - r), y1 = std::min(H->ny - 1, b.w + r);
    const size_t W1 = (size_t)H->nx + 1;
    return (double)(H->h_pre[(y1 + 1) * W1 + x1 + 1] - H->h_pre[(size_t)y0 * W1 + x1 + 1] -
                    H->h_pre[(y1 + 1) * W1 + x0] + H->h_pre[(size_t)y0 * W1 + x0]);
  };
  double win_bytes = 0;
  sa.gbox = H->windows ? H->d_gbox : nullptr;
  sa.band_rows = H->windows ? H->wband : 0;
  int64_t cur_step = 0;
  auto stage = [&](int k, const T *Uin, T *Uout, double alpha, double cs) -> dgdiff_status {
    sa.Uin = Uin;
    sa.U0 = u;
    sa.Uout = Uout;
    sa.alpha = alpha;
    sa.cs = cs;
    if (H->windows) {
      // output support radius (exact reach, or the 15-sigma clip)
      sa.wr = (int)std::min<int64_t>(1 << 30, win_radius(H, 3 * cur_step + k + 1, (double)(cur_step + 1) * dt));
      double px = 0;
      for (int g = 0; g < ngroups; g++) px += box_px(g, sa.wr);
      win_bytes += (k == 0 ? 2.0 : 3.0) * px * D2 * G * sizeof(T);
    }
    cudaError_t e = dgl::launch_stage(which, prec, P, k > 0, sa);
    if (e != cudaSuccess) return fail(DGDIFF_E_CUDA, "stage launch: %s", cudaGetErrorString(e));
    return DGDIFF_OK;
  };
  if (use_fused(H)) {
    // K3: one fused SSP-RK3 step per launch, ping-pong u <-> Ua
    sa.rowtab = H->d_rowtab3;
    sa.nstrips = H->nstrips3;
    sa.cs = c;
    T *cur = u, *nxt = Ua;
    for (int64_t s = 0; s < nsteps; s++) {
      sa.Uin = cur;
      sa.U0 = cur;
      sa.Uout = nxt;
      cudaError_t e = H->o.temporal_steps == 3 ? dgl::launch_dec_f64(sa) : dgl::launch_step_fused(prec, sa);
      if (e != cudaSuccess) return fail(DGDIFF_E_CUDA, "fused step launch: %s", cudaGetErrorString(e));
      std::swap(cur, nxt);
    }
    if (cur != u) std::swap(H->d_U[0], H->d_U[1]);   // the final state is always register 0
    u = (T *)H->d_U[0];
    if (e1) {
      CK(cudaEventRecord(e1, st));
      H->ev_launches_pending += nsteps;
    }
    H->st.launches += nsteps;
    H->st.stage_launches += nsteps;
    H->st.dom_launches += nsteps;
    H->st.dom_bytes += 2.0 * pass * nsteps;
    H->st.stage_bytes += 2.0 * pass * nsteps;
    H->st.stage_flops += fused_flops_per_step(H, chunk) * nsteps;
    goto after_stepping;
  }
  if (H->o.temporal_steps == 5) {
    // K3d: stage 1 on K2 (u -> Ua), stages 2 + 3 fused in one launch (Ua, u ->
    // Ub).  u' lands in another register than u (neighbouring strips read u in
    // their halo columns), so u and Ub trade places after every step.
    T *cu = u, *cb = Ub;
    dgl::StageArgs sp = sa;
    sp.rowtab = H->d_rowtab_pair;
    sp.nbs = H->d_nbs_pair;
    sp.nstrips = H->nstrips_pair;
    sp.cs = c;
    for (int64_t s = 0; s < nsteps; s++) {
      cur_step = s;
      dgdiff_status r;
      if ((r = stage(0, cu, Ua, 0.0, c)) != DGDIFF_OK) return r;
      sp.Uin = Ua;
      sp.U0 = cu;
      sp.Uout = cb;
      cudaEvent_t d0 = nullptr, d1 = nullptr;
      if (H->timing) {
        if (H->evd_used == H->evd.size()) {
          cudaEvent_t a, b;
          CK(cudaEventCreate(&a));
          CK(cudaEventCreate(&b));
          H->evd.push_back({a, b});
        }
        d0 = H->evd[H->evd_used].first;
        d1 = H->evd[H->evd_used].second;
        H->evd_used++;
        CK(cudaEventRecord(d0, st));
      }
      cudaError_t e = dgl::launch_pair(prec, P, sp);
      if (e != cudaSuccess) return fail(DGDIFF_E_CUDA, "stage-pair launch: %s", cudaGetErrorString(e));
      if (d1) CK(cudaEventRecord(d1, st));
      std::swap(cu, cb);
    }
    if (cu != u) std::swap(H->d_U[0], H->d_U[2]);   // the final state is always register 0
    u = (T *)H->d_U[0];
    if (e1) {
      CK(cudaEventRecord(e1, st));
      H->ev_launches_pending += 2 * nsteps;
    }
    H->st.launches += 2 * nsteps;
    H->st.stage_launches += 2 * nsteps;
    H->st.stage_bytes += 5.0 * pass * nsteps;   // stage 1: u in, U1 out; pair: U1, u in, u' out
    H->st.dom_bytes += 3.0 * pass * nsteps;     // the stage-pair kernel alone
    H->st.dom_launches += nsteps;
    H->st.stage_flops += fused_flops_per_step(H, chunk) * nsteps;
    goto after_stepping;
  }
  if (H->o.temporal_steps == 4 && !H->windows) {
    // K3c: one launch per SSP-RK3 step, stage items in wavefront order
    const int br = dgl::wave_band_rows();
    const int nb = (H->ny + br - 1) / br;
    const size_t ncnt = (size_t)ngroups * 3 * nb * H->nstrips;   // >= the strip-block count
    if (ncnt > H->wcnt_cap) {
      cudaFree(H->d_wcnt);
      H->d_wcnt = nullptr;
      CK(cudaMalloc(&H->d_wcnt, ncnt * sizeof(unsigned)));
      H->wcnt_cap = ncnt;
    }
    if (H->wtab_nb != nb) {
      std::vector<int2> wt;
      // stage k of band b in wavefront b + 2k: an item's inputs (stage k-1,
      // bands b-1..b+1) all belong to earlier wavefronts
      for (int w = 0; w < nb + 4; w++)
        for (int k = 0; k < 3; k++)
          if (w - 2 * k >= 0 && w - 2 * k < nb) wt.push_back(make_int2(k, w - 2 * k));
      cudaFree(H->d_wtab);
      H->d_wtab = nullptr;
      CK(cudaMalloc(&H->d_wtab, wt.size() * sizeof(int2)));
      CK(cudaMemcpy(H->d_wtab, wt.data(), wt.size() * sizeof(int2), cudaMemcpyHostToDevice));
      H->wtab_nb = nb;
    }
    CK(cudaMemsetAsync(H->d_wcnt, 0, ncnt * sizeof(unsigned), st));
    sa.Uin = u;
    sa.U0 = Ua;
    sa.Uout = Ub;
    sa.cs = c;
    sa.band_rows = br;
    sa.wave_cnt = H->d_wcnt;
    sa.wave_tab = H->d_wtab;
    for (int64_t s = 0; s < nsteps; s++) {
      sa.wave_epoch = (unsigned)(s + 1);
      cudaError_t e = dgl::launch_wave(prec, P, sa);
      if (e != cudaSuccess) return fail(DGDIFF_E_CUDA, "wavefront step launch: %s", cudaGetErrorString(e));
    }
    if (e1) {
      CK(cudaEventRecord(e1, st));
      H->ev_launches_pending += nsteps;
    }
    H->st.launches += nsteps;
    H->st.stage_launches += nsteps;
    H->st.dom_launches += nsteps;
    H->st.dom_bytes += 4.0 * pass * nsteps;
    H->st.stage_bytes += 4.0 * pass * nsteps;   // u read + u written + U1, U2 written back
    H->st.stage_flops += fused_flops_per_step(H, chunk) * nsteps;
    goto after_stepping;
  }
  for (int64_t s = 0; s < nsteps; s++) {
    const bool det = (s == 0);
    cur_step = s;
    dgdiff_status r;
    if (det && (r = stage_ev(0, true)) != DGDIFF_OK) return r;
    if ((r = stage(0, u, Ua, 0.0, c)) != DGDIFF_OK) return r;
    if (det && (r = stage_ev(0, false)) != DGDIFF_OK) return r;
    if (det && (r = stage_ev(1, true)) != DGDIFF_OK) return r;
    if ((r = stage(1, Ua, Ub, 0.75, 0.25 * c)) != DGDIFF_OK) return r;
    if (det && (r = stage_ev(1, false)) != DGDIFF_OK) return r;
    if (det && (r = stage_ev(2, true)) != DGDIFF_OK) return r;
    if ((r = stage(2, Ub, u, 1.0 / 3.0, (2.0 / 3.0) * c)) != DGDIFF_OK) return r;
    if (det && (r = stage_ev(2, false)) != DGDIFF_OK) return r;
  }
  if (e1) {
    CK(cudaEventRecord(e1, st));
    H->ev_launches_pending += 3 * nsteps;
  }
  H->st.launches += 3 * nsteps;
  H->st.stage_launches += 3 * nsteps;
  H->st.dom_launches += 3 * nsteps;   // K2: the stage kernel is the dominant kernel
  H->st.stage_bytes += H->windows ? win_bytes : 8.0 * pass * nsteps;
  H->st.dom_bytes += H->windows ? win_bytes : 8.0 * pass * nsteps;
  H->st.stage_flops += fused_flops_per_step(H, chunk) * nsteps * (H->windows ? win_bytes / std::max(1.0, 8.0 * pass * nsteps) : 1.0);
after_stepping:
  CK(cudaGetLastError());
  // K4
  const int mpx = 256;
  const int nblk = (nact + mpx - 1) / mpx;
  size_t need = (size_t)nblk * chunk * 6;
  if (need > H->partial_cap) {
    cudaFree(H->d_partial);
    H->d_partial = nullptr;
    CK(cudaMalloc(&H->d_partial, need * sizeof(double)));
    H->partial_cap = need;
  }
  dim3 mgrid(nblk, (ngroups + wpb - 1) / wpb);
  k_moments<T, NV, D2><<<mgrid, 32 * wpb, 0, st>>>(u, H->d_pix, H->d_src_xy, nact, ngroups, mpx, H->d_partial,
                                               chunk, H->windows ? H->d_grange : nullptr, H->momw);
  k_mom_reduce<<<(int)((nvalid + 7) / 8), 256, 0, st>>>(H->d_partial, nblk, chunk, nvalid, H->h, mom_rows,
                                                            H->windows ? H->d_perm + H->last_chunk_pos0 : nullptr,
                                                            H->d_mom);
  H->st.launches += 2;
  if (H->mix_R > 0 && !H->points) {   // the lattice is defined about pixel-centre sources (R20)
    const int nc = (2 * H->mix_R + 1) * (2 * H->mix_R + 1);
    k_mixture<T, NV, D2><<<(nc + 127) / 128, 128, 0, st>>>(u, H->d_aidx, H->nx, H->ny, nact, H->d_src_ij, mom_rows,
                                                         nvalid, H->mix_R, H->d_mix,
                                                         H->windows ? H->d_grange : nullptr, H->centw);
    H->st.launches++;
  }
  CK(cudaGetLastError());
  return DGDIFF_OK;
}

template <typename T>
static dgdiff_status run_chunk_p(dgdiff_s *H, int64_t nvalid, int64_t chunk, double dt, int64_t nsteps,
                                 double *mom_rows) {
  const int nv = lane_nv(H);
  if (nv == 1) {
    if (H->D2 == 6) return run_chunk<T, 1, 6>(H, nvalid, chunk, dt, nsteps, mom_rows);
    if (H->D2 == 20) return run_chunk<T, 1, 20>(H, nvalid, chunk, dt, nsteps, mom_rows);
    if (H->D2 == 4) return run_chunk<T, 1, 4>(H, nvalid, chunk, dt, nsteps, mom_rows);
    if (H->D2 == 9) return run_chunk<T, 1, 9>(H, nvalid, chunk, dt, nsteps, mom_rows);
    return run_chunk<T, 1, 12>(H, nvalid, chunk, dt, nsteps, mom_rows);
  }
  if (nv == 2) {
    if (H->D2 == 6) return run_chunk<T, 2, 6>(H, nvalid, chunk, dt, nsteps, mom_rows);
    if (H->D2 == 20) return run_chunk<T, 2, 20>(H, nvalid, chunk, dt, nsteps, mom_rows);
    if (H->D2 == 4) return run_chunk<T, 2, 4>(H, nvalid, chunk, dt, nsteps, mom_rows);
    if (H->D2 == 9) return run_chunk<T, 2, 9>(H, nvalid, chunk, dt, nsteps, mom_rows);
    return run_chunk<T, 2, 12>(H, nvalid, chunk, dt, nsteps, mom_rows);
  }
  if constexpr (sizeof(T) == 4) {
    if (H->D2 == 6) return run_chunk<T, 4, 6>(H, nvalid, chunk, dt, nsteps, mom_rows);
    return run_chunk<T, 4, 12>(H, nvalid, chunk, dt, nsteps, mom_rows);
  }
  return fail(DGDIFF_E_ARG, "internal: lane width");
}

// Adjoint moments (opts.adjoint): see k_adj_init.  The weight fields of up to
// 30 origins (a lattice over the box of the batch's sources, so that
// |x_s - x_o| stays small and the re-centring subtraction loses few digits:
// with 9 origins the worst c4 source's second moments differed from the
// per-source solve by 1.4e-10) fill ceil(30 / (G / 6)) source groups; they
// step with the transposed operator -- on the ring kernel with transposed
// compile-time tables (default), restricted to the sources' domain of
// dependence (stage k of the 3N computes only the box grown by 3N - 1 - k
// pixels: nothing outside can reach a source pixel by the end; pixels outside
// keep stale values that are never read), or on the v1 table kernel with the
// transposed table (opts.kernel = 1) -- then every source of the shard
// [b, b + nloc) is evaluated into its table row.
template <int D2, int G, int NT = 2>
static dgdiff_status adjoint_solve(dgdiff_s *H, const int32_t *sources, const double *px, int64_t n, int64_t b,
                                   int64_t nloc, double dt, int64_t nsteps) {
  constexpr int NG = adj_groups<G>();
  const int P = NT == 1 ? (D2 == 4 ? 101 : 102) : (D2 == 6 ? 1 : 2);
  const int nact = (int)H->nact;
  const bool ring = use_ring(H);
  cudaStream_t st = H->stream;
  if (nloc == 0) return DGDIFF_OK;   // an empty shard: its table rows stay zero
  if (H->chunk_cap < NG * G) {
    cudaFree(H->d_Ubase);
    H->d_Ubase = nullptr;
    const size_t reg = (size_t)nact * D2 * G * NG * sizeof(double);
    CK(cudaMalloc(&H->d_Ubase, 3 * reg));
    for (int r = 0; r < 3; r++) H->d_U[r] = (char *)H->d_Ubase + r * reg;
    H->chunk_cap = NG * G;
    H->chunk_cap_fit = false;
  }
  AdjOrigins org;
  org.n = 0;
  int4 box = make_int4(0, H->nx - 1, 0, H->ny - 1);
  if (nloc > 0) {
    // the origin lattice spans the WHOLE batch (every rank sees the same
    // list), so a source's moments do not depend on the rank count
    int x0 = INT32_MAX, x1 = INT32_MIN, y0 = INT32_MAX, y1 = INT32_MIN;
    for (int64_t k = 0; k < n; k++) {
      x0 = std::min(x0, sources[2 * k]);
      x1 = std::max(x1, sources[2 * k]);
      y0 = std::min(y0, sources[2 * k + 1]);
      y1 = std::max(y1, sources[2 * k + 1]);
    }
    box = make_int4(x0, x1, y0, y1);
    // a kx x ky lattice of cell centres (kx ky <= ADJ_MAXO), cells as square
    // as the box allows
    const double wx = x1 + 1 - x0, wy = y1 + 1 - y0;
    int kx = 1, ky = 1;
    for (int cx = 1; cx <= ADJ_MAXO; cx++) {
      const int cy = ADJ_MAXO / cx;
      if (cy < 1) break;
      if (std::max(wx / cx, wy / cy) < std::max(wx / kx, wy / ky)) { kx = cx; ky = cy; }
    }
    for (int oy = 0; oy < ky; oy++)
      for (int ox = 0; ox < kx; ox++) {
        org.x[org.n] = x0 + wx * (2 * ox + 1) / (2.0 * kx);
        org.y[org.n] = y0 + wy * (2 * oy + 1) / (2.0 * ky);
        org.n++;
      }
  }
  double *u = (double *)H->d_U[0], *Ua = (double *)H->d_U[1], *Ub = (double *)H->d_U[2];
  const int64_t total = (int64_t)nact * D2 * G * NG;
  k_adj_init<D2, G, NT><<<(int)std::min<int64_t>((total + 255) / 256, 148 * 64), 256, 0, st>>>(u, H->d_pix, nact, H->h,
                                                                                              H->momw, org);
  H->st.launches++;
  dgl::StageArgs sa;
  sa.nbr = H->d_nbr;
  sa.A = H->d_A;          // v1: the transposed table (dgdiff_create, adjoint)
  sa.nact = nact;
  sa.ny = H->ny;
  sa.ngroups = NG;
  sa.nsm = H->nsm;
  sa.px = 32;
  sa.wpb = std::min(NG, 4);
  sa.st = st;
  if (ring) {
    sa.rowtab = H->d_rowtab;
    sa.nstrips = H->nstrips;
    sa.rowtab_na = H->d_rowtab_na;
    sa.nstrips_na = H->nstrips_na;
    sa.n1_use = H->n1_use;
    sa.n1_use_na = H->n1_use > 0 ? H->n1_use : (int)(8.0 * H->mean_tile + 0.5);
    sa.n2_use = H->n2_use;
    sa.nbi = H->d_nbi[1];   // quads: item neighbour buffers
    sa.nbi_off = H->d_nbi_off[1];
    sa.nbi_na = H->d_nbi[0];
    sa.nbi_off_na = H->d_nbi_off[0];
    // every group clips to the sources' box grown by the remaining reach
    std::vector<int4> gb(NG, box);
    if (NG > H->gbox_cap) {
      cudaFree(H->d_gbox);
      cudaFree(H->d_grange);
      H->d_gbox = nullptr;
      H->d_grange = nullptr;
      CK(cudaMalloc(&H->d_gbox, sizeof(int4) * NG));
      CK(cudaMalloc(&H->d_grange, sizeof(int2) * NG));
      H->gbox_cap = NG;
    }
    CK(cudaMemcpyAsync(H->d_gbox, gb.data(), sizeof(int4) * NG, cudaMemcpyHostToDevice, st));
    sa.gbox = H->d_gbox;
    sa.band_rows = H->wband;
  }
  const double c = dt * H->D / (H->h * H->h);
  int64_t kst = 0;   // global stage index 0 .. 3N - 1
  auto stage = [&](const double *Uin, double *Uout, double alpha, double cs) -> dgdiff_status {
    sa.Uin = Uin;
    sa.U0 = u;
    sa.Uout = Uout;
    sa.alpha = alpha;
    sa.cs = cs;
    sa.wr = (int)std::min<int64_t>(1 << 30, H->halo * (3 * nsteps - 1 - kst));
    kst++;
    cudaError_t e = ring ? dgl::launch_ring_adj_f64(P, alpha != 0.0, sa) : dgl::launch_stage(0, 64, P, alpha != 0.0, sa);
    if (e != cudaSuccess) return fail(DGDIFF_E_CUDA, "adjoint stage launch: %s", cudaGetErrorString(e));
    return DGDIFF_OK;
  };
  for (int64_t step = 0; step < nsteps; step++) {   // SSP-RK3 increment form, as run_chunk
    dgdiff_status r;
    if ((r = stage(u, Ua, 0.0, c)) != DGDIFF_OK) return r;
    if ((r = stage(Ua, Ub, 0.75, 0.25 * c)) != DGDIFF_OK) return r;
    if ((r = stage(Ub, u, 1.0 / 3.0, (2.0 / 3.0) * c)) != DGDIFF_OK) return r;
  }
  H->st.launches += 3 * nsteps;
  H->st.stage_launches += 3 * nsteps;
  if (nloc > 0) {
    InitVals iv;
    const double ih2 = 1.0 / (H->h * H->h);
    for (int k = 0; k < D2; k++) iv.v[k] = H->tab.init[k] * ih2;
    const double *dpx = nullptr;
    if (px) {   // N4 points: this shard's rows (point + projected-Dirac row)
      const size_t PXS = 2 + D2;
      if (nloc > H->px_cap) {
        cudaFree(H->d_px);
        H->d_px = nullptr;
        CK(cudaMalloc(&H->d_px, sizeof(double) * PXS * nloc));
        H->px_cap = nloc;
      }
      CK(cudaMemcpyAsync(H->d_px, px + (size_t)b * PXS, sizeof(double) * PXS * nloc, cudaMemcpyHostToDevice, st));
      H->st.h2d_bytes += sizeof(double) * PXS * nloc;
      dpx = H->d_px;
    }
    k_adj_eval<D2, G><<<(int)((nloc + 127) / 128), 128, 0, st>>>(u, nact, H->d_src, b, nloc, H->d_aidx, H->nx, H->h,
                                                                 iv, org, H->d_mom, dpx);
    H->st.launches++;
  }
  CK(cudaGetLastError());
  H->st.chunk = NG * G;
  return DGDIFF_OK;
}

// sources: [n][2] pixel (i, j); px: nullable [n][2 + D2] sub-pixel points
// (pixel units) and their projected-Dirac rows (N4), in the same order
static dgdiff_status solve_impl(dgdiff_s *H, const int32_t *sources, const double *px, int64_t n, double dt,
                                int64_t nsteps) {
  if (!H) return fail(DGDIFF_E_ARG, "handle is NULL");
  if (n < 1 || !sources) return fail(DGDIFF_E_ARG, "need n >= 1 sources");
  if (n >= (1LL << 31)) return fail(DGDIFF_E_ARG, "too many sources");
  if (nsteps < 0 || !(dt > 0) || !std::isfinite(dt)) return fail(DGDIFF_E_ARG, "need dt > 0, nsteps >= 0");
  // quads: Bloch spectral radius of the 9-point-cross operator (N4; DESIGN
  // reading R22): rho_Q1 = 32, rho_Q2 = 130.7
  double dtmax = H->quad ? 2.5127453 / (H->p == 1 ? 32.0 : 130.7) * H->h * H->h / H->D
                         : dgdiff_dt_max(H->p, H->h, H->D);
  if (dt > dtmax)
    return fail(DGDIFF_E_UNSTABLE, "dt = %.17g exceeds the SSP-RK3 limit %.17g for P%d", dt, dtmax, H->p);
  for (int64_t s = 0; s < n; s++) {
    int i = sources[2 * s], j = sources[2 * s + 1];
    if (i < 0 || j < 0 || i >= H->nx || j >= H->ny)
      return fail(DGDIFF_E_SOURCE, "source %lld (%d,%d) is outside the %dx%d grid", (long long)s, i, j, H->nx, H->ny);
    if (H->h_aidx[(size_t)j * H->nx + i] < 0)
      return fail(DGDIFF_E_SOURCE, "source %lld (%d,%d) lies on an axon pixel (S:230)", (long long)s, i, j);
  }
  CK(cudaSetDevice(H->dev));
  H->solved = false;
  // no chunk of this solve kept yet (a rank whose shard is empty keeps none:
  // dgdiff_get_density must not see the previous solve's chunk)
  H->last_chunk_begin = -1;
  H->last_chunk_n = 0;
  H->last_chunk_pos0 = 0;
  H->h_spos.clear();
  H->st.h2d_bytes = 0;
  H->st.d2h_bytes = 0;
  int64_t b, e;
  dgdiff_shard(n, H->o.rank, H->o.nranks, &b, &e);
  const int64_t nloc = e - b;
  const int G = gsize(H);
  // zero-padded moment table for all n sources (K5 all-reduce input)
  if (n > H->mom_cap) {
    cudaFree(H->d_mom);
    H->d_mom = nullptr;
    CK(cudaMalloc(&H->d_mom, sizeof(double) * 6 * n));
    H->mom_cap = n;
  }
  CK(cudaMemsetAsync(H->d_mom, 0, sizeof(double) * 6 * n, H->stream));
  if (H->mix_R > 0) {
    const size_t nc = (size_t)(2 * H->mix_R + 1) * (2 * H->mix_R + 1);
    CK(cudaMemsetAsync(H->d_mix, 0, nc * sizeof(double), H->stream));
  }
  H->mix_reduced = false;
  H->mom_reduced = false;
  H->have_sigma = false;
  if (n > H->src_cap) {
    cudaFree(H->d_src);
    H->d_src = nullptr;
    CK(cudaMalloc(&H->d_src, sizeof(int32_t) * 2 * n));
    H->src_cap = n;
  }
  // inputs are staged through a pageable host copy: cudaMemcpyAsync from
  // pageable memory has consumed its source when it returns, so the caller may
  // reuse or free its (possibly pinned) buffer as soon as this call returns
  H->h_src_stage.assign(sources, sources + 2 * n);
  CK(cudaMemcpyAsync(H->d_src, H->h_src_stage.data(), sizeof(int32_t) * 2 * n, cudaMemcpyHostToDevice, H->stream));
  H->st.h2d_bytes += sizeof(int32_t) * 2 * n;
  if (H->o.adjoint) {
    // the adjoint fields are fp64 whatever the handle's precision (the
    // re-centring needs the digits): the fp64 lane width of the kernel used
    const int G = use_ring(H) ? (H->D2 == 6 ? 64 : 32) : 64;
    dgdiff_status r = H->quad ? (H->D2 == 4 ? adjoint_solve<4, 32, 1>(H, sources, px, n, b, nloc, dt, nsteps)
                                            : adjoint_solve<9, 32, 1>(H, sources, px, n, b, nloc, dt, nsteps))
                    : H->D2 == 6 ? (G == 64 ? adjoint_solve<6, 64>(H, sources, px, n, b, nloc, dt, nsteps)
                                            : adjoint_solve<6, 32>(H, sources, px, n, b, nloc, dt, nsteps))
                                 : (G == 64 ? adjoint_solve<12, 64>(H, sources, px, n, b, nloc, dt, nsteps)
                                            : adjoint_solve<12, 32>(H, sources, px, n, b, nloc, dt, nsteps));
    if (r != DGDIFF_OK) return r;
    H->solved = true;
    H->last_n = n;
    H->last_dt = dt;
    H->last_nsteps = nsteps;
    return DGDIFF_OK;
  }
  std::vector<int32_t> srt;   // N1: this rank's sources in Morton order
  // chunk order -> global source index: the contiguous shard [b, e), or under
  // N1 windows the shard [b, e) of the WHOLE batch in Morton order (every rank
  // sorts the same list the same way), so that each rank's source groups are
  // spatially compact whatever the number of ranks (sorting within a
  // contiguous shard of a random source list spreads each rank's sources over
  // the whole box: 8 logical ranks on c4 ran 1.6x the one-rank work)
  std::vector<int64_t> ord(std::max<int64_t>(nloc, 0));
  for (int64_t k = 0; k < nloc; k++) ord[k] = b + k;
  if (nloc > 0 && H->windows) {
    auto morton = [](uint32_t x, uint32_t y) {
      uint64_t k = 0;
      for (int bit = 0; bit < 16; bit++)
        k |= (uint64_t)((x >> bit) & 1) << (2 * bit) | (uint64_t)((y >> bit) & 1) << (2 * bit + 1);
      return k;
    };
    // (keys once, then one sort of (key, index) pairs: the index breaks ties,
    // i.e. a stable order)
    std::vector<std::pair<uint64_t, int64_t>> key(n);
    for (int64_t k = 0; k < n; k++) key[k] = {morton(sources[2 * k], sources[2 * k + 1]), k};
    std::sort(key.begin(), key.end());
    std::vector<int64_t> all(n);
    for (int64_t k = 0; k < n; k++) all[k] = key[k].second;
    for (int64_t k = 0; k < nloc; k++) ord[k] = all[b + k];
    srt.resize(2 * nloc);
    std::vector<int32_t> perm(nloc);
    H->h_spos.assign(n, -1);
    for (int64_t k = 0; k < nloc; k++) {
      srt[2 * k] = sources[2 * ord[k]];
      srt[2 * k + 1] = sources[2 * ord[k] + 1];
      perm[k] = (int32_t)ord[k];
      H->h_spos[ord[k]] = k;
    }
    if (nloc > H->srcw_cap) {
      cudaFree(H->d_srcw); cudaFree(H->d_perm);
      H->d_srcw = nullptr; H->d_perm = nullptr;
      CK(cudaMalloc(&H->d_srcw, sizeof(int32_t) * 2 * nloc));
      CK(cudaMalloc(&H->d_perm, sizeof(int32_t) * nloc));
      H->srcw_cap = nloc;
    }
    CK(cudaMemcpyAsync(H->d_srcw, srt.data(), sizeof(int32_t) * 2 * nloc, cudaMemcpyHostToDevice, H->stream));
    CK(cudaMemcpyAsync(H->d_perm, perm.data(), sizeof(int32_t) * nloc, cudaMemcpyHostToDevice, H->stream));
    H->st.h2d_bytes += sizeof(int32_t) * 3 * nloc;
  }
  // N4 sub-pixel points: point + projected-Dirac row per source, chunk order
  const int PXS = 2 + H->D2;
  H->points = px != nullptr;
  if (nloc > 0 && px) {
    std::vector<double> rows((size_t)nloc * PXS);
    for (int64_t k = 0; k < nloc; k++)
      memcpy(&rows[(size_t)k * PXS], px + (size_t)ord[k] * PXS, sizeof(double) * PXS);
    if (nloc > H->px_cap) {
      cudaFree(H->d_px);
      H->d_px = nullptr;
      CK(cudaMalloc(&H->d_px, sizeof(double) * PXS * nloc));
      H->px_cap = nloc;
    }
    CK(cudaMemcpyAsync(H->d_px, rows.data(), sizeof(double) * PXS * nloc, cudaMemcpyHostToDevice, H->stream));
    H->st.h2d_bytes += sizeof(double) * PXS * nloc;
  }
  if (nloc > 0) {
    // chunk size: fit 3 RK registers in free device memory
    const size_t per_src = 3 * (size_t)H->nact * H->D2 * tsize(H);
    int64_t want = (nloc + G - 1) / G * G;
    int64_t chunk = want;
    if (H->o.max_chunk > 0) chunk = std::min<int64_t>(chunk, std::max<int64_t>(G, H->o.max_chunk / G * G));
    // (a capacity that free memory limited is kept: re-allocating ~150 GB of
    // state on every solve larger than it cost ~0.13 s per call)
    if (chunk > H->chunk_cap && !H->chunk_cap_fit) {
      cudaFree(H->d_Ubase);
      H->d_Ubase = nullptr;
      for (int r = 0; r < 3; r++) H->d_U[r] = nullptr;
      cudaFree(H->d_src_a); H->d_src_a = nullptr;
      cudaFree(H->d_src_ij); H->d_src_ij = nullptr;
      cudaFree(H->d_src_xy); H->d_src_xy = nullptr;
      H->chunk_cap = 0;
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      int64_t fit = (int64_t)((double)fr * 0.85 / (double)per_src) / G * G;
      if (fit < G) return fail(DGDIFF_E_NOMEM, "one source group (%d sources) needs %.3g GB", G, per_src * G / 1e9);
      H->chunk_cap_fit = fit < chunk;
      chunk = std::min(chunk, fit);
      // the three RK registers live in one allocation; env DGDIFF_STAGGER=b
      // offsets register r by r*b extra bytes (layout experiments)
      {
        size_t reg = per_src / 3 * chunk, stag = 0;
        if (const char *e = tune_env("DGDIFF_STAGGER")) stag = (size_t)atoll(e) / 256 * 256;
        CK(cudaMalloc(&H->d_Ubase, 3 * reg + 3 * stag));
        for (int r = 0; r < 3; r++) H->d_U[r] = (char *)H->d_Ubase + r * (reg + stag);
      }
      CK(cudaMalloc(&H->d_src_a, sizeof(int) * chunk));
      CK(cudaMalloc(&H->d_src_ij, sizeof(int2) * chunk));
      CK(cudaMalloc(&H->d_src_xy, sizeof(double2) * chunk));
      H->chunk_cap = chunk;
    } else {
      chunk = std::min(chunk, H->chunk_cap);
    }
    H->st.chunk = chunk;
    for (int64_t c0 = 0; c0 < nloc; c0 += chunk) {
      int64_t nvalid = std::min(chunk, nloc - c0);
      int64_t cpad = (nvalid + G - 1) / G * G;
      const int32_t *srcp = H->windows ? H->d_srcw + 2 * c0 : H->d_src + 2 * (b + c0);
      H->cur_px = px ? H->d_px + (size_t)c0 * PXS : nullptr;
      k_src_prep<<<(int)((cpad + 127) / 128), 128, 0, H->stream>>>(srcp, nvalid, cpad, H->d_aidx, H->nx,
                                                                 H->d_src_a, H->d_src_ij, H->d_src_xy,
                                                                 H->cur_px, PXS);
      H->st.launches++;
      double *rows = H->d_mom + 6 * (b + c0);
      if (H->windows) {
        // per group: bounding box of its sources (padding repeats the last valid source)
        const int64_t ng = cpad / G;
        H->h_gbox.assign(ng, make_int4(INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN));
        for (int64_t sl = 0; sl < cpad; sl++) {
          const int64_t k = c0 + std::min(sl, nvalid - 1);
          int4 &bx = H->h_gbox[sl / G];
          bx.x = std::min(bx.x, srt[2 * k]);
          bx.y = std::max(bx.y, srt[2 * k]);
          bx.z = std::min(bx.z, srt[2 * k + 1]);
          bx.w = std::max(bx.w, srt[2 * k + 1]);
        }
        // maintained active range per group: whole rows the group's stages can
        // read, [y0 - R - 1, y1 + R + 1] with R = 3 nsteps (raster order: contiguous)
        std::vector<int2> rng(ng);
        const int64_t R = std::min<int64_t>(win_radius(H, 3 * nsteps, (double)nsteps * dt) + H->halo, H->ny);
        for (int64_t g = 0; g < ng; g++) {
          const int y0 = (int)std::max<int64_t>(0, H->h_gbox[g].z - R);
          const int y1 = (int)std::min<int64_t>(H->ny, H->h_gbox[g].w + R + 1);
          rng[g] = make_int2(H->h_pre[(size_t)y0 * (H->nx + 1) + H->nx], H->h_pre[(size_t)y1 * (H->nx + 1) + H->nx]);
        }
        if (ng > H->gbox_cap) {
          cudaFree(H->d_gbox);
          cudaFree(H->d_grange);
          H->d_gbox = nullptr;
          H->d_grange = nullptr;
          CK(cudaMalloc(&H->d_gbox, sizeof(int4) * ng));
          CK(cudaMalloc(&H->d_grange, sizeof(int2) * ng));
          H->gbox_cap = ng;
        }
        CK(cudaMemcpyAsync(H->d_gbox, H->h_gbox.data(), sizeof(int4) * ng, cudaMemcpyHostToDevice, H->stream));
        CK(cudaMemcpyAsync(H->d_grange, rng.data(), sizeof(int2) * ng, cudaMemcpyHostToDevice, H->stream));
        H->st.h2d_bytes += (sizeof(int4) + sizeof(int2)) * ng;
        if (cpad > H->momc_cap) {
          cudaFree(H->d_momc);
          H->d_momc = nullptr;
          CK(cudaMalloc(&H->d_momc, sizeof(double) * 6 * cpad));
          H->momc_cap = cpad;
        }
        rows = H->d_momc;   // chunk order; k_mom_reduce scatters to the input order
        H->last_chunk_pos0 = c0;
      }
      dgdiff_status s = H->o.precision == 32 ? run_chunk_p<float>(H, nvalid, cpad, dt, nsteps, rows)
                                             : run_chunk_p<double>(H, nvalid, cpad, dt, nsteps, rows);
      if (s != DGDIFF_OK) return s;
      H->last_chunk_begin = b + c0;
      H->last_chunk_n = nvalid;
      H->last_chunk_size = cpad;
    }
  }
  H->solved = true;
  H->last_n = n;
  H->last_dt = dt;
  H->last_nsteps = nsteps;
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_solve_batch(dgdiff_t H, const int32_t *sources, int64_t n, double dt,
                                            int64_t nsteps) {
  return solve_impl(H, sources, nullptr, n, dt, nsteps);
}

extern "C" dgdiff_status dgdiff_solve_batch_points(dgdiff_t H, const double *points, int64_t n, double dt,
                                                   int64_t nsteps) {
  if (!H) return fail(DGDIFF_E_ARG, "handle is NULL");
  if (n < 1 || !points) return fail(DGDIFF_E_ARG, "need n >= 1 points");
  if (n >= (1LL << 31)) return fail(DGDIFF_E_ARG, "too many sources");
  const int PXS = 2 + H->D2;
  std::vector<int32_t> pix((size_t)2 * n);
  std::vector<double> px((size_t)n * PXS);
  for (int64_t s = 0; s < n; s++) {
    const double x = points[2 * s] / H->h, y = points[2 * s + 1] / H->h;   // pixel units
    if (!std::isfinite(x) || !std::isfinite(y) || x < 0 || y < 0 || x >= H->nx || y >= H->ny)
      return fail(DGDIFF_E_SOURCE, "point %lld (%.17g, %.17g) is outside the grid", (long long)s, points[2 * s],
                  points[2 * s + 1]);
    const int i = std::min(H->nx - 1, (int)std::floor(x)), j = std::min(H->ny - 1, (int)std::floor(y));
    pix[2 * s] = i;
    pix[2 * s + 1] = j;
    double *r = &px[(size_t)s * PXS];
    r[0] = x;
    r[1] = y;
    if (H->quad) dgop::point_init_quad(H->qtab, x - i, y - j, r + 2);
    else dgop::point_init(H->tab, x - i, y - j, r + 2);
    const double ih2 = 1.0 / (H->h * H->h);
    for (int k = 0; k < H->D2; k++) r[2 + k] *= ih2;
  }
  return solve_impl(H, pix.data(), px.data(), n, dt, nsteps);
}

extern "C" dgdiff_status dgdiff_covariance(dgdiff_t H, double delta, double sigma[4], double mu[2]) {
  if (!H) return fail(DGDIFF_E_ARG, "handle is NULL");
  if (!sigma) return fail(DGDIFF_E_ARG, "sigma is NULL");
  if (!H->solved) return fail(DGDIFF_E_STATE, "dgdiff_covariance before dgdiff_solve_batch");
  double t = H->last_nsteps * H->last_dt;
  if (!(std::fabs(delta - t) <= 1e-12 * std::max(std::fabs(delta), std::fabs(t))))
    return fail(DGDIFF_E_STATE, "delta = %.17g but the last solve reached nsteps*dt = %.17g", delta, t);
  if (H->logical)
    return fail(DGDIFF_E_STATE, "logical rank %d of %d holds only its shard: sum the ranks' dgdiff_source_moments "
                "tables and call dgdiff_covariance_table", H->o.rank, H->o.nranks);
  CK(cudaSetDevice(H->dev));
  const int64_t n = H->last_n;
  if (H->comm && !H->mom_reduced) {
    // the one cross-GPU step: sum of disjoint zero-padded rows is exact (once
    // per solve: a second covariance call must not sum the reduced table again)
    ncclResult_t r = g_nccl.allReduce(H->d_mom, H->d_mom, (size_t)6 * n, ncclFloat64, ncclSum, H->comm, H->stream);
    if (r != ncclSuccess) return fail(DGDIFF_E_NCCL, "ncclAllReduce: %s", g_nccl.errStr(r));
    H->mom_reduced = true;
  }
  k_finalize<<<1, 256, 0, H->stream>>>(H->d_mom, n, H->o.centering, H->d_out);
  H->st.launches++;
  CK(cudaGetLastError());
  double out[6];
  CK(cudaMemcpyAsync(out, H->d_out, sizeof out, cudaMemcpyDeviceToHost, H->stream));
  CK(cudaStreamSynchronize(H->stream));
  H->st.d2h_bytes += sizeof out;
  int flags = (int)out[5];
  if (flags & 2) return fail(DGDIFF_E_NONFINITE, "non-finite moments (unstable run?)");
  if (flags & 1) return fail(DGDIFF_E_DEGENERATE, "a density has m00 <= 0");
  sigma[0] = out[0];
  sigma[1] = out[1];
  sigma[2] = out[1];
  sigma[3] = out[2];
  H->last_sigma[0] = out[0];
  H->last_sigma[1] = out[1];
  H->last_sigma[2] = out[2];
  H->last_mu[0] = out[3];
  H->last_mu[1] = out[4];
  H->have_sigma = true;
  if (mu) {
    mu[0] = out[3];
    mu[1] = out[4];
  }
  return DGDIFF_OK;
}

// K5 on a caller-provided table (logical ranks: the sum of the ranks' tables)
extern "C" dgdiff_status dgdiff_covariance_table(dgdiff_t H, const double *mom, int64_t n, double sigma[4],
                                                 double mu[2]) {
  if (!H || !mom || !sigma) return fail(DGDIFF_E_ARG, "NULL argument");
  if (n < 1 || n >= (1LL << 31)) return fail(DGDIFF_E_ARG, "need 1 <= n < 2^31 rows");
  CK(cudaSetDevice(H->dev));
  double *d_tab = nullptr, *d_o = nullptr;
  auto done = [&](dgdiff_status s) { cudaFree(d_tab); cudaFree(d_o); return s; };
  cudaError_t e = cudaMalloc(&d_tab, sizeof(double) * 6 * n);
  if (e == cudaSuccess) e = cudaMalloc(&d_o, sizeof(double) * 8);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_tab, mom, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, H->stream);
  if (e == cudaSuccess) {
    k_finalize<<<1, 256, 0, H->stream>>>(d_tab, n, H->o.centering, d_o);
    H->st.launches++;
    e = cudaGetLastError();
  }
  double out[6];
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d_o, sizeof out, cudaMemcpyDeviceToHost, H->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(H->stream);
  if (e != cudaSuccess) return done(fail(DGDIFF_E_CUDA, "covariance_table: %s", cudaGetErrorString(e)));
  const int flags = (int)out[5];
  if (flags & 2) return done(fail(DGDIFF_E_NONFINITE, "non-finite moments"));
  if (flags & 1) return done(fail(DGDIFF_E_DEGENERATE, "a density has m00 <= 0"));
  sigma[0] = out[0];
  sigma[1] = out[1];
  sigma[2] = out[1];
  sigma[3] = out[2];
  if (mu) { mu[0] = out[3]; mu[1] = out[4]; }
  return done(DGDIFF_OK);
}

extern "C" dgdiff_status dgdiff_mixture(dgdiff_t H, double *grid, double *residual) {
  if (!H) return fail(DGDIFF_E_ARG, "handle is NULL");
  if (H->mix_R <= 0) return fail(DGDIFF_E_STATE, "create the handle with opts.mixture_radius > 0");
  if (!H->solved || !H->have_sigma) return fail(DGDIFF_E_STATE, "dgdiff_mixture needs dgdiff_covariance first");
  if (H->points) return fail(DGDIFF_E_STATE, "the mixture lattice is defined for pixel-centre sources (dgdiff_solve_batch)");
  CK(cudaSetDevice(H->dev));
  const int R = H->mix_R;
  const size_t nc = (size_t)(2 * R + 1) * (2 * R + 1);
  if (H->comm && !H->mix_reduced) {
    ncclResult_t r = g_nccl.allReduce(H->d_mix, H->d_mix, nc, ncclFloat64, ncclSum, H->comm, H->stream);
    if (r != ncclSuccess) return fail(DGDIFF_E_NCCL, "ncclAllReduce (mixture): %s", g_nccl.errStr(r));
    H->mix_reduced = true;
  }
  k_mixture_final<<<1, 256, 0, H->stream>>>(H->d_mix, R, H->h, H->last_n, H->last_sigma[0], H->last_sigma[1],
                                            H->last_sigma[2], H->last_mu[0], H->last_mu[1], H->d_mix_out,
                                            H->d_mix_out + nc);
  H->st.launches++;
  CK(cudaGetLastError());
  if (grid) CK(cudaMemcpyAsync(grid, H->d_mix_out, nc * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  double res = 0;
  CK(cudaMemcpyAsync(&res, H->d_mix_out + nc, sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  CK(cudaStreamSynchronize(H->stream));
  if (residual) *residual = res;
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_mc_covariance(dgdiff_t H, const int32_t *sources, int64_t n,
                                              int32_t walkers_per_source, int64_t nsteps, double delta,
                                              uint32_t seed, double sigma[4], double mu[2], double se[3],
                                              double *disp) {
  if (!H || !sources || !sigma) return fail(DGDIFF_E_ARG, "NULL argument");
  if (n < 1 || walkers_per_source < 1 || nsteps < 1 || !(delta > 0))
    return fail(DGDIFF_E_ARG, "need n, walkers_per_source, nsteps >= 1 and delta > 0");
  const int64_t nwalk = n * (int64_t)walkers_per_source;
  if (nwalk >= (1LL << 32)) return fail(DGDIFF_E_ARG, "too many walkers");
  const double l = sqrt(4.0 * H->D * delta / (double)nsteps) / H->h;   // P:318, in pixels
  if (!(l < 1.0)) return fail(DGDIFF_E_ARG, "step length %.4g h >= h: use nsteps >= 4 D delta / h^2", l);
  for (int64_t s = 0; s < n; s++) {
    int i = sources[2 * s], j = sources[2 * s + 1];
    if (i < 0 || j < 0 || i >= H->nx || j >= H->ny || H->h_aidx[(size_t)j * H->nx + i] < 0)
      return fail(DGDIFF_E_SOURCE, "source %lld (%d,%d) is outside the grid or on an axon pixel", (long long)s, i, j);
  }
  CK(cudaSetDevice(H->dev));
  int32_t *d_src = nullptr;
  double *d_part = nullptr, *d_disp = nullptr, *d_res = nullptr;
  const int blocks = (int)((nwalk + 255) / 256);
  dgdiff_status st = DGDIFF_OK;
  auto cleanup = [&]() { cudaFree(d_src); cudaFree(d_part); cudaFree(d_disp); cudaFree(d_res); };
  cudaError_t e = cudaMalloc(&d_src, sizeof(int32_t) * 2 * n);
  if (e == cudaSuccess) e = cudaMalloc(&d_part, sizeof(double) * 5 * blocks);
  if (e == cudaSuccess) e = cudaMalloc(&d_res, sizeof(double) * 8);
  if (e == cudaSuccess && disp) e = cudaMalloc(&d_disp, sizeof(double) * 2 * nwalk);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_src, sources, sizeof(int32_t) * 2 * n, cudaMemcpyHostToDevice, H->stream);
  if (e == cudaSuccess) {
    dgk::k_mc_walk<<<blocks, 256, 0, H->stream>>>(H->d_aidx, H->nx, H->ny, d_src, nwalk, n, nsteps, l, seed,
                                                  d_part, d_disp);
    dgk::k_mc_final<<<1, 32, 0, H->stream>>>(d_part, blocks, nwalk, std::min(32, blocks), H->h, d_res);
    H->st.launches += 2;
    e = cudaGetLastError();
  }
  double out[8];
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d_res, sizeof out, cudaMemcpyDeviceToHost, H->stream);
  if (e == cudaSuccess && disp)
    e = cudaMemcpyAsync(disp, d_disp, sizeof(double) * 2 * nwalk, cudaMemcpyDeviceToHost, H->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(H->stream);
  if (e != cudaSuccess) st = fail(DGDIFF_E_CUDA, "mc: %s", cudaGetErrorString(e));
  cleanup();
  if (st != DGDIFF_OK) return st;
  sigma[0] = out[0];
  sigma[1] = out[1];
  sigma[2] = out[1];
  sigma[3] = out[2];
  if (mu) { mu[0] = out[3]; mu[1] = out[4]; }
  if (se) { se[0] = out[5]; se[1] = out[6]; se[2] = out[7]; }
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_absorb_table(int32_t degree, double *A) {
  if (degree < 1 || degree > 3) return fail(DGDIFF_E_ARG, "degree %d not supported (1..3)", degree);
  if (!A) return fail(DGDIFF_E_ARG, "A is NULL");
  try {
    std::vector<double> T = dgop::build_absorb(degree);
    memcpy(A, T.data(), T.size() * sizeof(double));
  } catch (std::exception &e) {
    return fail(DGDIFF_E_ARG, "operator precompute failed: %s", e.what());
  }
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_quad_table(int32_t degree, double *blocks) {
  if (degree < 1 || degree > 2) return fail(DGDIFF_E_ARG, "quadrilateral degree %d not supported (1 or 2)", degree);
  if (!blocks) return fail(DGDIFF_E_ARG, "NULL argument");
  try {
    dgop::QuadTable T = dgop::build_quad(degree);
    memcpy(blocks, T.blocks.data(), sizeof(double) * T.blocks.size());
  } catch (const std::exception &e) {
    return fail(DGDIFF_E_ARG, "K0 (quads): %s", e.what());
  }
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_centre_weights(int32_t degree, double *cw) {
  if (degree < 1 || degree > 3) return fail(DGDIFF_E_ARG, "degree %d not supported (1..3)", degree);
  if (!cw) return fail(DGDIFF_E_ARG, "cw is NULL");
  try {
    dgop::Table T = dgop::build(degree);
    memcpy(cw, T.cw.data(), T.cw.size() * sizeof(double));
  } catch (std::exception &e) {
    return fail(DGDIFF_E_ARG, "operator precompute failed: %s", e.what());
  }
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_source_moments(dgdiff_t H, double *out) {
  if (!H || !out) return fail(DGDIFF_E_ARG, "NULL argument");
  if (!H->solved) return fail(DGDIFF_E_STATE, "no solve yet");
  CK(cudaSetDevice(H->dev));
  CK(cudaMemcpyAsync(out, H->d_mom, sizeof(double) * 6 * H->last_n, cudaMemcpyDeviceToHost, H->stream));
  CK(cudaStreamSynchronize(H->stream));
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_get_density(dgdiff_t H, int64_t src, double *out) {
  if (!H || !out) return fail(DGDIFF_E_ARG, "NULL argument");
  if (!H->solved || !H->o.keep_density) return fail(DGDIFF_E_STATE, "needs keep_density and a solve");
  int64_t k = src - H->last_chunk_begin;
  if (H->windows) {
    // N1: chunks hold the rank's share of the Morton-ordered batch
    k = (src >= 0 && src < (int64_t)H->h_spos.size() && H->h_spos[src] >= 0) ? H->h_spos[src] - H->last_chunk_pos0 : -1;
  }
  if (k < 0 || k >= H->last_chunk_n)
    return fail(DGDIFF_E_STATE, "source %lld is not in this rank's last chunk", (long long)src);
  CK(cudaSetDevice(H->dev));
  const int G = gsize(H);
  int g = (int)(k / G), slot = (int)(k % G);
  const int64_t nel = H->nact * H->D2;
  double *d_tmp = nullptr;
  CK(cudaMalloc(&d_tmp, sizeof(double) * nel));
  int blocks = (int)((nel + 255) / 256);
  const int nv = lane_nv(H);
  const int2 *gr = H->windows ? H->d_grange : nullptr;
#define DG_GATHER(TT, NVV)                                                                                     \
  if (H->D2 == 6) k_gather<TT, NVV, 6><<<blocks, 256, 0, H->stream>>>((TT *)H->d_U[0], (int)H->nact, g, slot, d_tmp, gr); \
  else if (H->D2 == 20) k_gather<TT, NVV, 20><<<blocks, 256, 0, H->stream>>>((TT *)H->d_U[0], (int)H->nact, g, slot, d_tmp, gr); \
  else if (H->D2 == 4) k_gather<TT, NVV, 4><<<blocks, 256, 0, H->stream>>>((TT *)H->d_U[0], (int)H->nact, g, slot, d_tmp, gr); \
  else if (H->D2 == 9) k_gather<TT, NVV, 9><<<blocks, 256, 0, H->stream>>>((TT *)H->d_U[0], (int)H->nact, g, slot, d_tmp, gr); \
  else k_gather<TT, NVV, 12><<<blocks, 256, 0, H->stream>>>((TT *)H->d_U[0], (int)H->nact, g, slot, d_tmp, gr);
  if (H->o.precision == 32) {
    if (nv == 1) { DG_GATHER(float, 1) } else if (nv == 2) { DG_GATHER(float, 2) } else { DG_GATHER(float, 4) }
  } else {
    if (nv == 1) { DG_GATHER(double, 1) } else { DG_GATHER(double, 2) }
  }
#undef DG_GATHER
  std::vector<double> tmp(nel);
  cudaError_t e = cudaMemcpyAsync(tmp.data(), d_tmp, sizeof(double) * nel, cudaMemcpyDeviceToHost, H->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(H->stream);
  cudaFree(d_tmp);
  if (e != cudaSuccess) return fail(DGDIFF_E_CUDA, "get_density: %s", cudaGetErrorString(e));
  memset(out, 0, sizeof(double) * (size_t)H->nx * H->ny * H->D2);
  std::vector<int2> pix(H->nact);
  CK(cudaMemcpy(pix.data(), H->d_pix, sizeof(int2) * H->nact, cudaMemcpyDeviceToHost));
  for (int64_t a = 0; a < H->nact; a++)
    memcpy(out + ((size_t)pix[a].y * H->nx + pix[a].x) * H->D2, tmp.data() + a * H->D2, sizeof(double) * H->D2);
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_set_timing(dgdiff_t H, int32_t enable) {
  if (!H) return fail(DGDIFF_E_ARG, "handle is NULL");
  H->timing = enable != 0;
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_reset_stats(dgdiff_t H) {
  if (!H) return fail(DGDIFF_E_ARG, "handle is NULL");
  CK(cudaSetDevice(H->dev));
  CK(cudaStreamSynchronize(H->stream));
  int64_t na = H->st.n_active, ch = H->st.chunk;
  memset(&H->st, 0, sizeof H->st);
  H->st.n_active = na;
  H->st.chunk = ch;
  H->ev_used = 0;
  H->ev_launches_pending = 0;
  H->evd_used = 0;
  return DGDIFF_OK;
}

extern "C" dgdiff_status dgdiff_get_stats(dgdiff_t H, dgdiff_stats_t *out) {
  if (!H || !out) return fail(DGDIFF_E_ARG, "NULL argument");
  CK(cudaSetDevice(H->dev));
  if (H->ev_used) {
    CK(cudaStreamSynchronize(H->stream));
    double ms = 0;
    for (size_t k = 0; k < H->ev_used; k++) {
      float f = 0;
      CK(cudaEventElapsedTime(&f, H->ev[k].first, H->ev[k].second));
      ms += f;
    }
    H->st.stage_ms += ms;
    if (H->o.temporal_steps != 5) H->st.dom_ms += ms;   // K2: stage kernels = dominant kernel
    H->ev_used = 0;
    H->ev_launches_pending = 0;
  }
  if (H->evd_used) {
    CK(cudaStreamSynchronize(H->stream));
    double ms = 0;
    for (size_t k = 0; k < H->evd_used; k++) {
      float f = 0;
      CK(cudaEventElapsedTime(&f, H->evd[k].first, H->evd[k].second));
      ms += f;
    }
    H->st.dom_ms += ms;
    H->evd_used = 0;
  }
  if (H->stage_detail) {
    CK(cudaStreamSynchronize(H->stream));
    for (int k = 0; k < 3; k++)
      if (H->sev_pending[k]) {
        float f = 0;
        CK(cudaEventElapsedTime(&f, H->sev[k][0], H->sev[k][1]));
        H->sev_pending[k] = false;
        fprintf(stderr, "[dgdiff] stage %d: %.3f ms\n", k + 1, f);
      }
  }
  H->st.env_overrides = dgk::tune_overrides().load();
#ifdef DGDIFF_TUNING
  H->st.tuning_build = 1;
#else
  H->st.tuning_build = 0;
#endif
  *out = H->st;
  return DGDIFF_OK;
}
