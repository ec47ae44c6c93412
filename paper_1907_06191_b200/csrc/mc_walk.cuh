// mc_walk.cuh -- N3: Monte-Carlo random walk on the pixel substrate, an
// independent cross-check of the DG covariance (the paper's comparison,
// P:312-328, with its step-length relation l = sqrt(4 D t_s / T)).
//
// Walker w of source s = w mod S starts at the source pixel centre and takes T
// steps of length l (grid units) in uniform random directions.  A step whose
// straight segment would enter an axon pixel or leave the grid is rejected
// (the walker stays; SPEC's rejection rule, a reflecting barrier as l -> 0).
// l < 1 pixel, so a segment crosses at most one vertical and one horizontal
// pixel edge; the pixels it visits are checked in crossing order.
//
// Randomness: Philox4x32-10 (counter-based), key = (seed, walker), counter =
// (step low, step high, draw, 0x5eed5eed); a direction is (a, b)/sqrt(a^2 + b^2) with (a, b)
// uniform in the unit disk by rejection from the square (only IEEE-exact
// operations, so a CPU reimplementation reproduces trajectories bit for bit).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dgk {

struct Philox {
  __host__ __device__ static inline void mulhilo(uint32_t a, uint32_t b, uint32_t &hi, uint32_t &lo) {
    const uint64_t p = (uint64_t)a * (uint64_t)b;
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
  }
  // Philox4x32-10: counter c[4], key k[2]
  __host__ __device__ static inline void run(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; r++) {
      uint32_t hi0, lo0, hi1, lo1;
      mulhilo(0xD2511F53u, c[0], hi0, lo0);
      mulhilo(0xCD9E8D57u, c[2], hi1, lo1);
      const uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
      c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
};

// uniform in [0, 1) with 53 random bits from two 32-bit words
__host__ __device__ inline double u01(uint32_t hi, uint32_t lo) {
  const uint64_t m = ((uint64_t)(hi >> 5) << 26) | (uint64_t)(lo >> 6);   // 27 + 26 bits
  return (double)m * (1.0 / 9007199254740992.0);
}

// one walker: returns the displacement after T steps
__device__ inline void mc_walk_one(const int *__restrict__ aidx, int nx, int ny, double x0, double y0, int64_t T,
                                   double l, uint32_t seed, uint32_t walker, double &dx_out, double &dy_out) {
  double x = x0, y = y0;
  for (int64_t t = 0; t < T; t++) {
    double a = 0, b = 0, r2 = 0;
    for (uint32_t draw = 0;; draw++) {
      uint32_t c[4] = {(uint32_t)t, (uint32_t)(t >> 32), draw, 0x5eed5eedu};
      Philox::run(c, seed, walker);
      a = 2.0 * u01(c[0], c[1]) - 1.0;
      b = 2.0 * u01(c[2], c[3]) - 1.0;
      r2 = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));   // no FMA contraction: bit-reproducible
      if (r2 > 0.0 && r2 <= 1.0) break;
    }
    const double s = l / sqrt(r2);
    const double nxp = __dadd_rn(x, __dmul_rn(a, s)), nyp = __dadd_rn(y, __dmul_rn(b, s));
    // pixels visited by the segment (x, y) -> (nxp, nyp): start pixel, then
    // the crossings of the vertical / horizontal pixel edges in order
    int ci = (int)floor(x), cj = (int)floor(y);
    const int ei = (int)floor(nxp), ej = (int)floor(nyp);
    bool ok = true;
    if (ei != ci || ej != cj) {
      double tx = 2.0, ty = 2.0;   // parameters of the edge crossings (>1: none)
      if (ei != ci) tx = ((ei > ci ? (double)ei : (double)ci) - x) / (nxp - x);
      if (ej != cj) ty = ((ej > cj ? (double)ej : (double)cj) - y) / (nyp - y);
      // first crossing
      if (tx < ty) ci = ei; else if (ty < tx) cj = ej; else { ci = ei; cj = ej; }
      auto blocked = [&](int i, int j) {
        return i < 0 || j < 0 || i >= nx || j >= ny || __ldg(&aidx[(size_t)j * nx + i]) < 0;
      };
      if (blocked(ci, cj)) ok = false;
      if (ok && (ci != ei || cj != ej)) {   // second crossing
        ci = ei;
        cj = ej;
        if (blocked(ci, cj)) ok = false;
      }
    }
    if (ok) { x = nxp; y = nyp; }
  }
  dx_out = x - x0;
  dy_out = y - y0;
}

// walkers w = blockIdx.x * blockDim.x + threadIdx.x < S * K; per-block sums of
// (dx, dy, dx^2, dx dy, dy^2) in fixed order -> partial[block][5]
__global__ void __launch_bounds__(256) k_mc_walk(const int *__restrict__ aidx, int nx, int ny,
                                                 const int32_t *__restrict__ src, int64_t nwalk, int64_t S, int64_t T,
                                                 double l, uint32_t seed, double *__restrict__ partial,
                                                 double *__restrict__ disp /* nullable [nwalk][2] */) {
  __shared__ double sh[5][256];
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double v[5] = {0, 0, 0, 0, 0};
  if (w < nwalk) {
    const int64_t s = w % S;   // interleaved: every batch of walkers spans all sources
    const double x0 = src[2 * s] + 0.5, y0 = src[2 * s + 1] + 0.5;
    double dx, dy;
    mc_walk_one(aidx, nx, ny, x0, y0, T, l, seed, (uint32_t)w, dx, dy);
    v[0] = dx; v[1] = dy; v[2] = dx * dx; v[3] = dx * dy; v[4] = dy * dy;
    if (disp) { disp[2 * w] = dx; disp[2 * w + 1] = dy; }
  }
  for (int q = 0; q < 5; q++) sh[q][threadIdx.x] = v[q];
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int q = 0; q < 5; q++) sh[q][threadIdx.x] += sh[q][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < 5; q++) partial[(size_t)blockIdx.x * 5 + q] = sh[q][0];
}

// Sigma and its standard errors from nbatch equal batches of blocks (fixed
// order): out = {sxx, sxy, syy, mux, muy, se_xx, se_xy, se_yy}
__global__ void k_mc_final(const double *__restrict__ partial, int nblk, int64_t nwalk, int nbatch, double h,
                           double *__restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double tot[5] = {0, 0, 0, 0, 0}, bs[3] = {0, 0, 0}, bs2[3] = {0, 0, 0};
  const int per = (nblk + nbatch - 1) / nbatch;
  int used = 0;
  for (int b = 0; b < nbatch; b++) {
    double t[5] = {0, 0, 0, 0, 0};
    const int b0 = b * per, b1 = min(nblk, b0 + per);
    if (b0 >= b1) continue;
    for (int k = b0; k < b1; k++)
      for (int q = 0; q < 5; q++) t[q] += partial[(size_t)k * 5 + q];
    const int64_t wend = (int64_t)b1 * 256 < nwalk ? (int64_t)b1 * 256 : nwalk;
    const double nb = (double)(wend - (int64_t)b0 * 256);
    for (int q = 0; q < 5; q++) tot[q] += t[q];
    const double mx = t[0] / nb, my = t[1] / nb;
    const double c[3] = {t[2] / nb - mx * mx, t[3] / nb - mx * my, t[4] / nb - my * my};
    for (int q = 0; q < 3; q++) { bs[q] += c[q]; bs2[q] += c[q] * c[q]; }
    used++;
  }
  const double n = (double)nwalk, mx = tot[0] / n, my = tot[1] / n, h2 = h * h;
  out[0] = (tot[2] / n - mx * mx) * h2;
  out[1] = (tot[3] / n - mx * my) * h2;
  out[2] = (tot[4] / n - my * my) * h2;
  out[3] = mx * h;
  out[4] = my * h;
  for (int q = 0; q < 3; q++) {
    const double m = bs[q] / used, var = bs2[q] / used - m * m;
    out[5 + q] = used > 1 ? sqrt(fmax(var, 0.0) / (used - 1)) * h2 : 0.0;
  }
}

}  // namespace dgk
