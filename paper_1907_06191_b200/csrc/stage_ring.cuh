// stage_ring.cuh -- K2 v3: one SSP-RK3 stage, row-marching over a shared-memory
// byte ring filled by 1-D bulk TMA (cp.async.bulk + mbarrier).
//
// Work item = (column strip s of W pixels, source group g of G = 32 NV
// sources, band of rows [jb0, jb1)).  Because extracellular pixels are stored
// in raster order, the pixels of row j with x in [x0-1, x0+W+1) are one
// contiguous run of the state array for group g: one bulk copy per row
// ("row tile", rowtab[s][j] = {h0, c0, c1, h1} active-index bounds of the
// halo'd and computed ranges).  Row tiles enter a byte ring in order; thread 0
// keeps as many rows in flight as the ring holds (adaptive lookahead: sparse
// Gamma rows are ~40 % of a full row), so every pixel is read from HBM once
// per stage (plus the 2-column strip halo and 2 band-halo rows).  Warp w
// computes the w-th extracellular pixel of row j from rows j-1, j, j+1 in
// shared memory; u0 (the alpha term) and the neighbour indices of row j+1
// are prefetched into registers one row ahead; outputs go straight to HBM.
//
// Ring invariants (checked by construction): the ring is a circular buffer of
// NSLOT pixel tiles; a row tile may wrap (two bulk copies, one mbarrier), so
// no space is wasted.  At iteration j thread 0 may overwrite rows <= j-3 only
// (their last reader, compute(j-2), finished before the barrier of iteration
// j-1); NSLOT = 4 full rows, so row j+1 can always be issued; at most Q-2
// rows are live per mbarrier set.
#pragma once
#include "kernels.cuh"
#include "stage_imm.cuh"

namespace dgk {

constexpr int RING_Q = 16;        // row entries (mbarriers)
constexpr int RING_MAXBAND = 512; // max rows per band (+2 halo) for the rowtab cache

template <int P> struct RingCfg;  // warps per CTA = strip width W
template <> struct RingCfg<1> { static constexpr int W = 32; };
template <> struct RingCfg<2> { static constexpr int W = 16; };

template <typename T, int NV, int P>
struct RingGeom {
  static constexpr int G = 32 * NV;
  static constexpr int D2 = (P + 1) * (P + 2);
  static constexpr int W = RingCfg<P>::W;
  static constexpr int PXB = D2 * G * (int)sizeof(T);             // bytes of one pixel tile
  static constexpr int NSLOT = 4 * (W + 2);                       // ring capacity in pixel tiles
  static constexpr int RB = NSLOT * PXB;                          // ring bytes: 4 full rows
  static constexpr int SMEM = RB + RING_Q * 8 + RING_Q * 16 + (RING_MAXBAND + 2) * 16;
};

template <typename T, int NV, int P, bool HAS_ALPHA>
__global__ void __launch_bounds__(RingCfg<P>::W * 32, 1)
    k_stage_ring(const T *__restrict__ Uin, const T *U0, T *Uout, const int4 *__restrict__ nbr,
                 const int4 *__restrict__ rowtab, int nact, int ny, int nstrips, int ngroups, int band_rows,
                 int nitems, T alpha, T cs) {
  using Gm = RingGeom<T, NV, P>;
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, RB = Gm::RB, Q = RING_Q;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *ring = smem;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + RB);
  int4 *meta = reinterpret_cast<int4 *>(smem + RB + Q * 8);          // {phys off, h0, -, -}
  int4 *rt = reinterpret_cast<int4 *>(smem + RB + Q * 8 + Q * 16);   // band rowtab cache
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < Q; q++) mbar_init(&bars[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t Lbase = 0;               // loads issued by this CTA before the current item
  uint32_t vst[Q];                  // thread 0: virtual start offset per entry
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int s = item % nstrips;
    const int g = (item / nstrips) % ngroups;
    const int b = item / (nstrips * ngroups);
    const int jb0 = b * band_rows, jb1 = min(ny, jb0 + band_rows);
    const int lo = max(0, jb0 - 1), hi = min(ny - 1, jb1);
    for (int r = lo + tid; r <= hi; r += blockDim.x) rt[r - lo] = __ldg(&rowtab[(size_t)s * ny + r]);
    __syncthreads();
    const T *Ug = Uin + (size_t)g * nact * D2 * G;
    const T *U0g = U0 + (size_t)g * nact * D2 * G + lane * NV;
    T *Uog = Uout + (size_t)g * nact * D2 * G + lane * NV;
    // producer state (thread 0): wv = virtual pixel-slot counter
    int ld_row = lo;
    uint32_t wv = 0;
    // prefetch row jb0
    int a_n = -1;
    int4 nb_n = make_int4(-1, -1, -1, -1);
    T u0_n[D2][NV];
    {
      const int4 t = rt[jb0 - lo];
      if (t.y + w < t.z) {
        a_n = t.y + w;
        nb_n = __ldg(&nbr[a_n]);
        if (HAS_ALPHA)
#pragma unroll
          for (int k = 0; k < D2; k++) ldvc<T, NV>(U0g + ((size_t)a_n * D2 + k) * G, u0_n[k]);
      }
    }
    for (int j = jb0; j < jb1; j++) {
      if (tid == 0) {
        const int live = max(lo, j - 2);
        const uint32_t vlive = (ld_row > live) ? vst[(Lbase + (live - lo)) % Q] : wv;
        bool fenced = false;
        while (ld_row <= hi && ld_row - live < Q - 2) {
          const int4 t = rt[ld_row - lo];
          const uint32_t cnt = (uint32_t)(t.w - t.x);       // pixel tiles in this row
          if (wv + cnt - vlive > (uint32_t)Gm::NSLOT) break;
          const uint32_t L = Lbase + (ld_row - lo), q = L % Q;
          const uint32_t p0 = wv % Gm::NSLOT;
          meta[q] = make_int4((int)p0, t.x, 0, 0);
          vst[q] = wv;
          if (!fenced) { fence_proxy_async(); fenced = true; }
          mbar_expect_tx(&bars[q], cnt * PXB);
          const uint32_t c1 = min(cnt, (uint32_t)Gm::NSLOT - p0);
          const T *src = Ug + (size_t)t.x * D2 * G;
          if (c1) bulk_g2s(ring + (size_t)p0 * PXB, src, c1 * PXB, &bars[q]);
          if (cnt > c1) bulk_g2s(ring, src + (size_t)c1 * D2 * G, (cnt - c1) * PXB, &bars[q]);
          wv += cnt;
          ld_row++;
        }
      }
      __syncthreads();
      // rotate the prefetch registers and issue row j+1's
      const int a = a_n;
      const int4 nb = nb_n;
      T u0v[D2][NV];
      if (HAS_ALPHA)
#pragma unroll
        for (int k = 0; k < D2; k++)
#pragma unroll
          for (int e = 0; e < NV; e++) u0v[k][e] = u0_n[k][e];
      a_n = -1;
      if (j + 1 < jb1) {
        const int4 t = rt[j + 1 - lo];
        if (t.y + w < t.z) {
          a_n = t.y + w;
          nb_n = __ldg(&nbr[a_n]);
          if (HAS_ALPHA)
#pragma unroll
            for (int k = 0; k < D2; k++) ldvc<T, NV>(U0g + ((size_t)a_n * D2 + k) * G, u0_n[k]);
        }
      }
      // rows j-1, j, j+1 must have landed
      for (int r = max(lo, j - 1); r <= min(hi, j + 1); r++) {
        const uint32_t L = Lbase + (r - lo);
        mbar_wait(&bars[L % Q], (L / Q) & 1);
      }
      if (a >= 0) {
        // pixel tile address in the ring: slot (row start + index in row) mod NSLOT
        auto tile = [&](const int4 &m, int idx) -> const T * {
          int sl = m.x + (idx - m.y);
          if (sl >= Gm::NSLOT) sl -= Gm::NSLOT;
          return reinterpret_cast<const T *>(ring + (size_t)sl * PXB) + lane * NV;
        };
        const int4 mc = meta[(Lbase + (j - lo)) % Q];
        const T *ps = tile(mc, a);
        T xs[D2][NV], acc[D2][NV], xn[D2][NV];
#pragma unroll
        for (int k = 0; k < D2; k++) lds<T, NV>(ps + k * G, xs[k]);
#pragma unroll
        for (int k = 0; k < D2; k++)
#pragma unroll
          for (int e = 0; e < NV; e++) acc[k][e] = (T)0;
        mv_imm<T, NV, P, 0>(acc, xs);
        if (nb.x >= 0) {
          const T *pn = tile(mc, nb.x);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 1>(acc, xs);
          mv_imm<T, NV, P, 5>(acc, xn);
        }
        if (nb.y >= 0) {
          const T *pn = tile(mc, nb.y);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 2>(acc, xs);
          mv_imm<T, NV, P, 6>(acc, xn);
        }
        if (nb.z >= 0) {
          const int4 mn = meta[(Lbase + (j + 1 - lo)) % Q];
          const T *pn = tile(mn, nb.z);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 3>(acc, xs);
          mv_imm<T, NV, P, 7>(acc, xn);
        }
        if (nb.w >= 0) {
          const int4 ms = meta[(Lbase + (j - 1 - lo)) % Q];
          const T *pn = tile(ms, nb.w);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 4>(acc, xs);
          mv_imm<T, NV, P, 8>(acc, xn);
        }
        T *out = Uog + (size_t)a * D2 * G;
#pragma unroll
        for (int k = 0; k < D2; k++) {
          T y[NV];
#pragma unroll
          for (int e = 0; e < NV; e++)
            y[e] = HAS_ALPHA ? xs[k][e] + alpha * (u0v[k][e] - xs[k][e]) + cs * acc[k][e]
                             : xs[k][e] + cs * acc[k][e];
          stv<T, NV>(out + (size_t)k * G, y);
        }
      }
    }
    __syncthreads();  // item done: ring, rt cache and barriers quiescent
    Lbase += (uint32_t)(hi - lo + 1);
  }
}

}  // namespace dgk
