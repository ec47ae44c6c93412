// step_dec.cuh -- K3b: one whole SSP-RK3 step per pass (temporal blocking,
// T_b = 1) with DECOUPLED warp roles instead of K3's per-row lock-step.
//
//   producer warp   u row tiles (3-column strip halo) -> slot ring (bulk TMA)
//   A warps (NA)    U1(r) = u + c1 L(u)          rows i0..i1, from the u ring
//   B warps (NB)    U2(r) = U1 + 3/4 (u - U1) + c2 L(U1)      from U1 slots
//   C warps (NCW)   u'(r) = U2 + 1/3 (u - U2) + c3 L(U2)      from U2 slots
//
// Each role walks the rows in order and its warps split a row's pixels
// round-robin; rows are handed on through mbarriers instead of CTA barriers:
// f1/e1 (U1 slot full / empty, 4 slots), f2/e2 (U2, 4 slots) and the u
// ring's full/empty pairs.  A runs up to 3 rows ahead of B, B up to 3 ahead
// of C.  The alpha terms (u at the pixel) and the neighbour indices of B and
// C come from HBM/L2 (read-only), so only A touches the u ring.
// HBM traffic per step: u once through the ring (+ halo), u twice more as
// alpha terms (L2-resident: the same rows A just streamed), u' once.
#pragma once
#include <atomic>
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "launch.h"
#include "stage_imm.cuh"
#include "step_fused.cuh"

namespace dgk {

constexpr int DQ = 32;          // u-ring row entries
constexpr int DMAXBAND = 128;

struct DecGeom {
  using T = double;
#ifndef DEC_NA
#define DEC_NA 5
#define DEC_NB 4
#define DEC_NC 4
#endif
  static constexpr int D2 = 6, G = 32, W = 8, NA = DEC_NA, NB = DEC_NB, NCW = DEC_NC;
  static constexpr int NCONS = NA + NB + NCW, THREADS = (NCONS + 1) * 32;
  static constexpr int PXB = D2 * G * 8;
  static constexpr int SLOT1 = W + 4, SLOT2 = W + 2;
  static constexpr int U1B = 4 * SLOT1 * PXB, U2B = 4 * SLOT2 * PXB;
  static constexpr int SMEM_MAX = 232448;
  static constexpr int BARS = (2 * DQ + 16) * 8;
  static constexpr int EXTRA = BARS + DQ * 32 + (DMAXBAND + 8) * 32 + DQ * 4 + 64;
  static constexpr int N1 = (SMEM_MAX - U1B - U2B - EXTRA) / (PXB + 16);
  static constexpr int OFF_U1 = 0, OFF_U2 = U1B, OFF_R = U1B + U2B;
  static constexpr int OFF_NB = OFF_R + N1 * PXB;
  static constexpr int OFF_BAR = OFF_NB + N1 * 16;
  static constexpr int OFF_META = OFF_BAR + BARS;
  static constexpr int OFF_RT = OFF_META + DQ * 32;
  static constexpr int OFF_RV = OFF_RT + (DMAXBAND + 8) * 32;
  static constexpr int SMEM = OFF_RV + DQ * 4 + 64;
  static_assert(SMEM <= SMEM_MAX, "decoupled step does not fit in shared memory");
  static_assert(N1 >= 4 * (W + 6), "u ring too small for progress");
};

__global__ void __launch_bounds__(DecGeom::THREADS, 1)
    k_step_dec(const double *__restrict__ Uin, double *__restrict__ Uout, const int4 *__restrict__ nbr,
               const int4 *__restrict__ rowtab3, int nact, int ny, int nstrips, int ngroups, int band_rows,
               int nitems, double c1, double c2, double c3, int max_ahead) {
  using Gm = DecGeom;
  using T = double;
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, Q = DQ, NA = Gm::NA, NB = Gm::NB, NCW = Gm::NCW;
  constexpr int SLOT1 = Gm::SLOT1, SLOT2 = Gm::SLOT2;
  extern __shared__ __align__(128) unsigned char smem[];
  T *u1s = reinterpret_cast<T *>(smem + Gm::OFF_U1);
  T *u2s = reinterpret_cast<T *>(smem + Gm::OFF_U2);
  unsigned char *ring = smem + Gm::OFF_R;
  int4 *nring = reinterpret_cast<int4 *>(smem + Gm::OFF_NB);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Gm::OFF_BAR);
  uint64_t *empty = full + Q;
  uint64_t *f1 = empty + Q, *e1 = f1 + 4, *f2 = e1 + 4, *e2 = f2 + 4;
  FMeta *meta = reinterpret_cast<FMeta *>(smem + Gm::OFF_META);
  int4 *rt = reinterpret_cast<int4 *>(smem + Gm::OFF_RT);
  uint32_t *rv = reinterpret_cast<uint32_t *>(smem + Gm::OFF_RV);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < Q; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NA);
    }
    for (int s = 0; s < 4; s++) {
      mbar_init(&f1[s], NA);
      mbar_init(&e1[s], NB);
      mbar_init(&f2[s], NB);
      mbar_init(&e2[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t gstride = (size_t)nact * D2 * G;

  if (w == Gm::NCONS) {
    // ============ producer warp (as K3: batches of up to 32 rows) ============
    uint32_t L = 0, v1 = 0, rel = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      const int s = item % nstrips;
      const int g = (item / nstrips) % ngroups;
      const int b = item / (nstrips * ngroups);
      const int jb0 = b * band_rows, jb1 = min(ny, jb0 + band_rows);
      const int lo = max(0, jb0 - 3), hi = min(ny - 1, jb1 + 2);
      __syncwarp();
      for (int r = lo + lane; r <= hi; r += 32) {
        rt[2 * (r - lo)] = __ldg(&rowtab3[2 * ((size_t)s * ny + r)]);
        rt[2 * (r - lo) + 1] = __ldg(&rowtab3[2 * ((size_t)s * ny + r) + 1]);
      }
      __syncwarp();
      const T *Ug = Uin + g * gstride;
      for (int r0 = lo; r0 <= hi;) {
        const int r = r0 + lane;
        const bool valid = r <= hi;
        int4 ta = make_int4(0, 0, 0, 0), tb = make_int4(0, 0, 0, 0);
        if (valid) { ta = rt[2 * (r - lo)]; tb = rt[2 * (r - lo) + 1]; }
        const uint32_t n1 = valid ? (uint32_t)(tb.w - ta.x) : 0u;
        uint32_t e = n1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, e, o);
          if (lane >= o) e += y;
        }
        const uint32_t nvalid = (uint32_t)min(32, hi - r0 + 1);
        uint32_t take;
        for (;;) {
          const uint32_t s1 = rel ? rv[(rel - 1) % Q] : 0u;
          const bool fits = valid && (L + lane - rel < (uint32_t)max_ahead) && (v1 + e - s1 <= (uint32_t)Gm::N1);
          const uint32_t ok = __ballot_sync(0xffffffffu, fits);
          take = (ok == 0xffffffffu) ? 32u : (uint32_t)(__ffs(~ok) - 1);
          if (take > nvalid) take = nvalid;
          if (take > 0 || rel == L) break;
          mbar_wait(&empty[rel % Q], (rel / Q) & 1);
          rel++;
        }
        if (take == 0) take = 1;
        if ((uint32_t)lane < take) {
          const uint32_t Lr = L + lane, q = Lr % Q;
          if (Lr >= (uint32_t)Q) mbar_wait(&full[q], ((Lr - Q) / Q) & 1);
          const uint32_t b1v = v1 + e - n1, p1 = b1v % Gm::N1;
          FMeta m;
          m.p = (int)p1; m.h0 = ta.x; m.a1 = ta.y; m.a2 = ta.z;
          m.c0 = ta.w; m.c1 = tb.x; m.b2 = tb.y; m.b1 = tb.z;
          meta[q] = m;
          rv[q] = v1 + e;
          mbar_expect_tx(&full[q], n1 * (PXB + 16u));
          if (n1) {
            const uint32_t a1 = min(n1, (uint32_t)Gm::N1 - p1);
            const T *src = Ug + (size_t)ta.x * D2 * G;
            bulk_g2s(ring + (size_t)p1 * PXB, src, a1 * PXB, &full[q]);
            bulk_g2s(nring + p1, nbr + ta.x, a1 * 16u, &full[q]);
            if (n1 > a1) {
              bulk_g2s(ring, src + (size_t)a1 * D2 * G, (n1 - a1) * PXB, &full[q]);
              bulk_g2s(nring, nbr + ta.x + a1, (n1 - a1) * 16u, &full[q]);
            }
          }
        }
        v1 += __shfl_sync(0xffffffffu, e, take - 1);
        L += take;
        r0 += (int)take;
        __syncwarp();
      }
    }
    return;
  }

  // ================================ consumers ================================
  const int role = w < NA ? 0 : (w < NA + NB ? 1 : 2);
  const int rw = role == 0 ? w : (role == 1 ? w - NA : w - NA - NB);   // warp index within the role
  uint32_t Lbase = 0, S1 = 0, S2 = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int g = (item / nstrips) % ngroups;
    const int b = item / (nstrips * ngroups);
    const int jb0 = b * band_rows, jb1 = min(ny, jb0 + band_rows);
    const int lo = max(0, jb0 - 3), hi = min(ny - 1, jb1 + 2);
    const int i0 = max(0, jb0 - 2), i1 = min(ny - 1, jb1 + 1);      // U1 rows
    const int r2lo = max(0, jb0 - 1), r2hi = min(ny - 1, jb1);      // U2 rows
    const T *Ug = Uin + g * gstride + lane;
    T *Uog = Uout + g * gstride + lane;
    auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
    auto sq1 = [&](int r) { return S1 + (uint32_t)(r - i0); };
    auto sq2 = [&](int r) { return S2 + (uint32_t)(r - r2lo); };
    auto ut = [&](const FMeta &m, int idx) -> const T * {
      int sl = m.p + (idx - m.h0);
      if (sl >= Gm::N1) sl -= Gm::N1;
      return reinterpret_cast<const T *>(ring + (size_t)sl * PXB) + lane;
    };
    auto unb = [&](const FMeta &m, int idx) -> int4 {
      int sl = m.p + (idx - m.h0);
      if (sl >= Gm::N1) sl -= Gm::N1;
      return nring[sl];
    };
    auto u1t = [&](int r, int idx) -> T * {
      return u1s + ((size_t)(sq1(r) % 4) * SLOT1 + (idx - meta[seq(r) % Q].a1)) * D2 * G + lane;
    };
    auto u2t = [&](int r, int idx) -> T * {
      return u2s + ((size_t)(sq2(r) % 4) * SLOT2 + (idx - meta[seq(r) % Q].a2)) * D2 * G + lane;
    };
    auto body = [&](const T *ps, const T *pe, const T *pw, const T *pn, const T *pq, int4 nb, const T *z, T alpha,
                    T cc, T *out) {
      T xs[6][1], acc[6][1];
#pragma unroll
      for (int k = 0; k < 6; k++) { xs[k][0] = ps[k * G]; acc[k][0] = (T)0; }
      fused_apply<T>(acc, xs, nb, pe, pw, pn, pq);
#pragma unroll
      for (int k = 0; k < 6; k++) {
        const T zk = z ? z[k] : xs[k][0];
        out[k * G] = xs[k][0] + alpha * (zk - xs[k][0]) + cc * acc[k][0];
      }
    };
    if (role == 0) {
      // ------------------------------- A: U1 --------------------------------
      for (int r = i0; r <= i1; r++) {
        for (int rr = max(lo, r - 1); rr <= min(hi, r + 1); rr++) {
          const uint32_t L = seq(rr);
          mbar_wait(&full[L % Q], (L / Q) & 1);
        }
        const uint32_t q1 = sq1(r);
        if (q1 >= 4) mbar_wait(&e1[q1 % 4], ((q1 / 4) - 1) & 1);
        const FMeta m = meta[seq(r) % Q];
        const FMeta mn = (r + 1 <= hi) ? meta[seq(r + 1) % Q] : m;
        const FMeta ms = (r - 1 >= lo) ? meta[seq(r - 1) % Q] : m;
        T *slot = u1s + (size_t)(q1 % 4) * SLOT1 * D2 * G + lane;
        for (int it = rw; it < m.b1 - m.a1; it += NA) {
          const int a = m.a1 + it;
          const int4 nb = unb(m, a);
          const T *ps = ut(m, a);
          body(ps, nb.x >= 0 ? ut(m, nb.x) : ps, nb.y >= 0 ? ut(m, nb.y) : ps, nb.z >= 0 ? ut(mn, nb.z) : ps,
               nb.w >= 0 ? ut(ms, nb.w) : ps, nb, nullptr, (T)0, c1, slot + (size_t)it * D2 * G);
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&f1[q1 % 4]);
          if (r - 1 >= lo) mbar_arrive(&empty[seq(r - 1) % Q]);   // u row r-1: last reader was U1(r)
        }
      }
      // u rows the loop did not release (it released i0-1 .. i1-1)
      __syncwarp();
      if (lane == 0)
        for (int r = lo; r <= hi; r++)
          if (!(r >= i0 - 1 && r <= i1 - 1)) {
            const uint32_t L = seq(r);
            mbar_wait(&full[L % Q], (L / Q) & 1);
            mbar_arrive(&empty[L % Q]);
          }
    } else if (role == 1) {
      // ------------------------------- B: U2 --------------------------------
      for (int r = r2lo; r <= r2hi; r++) {
        for (int rr = max(i0, r - 1); rr <= min(i1, r + 1); rr++) {
          const uint32_t q = sq1(rr);
          mbar_wait(&f1[q % 4], (q / 4) & 1);
        }
        const uint32_t q2 = sq2(r);
        if (q2 >= 4) mbar_wait(&e2[q2 % 4], ((q2 / 4) - 1) & 1);
        const FMeta m = meta[seq(r) % Q];
        T *slot = u2s + (size_t)(q2 % 4) * SLOT2 * D2 * G + lane;
        for (int it = rw; it < m.b2 - m.a2; it += NB) {
          const int a = m.a2 + it;
          const int4 nb = __ldg(&nbr[a]);
          T z[6];
#pragma unroll
          for (int k = 0; k < 6; k++) z[k] = __ldg(Ug + ((size_t)a * D2 + k) * G);
          const T *ps = u1t(r, a);
          body(ps, nb.x >= 0 ? u1t(r, nb.x) : ps, nb.y >= 0 ? u1t(r, nb.y) : ps,
               nb.z >= 0 ? u1t(r + 1, nb.z) : ps, nb.w >= 0 ? u1t(r - 1, nb.w) : ps, nb, z, (T)0.75, c2,
               slot + (size_t)it * D2 * G);
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&f2[q2 % 4]);
          if (r - 1 >= i0) mbar_arrive(&e1[sq1(r - 1) % 4]);      // U1 row r-1: last reader was U2(r)
        }
      }
      __syncwarp();
      if (lane == 0)
        for (int r = i0; r <= i1; r++)
          if (!(r >= r2lo - 1 && r <= r2hi - 1)) mbar_arrive(&e1[sq1(r) % 4]);
    } else {
      // ------------------------------- C: u' --------------------------------
      for (int r = jb0; r < jb1; r++) {
        for (int rr = max(r2lo, r - 1); rr <= min(r2hi, r + 1); rr++) {
          const uint32_t q = sq2(rr);
          mbar_wait(&f2[q % 4], (q / 4) & 1);
        }
        const FMeta m = meta[seq(r) % Q];
        for (int it = rw; it < m.c1 - m.c0; it += NCW) {
          const int a = m.c0 + it;
          const int4 nb = __ldg(&nbr[a]);
          T z[6];
#pragma unroll
          for (int k = 0; k < 6; k++) z[k] = __ldg(Ug + ((size_t)a * D2 + k) * G);
          const T *ps = u2t(r, a);
          body(ps, nb.x >= 0 ? u2t(r, nb.x) : ps, nb.y >= 0 ? u2t(r, nb.y) : ps,
               nb.z >= 0 ? u2t(r + 1, nb.z) : ps, nb.w >= 0 ? u2t(r - 1, nb.w) : ps, nb, z,
               (T)(1.0 / 3.0), c3, Uog + (size_t)a * D2 * G);
        }
        __syncwarp();
        if (lane == 0 && r - 1 >= r2lo) mbar_arrive(&e2[sq2(r - 1) % 4]);   // U2 row r-1: last reader u'(r)
      }
      __syncwarp();
      if (lane == 0)
        for (int r = r2lo; r <= r2hi; r++)
          if (!(r >= jb0 - 1 && r <= jb1 - 2)) mbar_arrive(&e2[sq2(r) % 4]);
    }
    Lbase += (uint32_t)(hi - lo + 1);
    S1 += (uint32_t)(i1 - i0 + 1);
    S2 += (uint32_t)(r2hi - r2lo + 1);
  }
}

inline cudaError_t launch_step_dec(const dgl::StageArgs &a) {
  using Gm = DecGeom;
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!(attr_set.load() >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_step_dec, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(uint64_t(1) << dev);
  }
  const int per_band = a.nstrips * a.ngroups;
  int nbands = std::max(1, std::min(a.ny, (8 * a.nsm + per_band - 1) / per_band));
  int band_rows = (a.ny + nbands - 1) / nbands;
  if (band_rows > DMAXBAND) band_rows = DMAXBAND;
  nbands = (a.ny + band_rows - 1) / band_rows;
  const int nitems = per_band * nbands;
  const int grid = std::min(nitems, a.nsm);
  k_step_dec<<<grid, Gm::THREADS, Gm::SMEM, a.st>>>(
      (const double *)a.Uin, (double *)a.Uout, a.nbr, a.rowtab, a.nact, a.ny, a.nstrips, a.ngroups, band_rows,
      nitems, a.cs, 0.25 * a.cs, (2.0 / 3.0) * a.cs,
      std::max(6, std::min(DQ - 12, a.ahead_alpha > 0 ? a.ahead_alpha : DQ - 12)));
  return cudaGetLastError();
}

}  // namespace dgk
