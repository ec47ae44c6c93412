// stage_pair.cuh -- K3d: SSP-RK3 stages 2 AND 3 in one launch (temporal
// blocking over the stage pair; stage 1 stays on K2).  temporal_steps = 5.
//
//   U2 = U1 + 3/4 (u - U1) + c2 L(U1)      (stage 2, reading U1 from HBM)
//   u' = U2 + 1/3 (u - U2) + c3 L(U2)      (stage 3, U2 never leaves the SM)
//
// HBM traffic of a step: stage 1 (K2) reads u and writes U1 (2 passes); this
// kernel reads U1 (ring, 2-column strip halo) and u (alpha terms, direct
// loads) and writes u' (3 passes): 5 state passes per step instead of K2's 8.
// The price is recomputing U2 on a 1-column strip halo (W + 2 of W columns)
// and one band-halo row each side.  Per pixel the arithmetic is K2's (same
// compile-time operator, same order: self block, then E, W, N, S neighbours,
// then the RK combination), so the result is bitwise K2's.
//
// Work item = (strip s of W = 8 columns, source group g, band [jb0, jb1)).
//
//   producer warp   U1 row tiles of rows jb0-2 .. jb1+1, columns
//                   [x0-2, x0+W+2), into ring 1 (bulk TMA), and the neighbour
//                   indices of the U2 pixels [x0-1, x0+W+1) into ring 2; one
//                   row entry per row (full / empty mbarriers as K2, plus
//                   full3 / empty3 for the U2 rows); the row's U2 tiles get
//                   consecutive virtual slots of ring 3 (meta.v3)
//   B warps (NB)    U2 of rows jb0-1 .. jb1 on the U2 columns, pixels dealt
//                   round-robin in raster order across rows (K2's cursor):
//                   U1 from ring 1, u from HBM, result into ring 3; a warp
//                   arrives on full3[row] when its cursor leaves the row and
//                   releases U1 rows (empty) once past their last reader
//   C warps (NCW)   u' of rows jb0 .. jb1-1 on the W columns, same dealing:
//                   U2 from ring 3 (rows r-1..r+1 complete: full3), u and the
//                   neighbour indices from HBM/L2, u' to HBM (a different
//                   register than u: the neighbouring strips still read u in
//                   their halo columns); C releases U2 rows through empty3 and
//                   publishes its released ring-3 frontier (relv) for B
//
// Ring 3 is allocated lazily by B: a U2 row's tiles may be written once C has
// released everything older than two rows before it, so ring 3 needs three
// full U2 rows and ring 1 three full U1 rows for progress (static_asserts);
// the producer reuses a row entry only after both B and C released it.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include "kernels.cuh"
#include "stage_imm.cuh"
#include "launch.h"

namespace dgk {

constexpr int PAIR_Q = 16;          // row entries
constexpr int PAIR_MAXBAND = 128;   // rows per band
#ifndef DGDIFF_PAIR_NB
#define DGDIFF_PAIR_NB 6            // U2 warps
#endif
#ifndef DGDIFF_PAIR_NC
#define DGDIFF_PAIR_NC 5            // u' warps
#endif

struct PairMeta {
  int p1, h0, c0, c1;   // ring-1 slot of the tile start; tile [h0, ..), U2 pixels [c0, c1)
  int p2, o0, o1;       // ring-2 slot of the neighbour run; u' pixels [o0, o1)
  uint32_t v3;          // virtual ring-3 slot of U2 pixel c0
};

template <typename T, int NV, int P>
struct PairGeom {
  static constexpr int G = 32 * NV;
  static constexpr int D2 = ndof_px<P>();
  static constexpr int PXB = D2 * G * (int)sizeof(T);
  static constexpr int W = 8;
  static constexpr int NB = DGDIFF_PAIR_NB, NCW = DGDIFF_PAIR_NC;
  static constexpr int THREADS = (NB + NCW + 1) * 32;
  static constexpr int SMEM_MAX = 232448;
  static constexpr int N2 = 8 * (W + 2);                             // neighbour entries (int4)
  static constexpr int OFF_NB = 0;
  static constexpr int OFF_BAR = OFF_NB + N2 * 16;
  static constexpr int OFF_META = OFF_BAR + 4 * PAIR_Q * 8;
  static constexpr int OFF_RT = OFF_META + PAIR_Q * (int)sizeof(PairMeta);
  static constexpr int OFF_RV = OFF_RT + (PAIR_MAXBAND + 4) * 2 * 16;
  static constexpr int OFF_RELV = OFF_RV + 2 * PAIR_Q * 4;
  static constexpr int OFF_TILES = (OFF_RELV + NCW * 4 + 127) / 128 * 128;
  static constexpr int NT = (SMEM_MAX - OFF_TILES) / PXB;            // pixel tiles for rings 1 and 3
  static constexpr int N1MIN = 3 * (W + 4), N3MIN = 3 * (W + 2);
  static constexpr int N3 = N3MIN + (NT - N1MIN - N3MIN) / 2;
  static constexpr int N1 = NT - N3;
  static constexpr int OFF_R1 = OFF_TILES, OFF_R3 = OFF_R1 + N1 * PXB;
  static constexpr int SMEM = OFF_R3 + N3 * PXB;
  static_assert(N1 >= N1MIN && N3 >= N3MIN, "stage pair: rings too small for progress");
  static_assert(N2 >= 3 * (W + 2), "stage pair: neighbour ring too small");
  static_assert(SMEM <= SMEM_MAX, "stage pair does not fit in shared memory");
};

__device__ __forceinline__ void st_release_cta(uint32_t *p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// acc += L(x) at one pixel with K2's operator and order: self block of the
// open-face code, then the E, W, N, S neighbour blocks of the open faces
template <typename T, int NV, int P>
__device__ __forceinline__ void pair_apply(T (&acc)[ndof_px<P>()][NV], const T (&xs)[ndof_px<P>()][NV], int4 nb,
                                           const T *pe, const T *pw, const T *pn, const T *ps_, int G) {
  constexpr int D2 = ndof_px<P>();
  T xn[D2][NV];
  mv_self<T, NV, P>(open_code(nb), acc, xs);
  if (nb.x >= 0) {
#pragma unroll
    for (int k = 0; k < D2; k++) lds<T, NV>(pe + k * G, xn[k]);
    mv_imm<T, NV, P, 5>(acc, xn);
  }
  if (nb.y >= 0) {
#pragma unroll
    for (int k = 0; k < D2; k++) lds<T, NV>(pw + k * G, xn[k]);
    mv_imm<T, NV, P, 6>(acc, xn);
  }
  if (nb.z >= 0) {
#pragma unroll
    for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
    mv_imm<T, NV, P, 7>(acc, xn);
  }
  if (nb.w >= 0) {
#pragma unroll
    for (int k = 0; k < D2; k++) lds<T, NV>(ps_ + k * G, xn[k]);
    mv_imm<T, NV, P, 8>(acc, xn);
  }
}

template <typename T, int NV, int P>
__global__ void __launch_bounds__(PairGeom<T, NV, P>::THREADS, 1)
    k_stage_pair(const T *__restrict__ U1, const T *__restrict__ U0, T *__restrict__ Uout,
                 const int4 *__restrict__ nbr, const int4 *__restrict__ rowtab /* [nstrips][ny][2] */, int nact,
                 int ny, int nstrips, int ngroups, int band_rows, int nitems, T a2, T c2, T a3, T c3,
                 int max_ahead) {
  using Gm = PairGeom<T, NV, P>;
  static_assert(!is_quad<P>(), "stage pair: triangles");
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, Q = PAIR_Q, NB = Gm::NB, NCW = Gm::NCW;
  constexpr int N1 = Gm::N1, N2 = Gm::N2, N3 = Gm::N3;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *ring1 = smem + Gm::OFF_R1;
  unsigned char *ring3 = smem + Gm::OFF_R3;
  int4 *nbr_ring = reinterpret_cast<int4 *>(smem + Gm::OFF_NB);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Gm::OFF_BAR);
  uint64_t *empty = full + Q, *full3 = empty + Q, *empty3 = full3 + Q;
  PairMeta *meta = reinterpret_cast<PairMeta *>(smem + Gm::OFF_META);
  int4 *rt = reinterpret_cast<int4 *>(smem + Gm::OFF_RT);
  uint32_t *rv = reinterpret_cast<uint32_t *>(smem + Gm::OFF_RV);      // [2][Q] producer's virtual ends
  uint32_t *relv = reinterpret_cast<uint32_t *>(smem + Gm::OFF_RELV);  // [NCW] ring-3 frontier per C warp
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < Q; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NB);
      mbar_init(&full3[q], NB);
      mbar_init(&empty3[q], NCW);
    }
    for (int c = 0; c < NCW; c++) relv[c] = 0u;
    fence_mbar_init();
  }
  __syncthreads();
  const size_t gstride = (size_t)nact * D2 * G;
  auto decode = [&](int item, int &s, int &g, int &jb0, int &jb1) {
    s = item % nstrips;
    g = (item / nstrips) % ngroups;
    jb0 = (item / (nstrips * ngroups)) * band_rows;
    jb1 = min(ny, jb0 + band_rows);
  };

  if (w == NB + NCW) {
    // =========================== producer warp ===========================
    uint32_t L = 0, v1 = 0, v2 = 0, relB = 0, relC = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int s, g, jb0, jb1;
      decode(item, s, g, jb0, jb1);
      const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
      const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
      __syncwarp();
      for (int r = lo + lane; r <= hi; r += 32) {
        rt[2 * (r - lo)] = __ldg(&rowtab[2 * ((size_t)s * ny + r)]);
        rt[2 * (r - lo) + 1] = __ldg(&rowtab[2 * ((size_t)s * ny + r) + 1]);
      }
      __syncwarp();
      const T *Ug = U1 + g * gstride;
      for (int r0 = lo; r0 <= hi;) {
        const int r = r0 + lane;
        const bool valid = r <= hi;
        int4 t = make_int4(0, 0, 0, 0), t2 = make_int4(0, 0, 0, 0);
        if (valid) {
          t = rt[2 * (r - lo)];
          t2 = rt[2 * (r - lo) + 1];
        }
        const bool comp = valid && r >= u2lo && r <= u2hi;
        const uint32_t n1 = valid ? (uint32_t)(t.w - t.x) : 0u;
        const uint32_t n2 = comp ? (uint32_t)(t.z - t.y) : 0u;
        uint32_t e1 = n1, e2 = n2;   // inclusive scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y1 = __shfl_up_sync(0xffffffffu, e1, o), y2 = __shfl_up_sync(0xffffffffu, e2, o);
          if (lane >= o) { e1 += y1; e2 += y2; }
        }
        const uint32_t nvalid = (uint32_t)min(32, hi - r0 + 1);
        uint32_t take;
        for (;;) {
          const uint32_t s1 = relB ? rv[(relB - 1) % Q] : 0u, s2 = relB ? rv[Q + (relB - 1) % Q] : 0u;
          const bool fitsB = valid && (L + lane - relB < (uint32_t)max_ahead) && (v1 + e1 - s1 <= (uint32_t)N1) &&
                             (v2 + e2 - s2 <= (uint32_t)N2);
          const bool fitsC = L + lane - relC < (uint32_t)max_ahead;
          const uint32_t ok = __ballot_sync(0xffffffffu, fitsB && fitsC);
          take = __ffs(~ok) - 1;
          if (ok == 0xffffffffu) take = 32;
          if (take > nvalid) take = nvalid;
          if (take > 0 || (relB == L && relC == L)) break;
          // the first row does not fit: wait for the release it lacks
          const bool b0 = __shfl_sync(0xffffffffu, fitsB, 0);
          if (!b0 && relB < L) {
            mbar_wait(&empty[relB % Q], (relB / Q) & 1);
            relB++;
          } else {
            mbar_wait(&empty3[relC % Q], (relC / Q) & 1);
            relC++;
          }
        }
        if (take == 0) take = 1;   // everything released: the ring is empty
        if ((uint32_t)lane < take) {
          const uint32_t Lr = L + lane, q = Lr % Q;
          const uint32_t b1 = v1 + e1 - n1, b2 = v2 + e2 - n2;   // virtual starts
          const uint32_t p1 = b1 % N1, p2 = b2 % N2;
          PairMeta m;
          m.p1 = (int)p1; m.h0 = t.x; m.c0 = t.y; m.c1 = comp ? t.z : t.y;
          m.p2 = (int)p2; m.o0 = t2.x; m.o1 = t2.y; m.v3 = b2;
          meta[q] = m;
          rv[q] = v1 + e1;
          rv[Q + q] = v2 + e2;
          mbar_expect_tx(&full[q], n1 * PXB + n2 * 16u);
          if (n1) {
            const uint32_t a1 = min(n1, (uint32_t)N1 - p1);
            const T *src = Ug + (size_t)t.x * D2 * G;
            bulk_g2s(ring1 + (size_t)p1 * PXB, src, a1 * PXB, &full[q]);
            if (n1 > a1) bulk_g2s(ring1, src + (size_t)a1 * D2 * G, (n1 - a1) * PXB, &full[q]);
          }
          if (n2) {
            const uint32_t a2n = min(n2, (uint32_t)N2 - p2);
            bulk_g2s(nbr_ring + p2, nbr + t.y, a2n * 16u, &full[q]);
            if (n2 > a2n) bulk_g2s(nbr_ring, nbr + t.y + a2n, (n2 - a2n) * 16u, &full[q]);
          }
        }
        v1 += __shfl_sync(0xffffffffu, e1, take - 1);
        v2 += __shfl_sync(0xffffffffu, e2, take - 1);
        L += take;
        r0 += (int)take;
        __syncwarp();
      }
    }
    return;
  }

  if (w < NB) {
    // ============================ B warps: U2 =============================
    uint32_t Lbase = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int s_, g, jb0, jb1;
      decode(item, s_, g, jb0, jb1);
      const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
      const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
      const T *U0l = U0 + g * gstride + lane * NV;
      auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
      auto wait_row = [&](int r) {
        if (r >= lo && r <= hi) {
          const uint32_t L = seq(r);
          mbar_wait(&full[L % Q], (L / Q) & 1);
        }
      };
      auto tile1 = [&](const PairMeta &m, int idx) -> const T * {
        int sl = m.p1 + (idx - m.h0);
        if (sl >= N1) sl -= N1;
        return reinterpret_cast<const T *>(ring1 + (size_t)sl * PXB) + lane * NV;
      };
      int j = u2lo, rel_next = lo, cum = 0;
      for (int r = u2lo - 1; r <= u2lo + 1; r++) wait_row(r);
      // the halo row above the U2 rows has no U2 part: complete its full3
      // phase (after its full wait, so the arrival lands in this row's phase)
      __syncwarp();
      if (lane == 0)
        for (int r = lo; r < u2lo; r++) mbar_arrive(&full3[seq(r) % Q]);
      PairMeta mc = meta[seq(j) % Q];
      bool space_ok = false;
      for (int f = w;; f += NB) {
        while (f >= cum + (mc.c1 - mc.c0)) {
          cum += mc.c1 - mc.c0;
          __syncwarp();
          if (lane == 0) mbar_arrive(&full3[seq(j) % Q]);   // this warp's U2 tiles of row j are written
          if (++j > u2hi) break;
          if (rel_next <= j - 2) {   // U1 rows <= j-2 have had their last reader
            if (lane == 0)
              for (int r = rel_next; r <= j - 2; r++) mbar_arrive(&empty[seq(r) % Q]);
            rel_next = j - 1;
          }
          wait_row(j + 1);
          mc = meta[seq(j) % Q];
          space_ok = false;
        }
        if (j > u2hi) break;
        if (!space_ok) {
          // ring-3 room for all of row j: C must have released everything
          // older than row j-2 (lazy allocation; see the header)
          const uint32_t need = mc.v3 + (uint32_t)(mc.c1 - mc.c0);
          for (;;) {
            uint32_t mn = 0xffffffffu;
            bool first = true;
#pragma unroll
            for (int c = 0; c < NCW; c++) {
              const uint32_t v = ld_acquire_cta(&relv[c]);
              if (first || (int)(v - mn) < 0) mn = v;
              first = false;
            }
            if ((int)(need - mn) <= N3) break;
            __nanosleep(32);
          }
          space_ok = true;
        }
        const int a = mc.c0 + (f - cum);
        int sl2 = mc.p2 + (f - cum);
        if (sl2 >= N2) sl2 -= N2;
        const int4 nb = nbr_ring[sl2];
        T xs[D2][NV], acc[D2][NV], z[D2][NV];
#pragma unroll
        for (int k = 0; k < D2; k++) ldv<T, NV>(U0l + ((size_t)a * D2 + k) * G, z[k]);
        const T *ps = tile1(mc, a);
#pragma unroll
        for (int k = 0; k < D2; k++) lds<T, NV>(ps + k * G, xs[k]);
#pragma unroll
        for (int k = 0; k < D2; k++)
#pragma unroll
          for (int e = 0; e < NV; e++) acc[k][e] = (T)0;
        const T *pe = nb.x >= 0 ? tile1(mc, nb.x) : ps;
        const T *pw = nb.y >= 0 ? tile1(mc, nb.y) : ps;
        const T *pn = nb.z >= 0 ? tile1(meta[seq(j + 1) % Q], nb.z) : ps;
        const T *pq = nb.w >= 0 ? tile1(meta[seq(j - 1) % Q], nb.w) : ps;
        pair_apply<T, NV, P>(acc, xs, nb, pe, pw, pn, pq, G);
        uint32_t sl3 = (mc.v3 + (uint32_t)(f - cum)) % (uint32_t)N3;
        T *out = reinterpret_cast<T *>(ring3 + (size_t)sl3 * PXB) + lane * NV;
#pragma unroll
        for (int k = 0; k < D2; k++) {
          T y[NV];
#pragma unroll
          for (int e = 0; e < NV; e++) y[e] = xs[k][e] + a2 * (z[k][e] - xs[k][e]) + c2 * acc[k][e];
          stv<T, NV>(out + (size_t)k * G, y);
        }
      }
      __syncwarp();
      if (lane == 0) {
        for (int r = u2hi + 1; r <= hi; r++) mbar_arrive(&full3[seq(r) % Q]);   // halo row below: no U2
        for (int r = rel_next; r <= hi; r++) mbar_arrive(&empty[seq(r) % Q]);
      }
      Lbase += (uint32_t)(hi - lo + 1);
    }
    return;
  }

  // ============================== C warps: u' ==============================
  const int wc = w - NB;
  uint32_t Lbase = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    int s_, g, jb0, jb1;
    decode(item, s_, g, jb0, jb1);
    const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
    const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
    const T *U0l = U0 + g * gstride + lane * NV;
    T *Uog = Uout + g * gstride + lane * NV;
    auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
    auto wait3 = [&](int r) {
      if (r >= u2lo && r <= u2hi) {
        const uint32_t L = seq(r);
        mbar_wait(&full3[L % Q], (L / Q) & 1);
      }
    };
    auto tile3 = [&](const PairMeta &m, int idx) -> const T * {
      const uint32_t sl = (m.v3 + (uint32_t)(idx - m.c0)) % (uint32_t)N3;
      return reinterpret_cast<const T *>(ring3 + (size_t)sl * PXB) + lane * NV;
    };
    auto release3 = [&](int r) {   // lane 0: C is done with U2 row r (and with entry seq(r))
      // every row's full3 phase completes before its entry is released (halo
      // rows without U2 included), so B's next arrival on the entry cannot
      // fall into an older phase
      const uint32_t L = seq(r);
      mbar_wait(&full3[L % Q], (L / Q) & 1);
      const PairMeta m = meta[seq(r) % Q];
      st_release_cta(&relv[wc], m.v3 + (uint32_t)(m.c1 - m.c0));
      mbar_arrive(&empty3[seq(r) % Q]);
    };
    int j = jb0, rel_next = lo, cum = 0;
    for (int r = jb0 - 1; r <= jb0 + 1; r++) wait3(r);
    PairMeta mc = meta[seq(j) % Q];
    for (int f = wc;; f += NCW) {
      while (f >= cum + (mc.o1 - mc.o0)) {
        cum += mc.o1 - mc.o0;
        if (++j >= jb1) break;
        if (rel_next <= j - 2) {   // U2 rows <= j-2 have had their last reader
          __syncwarp();
          if (lane == 0)
            for (int r = rel_next; r <= j - 2; r++) release3(r);
          rel_next = j - 1;
        }
        wait3(j + 1);
        mc = meta[seq(j) % Q];
      }
      if (j >= jb1) break;
      const int a = mc.o0 + (f - cum);
      const int4 nb = __ldg(&nbr[a]);
      T xs[D2][NV], acc[D2][NV], z[D2][NV];
#pragma unroll
      for (int k = 0; k < D2; k++) ldv<T, NV>(U0l + ((size_t)a * D2 + k) * G, z[k]);
      const T *ps = tile3(mc, a);
#pragma unroll
      for (int k = 0; k < D2; k++) lds<T, NV>(ps + k * G, xs[k]);
#pragma unroll
      for (int k = 0; k < D2; k++)
#pragma unroll
        for (int e = 0; e < NV; e++) acc[k][e] = (T)0;
      const T *pe = nb.x >= 0 ? tile3(mc, nb.x) : ps;
      const T *pw = nb.y >= 0 ? tile3(mc, nb.y) : ps;
      const T *pn = nb.z >= 0 ? tile3(meta[seq(j + 1) % Q], nb.z) : ps;
      const T *pq = nb.w >= 0 ? tile3(meta[seq(j - 1) % Q], nb.w) : ps;
      pair_apply<T, NV, P>(acc, xs, nb, pe, pw, pn, pq, G);
      T *out = Uog + (size_t)a * D2 * G;
#pragma unroll
      for (int k = 0; k < D2; k++) {
        T y[NV];
#pragma unroll
        for (int e = 0; e < NV; e++) y[e] = xs[k][e] + a3 * (z[k][e] - xs[k][e]) + c3 * acc[k][e];
        stv<T, NV>(out + (size_t)k * G, y);
      }
    }
    __syncwarp();
    if (lane == 0)
      for (int r = rel_next; r <= hi; r++) release3(r);
    Lbase += (uint32_t)(hi - lo + 1);
  }
}

// stages 2 + 3 of one step: a.Uin = U1, a.U0 = u (read only), a.Uout = u'
// (must not alias u), a.rowtab = the pair row table [nstrips][ny][2]
// {c(x0-2), c(x0-1), c(x0+W+1), c(x0+W+2)}, {c(x0), c(x0+W)}, a.cs = dt D/h^2
template <typename T, int NV, int P>
cudaError_t launch_pair(const dgl::StageArgs &a) {
  using Gm = PairGeom<T, NV, P>;
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!(attr_set.load() >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_stage_pair<T, NV, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(uint64_t(1) << dev);
  }
  const int per_band = a.nstrips * a.ngroups;
  int nbands = std::max(1, std::min(a.ny, (8 * a.nsm + per_band - 1) / per_band));
  int band_rows = (a.ny + nbands - 1) / nbands;
  if (band_rows > PAIR_MAXBAND) band_rows = PAIR_MAXBAND;
  nbands = (a.ny + band_rows - 1) / band_rows;
  const int nitems = per_band * nbands;
  const int grid = std::min(nitems, a.nsm);
  const double c = a.cs;
  k_stage_pair<T, NV, P><<<grid, Gm::THREADS, Gm::SMEM, a.st>>>(
      (const T *)a.Uin, (const T *)a.U0, (T *)a.Uout, a.nbr, a.rowtab, a.nact, a.ny, a.nstrips, a.ngroups, band_rows,
      nitems, (T)0.75, (T)(0.25 * c), (T)(1.0 / 3.0), (T)((2.0 / 3.0) * c), PAIR_Q - 1);
  return cudaGetLastError();
}

}  // namespace dgk
