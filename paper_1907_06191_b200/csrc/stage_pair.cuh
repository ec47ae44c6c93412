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
//   producer warp   per item ONE bulk copy of the item's 16-bit neighbour
//                   table (nbS, strip-major: open-face code and the tile
//                   positions of the N and S neighbours of every U2 pixel)
//                   into one of two item buffers; per row ONE bulk copy of the
//                   U1 row tile [x0-2, x0+W+2) into ring 1 (rows jb0-2 ..
//                   jb1+1); one row entry per row (full / empty mbarriers as
//                   K2, plus full3 / empty3 for the U2 rows); the row's U2
//                   tiles get consecutive virtual slots of ring 3 (meta.v3).
//                   (A 1-D bulk copy costs the SM's TMA ~0.25 us whatever its
//                   size up to 12 KB -- profiles/r02_tma_bw.json -- so a row
//                   must cost one copy, not the four of the first version.)
//   B warps (NB)    U2 of rows jb0-1 .. jb1 on the U2 columns [x0-1, x0+W+1),
//                   pixels dealt round-robin in raster order across rows
//                   (K2's cursor): U1 from ring 1, u from HBM, result into
//                   ring 3; a warp arrives on full3[row] when its cursor leaves
//                   the row and releases U1 rows (empty) once past their last
//                   reader
//   C warps (NCW)   u' of rows jb0 .. jb1-1 on the W columns, same dealing:
//                   U2 from ring 3 (rows r-1..r+1 complete: full3), u from
//                   HBM/L2, u' to HBM (a different register than u: the
//                   neighbouring strips still read u in their halo columns);
//                   C releases U2 rows through empty3 and publishes its
//                   released ring-3 frontier (relv) for B
//
// Ring 3 is allocated lazily by B: a U2 row's tiles may be written once C has
// released everything older than two rows before it, so ring 3 needs three
// full U2 rows and ring 1 three full U1 rows for progress (static_asserts);
// the producer reuses a row entry only after both B and C released it, and an
// item buffer only after both finished the item that used it.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include "kernels.cuh"
#include "stage_imm.cuh"
#include "launch.h"

namespace dgk {

constexpr int PAIR_Q = 32;          // row entries
constexpr int PAIR_MAXBAND = 128;   // rows per band
#ifndef DGDIFF_PAIR_NB
#define DGDIFF_PAIR_NB 7            // U2 warps (product default; swept 6-10: 7/4 best, B has the HBM alpha loads)
#endif
#ifndef DGDIFF_PAIR_NC
#define DGDIFF_PAIR_NC 4            // u' warps (swept 4-7)
#endif
#ifndef DGDIFF_PAIR_W
#define DGDIFF_PAIR_W 8
#endif
constexpr int PAIR_W = DGDIFF_PAIR_W;   // strip width (columns of u' per item)
// item neighbour buffer: U2 pixels of the band's rows (+ 2 halo rows) plus
// the 16-byte alignment slack of the bulk copy, in 16-bit entries
constexpr int PAIR_NBUF = ((PAIR_MAXBAND + 2) * (PAIR_W + 2) + 16 + 7) / 8 * 8;

struct PairMeta {
  int p1, h0, c0, c1;   // ring-1 slot of the tile start; tile [h0, ..), U2 pixels [c0, c1)
  int o0, o1;           // u' pixels [o0, o1)
  int nbo;              // item-buffer index of the neighbour entry of U2 pixel c0
  uint32_t v3;          // virtual ring-3 slot of U2 pixel c0
};

template <typename T, int NV, int P, int NB_ = DGDIFF_PAIR_NB, int NC_ = DGDIFF_PAIR_NC>
struct PairGeom {
  static constexpr int G = 32 * NV;
  static constexpr int D2 = ndof_px<P>();
  static constexpr int PXB = D2 * G * (int)sizeof(T);
  static constexpr int W = PAIR_W;
  static constexpr int NB = NB_, NCW = NC_;
  static constexpr int THREADS = (NB + NCW + 1) * 32;
  static constexpr int SMEM_MAX = 232448;
  static constexpr int OFF_NBUF = 0;                                        // [2][PAIR_NBUF] uint16
  static constexpr int OFF_BAR = OFF_NBUF + 2 * PAIR_NBUF * 2;
  static constexpr int OFF_META = OFF_BAR + (4 * PAIR_Q + 4) * 8;
  static constexpr int OFF_RT = OFF_META + PAIR_Q * (int)sizeof(PairMeta);
  static constexpr int OFF_RV = OFF_RT + (PAIR_MAXBAND + 4) * 2 * 16;
  static constexpr int OFF_RELV = OFF_RV + PAIR_Q * 4;
  static constexpr int OFF_TILES = (OFF_RELV + NCW * 4 + 127) / 128 * 128;
  static constexpr int NT = (SMEM_MAX - OFF_TILES) / PXB;            // pixel tiles for rings 1 and 3
  static constexpr int N1MIN = 3 * (W + 4), N3MIN = 3 * (W + 2);
  static constexpr int N3 = N3MIN + (NT - N1MIN - N3MIN) / 2;
  static constexpr int N1 = NT - N3;
  static constexpr int OFF_R1 = OFF_TILES, OFF_R3 = OFF_R1 + N1 * PXB;
  static constexpr int SMEM = OFF_R3 + N3 * PXB;
  static_assert(N1 >= N1MIN && N3 >= N3MIN, "stage pair: rings too small for progress");
  static_assert(SMEM <= SMEM_MAX, "stage pair does not fit in shared memory");
  static_assert(W + 4 <= 16, "tile positions must fit the 4-bit fields of the neighbour table");
};

__device__ __forceinline__ void st_release_cta(uint32_t *p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// shared-memory vector load / store at a 32-bit shared address
template <typename T, int NV>
__device__ __forceinline__ void lds_a(uint32_t a, T (&x)[NV]) {
  if constexpr (sizeof(T) == 8 && NV == 2) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x[0]), "=d"(x[1]) : "r"(a));
  } else if constexpr (sizeof(T) == 8 && NV == 1) {
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x[0]) : "r"(a));
  } else if constexpr (sizeof(T) == 4 && NV == 4) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]) : "r"(a));
  } else {
    static_assert(sizeof(T) == 4 && NV == 2, "lane width");
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x[0]), "=f"(x[1]) : "r"(a));
  }
}
template <typename T, int NV>
__device__ __forceinline__ void sts_a(uint32_t a, const T (&x)[NV]) {
  if constexpr (sizeof(T) == 8 && NV == 2) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x[0]), "d"(x[1]) : "memory");
  } else if constexpr (sizeof(T) == 8 && NV == 1) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x[0]) : "memory");
  } else if constexpr (sizeof(T) == 4 && NV == 4) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3])
                 : "memory");
  } else {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x[0]), "f"(x[1]) : "memory");
  }
}

// One pixel of an alpha stage, shared by the U2 (B) and u' (C) warps so that
// the operator's code exists once (two inlined copies overflowed the
// instruction cache: 20 % "no instruction" stalls):
//   out = x + alpha (z - x) + cs L(x),  L with K2's operator and order (self
//   block of the open-face code, then the E, W, N, S neighbour blocks)
// x and its neighbours are this lane's data in shared-memory tiles (32-bit
// addresses, dof stride G values); z is read from global memory; out goes to
// shared memory (out_s, B) or to global memory (out_g != nullptr, C).
template <typename T, int NV, int P>
__device__ __noinline__ void pair_pixel(uint32_t xs_a, uint32_t xe_a, uint32_t xw_a, uint32_t xn_a, uint32_t xq_a,
                                        int code, const T *__restrict__ zsrc, T *out_g, uint32_t out_s, T alpha,
                                        T cs, const T *pf /* nullable: the warp's next alpha term, into L2 */) {
  constexpr int D2 = ndof_px<P>(), G = 32 * NV, DS = G * (int)sizeof(T);
  // shared-memory loads run one block ahead of the MACs that consume them
  // (two neighbour buffers; a closed face's buffer is filled from the own
  // tile and not used), so the LDS latency hides behind the previous block
  T xs[D2][NV], acc[D2][NV], b0[D2][NV], b1[D2][NV], z[D2][NV];
#pragma unroll
  for (int k = 0; k < D2; k++) ldv<T, NV>(zsrc + (size_t)k * G, z[k]);
  if (pf) {
#pragma unroll
    for (int k = 0; k < D2; k++) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (size_t)k * G));
  }
#pragma unroll
  for (int k = 0; k < D2; k++) lds_a<T, NV>(xs_a + k * DS, xs[k]);
#pragma unroll
  for (int k = 0; k < D2; k++) lds_a<T, NV>(((code & 1) ? xe_a : xs_a) + k * DS, b0[k]);
#pragma unroll
  for (int k = 0; k < D2; k++)
#pragma unroll
    for (int e = 0; e < NV; e++) acc[k][e] = (T)0;
  mv_self<T, NV, P>(code, acc, xs);
#pragma unroll
  for (int k = 0; k < D2; k++) lds_a<T, NV>(((code & 2) ? xw_a : xs_a) + k * DS, b1[k]);
  if (code & 1) mv_imm<T, NV, P, 5>(acc, b0);
#pragma unroll
  for (int k = 0; k < D2; k++) lds_a<T, NV>(((code & 4) ? xn_a : xs_a) + k * DS, b0[k]);
  if (code & 2) mv_imm<T, NV, P, 6>(acc, b1);
#pragma unroll
  for (int k = 0; k < D2; k++) lds_a<T, NV>(((code & 8) ? xq_a : xs_a) + k * DS, b1[k]);
  if (code & 4) mv_imm<T, NV, P, 7>(acc, b0);
  if (code & 8) mv_imm<T, NV, P, 8>(acc, b1);
#pragma unroll
  for (int k = 0; k < D2; k++) {
    T y[NV];
#pragma unroll
    for (int e = 0; e < NV; e++) y[e] = xs[k][e] + alpha * (z[k][e] - xs[k][e]) + cs * acc[k][e];
    if (out_g) stv<T, NV>(out_g + (size_t)k * G, y);
    else sts_a<T, NV>(out_s + k * DS, y);
  }
}

template <typename T, int NV, int P, int NB_, int NC_>
__global__ void __launch_bounds__(PairGeom<T, NV, P, NB_, NC_>::THREADS, 1)
    k_stage_pair(const T *__restrict__ U1, const T *__restrict__ U0, T *__restrict__ Uout,
                 const uint16_t *__restrict__ nbs /* strip-major neighbour table */,
                 const int4 *__restrict__ rowtab /* [nstrips][ny][2] */, int nact, int ny, int nstrips, int ngroups,
                 int band_rows, int nitems, T a2, T c2, T a3, T c3, int max_ahead,
                 int diag /* tuning builds only: 1 skip B math, 2 skip C math, 8 no C warps */) {
  using Gm = PairGeom<T, NV, P, NB_, NC_>;
  static_assert(!is_quad<P>(), "stage pair: triangles");
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, Q = PAIR_Q, NB = Gm::NB, NCW = Gm::NCW;
  constexpr int N1 = Gm::N1, N3 = Gm::N3;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *ring1 = smem + Gm::OFF_R1;
  unsigned char *ring3 = smem + Gm::OFF_R3;
  uint16_t *nbuf = reinterpret_cast<uint16_t *>(smem + Gm::OFF_NBUF);   // [2][PAIR_NBUF]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Gm::OFF_BAR);
  uint64_t *empty = full + Q, *full3 = empty + Q, *empty3 = full3 + Q;
  uint64_t *nbf = empty3 + Q, *nbe = nbf + 2;                           // item buffers: full / empty
  PairMeta *meta = reinterpret_cast<PairMeta *>(smem + Gm::OFF_META);
  int4 *rt = reinterpret_cast<int4 *>(smem + Gm::OFF_RT);
  uint32_t *rv = reinterpret_cast<uint32_t *>(smem + Gm::OFF_RV);      // [Q] producer's ring-1 virtual ends
  uint32_t *relv = reinterpret_cast<uint32_t *>(smem + Gm::OFF_RELV);  // [NCW] ring-3 frontier per C warp
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t r1 = smem_u32(ring1), r3 = smem_u32(ring3), lane_b = (uint32_t)(lane * NV * sizeof(T));
  if (tid == 0) {
    for (int q = 0; q < Q; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NB);
      mbar_init(&full3[q], NB);
      mbar_init(&empty3[q], NCW);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&nbf[b], 1);
      mbar_init(&nbe[b], NB + NCW);
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
    uint32_t L = 0, v1 = 0, v3 = 0, relB = 0, relC = 0, it = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, it++) {
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
      // the item's neighbour table: one bulk copy of the U2 rows' entries
      const int ib = (int)(it & 1);
      const int nb_first = rt[2 * (u2lo - lo) + 1].z;
      const int nb_last = rt[2 * (u2hi - lo) + 1].z + (rt[2 * (u2hi - lo)].z - rt[2 * (u2hi - lo)].y);
      const int nb_base = nb_first & ~7;                      // 16-byte aligned start (entries)
      const uint32_t nb_bytes = (uint32_t)(((nb_last + 7) & ~7) - nb_base) * 2u;
      if (lane == 0) {
        if (it >= 2 && !(diag & 8)) mbar_wait(&nbe[ib], ((it / 2) - 1) & 1);   // both roles finished item it-2
        mbar_expect_tx(&nbf[ib], nb_bytes);
        if (nb_bytes) bulk_g2s(nbuf + ib * PAIR_NBUF, nbs + nb_base, nb_bytes, &nbf[ib]);
      }
      // rows are issued by one lane, one row at a time: the warp-wide batch
      // issue of K2 (scan + ballot per batch) re-ran for every released row
      // once the ring was full and made the producer the bottleneck
      // (profiles/r02_pair_diag3: the producer warp never idle)
      if (lane == 0) {
        const T *Ug = U1 + g * gstride;
        for (int r = lo; r <= hi; r++) {
          const int4 t = rt[2 * (r - lo)], t2 = rt[2 * (r - lo) + 1];
          const bool comp = r >= u2lo && r <= u2hi;
          const uint32_t n1 = (uint32_t)(t.w - t.x), n3 = comp ? (uint32_t)(t.z - t.y) : 0u;
          // entry reuse (B and C released the entry's previous row) and
          // ring-1 room (B released enough U1 rows)
          for (;;) {
            const uint32_t s1 = relB ? rv[(relB - 1) % Q] : 0u;
            if (L - relB < (uint32_t)max_ahead && v1 + n1 - s1 <= (uint32_t)N1) break;
            mbar_wait(&empty[relB % Q], (relB / Q) & 1);
            relB++;
          }
          while (!(diag & 8) && L - relC >= (uint32_t)max_ahead) {
            mbar_wait(&empty3[relC % Q], (relC / Q) & 1);
            relC++;
          }
          const uint32_t q = L % Q, p1 = v1 % N1;
          PairMeta m;
          m.p1 = (int)p1; m.h0 = t.x; m.c0 = t.y; m.c1 = comp ? t.z : t.y;
          m.o0 = t2.x; m.o1 = t2.y; m.nbo = t2.z - nb_base; m.v3 = v3;
          meta[q] = m;
          v1 += n1;
          v3 += n3;
          rv[q] = v1;
          mbar_expect_tx(&full[q], n1 * PXB);
          if (n1) {
            const uint32_t a1 = min(n1, (uint32_t)N1 - p1);
            const T *src = Ug + (size_t)t.x * D2 * G;
            bulk_g2s(ring1 + (size_t)p1 * PXB, src, a1 * PXB, &full[q]);
            if (n1 > a1) bulk_g2s(ring1, src + (size_t)a1 * D2 * G, (n1 - a1) * PXB, &full[q]);
          }
          L++;
        }
      }
      __syncwarp();
    }
    return;
  }

  // neighbour entry of a pixel: bits 0-3 open-face code (E, W, N, S), 4-7 the
  // N neighbour's position in row j+1's tile, 8-11 the S neighbour's in row
  // j-1's tile (tile positions count from column x0-2)
  if (w < NB) {
    // ============================ B warps: U2 =============================
    uint32_t Lbase = 0, it = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, it++) {
      int s_, g, jb0, jb1;
      decode(item, s_, g, jb0, jb1);
      const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
      const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
      const T *U0l = U0 + g * gstride + lane * NV;
      const uint16_t *nbi = nbuf + (it & 1) * PAIR_NBUF;
      auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
      auto wait_row = [&](int r) {
        if (r >= lo && r <= hi) {
          const uint32_t L = seq(r);
          mbar_wait(&full[L % Q], (L / Q) & 1);
        }
      };
      auto tile1 = [&](const PairMeta &m, int pos) -> uint32_t {   // pos = position in the row tile
        int sl = m.p1 + pos;
        if (sl >= N1) sl -= N1;
        return r1 + (uint32_t)sl * PXB + lane_b;
      };
      mbar_wait(&nbf[it & 1], (it / 2) & 1);
      int j = u2lo, rel_next = lo, cum = 0;
      for (int r = u2lo - 1; r <= u2lo + 1; r++) wait_row(r);
      // the halo row above the U2 rows has no U2 part: complete its full3
      // phase (after its full wait, so the arrival lands in this row's phase)
      __syncwarp();
      if (lane == 0)
        for (int r = lo; r < u2lo; r++) mbar_arrive(&full3[seq(r) % Q]);
      PairMeta mc = meta[seq(j) % Q];
      // metas of the rows above / below, cached per row (rows lo..hi exist)
      PairMeta mN = j + 1 <= hi ? meta[seq(j + 1) % Q] : mc, mS = j - 1 >= lo ? meta[seq(j - 1) % Q] : mc;
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
          mS = mc;
          mc = mN;
          mN = j + 1 <= hi ? meta[seq(j + 1) % Q] : mc;
          space_ok = false;
        }
        if (j > u2hi) break;
        if (!space_ok && !(diag & 8)) {
          // ring-3 room for all of row j: C must have released everything
          // older than row j-2 (lazy allocation; see the header)
          const uint32_t need = mc.v3 + (uint32_t)(mc.c1 - mc.c0);
          const long long t0 = clock64();
          for (;;) {
            uint32_t mn = ld_acquire_cta(&relv[0]);
#pragma unroll
            for (int c = 1; c < NCW; c++) {
              const uint32_t v = ld_acquire_cta(&relv[c]);
              if ((int)(v - mn) < 0) mn = v;
            }
            if ((int)(need - mn) <= N3) break;
            __nanosleep(32);
            if (clock64() - t0 > (1LL << 34)) __trap();   // watchdog, as mbar_wait
          }
          space_ok = true;
        }
        const int k = f - cum;                         // U2 pixel k of row j
        const int a = mc.c0 + k;
        const int nbw = nbi[mc.nbo + k];
        const int code = nbw & 15, pos = a - mc.h0;
        const uint32_t xs_a = tile1(mc, pos);
        const uint32_t sl3 = (mc.v3 + (uint32_t)k) % (uint32_t)N3;
        if (diag & 1) continue;
        // the alpha term of this warp's next pixel (f + NB), if its row is known
        const T *pfn = nullptr;
        {
          const int kn = k + NB, szj = mc.c1 - mc.c0;
          if (kn < szj) {
            pfn = U0l + (size_t)(mc.c0 + kn) * D2 * G;
          } else if (j + 1 <= u2hi && kn - szj < mN.c1 - mN.c0) {
            pfn = U0l + (size_t)(mN.c0 + kn - szj) * D2 * G;
          }
        }
        pair_pixel<T, NV, P>(xs_a, tile1(mc, pos + 1), tile1(mc, pos - 1 < 0 ? 0 : pos - 1),
                             (code & 4) ? tile1(mN, (nbw >> 4) & 15) : xs_a,
                             (code & 8) ? tile1(mS, (nbw >> 8) & 15) : xs_a, code, U0l + (size_t)a * D2 * G, nullptr,
                             r3 + sl3 * PXB + lane_b, a2, c2, pfn);
      }
      __syncwarp();
      if (lane == 0) {
        for (int r = u2hi + 1; r <= hi; r++) mbar_arrive(&full3[seq(r) % Q]);   // halo row below: no U2
        for (int r = rel_next; r <= hi; r++) mbar_arrive(&empty[seq(r) % Q]);
        mbar_arrive(&nbe[it & 1]);
      }
      Lbase += (uint32_t)(hi - lo + 1);
    }
    return;
  }

  // ============================== C warps: u' ==============================
  if (diag & 8) return;   // diagnostic: no C warps at all
  const int wc = w - NB;
  uint32_t Lbase = 0, it = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, it++) {
    int s_, g, jb0, jb1;
    decode(item, s_, g, jb0, jb1);
    const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
    const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
    const T *U0l = U0 + g * gstride + lane * NV;
    T *Uog = Uout + g * gstride + lane * NV;
    const uint16_t *nbi = nbuf + (it & 1) * PAIR_NBUF;
    auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
    auto wait3 = [&](int r) {
      if (r >= u2lo && r <= u2hi) {
        const uint32_t L = seq(r);
        mbar_wait(&full3[L % Q], (L / Q) & 1);
      }
    };
    auto tile3 = [&](const PairMeta &m, int pos) -> uint32_t {   // pos = position in the row tile
      const uint32_t sl = (m.v3 + (uint32_t)(pos - (m.c0 - m.h0))) % (uint32_t)N3;
      return r3 + sl * PXB + lane_b;
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
    mbar_wait(&nbf[it & 1], (it / 2) & 1);
    int j = jb0, rel_next = lo, cum = 0;
    for (int r = jb0 - 1; r <= jb0 + 1; r++) wait3(r);
    PairMeta mc = meta[seq(j) % Q];
    PairMeta mN = meta[seq(j + 1) % Q], mS = meta[seq(j - 1 >= lo ? j - 1 : j) % Q];   // U2 rows j-1..j+1 exist
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
        mS = mc;
        mc = mN;
        mN = meta[seq(j + 1) % Q];
      }
      if (j >= jb1) break;
      const int a = mc.o0 + (f - cum);
      const int nbw = nbi[mc.nbo + (a - mc.c0)];
      const int code = nbw & 15, pos = a - mc.h0;
      const uint32_t xs_a = tile3(mc, pos);
      if (diag & 2) continue;
      pair_pixel<T, NV, P>(xs_a, tile3(mc, pos + 1), tile3(mc, pos - 1),
                           (code & 4) ? tile3(mN, (nbw >> 4) & 15) : xs_a,
                           (code & 8) ? tile3(mS, (nbw >> 8) & 15) : xs_a, code, U0l + (size_t)a * D2 * G,
                           Uog + (size_t)a * D2 * G, 0u, a3, c3, nullptr);
    }
    __syncwarp();
    if (lane == 0) {
      for (int r = rel_next; r <= hi; r++) release3(r);
      mbar_arrive(&nbe[it & 1]);
    }
    Lbase += (uint32_t)(hi - lo + 1);
  }
}

// stages 2 + 3 of one step: a.Uin = U1, a.U0 = u (read only), a.Uout = u'
// (must not alias u), a.rowtab = the pair row table [nstrips][ny][2]
// {c(x0-2), c(x0-1), c(x0+W+1), c(x0+W+2)}, {c(x0), c(x0+W), nbS offset, 0},
// a.nbs = the strip-major neighbour table, a.cs = dt D/h^2
template <typename T, int NV, int P, int NB_ = DGDIFF_PAIR_NB, int NC_ = DGDIFF_PAIR_NC>
cudaError_t launch_pair(const dgl::StageArgs &a, int diag = 0) {
  using Gm = PairGeom<T, NV, P, NB_, NC_>;
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!(attr_set.load() >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_stage_pair<T, NV, P, NB_, NC_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Gm::SMEM);
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
  k_stage_pair<T, NV, P, NB_, NC_><<<grid, Gm::THREADS, Gm::SMEM, a.st>>>(
      (const T *)a.Uin, (const T *)a.U0, (T *)a.Uout, a.nbs, a.rowtab, a.nact, a.ny, a.nstrips, a.ngroups, band_rows,
      nitems, (T)0.75, (T)(0.25 * c), (T)(1.0 / 3.0), (T)((2.0 / 3.0) * c), PAIR_Q - 1, diag);
  return cudaGetLastError();
}

}  // namespace dgk
