// stage_ring.cuh -- K2 v3: one SSP-RK3 stage, row-marching through shared
// memory, fed by 1-D bulk TMA (cp.async.bulk) in a warp-specialised
// producer/consumer pipeline with full/empty mbarriers.
//
// Work item = (column strip s of W pixels, source group g of G = 32 NV
// sources, band of rows [jb0, jb1)).  Extracellular pixels are stored in
// raster order, so the pixels of row j with x in [x0-1, x0+W+1) are one
// contiguous run of group g's state: one bulk copy per row ("row tile";
// rowtab[s][j] = {h0, c0, c1, h1}: active-index bounds of the halo'd and the
// computed ranges).
//
//   producer warp            for every row r of every item of this CTA, in
//       batches of up to 32 rows (one per lane): wait until the ring slots are
//       released (empty barriers), write the row's metadata, arm full[r] with
//       the byte count and issue the bulk copies: U_in tile [h0, h1) into
//       ring 1, and -- for rows that are computed -- the neighbour indices
//       nbr[c0, c1) (and, staged variant only, the u0 tile) into ring 2.
//   consumer warps           the band's computed pixels, dealt out round-robin
//       in raster order (warp w: pixels w, w+NC, ...): for a pixel of row j,
//       wait full[j-1..j+1]; apply the 5-point composite operator with
//       compile-time immediates (stage_imm.cuh) from shared memory, add the
//       RK combination with u0 (alpha stages: loaded from HBM at the start of
//       the pixel), store to HBM; release rows whose last reader has passed.
//
// No CTA-wide barrier: warps drift within the ring, the producer keeps as many
// rows in flight as the rings hold (adaptive lookahead: Gamma rows are ~40 %
// full), and every pixel is read from HBM once per stage plus the 2-column
// strip halo and 2 band-halo rows.  Rings are circular buffers of pixel tiles
// (a tile copy may wrap: two bulk copies on one barrier); ring 1 holds >= 4
// full row tiles and ring 2 >= 4 full compute rows, so row j+1 can always be
// issued while rows j-1 and j are held (no deadlock).
#pragma once
#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cstdlib>
#include "kernels.cuh"
#include "stage_imm.cuh"
#include "launch.h"

namespace dgk {

constexpr int RING_Q = 16;         // row entries (full/empty barrier pairs)
#ifndef RING_N1_NOALPHA            // ring-1 slots without the alpha term
#define RING_N1_NOALPHA(W, PXB, budget) ((budget) / (PXB))
#endif
constexpr int RING_MAXBAND = 256;  // max rows per band (+2 halo rows)
// alpha stages: u0 is read by the consumer straight from HBM (issued before
// the pixel's MACs, so its latency hides behind them) instead of being staged
// in ring 2; the freed shared memory buys the stage-1 geometry (W = 16 for
// P1, deeper ring 1).  -DDGDIFF_U0_RING restores the staged variant.
#ifdef DGDIFF_U0_RING
template <int P> constexpr bool ring_u0_direct() { return false; }
#else
template <int P> constexpr bool ring_u0_direct() { return true; }
#endif

// strip width W and consumer warps NC per (degree, lane bytes, mode): a pixel
// tile is 2d x 32 lanes x lane bytes; four full halo'd rows must fit in ring
// 1.  Modes: RING_PLAIN (stage 1, no alpha term: ring 2 only holds neighbour
// indices, so P1 affords W = 16, half the rows per byte of W = 8),
// RING_U0_STAGED (u0 tiles in ring 2), RING_U0_DIRECT (u0 from HBM into
// registers: P2 runs it with 12 consumer warps so the extra registers fit).
enum { RING_PLAIN = 0, RING_U0_STAGED = 1, RING_U0_DIRECT = 2 };
template <int P, int LB, int MODE> struct RingCfg;
template <> struct RingCfg<1, 16, RING_PLAIN> { static constexpr int W = 16, NC = 8; };   // NC swept 4/8/12/16
template <> struct RingCfg<1, 16, RING_U0_STAGED> { static constexpr int W = 8, NC = 8; };
template <> struct RingCfg<1, 16, RING_U0_DIRECT> { static constexpr int W = 16, NC = 8; };
template <> struct RingCfg<2, 8, RING_PLAIN> { static constexpr int W = 16, NC = 16; };   // c5: W 8 -> 16 -29 %
template <> struct RingCfg<2, 8, RING_U0_STAGED> { static constexpr int W = 8, NC = 16; };
template <> struct RingCfg<2, 8, RING_U0_DIRECT> { static constexpr int W = 16, NC = 12; };   // c5: NC 8 -> 12 -4 %
// P3 (N4): 5 KB pixel tiles (fp64), four halo'd rows of W = 8 fill ring 1
template <> struct RingCfg<3, 8, RING_PLAIN> { static constexpr int W = 8, NC = 12; };   // c5: NC 8 -> 12 -10 %
template <> struct RingCfg<3, 8, RING_U0_STAGED> { static constexpr int W = 8, NC = 8; };
template <> struct RingCfg<3, 8, RING_U0_DIRECT> { static constexpr int W = 8, NC = 8; };
// N4 quadrilaterals: degree codes 101 (Q1), 102 (Q2); their composite
// operator is a 9-point cross, so strips carry a 2-column halo, a pixel of
// row j reads rows j-2..j+2 and each pixel has 8 neighbour indices
// (Q1 with item neighbour buffers, c5: 8 / 11 / 15 / 19 / 23 / 31 consumer
// warps -> 0.76 / 0.63 / 0.57 / 0.57 / 0.59 / 0.65 ms stage 1)
#ifndef DGDIFF_Q1_NC
#define DGDIFF_Q1_NC 15
#endif
template <> struct RingCfg<101, 8, RING_PLAIN> { static constexpr int W = 16, NC = DGDIFF_Q1_NC; };
template <> struct RingCfg<101, 8, RING_U0_STAGED> { static constexpr int W = 16, NC = 8; };
template <> struct RingCfg<101, 8, RING_U0_DIRECT> { static constexpr int W = 16, NC = DGDIFF_Q1_NC; };
// (Q2 with item neighbour buffers, c5: 6 / 8 / 11 / 15 consumer warps ->
// 1.34 / 1.22 / 1.11 / 1.11 ms stage 1)
#ifndef DGDIFF_Q2_NC
#define DGDIFF_Q2_NC 11
#endif
#ifndef DGDIFF_Q2_NCA
#define DGDIFF_Q2_NCA 11
#endif
template <> struct RingCfg<102, 8, RING_PLAIN> { static constexpr int W = 8, NC = DGDIFF_Q2_NC; };
template <> struct RingCfg<102, 8, RING_U0_STAGED> { static constexpr int W = 8, NC = 8; };
template <> struct RingCfg<102, 8, RING_U0_DIRECT> { static constexpr int W = 8, NC = DGDIFF_Q2_NCA; };
// P3 operator application: column loops over a shared-memory table (round
// 2, default) or the round-1 straight-line immediates (-DDGDIFF_P3_IMM)
// (fp64 only: fp32 coefficients are 32-bit FFMA immediates, so the fp32
// straight-line code is half the size and runs faster than the loops, c5:
// 2.2 vs 3.8 ms per stage)
#ifdef DGDIFF_P3_IMM
template <typename T, int P> constexpr bool ring_p3_columns() { return false; }
#else
template <typename T, int P> constexpr bool ring_p3_columns() { return P == 3 && sizeof(T) == 8; }
#endif

#ifndef DGDIFF_P3COL_NC
#define DGDIFF_P3COL_NC 11
#endif
#ifndef DGDIFF_P3COL_UNROLL   // column-loop unroll of the pair loop (c5: 1 / 2 / 4 swept)
#define DGDIFF_P3COL_UNROLL 2
#endif
#ifndef DGDIFF_P3COL_NCA   // alpha stages (u0 loads): 8 warps, 255 registers
#define DGDIFF_P3COL_NCA 7
#endif

template <int P> constexpr int ring_mode(bool alpha) {
  return alpha ? (ring_u0_direct<P>() ? RING_U0_DIRECT : RING_U0_STAGED) : RING_PLAIN;
}

template <typename T, int NV, int P, bool ALPHA>
struct RingGeom {
  static constexpr int G = 32 * NV;
  static constexpr int D2 = ndof_px<P>();
  static constexpr int HALO = halo_of<P>();                     // strip / band halo (quads: 2)
  static constexpr int NBW = HALO;                               // int4 neighbour entries per pixel
  static constexpr bool R2U = ALPHA && !ring_u0_direct<P>();   // u0 tiles staged in ring 2
  static constexpr int W = RingCfg<P, NV * (int)sizeof(T), ring_mode<P>(ALPHA)>::W;
  // (P3 column form: pixel pairs hold two 20-dof accumulators; the register
  // file is split over the 4 SM sub-partitions, so 12 warps per CTA leave 168
  // registers per thread and 8 warps 255)
  static constexpr int NC = ring_p3_columns<T, P>() ? (ALPHA ? DGDIFF_P3COL_NCA : DGDIFF_P3COL_NC)
                                                   : RingCfg<P, NV * (int)sizeof(T), ring_mode<P>(ALPHA)>::NC;
  static constexpr int PXB = D2 * G * (int)sizeof(T);  // one pixel tile (one group)
  static constexpr int SMEM_MAX = 232448;
  static constexpr int EXTRA = 2 * RING_Q * 8 + 4 * 8 + RING_Q * 32 + (RING_MAXBAND + 4) * 16 + 2 * RING_Q * 4;
  // ring 2 holds staged u0 tiles (R2U) and neighbour indices; otherwise it
  // only holds the 16-byte indices and ring 1 takes the rest
  static constexpr int N2 = R2U ? 4 * W : 16 * W;
  static constexpr int ROWS_MIN = 2 * HALO + 2;                 // rows held + 1 in flight
  // item neighbour buffer (quads, round 2): the neighbour indices of an
  // item's computed pixels arrive in ONE bulk copy per item from a strip-major
  // copy of the table (nbi), into one of two item buffers of NBI_CAP pixels,
  // instead of one copy per row into ring 2: a row then costs one bulk copy
  // (a 1-D bulk copy costs the SM's TMA ~0.3 us whatever its size, and the
  // quad kernels were bound by that row pipeline: c5 Q2 streams its rows in
  // 1.08 of 1.28 ms without computing).  Bands are capped at NBI_ROWS rows.
  static constexpr bool NBI = is_quad<P>() && !R2U;
  static constexpr int NBI_ROWS = 64;
  static constexpr int NBI_CAP = NBI ? NBI_ROWS * W : 0;
  static constexpr int NBR_BYTES = NBI ? 2 * NBI_CAP * 16 * NBW : N2 * 16 * NBW;
  // P3: the column-form operator (tables.inc P3COL_*) and its column lists
  // live in shared memory (ring_p3_columns())
  // (+ one zero lane vector: the x operand of a closed face in a pixel pair)
  static constexpr int COLB = ring_p3_columns<T, P>()
                                  ? ((P3COL_N * (int)sizeof(T) + 4 * (P3COL_NCF + P3COL_NCN) + 32 * NV * (int)sizeof(T) + 127) / 128) * 128
                                  : 0;
  // pixels per consumer work unit: P3 column form pairs (shared coefficient
  // loads).  (Units of 2-4 consecutive quad pixels, one after the other, were
  // measured for Q1/Q2 on c5 and were 0-7 % slower.)
  static constexpr int UPX = COLB ? 2 : 1;
  static_assert(!(NBI && UPX != 1), "item neighbour buffers index pixels by their unit");
  static constexpr int N1 = R2U ? ROWS_MIN * (W + 2 * HALO) : RING_N1_NOALPHA(W, PXB, SMEM_MAX - EXTRA - COLB - NBR_BYTES);
  static constexpr int OFF_R2 = N1 * PXB;
  static constexpr int OFF_NB = OFF_R2 + (R2U ? N2 * PXB : 0);
  static constexpr int OFF_BAR = OFF_NB + NBR_BYTES;
  static constexpr int OFF_META = OFF_BAR + 2 * RING_Q * 8 + 4 * 8;   // + item full / empty barriers
  static constexpr int OFF_RT = OFF_META + RING_Q * 32;
  static constexpr int OFF_COL = OFF_RT + (RING_MAXBAND + 4) * 16 + 2 * RING_Q * 4;   // rows of a band + 2 halos
  static constexpr int SMEM = OFF_COL + COLB;
  static constexpr int THREADS = (NC + 1) * 32;
  static_assert(SMEM <= SMEM_MAX, "ring does not fit in shared memory");
  static_assert(N1 >= ROWS_MIN * (W + 2 * HALO) && N2 >= ROWS_MIN * W, "rings too small for progress");
};

// Work item -> (strip s, group g, computed rows [jb0, jb1)); false if the item
// has nothing to compute.  With active windows (N1, gbox != nullptr) the rows
// and strips are clipped to group g's source box grown by wr pixels: outside
// it the stage's output is exactly zero (the 5-point operator spreads support
// by one pixel per stage) and the registers already hold zeros there.
template <int W>
__device__ __forceinline__ bool ring_item(int item, int nstrips, int ngroups, int band_rows, int ny,
                                          const int4 *__restrict__ gbox, int wr, int &s, int &g, int &jb0,
                                          int &jb1) {
  s = item % nstrips;
  g = (item / nstrips) % ngroups;
  const int b = item / (nstrips * ngroups);
  jb0 = b * band_rows;
  jb1 = min(ny, jb0 + band_rows);
  if (gbox) {
    const int4 bx = __ldg(&gbox[g]);
    if (s * W > bx.y + wr || s * W + W - 1 < bx.x - wr) return false;
    jb0 = max(jb0, bx.z - wr);
    jb1 = min(jb1, bx.w + wr + 1);
  }
  return jb0 < jb1;
}

struct RowMeta {
  int p1, h0, c0, c1;   // ring-1 slot of tile start, active-index bounds
  int p2, pad0, pad1, pad2;
};


// acc[R0 .. R0+R) += C x over the columns of a column-form block (P3): column
// jj of C is the R contiguous coefficients cf[jj*R ..], applied to the dof
// cols[jj] (identity when cols is null) of the pixel tile x (ring-1 slot,
// this lane's sources).  A runtime loop: one warp-uniform (broadcast) shared-
// memory load per two coefficients, so the code stays in the instruction
// cache whatever the block; the loop is unrolled by two so the next column's
// loads overlap this column's FMAs.
template <typename T, int NV, int D2, int G, int R, int R0>
__device__ __forceinline__ void colmv(T (&acc)[D2][NV], const T *__restrict__ cf, const unsigned char *__restrict__ cols,
                                      int ncol, const T *__restrict__ x) {
  typedef typename VT<T, 2>::type T2;
#pragma unroll 2
  for (int jj = 0; jj < ncol; jj++) {
    const int c = cols ? (int)cols[jj] : jj;
    T xv[NV];
    lds<T, NV>(x + c * G, xv);
    const T *cp = cf + jj * R;
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const T2 cc = *reinterpret_cast<const T2 *>(cp + r);
      fma_bc<T, NV>(cc.x, xv, acc[R0 + r]);
      fma_bc<T, NV>(cc.y, xv, acc[R0 + r + 1]);
    }
  }
}

// The same for two pixels at once (a warp's pixel pair): each coefficient
// load feeds both pixels' FMAs, which halves the shared-memory wavefronts per
// FMA (one broadcast wavefront per coefficient is the limit of the one-pixel
// loop: ncu, c5, L1 at 85 %).  A side whose face is closed reads the zero
// vector (stride 0): it adds exact zeros.
template <typename T, int NV, int D2, int R, int R0>
__device__ __forceinline__ void colmv2(T (&accA)[D2][NV], T (&accB)[D2][NV], const T *__restrict__ cf,
                                       const unsigned char *__restrict__ cols, int ncol, const T *__restrict__ xA,
                                       int sA, const T *__restrict__ xB, int sB) {
  typedef typename VT<T, 2>::type T2;
  constexpr int kUnroll = DGDIFF_P3COL_UNROLL;
#pragma unroll kUnroll
  for (int jj = 0; jj < ncol; jj++) {
    const int c = cols ? (int)cols[jj] : jj;
    T va[NV], vb[NV];
    lds<T, NV>(xA + c * sA, va);
    lds<T, NV>(xB + c * sB, vb);
    const T *cp = cf + jj * R;
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const T2 cc = *reinterpret_cast<const T2 *>(cp + r);
      fma_bc<T, NV>(cc.x, va, accA[R0 + r]);
      fma_bc<T, NV>(cc.x, vb, accB[R0 + r]);
      fma_bc<T, NV>(cc.y, va, accA[R0 + r + 1]);
      fma_bc<T, NV>(cc.y, vb, accB[R0 + r + 1]);
    }
  }
}

// TR: apply the transposed operator L^T (adjoint moments; P1/P2, REFLECT)
template <typename T, int NV, int P, bool HAS_ALPHA, bool TR = false>
__global__ void __launch_bounds__(RingGeom<T, NV, P, HAS_ALPHA>::THREADS, 1)
    k_stage_ring(const T *__restrict__ Uin, const T *U0, T *Uout, const int4 *__restrict__ nbr,
                 const int4 *__restrict__ rowtab, int nact, int ny, int nstrips, int ngroups, int band_rows,
                 int nitems, T alpha, T cs, int diag, int max_ahead, int n1_use, int n2_use,
                 const T *__restrict__ Aabs, const int4 *__restrict__ gbox, int wr, int serial,
                 const int4 *__restrict__ nbi, const int *__restrict__ nbi_off) {
  using Gm = RingGeom<T, NV, P, HAS_ALPHA>;
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, Q = RING_Q, NC = Gm::NC;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *ring1 = smem;
  unsigned char *ring2 = smem + Gm::OFF_R2;
  int4 *nbr_ring = reinterpret_cast<int4 *>(smem + Gm::OFF_NB);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Gm::OFF_BAR);
  uint64_t *empty = full + Q;
  uint64_t *ifull = full + 2 * Q, *iempty = ifull + 2;   // item neighbour buffers (Gm::NBI)
  RowMeta *meta = reinterpret_cast<RowMeta *>(smem + Gm::OFF_META);
  int4 *rt = reinterpret_cast<int4 *>(smem + Gm::OFF_RT);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < Q; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NC);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&ifull[b], 1);
      mbar_init(&iempty[b], NC);
    }
    fence_mbar_init();
  }
  T *colA = reinterpret_cast<T *>(smem + Gm::OFF_COL);
  T *colZ = colA + (Gm::COLB ? P3COL_N : 0);   // 32 NV zeros (a closed face's x in a pair)
  unsigned char *colI = smem + Gm::OFF_COL + (Gm::COLB ? (P3COL_N + 32 * NV) * (int)sizeof(T) : 0);
  if constexpr (Gm::COLB > 0) {
    // P3 column-form operator (state precision) and its column lists
    for (int i = tid; i < P3COL_N; i += blockDim.x) colA[i] = (T)P3COL_D[i];
    for (int i = tid; i < 32 * NV; i += blockDim.x) colZ[i] = (T)0;
    for (int i = tid; i < 4 * (P3COL_NCF + P3COL_NCN); i += blockDim.x)
      colI[i] = i < 4 * P3COL_NCF ? P3COL_CF[i / P3COL_NCF][i % P3COL_NCF]
                                  : P3COL_CN[(i - 4 * P3COL_NCF) / P3COL_NCN][(i - 4 * P3COL_NCF) % P3COL_NCN];
  }
  __syncthreads();
  const size_t gstride = (size_t)nact * D2 * G;

  if (w == NC) {
    // =========================== producer warp ===========================
    // Rows are issued in batches of up to 32, one row per lane: a warp scan
    // gives every row its ring offsets, the longest prefix that fits is
    // issued at once (each lane arms its row's barrier and issues its own
    // bulk copies), and releases are awaited in row order only when the
    // rings are full.  rv1/rv2[q] = virtual end of the row in entry q.
    uint32_t *rv = reinterpret_cast<uint32_t *>(rt + RING_MAXBAND + 4);   // [2][Q]
    uint32_t L = 0;                 // row loads issued by this CTA
    uint32_t v1 = 0, v2 = 0;        // virtual slot counters of rings 1 and 2
    uint32_t rel = 0;               // rows whose release has been observed
    uint32_t icount = 0;            // items issued (NBI buffers)
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int s, g, jb0, jb1;
      if (!ring_item<Gm::W>(item, nstrips, ngroups, band_rows, ny, gbox, wr, s, g, jb0, jb1)) continue;
      const int lo = max(0, jb0 - Gm::HALO), hi = min(ny - 1, jb1 - 1 + Gm::HALO);
      __syncwarp();
      for (int r = lo + lane; r <= hi; r += 32) rt[r - lo] = __ldg(&rowtab[(size_t)s * ny + r]);
      __syncwarp();
      const T *Ug = Uin + g * gstride;
      const T *U0g = U0 + g * gstride;
      if constexpr (Gm::NBI) {
        // the item's neighbour entries: one bulk copy into item buffer b once
        // the consumers are done with the item that used it two items ago
        if (lane == 0) {
          const uint32_t b = icount & 1;
          if (icount >= 2) mbar_wait(&iempty[b], ((icount - 2) >> 1) & 1);
          const int o0 = __ldg(&nbi_off[(size_t)s * (ny + 1) + jb0]), o1 = __ldg(&nbi_off[(size_t)s * (ny + 1) + jb1]);
          if (o1 - o0 > Gm::NBI_CAP) __trap();   // the launcher caps the bands
          const uint32_t bytes = (uint32_t)(o1 - o0) * 16u * Gm::NBW;
          mbar_expect_tx(&ifull[b], bytes);
          if (bytes) bulk_g2s(nbr_ring + (size_t)b * Gm::NBI_CAP * Gm::NBW, nbi + (size_t)o0 * Gm::NBW, bytes, &ifull[b]);
        }
        icount++;
      }
      if (serial || Gm::NBI) {
        // one lane issues the rows one at a time (see k_stage_pair: the batch
        // issue re-runs its scan for every released row once the ring is full)
        if (lane == 0) {
          for (int r = lo; r <= hi; r++) {
            const int4 t = rt[r - lo];
            const bool comp = r >= jb0 && r < jb1;
            const uint32_t n1 = (uint32_t)(t.w - t.x), n2 = comp && !Gm::NBI ? (uint32_t)(t.z - t.y) : 0u;
            for (;;) {
              const uint32_t s1 = rel ? rv[(rel - 1) % Q] : 0u, s2 = rel ? rv[Q + (rel - 1) % Q] : 0u;
              if ((L - rel < (uint32_t)max_ahead && v1 + n1 - s1 <= (uint32_t)n1_use && v2 + n2 - s2 <= (uint32_t)n2_use) ||
                  rel == L)
                break;
              mbar_wait(&empty[rel % Q], (rel / Q) & 1);
              rel++;
            }
            const uint32_t q = L % Q, p1 = v1 % Gm::N1, p2 = v2 % Gm::N2;
            RowMeta m;
            m.p1 = (int)p1; m.h0 = t.x; m.c0 = t.y; m.c1 = comp ? t.z : t.y; m.p2 = (int)p2;
            m.pad0 = m.pad1 = m.pad2 = 0;
            meta[q] = m;
            v1 += n1;
            v2 += n2;
            rv[q] = v1;
            rv[Q + q] = v2;
            const uint32_t bytes = n1 * PXB + (Gm::R2U ? n2 * PXB : 0u) + n2 * 16u * Gm::NBW;
            mbar_expect_tx(&full[q], bytes);
            if (n1) {
              const uint32_t a1 = min(n1, (uint32_t)Gm::N1 - p1);
              const T *src = Ug + (size_t)t.x * D2 * G;
              bulk_g2s(ring1 + (size_t)p1 * PXB, src, a1 * PXB, &full[q]);
              if (n1 > a1) bulk_g2s(ring1, src + (size_t)a1 * D2 * G, (n1 - a1) * PXB, &full[q]);
            }
            if (n2) {
              const uint32_t a2 = min(n2, (uint32_t)Gm::N2 - p2);
              if (Gm::R2U) {
                const T *src = U0g + (size_t)t.y * D2 * G;
                bulk_g2s(ring2 + (size_t)p2 * PXB, src, a2 * PXB, &full[q]);
                if (n2 > a2) bulk_g2s(ring2, src + (size_t)a2 * D2 * G, (n2 - a2) * PXB, &full[q]);
              }
              bulk_g2s(nbr_ring + (size_t)p2 * Gm::NBW, nbr + (size_t)t.y * Gm::NBW, a2 * 16u * Gm::NBW, &full[q]);
              if (n2 > a2)
                bulk_g2s(nbr_ring, nbr + ((size_t)t.y + a2) * Gm::NBW, (n2 - a2) * 16u * Gm::NBW, &full[q]);
            }
            L++;
          }
        }
        __syncwarp();
        continue;
      }
      for (int r0 = lo; r0 <= hi;) {
        const int r = r0 + lane;
        const bool valid = r <= hi;
        int4 t = make_int4(0, 0, 0, 0);
        if (valid) t = rt[r - lo];
        const bool comp = valid && r >= jb0 && r < jb1;
        const uint32_t n1 = valid ? (uint32_t)(t.w - t.x) : 0u;
        const uint32_t n2 = comp ? (uint32_t)(t.z - t.y) : 0u;
        uint32_t e1 = n1, e2 = n2;                      // inclusive scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y1 = __shfl_up_sync(0xffffffffu, e1, o), y2 = __shfl_up_sync(0xffffffffu, e2, o);
          if (lane >= o) { e1 += y1; e2 += y2; }
        }
        const uint32_t nvalid = (uint32_t)min(32, hi - r0 + 1);
        // wait (in row order) until at least the first row fits, then take
        // the longest prefix that fits
        uint32_t take;
        for (;;) {
          const uint32_t s1 = rel ? rv[(rel - 1) % Q] : 0u, s2 = rel ? rv[Q + (rel - 1) % Q] : 0u;
          // L + lane - rel < max_ahead <= Q - 1: rows in flight are capped, and entry
          // (rel-1) % Q (the live start) is never reused early
          const bool fits = valid && (L + lane - rel < (uint32_t)max_ahead) && (v1 + e1 - s1 <= (uint32_t)n1_use) &&
                            (v2 + e2 - s2 <= (uint32_t)n2_use);
          const uint32_t ok = __ballot_sync(0xffffffffu, fits);
          take = __ffs(~ok) - 1;                         // length of the fitting prefix
          if (ok == 0xffffffffu) take = 32;
          if (take > nvalid) take = nvalid;
          if (take > 0 || rel == L) break;
          mbar_wait(&empty[rel % Q], (rel / Q) & 1);
          rel++;
        }
        if (take == 0) take = 1;                         // rel == L: the ring is empty
        if ((uint32_t)lane < take) {
          const uint32_t Lr = L + lane, q = Lr % Q;
          const uint32_t b1 = v1 + e1 - n1, b2 = v2 + e2 - n2;   // virtual starts
          const uint32_t p1 = b1 % Gm::N1, p2 = b2 % Gm::N2;
          RowMeta m;
          m.p1 = (int)p1; m.h0 = t.x; m.c0 = t.y; m.c1 = comp ? t.z : t.y; m.p2 = (int)p2;
          m.pad0 = m.pad1 = m.pad2 = 0;
          meta[q] = m;
          rv[q] = v1 + e1;
          rv[Q + q] = v2 + e2;
          const uint32_t bytes = n1 * PXB + (Gm::R2U ? n2 * PXB : 0u) + n2 * 16u * Gm::NBW;
          mbar_expect_tx(&full[q], bytes);
          if (n1) {
            const uint32_t a1 = min(n1, (uint32_t)Gm::N1 - p1);
            const T *src = Ug + (size_t)t.x * D2 * G;
            bulk_g2s(ring1 + (size_t)p1 * PXB, src, a1 * PXB, &full[q]);
            if (n1 > a1) bulk_g2s(ring1, src + (size_t)a1 * D2 * G, (n1 - a1) * PXB, &full[q]);
          }
          if (n2) {
            const uint32_t a2 = min(n2, (uint32_t)Gm::N2 - p2);
            if (Gm::R2U) {
              const T *src = U0g + (size_t)t.y * D2 * G;
              bulk_g2s(ring2 + (size_t)p2 * PXB, src, a2 * PXB, &full[q]);
              if (n2 > a2) bulk_g2s(ring2, src + (size_t)a2 * D2 * G, (n2 - a2) * PXB, &full[q]);
            }
            bulk_g2s(nbr_ring + (size_t)p2 * Gm::NBW, nbr + (size_t)t.y * Gm::NBW, a2 * 16u * Gm::NBW, &full[q]);
            if (n2 > a2)
              bulk_g2s(nbr_ring, nbr + ((size_t)t.y + a2) * Gm::NBW, (n2 - a2) * 16u * Gm::NBW, &full[q]);
          }
        }
        // advance by the issued prefix
        v1 += __shfl_sync(0xffffffffu, e1, take - 1);
        v2 += __shfl_sync(0xffffffffu, e2, take - 1);
        L += take;
        r0 += (int)take;
        __syncwarp();
      }
    }
    return;
  }

  // ============================= consumer warps ============================
  // The band's computed pixels are dealt out flattened across rows: warp w
  // takes pixels w, w + NC, w + 2 NC, ... in raster order, so on sparse rows
  // the warps work on several rows at once.  A warp releases row r once its
  // cursor has passed row r + 1.
  uint32_t Lbase = 0;
  uint32_t icount = 0;   // items consumed (NBI buffers)
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    int s_, g, jb0, jb1;
    if (!ring_item<Gm::W>(item, nstrips, ngroups, band_rows, ny, gbox, wr, s_, g, jb0, jb1)) continue;
    // (NBI: the item's neighbour entries, indexed by the pixel's position f in
    // the band's computed pixels)
    const int4 *nbb = nbr_ring + (size_t)(icount & 1) * Gm::NBI_CAP * Gm::NBW;
    if constexpr (Gm::NBI) mbar_wait(&ifull[icount & 1], (icount >> 1) & 1);
    const int lo = max(0, jb0 - Gm::HALO), hi = min(ny - 1, jb1 - 1 + Gm::HALO);
    T *Uog = Uout + g * gstride + lane * NV;
    const T *U0l = U0 + g * gstride + lane * NV;
    auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
    auto wait_row = [&](int r) {
      if (r >= lo && r <= hi) {
        const uint32_t L = seq(r);
        mbar_wait(&full[L % Q], (L / Q) & 1);
      }
    };
    auto tile1 = [&](const RowMeta &m, int idx) -> const T * {
      int sl = m.p1 + (idx - m.h0);
      if (sl >= Gm::N1) sl -= Gm::N1;
      return reinterpret_cast<const T *>(ring1 + (size_t)sl * PXB) + lane * NV;
    };
    int j = jb0, rel_next = lo, cum = 0;
    for (int r = jb0 - Gm::HALO; r <= jb0 + Gm::HALO; r++) wait_row(r);
    RowMeta mc = meta[seq(j) % Q];
    constexpr int UPX = Gm::UPX;
    for (int f = w;; f += NC) {
      // (work units: pixels, or pixel pairs within a row for the P3 column form)
      while (f >= cum + (mc.c1 - mc.c0 + UPX - 1) / UPX) {      // advance the cursor to f's row
        cum += (mc.c1 - mc.c0 + UPX - 1) / UPX;
        if (++j >= jb1) break;
        // this warp's remaining pixels lie in rows >= j: rows <= j-1-HALO have
        // had their last reader; release them before waiting for row j+HALO (a
        // warp must never hold old rows while it waits for new ones)
        if (rel_next <= j - 1 - Gm::HALO) {
          __syncwarp();
          if (lane == 0)
            for (int r = rel_next; r <= j - 1 - Gm::HALO; r++) mbar_arrive(&empty[seq(r) % Q]);
          rel_next = j - Gm::HALO;
        }
        wait_row(j + Gm::HALO);
        mc = meta[seq(j) % Q];
      }
      if (j >= jb1) break;
      if (diag == 1) continue;   // diagnostic: stream through the ring without computing
      auto pixel = [&](const int a) {
      int sl2 = mc.p2 + (a - mc.c0);
      if (sl2 >= Gm::N2) sl2 -= Gm::N2;
      const int4 *nbp = Gm::NBI ? nbb + (size_t)f * Gm::NBW : nbr_ring + (size_t)sl2 * Gm::NBW;
      const int4 nb = nbp[0];
      const T *ps = tile1(mc, a);
      T xs[D2][NV], acc[D2][NV], xn[D2][NV], z[D2][NV];
      if constexpr (HAS_ALPHA && !Gm::R2U) {
        // u0 straight from HBM (coherent load: stage 3 writes u in place; this
        // lane reads its elements before it writes them)
#pragma unroll
        for (int k = 0; k < D2; k++) ldvc<T, NV>(U0l + ((size_t)a * D2 + k) * G, z[k]);
      }
      // (column form: xs is read per column and again for the RK combination)
      if constexpr (!Gm::COLB) {
#pragma unroll
        for (int k = 0; k < D2; k++) lds<T, NV>(ps + k * G, xs[k]);
      }
#pragma unroll
      for (int k = 0; k < D2; k++)
#pragma unroll
        for (int e = 0; e < NV; e++) acc[k][e] = (T)0;
      // faces on the outer square under ABSORB (Eq. (4)) are marked -2
      const int outer = (nb.x == -2) | ((nb.y == -2) << 1) | ((nb.z == -2) << 2) | ((nb.w == -2) << 3);
      if constexpr (is_quad<P>()) {
        // N4 Q_p: self[code] + per open face the neighbour block (two variants:
        // opposite face open / closed) and the far block of the pixel two
        // steps on (when extracellular); the corners couple to nothing
        const int4 nb2 = nbp[1];
        const int code = open_code(nb);
        const int far_out = (nb2.x == -2) | ((nb2.y == -2) << 1) | ((nb2.z == -2) << 2) | ((nb2.w == -2) << 3);
        if (__builtin_expect((outer | far_out) != 0, 0)) {
          // ABSORB within two pixels of the outer square: K0's runtime blocks
          // (self by (code, outer); neighbour by (opposite-face state, far
          // face outer); far block fixed), see build_quad_absorb
          const T *Ab = Aabs;
          mv_gen<T, NV, D2>(acc, Ab + (size_t)(code * 16 + outer) * D2 * D2, xs);
          const int nbv[4] = {nb.x, nb.y, nb.z, nb.w}, far[4] = {nb2.x, nb2.y, nb2.z, nb2.w};
#pragma unroll 1
          for (int f = 0; f < 4; f++) {
            if (nbv[f] < 0) continue;
            const int o = f ^ 1;   // opposite face (E<->W, N<->S)
            const int os = nbv[o] >= 0 ? 1 : (nbv[o] == -2 ? 2 : 0);
            const RowMeta mf = f < 2 ? mc : meta[seq(f == 2 ? j + 1 : j - 1) % Q];
            const T *pn = tile1(mf, nbv[f]);
#pragma unroll
            for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
            mv_gen<T, NV, D2>(acc, Ab + (size_t)(256 + (f * 3 + os) * 2 + (far[f] == -2)) * D2 * D2, xn);
            if (far[f] >= 0) {
              const RowMeta mff = f < 2 ? mc : meta[seq(f == 2 ? j + 2 : j - 2) % Q];
              const T *pf = tile1(mff, far[f]);
#pragma unroll
              for (int k = 0; k < D2; k++) lds<T, NV>(pf + k * G, xn[k]);
              mv_gen<T, NV, D2>(acc, Ab + (size_t)(280 + f) * D2 * D2, xn);
            }
          }
        } else {
        // (TR, the transposed operator: the face-f block's variant follows the
        // state of the pixel two steps on, whose face decides L's block there)
        mv_self<T, NV, P, TR>(code, acc, xs);
        if (nb.x >= 0) {
          const T *pn = tile1(mc, nb.x);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          if (TR ? nb2.x >= 0 : nb.y >= 0) mv_imm<T, NV, P, 16, TR>(acc, xn); else mv_imm<T, NV, P, 20, TR>(acc, xn);
          if (nb2.x >= 0) {
            const T *pf = tile1(mc, nb2.x);
#pragma unroll
            for (int k = 0; k < D2; k++) lds<T, NV>(pf + k * G, xn[k]);
            mv_imm<T, NV, P, 24, TR>(acc, xn);
          }
        }
        if (nb.y >= 0) {
          const T *pn = tile1(mc, nb.y);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          if (TR ? nb2.y >= 0 : nb.x >= 0) mv_imm<T, NV, P, 17, TR>(acc, xn); else mv_imm<T, NV, P, 21, TR>(acc, xn);
          if (nb2.y >= 0) {
            const T *pf = tile1(mc, nb2.y);
#pragma unroll
            for (int k = 0; k < D2; k++) lds<T, NV>(pf + k * G, xn[k]);
            mv_imm<T, NV, P, 25, TR>(acc, xn);
          }
        }
        if (nb.z >= 0) {
          const T *pn = tile1(meta[seq(j + 1) % Q], nb.z);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          if (TR ? nb2.z >= 0 : nb.w >= 0) mv_imm<T, NV, P, 18, TR>(acc, xn); else mv_imm<T, NV, P, 22, TR>(acc, xn);
          if (nb2.z >= 0) {
            const T *pf = tile1(meta[seq(j + 2) % Q], nb2.z);
#pragma unroll
            for (int k = 0; k < D2; k++) lds<T, NV>(pf + k * G, xn[k]);
            mv_imm<T, NV, P, 26, TR>(acc, xn);
          }
        }
        if (nb.w >= 0) {
          const T *pn = tile1(meta[seq(j - 1) % Q], nb.w);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          if (TR ? nb2.w >= 0 : nb.z >= 0) mv_imm<T, NV, P, 19, TR>(acc, xn); else mv_imm<T, NV, P, 23, TR>(acc, xn);
          if (nb2.w >= 0) {
            const T *pf = tile1(meta[seq(j - 2) % Q], nb2.w);
#pragma unroll
            for (int k = 0; k < D2; k++) lds<T, NV>(pf + k * G, xn[k]);
            mv_imm<T, NV, P, 27, TR>(acc, xn);
          }
        }
        }   // interior / REFLECT quads
      } else if (Gm::COLB && __builtin_expect(outer == 0, 1)) {
        // P3 column form: V, then per open face F_f (the RF rows of the
        // triangle owning face f) and N_f, each a loop over its columns
        if constexpr (Gm::COLB > 0) {
          constexpr int RF = P3COL_RF, NCF = P3COL_NCF, NCN = P3COL_NCN;
          const T *cV = colA, *cF = colA + D2 * D2;
          constexpr int FB = NCF * RF + NCN * D2;   // per-face block size
          colmv<T, NV, D2, G, D2, 0>(acc, cV, nullptr, D2, ps);
          if (nb.x >= 0) {
            colmv<T, NV, D2, G, RF, P3COL_R0F[0]>(acc, cF + 0 * FB, colI + 0 * NCF, NCF, ps);
            colmv<T, NV, D2, G, D2, 0>(acc, cF + 0 * FB + NCF * RF, colI + 4 * NCF + 0 * NCN, NCN, tile1(mc, nb.x));
          }
          if (nb.y >= 0) {
            colmv<T, NV, D2, G, RF, P3COL_R0F[1]>(acc, cF + 1 * FB, colI + 1 * NCF, NCF, ps);
            colmv<T, NV, D2, G, D2, 0>(acc, cF + 1 * FB + NCF * RF, colI + 4 * NCF + 1 * NCN, NCN, tile1(mc, nb.y));
          }
          if (nb.z >= 0) {
            colmv<T, NV, D2, G, RF, P3COL_R0F[2]>(acc, cF + 2 * FB, colI + 2 * NCF, NCF, ps);
            colmv<T, NV, D2, G, D2, 0>(acc, cF + 2 * FB + NCF * RF, colI + 4 * NCF + 2 * NCN, NCN,
                                       tile1(meta[seq(j + 1) % Q], nb.z));
          }
          if (nb.w >= 0) {
            colmv<T, NV, D2, G, RF, P3COL_R0F[3]>(acc, cF + 3 * FB, colI + 3 * NCF, NCF, ps);
            colmv<T, NV, D2, G, D2, 0>(acc, cF + 3 * FB + NCF * RF, colI + 4 * NCF + 3 * NCN, NCN,
                                       tile1(meta[seq(j - 1) % Q], nb.w));
          }
        }
      } else if (__builtin_expect(outer == 0, 1)) {
        // self block of this pixel's open-face code (compile-time immediates),
        // then the fixed neighbour blocks of the open faces
        // (P3: 400-entry blocks; a 16-variant switch would not fit the
        // instruction cache, so the self block is applied as V + sum F_f)
        if constexpr (P <= 2) mv_self<T, NV, P, TR>(open_code(nb), acc, xs);
        else mv_imm<T, NV, P, 0>(acc, xs);
        if (nb.x >= 0) {
          if constexpr (P == 3) mv_imm<T, NV, P, 1>(acc, xs);
          const T *pn = tile1(mc, nb.x);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 5, TR>(acc, xn);
        }
        if (nb.y >= 0) {
          if constexpr (P == 3) mv_imm<T, NV, P, 2>(acc, xs);
          const T *pn = tile1(mc, nb.y);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 6, TR>(acc, xn);
        }
        if (nb.z >= 0) {
          if constexpr (P == 3) mv_imm<T, NV, P, 3>(acc, xs);
          const RowMeta mn = meta[seq(j + 1) % Q];
          const T *pn = tile1(mn, nb.z);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 7, TR>(acc, xn);
        }
        if (nb.w >= 0) {
          if constexpr (P == 3) mv_imm<T, NV, P, 4>(acc, xs);
          const RowMeta ms = meta[seq(j - 1) % Q];
          const T *pn = tile1(ms, nb.w);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_imm<T, NV, P, 8, TR>(acc, xn);
        }
      } else {
        // boundary pixel with absorbing outer faces: blocks of (code, outer)
        // read from the K0 table in global memory (rare: grid-edge pixels)
        const T *Ab = Aabs + (size_t)((open_code(nb) * 16 + outer) * 5) * D2 * D2;
        if constexpr (Gm::COLB > 0) {
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(ps + k * G, xs[k]);
        }
        mv_gen<T, NV, D2>(acc, Ab, xs);
        const int nbv[4] = {nb.x, nb.y, nb.z, nb.w};
#pragma unroll 1
        for (int f = 0; f < 4; f++) {
          if (nbv[f] < 0) continue;
          const T *pn = f < 2 ? tile1(mc, nbv[f]) : tile1(meta[seq(f == 2 ? j + 1 : j - 1) % Q], nbv[f]);
#pragma unroll
          for (int k = 0; k < D2; k++) lds<T, NV>(pn + k * G, xn[k]);
          mv_gen<T, NV, D2>(acc, Ab + (size_t)(f + 1) * D2 * D2, xn);
        }
      }
      const T *pu = reinterpret_cast<const T *>(ring2 + (size_t)sl2 * PXB) + lane * NV;
      T *out = Uog + (size_t)a * D2 * G;
#pragma unroll
      for (int k = 0; k < D2; k++) {
        T y[NV];
        if constexpr (Gm::COLB > 0) lds<T, NV>(ps + k * G, xs[k]);
        if (HAS_ALPHA) {
          if constexpr (Gm::R2U) lds<T, NV>(pu + k * G, z[k]);
#pragma unroll
          for (int e = 0; e < NV; e++) y[e] = xs[k][e] + alpha * (z[k][e] - xs[k][e]) + cs * acc[k][e];
        } else {
#pragma unroll
          for (int e = 0; e < NV; e++) y[e] = xs[k][e] + cs * acc[k][e];
        }
        stv<T, NV>(out + (size_t)k * G, y);
      }
      };   // pixel
      if constexpr (UPX == 1) {
        pixel(mc.c0 + (f - cum));
      } else {
        const int a = mc.c0 + 2 * (f - cum);
        if (a + 1 < mc.c1) {
          int sl2 = mc.p2 + (a - mc.c0), sl2b = sl2 + 1;
          if (sl2 >= Gm::N2) sl2 -= Gm::N2;
          if (sl2b >= Gm::N2) sl2b -= Gm::N2;
          const int4 nA = nbr_ring[(size_t)sl2 * Gm::NBW], nB = nbr_ring[(size_t)sl2b * Gm::NBW];
          const bool outer = nA.x == -2 || nA.y == -2 || nA.z == -2 || nA.w == -2 || nB.x == -2 || nB.y == -2 ||
                             nB.z == -2 || nB.w == -2;
          if (__builtin_expect(!outer, 1)) {
            if constexpr (Gm::COLB > 0) {
              // pixel pair (a, a + 1) of row j, P3 column form
              constexpr int RF = P3COL_RF, NCF = P3COL_NCF, NCN = P3COL_NCN;
              constexpr int FB = NCF * RF + NCN * D2;
              const T *cV = colA, *cF = colA + D2 * D2;
              const T *pA = tile1(mc, a), *pB = tile1(mc, a + 1);
              T accA[D2][NV], accB[D2][NV];
#pragma unroll
              for (int k = 0; k < D2; k++)
#pragma unroll
                for (int e = 0; e < NV; e++) accA[k][e] = accB[k][e] = (T)0;
              colmv2<T, NV, D2, D2, 0>(accA, accB, cV, nullptr, D2, pA, G, pB, G);
              const T *zv = colZ + lane * NV;
              // per face: F_f on the self tile and N_f on the neighbour tile of
              // each pixel whose face is open (zeros for the other)
              auto face = [&](auto fc, int ia, int ib, const RowMeta &mn) {
                constexpr int fi = decltype(fc)::value;
                if (ia < 0 && ib < 0) return;
                colmv2<T, NV, D2, RF, P3COL_R0F[fi]>(accA, accB, cF + fi * FB, colI + fi * NCF, NCF, ia >= 0 ? pA : zv,
                                                     ia >= 0 ? G : 0, ib >= 0 ? pB : zv, ib >= 0 ? G : 0);
                colmv2<T, NV, D2, D2, 0>(accA, accB, cF + fi * FB + NCF * RF, colI + 4 * NCF + fi * NCN, NCN,
                                         ia >= 0 ? tile1(mn, ia) : zv, ia >= 0 ? G : 0, ib >= 0 ? tile1(mn, ib) : zv,
                                         ib >= 0 ? G : 0);
              };
              face(std::integral_constant<int, 0>(), nA.x, nB.x, mc);
              face(std::integral_constant<int, 1>(), nA.y, nB.y, mc);
              face(std::integral_constant<int, 2>(), nA.z, nB.z, meta[seq(j + 1) % Q]);
              face(std::integral_constant<int, 3>(), nA.w, nB.w, meta[seq(j - 1) % Q]);
              auto finish = [&](int ap, const T *pp, const T (&ac)[D2][NV]) {
                T *out = Uog + (size_t)ap * D2 * G;
#pragma unroll
                for (int k = 0; k < D2; k++) {
                  T xk[NV], y[NV];
                  lds<T, NV>(pp + k * G, xk);
                  if constexpr (HAS_ALPHA) {
                    T zk[NV];
                    ldvc<T, NV>(U0l + ((size_t)ap * D2 + k) * G, zk);
#pragma unroll
                    for (int e = 0; e < NV; e++) y[e] = xk[e] + alpha * (zk[e] - xk[e]) + cs * ac[k][e];
                  } else {
#pragma unroll
                    for (int e = 0; e < NV; e++) y[e] = xk[e] + cs * ac[k][e];
                  }
                  stv<T, NV>(out + (size_t)k * G, y);
                }
              };
              finish(a, pA, accA);
              finish(a + 1, pB, accB);
            }
          } else {
            pixel(a);
            pixel(a + 1);
          }
        } else {
          pixel(a);
        }
      }
    }
    // release every row of the item not yet released by this warp
    __syncwarp();
    if (lane == 0) {
      for (int r = rel_next; r <= hi; r++) mbar_arrive(&empty[seq(r) % Q]);
      if constexpr (Gm::NBI) mbar_arrive(&iempty[icount & 1]);
    }
    icount++;
    Lbase += (uint32_t)(hi - lo + 1);
  }
}

// producer mode: 1 = rows issued one at a time by one lane, 0 = warp-wide
// batches.  Measured on c5 (64 sources, ms per stage, round 2): Q2 1.42 -> 1.32
// with the serial issue, Q1 0.835 -> 0.829, P2 1.18 -> 1.22, P1 / P3 / c4 and
// windows unchanged: serial for the quadrilaterals (DGDIFF_RING_SERIAL
// overrides in tuning builds)
template <int P>
inline int ring_serial_producer() {
  static const int v = [] {
    const char *e = tune_env("DGDIFF_RING_SERIAL");
    return e ? atoi(e) : (is_quad<P>() ? 1 : 0);
  }();
  return v;
}

// rows in flight per CTA (issued, not yet released): sparse rows stream best
// with ~8 rows of lookahead, dense rows are limited by ring bytes first
inline int alpha_max_ahead(const dgl::StageArgs &a, bool alpha) {
  return alpha ? (a.ahead_alpha > 0 ? a.ahead_alpha : RING_Q - 1) : (a.ahead_noalpha > 0 ? a.ahead_noalpha : RING_Q - 1);
}

template <typename T, int NV, int P, bool ALPHA, bool TR = false>
cudaError_t launch_ring(const dgl::StageArgs &a) {
  using Gm = RingGeom<T, NV, P, ALPHA>;
  // the dynamic shared-memory opt-in is per device: one bit per ordinal
  static std::atomic<uint64_t> attr_set{0};
  static const int pad = [] {
    int v = 0;
    if (const char *e = tune_env("DGDIFF_SMEM_PAD")) v = atoi(e);
    return Gm::SMEM + v > Gm::SMEM_MAX ? Gm::SMEM_MAX - Gm::SMEM : std::max(0, v);
  }();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!(attr_set.load() >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_stage_ring<T, NV, P, ALPHA, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Gm::SMEM + pad);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(uint64_t(1) << dev);
  }
  const int per_band = (ALPHA ? a.nstrips : a.nstrips_na) * a.ngroups;
  int nbands = std::max(1, std::min(a.ny, (8 * a.nsm + per_band - 1) / per_band));
  int band_rows = (a.ny + nbands - 1) / nbands;
  if (a.band_rows > 0) band_rows = std::min(band_rows, a.band_rows);   // N1 windows: finer items
  static const int env_band = tune_env("DGDIFF_K2_BAND") ? atoi(tune_env("DGDIFF_K2_BAND")) : 0;   // diagnostic
  if (env_band > 0) band_rows = std::min(band_rows, env_band);
  if (band_rows > RING_MAXBAND) band_rows = RING_MAXBAND;
  if (Gm::NBI) {
    if (!(ALPHA ? a.nbi : a.nbi_na)) return cudaErrorInvalidValue;
    band_rows = std::min(band_rows, Gm::NBI_ROWS);   // the item buffer holds NBI_ROWS full rows
  }
  nbands = (a.ny + band_rows - 1) / band_rows;
  const int nitems = per_band * nbands;
  const int grid = std::min(nitems, a.nsm);
  k_stage_ring<T, NV, P, ALPHA, TR><<<grid, Gm::THREADS, Gm::SMEM + pad, a.st>>>(
      (const T *)a.Uin, (const T *)a.U0, (T *)a.Uout, a.nbr, ALPHA ? a.rowtab : a.rowtab_na, a.nact, a.ny,
      ALPHA ? a.nstrips : a.nstrips_na, a.ngroups,
      band_rows, nitems, (T)a.alpha, (T)a.cs, a.diag,
      std::max(Gm::ROWS_MIN, std::min(RING_Q - 1, alpha_max_ahead(a, ALPHA))),
      // (never below the progress minimum: ROWS_MIN full halo'd rows)
      Gm::R2U ? Gm::N1
              : std::max(Gm::ROWS_MIN * (Gm::W + 2 * Gm::HALO), std::min(Gm::N1, a.n1_use_na > 0 ? a.n1_use_na : Gm::N1)),
      std::max(Gm::ROWS_MIN * Gm::W, std::min(Gm::N2, a.n2_use > 0 ? a.n2_use : Gm::N2)), (const T *)a.Aabs, a.gbox, a.wr,
      ring_serial_producer<P>(), ALPHA ? a.nbi : a.nbi_na, ALPHA ? a.nbi_off : a.nbi_off_na);
  return cudaGetLastError();
}

}  // namespace dgk
