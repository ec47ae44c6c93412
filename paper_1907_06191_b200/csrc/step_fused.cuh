// step_fused.cuh -- K3: one whole SSP-RK3 step per pass (temporal blocking,
// T_b = 1), row-marching through shared memory.
//
//   U1 = u  + c L(u)                      (beta 1)
//   U2 = U1 + 3/4 (u - U1) + 1/4 c L(U1)
//   u' = U2 + 1/3 (u - U2) + 2/3 c L(U2)  (increment form, R7)
//
// HBM traffic per step: read u once (bulk TMA, strip halo of 3 columns) and
// write u' once -- 2 passes instead of the 8 of three per-stage launches.
// The work becomes FP64-bound; the price is recomputing U1 on W+4 and U2 on
// W+2 columns for W output columns (W = 8: 1.25x flops).
//
// Work item = (strip s of W output columns, source group g of 32 sources,
// band of output rows [jb0, jb1)).  Row tiles of u cover columns
// [x0-3, x0+W+3) and arrive, with their neighbour indices, in a slot ring
// (producer warp, batches of up to 32 rows, full/empty mbarriers).  U1 rows
// live in 3 and U2 rows in 4 fixed shared-memory slots.  Iteration i:
//   phase A   U1(i)            needs u(i-1..i+1)                 (ring)
//   -- named barrier (consumers) --
//   phase B   U2(i-1)          needs U1(i-2..i), u(i-1) (ring)
//             u'(i-3)          needs U2(i-4..i-2), u(i-3) and nbr (global/L2)
//   -- named barrier -- release u row i-1 (its last reader was phase B of i)
// rowtab3[s][r] = {h0, a1, a2, c0} {c1, b2, b1, h1}: active-index bounds of
// the u / U1 / U2 / output ranges of strip s, row r.
#pragma once
#include <atomic>
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "launch.h"
#include "stage_imm.cuh"

namespace dgk {

constexpr int FQ = 16;                // row entries
constexpr int FMAXBAND = 256;

template <typename T> struct FusedCfg;
template <> struct FusedCfg<double> { static constexpr int W = 8, NC = 8; };
template <> struct FusedCfg<float> { static constexpr int W = 16, NC = 8; };

template <typename T>
struct FusedGeom {
  static constexpr int P = 1, D2 = 6, NV = 1, G = 32;
  static constexpr int W = FusedCfg<T>::W, NC = FusedCfg<T>::NC;
  static constexpr int PXB = D2 * G * (int)sizeof(T);
  static constexpr int SMEM_MAX = 232448;
  static constexpr int U1B = 3 * (W + 4) * PXB, U2B = 4 * (W + 2) * PXB;
  static constexpr int EXTRA = 2 * FQ * 8 + FQ * 32 + (FMAXBAND + 8) * 32 + 2 * FQ * 4 + 64;
  static constexpr int N1 = (SMEM_MAX - U1B - U2B - EXTRA) / (PXB + 16);   // u ring slots
  static constexpr int OFF_U1 = 0, OFF_U2 = U1B, OFF_R = U1B + U2B;
  static constexpr int OFF_NB = OFF_R + N1 * PXB;
  static constexpr int OFF_BAR = OFF_NB + N1 * 16;
  static constexpr int OFF_META = OFF_BAR + 2 * FQ * 8;
  static constexpr int OFF_RT = OFF_META + FQ * 32;
  static constexpr int OFF_RV = OFF_RT + (FMAXBAND + 8) * 32;
  static constexpr int SMEM = OFF_RV + 2 * FQ * 4 + 64;
  static constexpr int THREADS = (NC + 1) * 32;
  static_assert(SMEM <= SMEM_MAX, "fused step does not fit in shared memory");
  static_assert(N1 >= 4 * (W + 6), "u ring too small for progress");
};

struct FMeta {
  int p, h0, a1, a2;   // ring slot of the tile start; range starts
  int c0, c1, b2, b1;  // output range, U2/U1 range ends
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// out = base + alpha (u0 - base) + cs * L(x) at one pixel; x/acc in registers
template <typename T>
__device__ __forceinline__ void fused_apply(T (&acc)[6][1], const T (&xs)[6][1], int4 nb,
                                            const T *pe, const T *pw, const T *pn, const T *ps) {
  mv_self<T, 1, 1>(open_code(nb), acc, xs);
  T xn[6][1];
  if (nb.x >= 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) xn[k][0] = pe[k * 32];
    mv_imm<T, 1, 1, 5>(acc, xn);
  }
  if (nb.y >= 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) xn[k][0] = pw[k * 32];
    mv_imm<T, 1, 1, 6>(acc, xn);
  }
  if (nb.z >= 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) xn[k][0] = pn[k * 32];
    mv_imm<T, 1, 1, 7>(acc, xn);
  }
  if (nb.w >= 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) xn[k][0] = ps[k * 32];
    mv_imm<T, 1, 1, 8>(acc, xn);
  }
}

template <typename T>
__global__ void __launch_bounds__(FusedGeom<T>::THREADS, 1)
    k_step_fused(const T *__restrict__ Uin, T *__restrict__ Uout, const int4 *__restrict__ nbr,
                 const int4 *__restrict__ rowtab3, int nact, int ny, int nstrips, int ngroups, int band_rows,
                 int nitems, T c1, T c2, T c3, int max_ahead) {
  using Gm = FusedGeom<T>;
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, Q = FQ, NC = Gm::NC, W = Gm::W;
  constexpr int SLOT1 = W + 4, SLOT2 = W + 2;
  extern __shared__ __align__(128) unsigned char smem[];
  T *u1s = reinterpret_cast<T *>(smem + Gm::OFF_U1);
  T *u2s = reinterpret_cast<T *>(smem + Gm::OFF_U2);
  unsigned char *ring = smem + Gm::OFF_R;
  int4 *nring = reinterpret_cast<int4 *>(smem + Gm::OFF_NB);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Gm::OFF_BAR);
  uint64_t *empty = full + Q;
  FMeta *meta = reinterpret_cast<FMeta *>(smem + Gm::OFF_META);
  int4 *rt = reinterpret_cast<int4 *>(smem + Gm::OFF_RT);                 // [rows][2]
  uint32_t *rv = reinterpret_cast<uint32_t *>(smem + Gm::OFF_RV);        // [Q] ring ends
  int *rowinfo = reinterpret_cast<int *>(smem + Gm::OFF_RV + 2 * Q * 4); // U1/U2 slot bases [3+4]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < Q; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t gstride = (size_t)nact * D2 * G;

  if (w == NC) {
    // ============================ producer warp ============================
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
        uint32_t e1 = n1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, e1, o);
          if (lane >= o) e1 += y;
        }
        const uint32_t nvalid = (uint32_t)min(32, hi - r0 + 1);
        uint32_t take;
        for (;;) {
          const uint32_t s1 = rel ? rv[(rel - 1) % Q] : 0u;
          const bool fits = valid && (L + lane - rel < (uint32_t)max_ahead) && (v1 + e1 - s1 <= (uint32_t)Gm::N1);
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
          // the previous row in this entry must have landed before re-arming
          if (Lr >= (uint32_t)Q) mbar_wait(&full[q], ((Lr - Q) / Q) & 1);
          const uint32_t b1v = v1 + e1 - n1, p1 = b1v % Gm::N1;
          FMeta m;
          m.p = (int)p1; m.h0 = ta.x; m.a1 = ta.y; m.a2 = ta.z;
          m.c0 = ta.w; m.c1 = tb.x; m.b2 = tb.y; m.b1 = tb.z;
          meta[q] = m;
          rv[q] = v1 + e1;
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
        v1 += __shfl_sync(0xffffffffu, e1, take - 1);
        L += take;
        r0 += (int)take;
        __syncwarp();
      }
    }
    return;
  }

  // ============================== consumers ==============================
  uint32_t Lbase = 0;
  const int NT = NC * 32;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int g = (item / nstrips) % ngroups;
    const int b = item / (nstrips * ngroups);
    const int jb0 = b * band_rows, jb1 = min(ny, jb0 + band_rows);
    const int lo = max(0, jb0 - 3), hi = min(ny - 1, jb1 + 2);
    const T *Ug = Uin + g * gstride + lane;   // u rows outside the ring (alpha of u')
    T *Uog = Uout + g * gstride + lane;
    auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
    auto ut = [&](const FMeta &m, int idx) -> const T * {   // u tile of a pixel in the ring
      int sl = m.p + (idx - m.h0);
      if (sl >= Gm::N1) sl -= Gm::N1;
      return reinterpret_cast<const T *>(ring + (size_t)sl * PXB) + lane;
    };
    auto unb = [&](const FMeta &m, int idx) -> int4 {
      int sl = m.p + (idx - m.h0);
      if (sl >= Gm::N1) sl -= Gm::N1;
      return nring[sl];
    };
    // U1 row r lives in slot r mod 3 (base index a1), U2 row r in slot r mod 4 (a2)
    // (slot bases come from the row's ring metadata, valid while its u row
    // or a later one is held: no shared base table, so no barrier to publish it)
    auto u1t = [&](int r, int idx) -> T * {
      const int sl = ((r % 3) + 3) % 3;
      return u1s + ((size_t)sl * SLOT1 + (idx - meta[seq(r) % Q].a1)) * D2 * G + lane;
    };
    auto u2t = [&](int r, int idx) -> T * {
      const int sl = ((r % 4) + 4) % 4;
      return u2s + ((size_t)sl * SLOT2 + (idx - meta[seq(r) % Q].a2)) * D2 * G + lane;
    };
    const int i0 = max(0, jb0 - 2), i1 = min(ny - 1, jb1 + 1);   // U1 rows
    const int iend = jb1 + 2;                                      // u'(jb1-1) is done at i = jb1+2
    const int r2lo = max(0, jb0 - 1), r2hi = min(ny - 1, jb1);     // U2 rows
    // phase-B work list of iteration i: U2 row i-1 ([a2, b2) of its u tile)
    // then output row i-3 ([c0, c1)); both bounds come from the ring metadata
    // (row i-3's entry stays valid: max_ahead <= Q-4)
    auto items = [&](int i, int &n2, int &c0, int &n3) {
      const int r2 = i - 1, r3 = i - 3;
      n2 = 0; c0 = 0; n3 = 0;
      if (r2 >= r2lo && r2 <= r2hi) { const FMeta m = meta[seq(r2) % Q]; n2 = m.b2 - m.a2; }
      if (r3 >= jb0 && r3 < jb1) { const FMeta m = meta[seq(r3) % Q]; c0 = m.c0; n3 = m.c1 - m.c0; }
    };
    // registers prefetched one iteration ahead for this warp's first output
    // pixel of the next phase B: neighbour indices and the u alpha-term
    int pf_a = -1;
    int4 pf_nb = make_int4(-1, -1, -1, -1);
    T pf_z[6];
    auto prefetch = [&](int i) {     // for phase B of iteration i (metadata of rows i-1, i-3 known)
      int n2, c0, n3;
      items(i, n2, c0, n3);
      pf_a = -1;
      if (w >= n2 && w - n2 < n3) {
        pf_a = c0 + (w - n2);
        pf_nb = __ldg(&nbr[pf_a]);
#pragma unroll
        for (int k = 0; k < 6; k++) pf_z[k] = __ldg(Ug + ((size_t)pf_a * D2 + k) * G);
      }
    };
    // one code path for all three kinds of work (U1, U2, u'): per item the
    // pixel's five operand tiles, neighbour indices, alpha term and
    // destination are set up, then a single operator body runs (one copy of
    // the 16-way self-block switch in the instruction stream)
    int cur_a = -1;
    int4 cur_nb = make_int4(-1, -1, -1, -1);
    T cur_z[6];
    for (int i = i0; i <= iend; i++) {
      int n2 = 0, c0 = 0, n3 = 0;
      FMeta m = meta[seq(max(lo, min(hi, i))) % Q], mn = m, ms = m, m2 = m;
#pragma unroll 1
      for (int phase = 0; phase < 2; phase++) {
        int nitem = 0;
        if (phase == 0) {
          // ---- phase A: U1(i) over [a1, b1)
          if (i <= i1) {
            for (int r = max(lo, i - 1); r <= min(hi, i + 1); r++) {
              const uint32_t L = seq(r);
              mbar_wait(&full[L % Q], (L / Q) & 1);
            }
            m = meta[seq(i) % Q];
            mn = (i + 1 <= hi) ? meta[seq(i + 1) % Q] : m;
            ms = (i - 1 >= lo) ? meta[seq(i - 1) % Q] : m;
            nitem = m.b1 - m.a1;
          }
          if (i == i0) prefetch(i);
        } else {
          // ---- phase B: U2(i-1) over [a2, b2), then u'(i-3) over [c0, c1)
          items(i, n2, c0, n3);
          m2 = meta[seq(max(lo, min(hi, i - 1))) % Q];
          cur_a = pf_a;
          cur_nb = pf_nb;
#pragma unroll
          for (int k = 0; k < 6; k++) cur_z[k] = pf_z[k];
          if (i + 1 <= iend) prefetch(i + 1);
          nitem = n2 + n3;
        }
        // (no barrier here: the slot a phase writes was last read before the
        // barrier that ended the previous phase)
        for (int it = w; it < nitem; it += NC) {
          const T *ps, *pe, *pw, *pn, *pq, *zs = nullptr;
          T *out;
          int4 nb;
          T z[6], alpha, cc;
          bool zreg = false;
          if (phase == 0) {                         // U1(i) = u + c1 L(u)
            const int a = m.a1 + it;
            nb = unb(m, a);
            ps = ut(m, a);
            pe = nb.x >= 0 ? ut(m, nb.x) : ps;
            pw = nb.y >= 0 ? ut(m, nb.y) : ps;
            pn = nb.z >= 0 ? ut(mn, nb.z) : ps;
            pq = nb.w >= 0 ? ut(ms, nb.w) : ps;
            alpha = (T)0;
            cc = c1;
            out = u1t(i, a);
          } else if (it < n2) {                     // U2(r2) = U1 + 3/4 (u - U1) + c2 L(U1)
            const int r2 = i - 1, a = m2.a2 + it;
            nb = unb(m2, a);
            ps = u1t(r2, a);
            pe = nb.x >= 0 ? u1t(r2, nb.x) : ps;
            pw = nb.y >= 0 ? u1t(r2, nb.y) : ps;
            pn = nb.z >= 0 ? u1t(r2 + 1, nb.z) : ps;
            pq = nb.w >= 0 ? u1t(r2 - 1, nb.w) : ps;
            zs = ut(m2, a);
            alpha = (T)0.75;
            cc = c2;
            out = u2t(r2, a);
          } else {                                  // u'(r3) = U2 + 1/3 (u - U2) + c3 L(U2)
            const int r3 = i - 3, a = c0 + (it - n2);
            if (it == w && a == cur_a) {            // first item of this warp: prefetched
              nb = cur_nb;
#pragma unroll
              for (int k = 0; k < 6; k++) z[k] = cur_z[k];
            } else {
              nb = __ldg(&nbr[a]);
#pragma unroll
              for (int k = 0; k < 6; k++) z[k] = __ldg(Ug + ((size_t)a * D2 + k) * G);
            }
            zreg = true;
            ps = u2t(r3, a);
            pe = nb.x >= 0 ? u2t(r3, nb.x) : ps;
            pw = nb.y >= 0 ? u2t(r3, nb.y) : ps;
            pn = nb.z >= 0 ? u2t(r3 + 1, nb.z) : ps;
            pq = nb.w >= 0 ? u2t(r3 - 1, nb.w) : ps;
            alpha = (T)(1.0 / 3.0);
            cc = c3;
            out = Uog + (size_t)a * D2 * G;
          }
          T xs[6][1], acc[6][1];
#pragma unroll
          for (int k = 0; k < 6; k++) { xs[k][0] = ps[k * G]; acc[k][0] = (T)0; }
          fused_apply<T>(acc, xs, nb, pe, pw, pn, pq);
#pragma unroll
          for (int k = 0; k < 6; k++) {
            const T zk = zreg ? z[k] : (zs ? zs[k * G] : xs[k][0]);
            out[k * G] = xs[k][0] + alpha * (zk - xs[k][0]) + cc * acc[k][0];
          }
        }
        if (phase == 0) named_bar(1, NT);
      }
      named_bar(1, NT);
      // u row i-1 had its last reader (phase B above): release it
      if (tid == 0 && i - 1 >= lo && i - 1 <= hi) mbar_arrive(&empty[seq(i - 1) % Q]);
    }
    // release the u rows the loop did not release (it released i0-1 .. iend-1)
    if (tid == 0) {
      for (int r = lo; r <= hi; r++) {
        const bool released = (r >= i0 - 1 && r <= iend - 1);
        if (!released) {
          const uint32_t L = seq(r);
          mbar_wait(&full[L % Q], (L / Q) & 1);
          mbar_arrive(&empty[L % Q]);
        }
      }
    }
    named_bar(1, NT);
    Lbase += (uint32_t)(hi - lo + 1);
  }
}

template <typename T>
cudaError_t launch_fused(const dgl::StageArgs &a) {
  using Gm = FusedGeom<T>;
  static std::atomic<uint64_t> attr_set{0};   // per-device opt-in, one bit per ordinal
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!(attr_set.load() >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_step_fused<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(uint64_t(1) << dev);
  }
  const int per_band = a.nstrips * a.ngroups;
  int nbands = std::max(1, std::min(a.ny, (8 * a.nsm + per_band - 1) / per_band));
  int band_rows = (a.ny + nbands - 1) / nbands;
  if (band_rows > FMAXBAND) band_rows = FMAXBAND;
  nbands = (a.ny + band_rows - 1) / band_rows;
  const int nitems = per_band * nbands;
  const int grid = std::min(nitems, a.nsm);
  k_step_fused<T><<<grid, Gm::THREADS, Gm::SMEM, a.st>>>(
      (const T *)a.Uin, (T *)a.Uout, a.nbr, a.rowtab, a.nact, a.ny, a.nstrips, a.ngroups, band_rows, nitems,
      (T)a.cs, (T)(0.25 * a.cs), (T)((2.0 / 3.0) * a.cs),
      std::max(6, std::min(FQ - 4, a.ahead_alpha > 0 ? a.ahead_alpha : FQ - 4)));
  return cudaGetLastError();
}

}  // namespace dgk
