// EXPERIMENT, NOT BUILT (round 2): kept for the record of profiles/r02_k3d_sweeps.txt
// ("K3e").  It was wired as temporal_steps = 6 with StageArgs::split_pairs and a
// pair_pixel<..., REMOTE = true> variant whose output used st.shared::cluster;
// bitwise equal to K2, 1.6x slower than K3d on c4 fp64, so it was removed from
// the library.
// stage_pair_split.cuh -- K3e: SSP-RK3 stages 2 + 3 of one step with the two
// roles of K3d on the two CTAs of a 2-CTA cluster (temporal_steps = 6).
//
//   CTA 0 ("B")  U2 = U1 + 3/4 (u - U1) + c2 L(U1): a producer warp brings
//                the U1 row tiles into a ~220 KB shared-memory ring (one 1-D
//                bulk copy per row); 10 compute warps write each U2 pixel
//                tile straight into the C CTA's shared memory (DSMEM stores)
//   CTA 1 ("C")  u' = U2 + 1/3 (u - U2) + c3 L(U2): 11 compute warps read U2
//                from the ~220 KB ring B fills; a meta warp prepares the row
//                descriptors and the item's neighbour table; u' to HBM
//
// Compared with K3d (both roles in one SM, 3 KB pixel tiles in 227 KB of
// shared memory) each role gets a whole SM: twice the ring depth for the U1
// pipeline and for U2, and twice the issue slots per pixel.  The hand-off is
// K3d's, across the cluster: B warps arrive on C's per-row barriers
// (mbarrier.arrive.release.cluster on a shared::cluster address), C warps
// publish their ring frontier (read by B with ld.acquire.cluster) and arrive
// on B's entry-reuse barriers.  No global memory and no gpu-scope fence is
// involved (a first version passed U2 through an L2 ring with gpu-scope
// release / acquire counters: the fences cost ~2 us each and made it 6x
// slower than K3d).  Per pixel the arithmetic is K2's (pair_pixel), so the
// result is bitwise K2's.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include "kernels.cuh"
#include "stage_imm.cuh"
#include "stage_pair.cuh"
#include "launch.h"

namespace dgk {

constexpr int SPL_Q = 32;        // row entries per CTA
constexpr int SPL_NB = 10;       // B compute warps
constexpr int SPL_NC = 10;       // C compute warps

template <typename T, int NV, int P>
struct SplitGeom {
  static constexpr int G = 32 * NV;
  static constexpr int D2 = ndof_px<P>();
  static constexpr int PXB = D2 * G * (int)sizeof(T);
  static constexpr int W = PAIR_W;
  static constexpr int THREADS = 12 * 32;   // B: 10 + producer + forwarder, C: 10 + meta + forwarder
  static constexpr int SMEM_MAX = 232448;
  static constexpr int OFF_NBUF = 0;                                        // [2][PAIR_NBUF] uint16
  static constexpr int OFF_BAR = OFF_NBUF + 2 * PAIR_NBUF * 2;             // [4][Q] + [4] barriers
  static constexpr int OFF_META = OFF_BAR + (4 * SPL_Q + 4) * 8;
  static constexpr int OFF_RT = OFF_META + SPL_Q * (int)sizeof(PairMeta);
  static constexpr int OFF_RV = OFF_RT + (PAIR_MAXBAND + 4) * 2 * 16;      // [2][Q] B: ring-1 / C-ring ends
  static constexpr int OFF_TILES = (OFF_RV + 2 * SPL_Q * 4 + 127) / 128 * 128;
  static constexpr int NT = (SMEM_MAX - OFF_TILES) / PXB;                  // B: U1 tiles; C: U2 tiles
  static constexpr int SMEM = OFF_TILES + NT * PXB;
  static_assert(NT >= 4 * (W + 4), "split pair: ring too small for progress");
  static_assert(SPL_NB + 2 <= THREADS / 32 && SPL_NC + 2 <= THREADS / 32, "split pair: warps");
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_cl(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t remote) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl_relaxed(uint32_t remote) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ bool mbar_try_cl(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
// watchdog of the split kernel's waits: tuning builds name the wait that
// timed out (tag, row) before the trap
__device__ __noinline__ void spl_stuck(int tag, uint32_t row) {
#ifdef DGDIFF_TUNING
  printf("K3e stuck: block %d warp %d tag %d row %u\n", (int)blockIdx.x, (int)(threadIdx.x >> 5), tag, row);
#endif
  __trap();
}
// wait for a phase completed by arrivals from the other CTA (cluster acquire)
__device__ __forceinline__ void mbar_wait_cl(uint64_t *bar, uint32_t parity, int tag = 0, uint32_t row = 0) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_cl(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_cl(a, parity)) {
    if (clock64() - t0 > (1LL << 32)) spl_stuck(tag, row);
  }
}
__device__ __forceinline__ void mbar_wait_t(uint64_t *bar, uint32_t parity, int tag, uint32_t row) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(a, parity)) {
    if (clock64() - t0 > (1LL << 32)) spl_stuck(tag, row);
  }
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#ifdef DGDIFF_TUNING
// tuning builds: cycles spent in each wait, per warp kind (0 B compute, 1 B
// producer, 2 C meta, 3 C compute) x (3 wait slots + total)
__device__ unsigned long long g_split_dbg[4][4];
#define SPL_TW(slot, ...)                 \
  do {                                    \
    const long long _t = clock64();       \
    __VA_ARGS__;                          \
    tacc[slot] += clock64() - _t;         \
  } while (0)
#else
#define SPL_TW(slot, ...) __VA_ARGS__
#endif

template <typename T, int NV, int P>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SplitGeom<T, NV, P>::THREADS, 1)
    k_stage_pair_split(const T *__restrict__ U1, const T *__restrict__ U0, T *__restrict__ Uout,
                       const uint16_t *__restrict__ nbs, const int4 *__restrict__ rowtab, int nact, int ny,
                       int nstrips, int ngroups, int band_rows, int nitems, T a2, T c2, T a3, T c3,
                       int relax /* tuning diagnostic: 2 = B's forwarded arrivals relaxed */) {
  using Gm = SplitGeom<T, NV, P>;
  static_assert(!is_quad<P>(), "split pair: triangles");
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, Q = SPL_Q, NT = Gm::NT;
  constexpr int NB = SPL_NB, NC = SPL_NC;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *ring = smem + Gm::OFF_TILES;
  uint16_t *nbuf = reinterpret_cast<uint16_t *>(smem + Gm::OFF_NBUF);
  // B: full = U1 row landed, empty = B warps done with the U1 row, full3 =
  //    B warps wrote the row's U2 tiles (into C), cfree = C done with the
  //    row (one arrival from C's forwarder)
  // C: full = row descriptor ready, empty = C warps done with the row,
  //    full3 = the row's U2 tiles are in (one arrival from B's forwarder)
  // The compute warps only touch barriers of their own CTA; one forwarder
  // warp per CTA turns each completed local phase into one remote arrival
  // (mbarrier.arrive.release.cluster), in row order.
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Gm::OFF_BAR);
  uint64_t *empty = full + Q, *full3 = empty + Q, *cfree = full3 + Q, *nbf = cfree + Q, *nbe = nbf + 2;
  PairMeta *meta = reinterpret_cast<PairMeta *>(smem + Gm::OFF_META);
  int4 *rt = reinterpret_cast<int4 *>(smem + Gm::OFF_RT);
  uint32_t *rv = reinterpret_cast<uint32_t *>(smem + Gm::OFF_RV);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t role = cluster_ctarank();                          // 0 = B, 1 = C
  const int pair = (int)(blockIdx.x >> 1), npairs = (int)(gridDim.x >> 1);
  const uint32_t rbase = smem_u32(ring), lane_b = (uint32_t)(lane * NV * sizeof(T));
  const int ncomp = role == 0 ? NB : NC;
  if (tid == 0) {
    for (int q = 0; q < Q; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], ncomp);
      mbar_init(&full3[q], role == 0 ? NB : 1);
      mbar_init(&cfree[q], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&nbf[b], 1);
      mbar_init(&nbe[b], ncomp);
    }
    fence_mbar_init();
  }
  cluster_sync_all();   // both CTAs' barriers exist before any remote arrival
  const size_t gstride = (size_t)nact * D2 * G;
#ifdef DGDIFF_TUNING
  unsigned long long tacc[3] = {0, 0, 0};
  const long long tstart = clock64();
  auto flush = [&](int kind) {
    if (lane == 0) {
      for (int k = 0; k < 3; k++) atomicAdd(&g_split_dbg[kind][k], tacc[k]);
      atomicAdd(&g_split_dbg[kind][3], (unsigned long long)(clock64() - tstart));
    }
  };
#else
  auto flush = [](int) {};
#endif
  auto decode = [&](int item, int &s, int &g, int &jb0, int &jb1) {
    s = item % nstrips;
    g = (item / nstrips) % ngroups;
    jb0 = (item / (nstrips * ngroups)) * band_rows;
    jb1 = min(ny, jb0 + band_rows);
  };
  auto load_rt = [&](int s, int lo, int hi) {
    __syncwarp();
    for (int r = lo + lane; r <= hi; r += 32) {
      rt[2 * (r - lo)] = __ldg(&rowtab[2 * ((size_t)s * ny + r)]);
      rt[2 * (r - lo) + 1] = __ldg(&rowtab[2 * ((size_t)s * ny + r) + 1]);
    }
    __syncwarp();
  };
  // the item's neighbour table (one bulk copy into item buffer ib), lane 0
  auto copy_nb = [&](int lo, int u2lo, int u2hi, int ib) -> int {
    const int nb_first = rt[2 * (u2lo - lo) + 1].z;
    const int nb_last = rt[2 * (u2hi - lo) + 1].z + (rt[2 * (u2hi - lo)].z - rt[2 * (u2hi - lo)].y);
    const int nb_base = nb_first & ~7;
    const uint32_t nb_bytes = (uint32_t)(((nb_last + 7) & ~7) - nb_base) * 2u;
    mbar_expect_tx(&nbf[ib], nb_bytes);
    if (nb_bytes) bulk_g2s(nbuf + ib * PAIR_NBUF, nbs + nb_base, nb_bytes, &nbf[ib]);
    return nb_base;
  };

  [&] {
    if (role == 0) {
      // =============================== B CTA ==============================
      if (w == NB) {
        // ----- producer: U1 row tiles, one bulk copy per row, one lane -----
        uint32_t L = 0, v1 = 0, v3 = 0, relB = 0, relC = 0, it = 0;
        for (int item = pair; item < nitems; item += npairs, it++) {
          int s, g, jb0, jb1;
          decode(item, s, g, jb0, jb1);
          const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
          const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
          const int ib = (int)(it & 1);
          if (lane == 0 && it >= 2) SPL_TW(2, mbar_wait_t(&nbe[ib], ((it / 2) - 1) & 1, 1, it));
          load_rt(s, lo, hi);
          if (lane == 0) {
            const int nb_base = copy_nb(lo, u2lo, u2hi, ib);
            const T *Ug = U1 + g * gstride;
            for (int r = lo; r <= hi; r++) {
              const int4 t = rt[2 * (r - lo)], t2 = rt[2 * (r - lo) + 1];
              const bool comp = r >= u2lo && r <= u2hi;
              const uint32_t n1 = (uint32_t)(t.w - t.x), n3 = comp ? (uint32_t)(t.z - t.y) : 0u;
              // entry reuse + ring-1 room (B warps released U1 rows)
              for (;;) {
                const uint32_t s1 = relB ? rv[(relB - 1) % Q] : 0u;
                if (L - relB < (uint32_t)(Q - 1) && v1 + n1 - s1 <= (uint32_t)NT) break;
                SPL_TW(0, mbar_wait_t(&empty[relB % Q], (relB / Q) & 1, 2, relB));
                relB++;
              }
              // C's entry of the same row index is free (its full3 phase done)
              // and C's ring has room for the row's U2 tiles (C released
              // rows up to relC-1: its ring is free up to their end)
              for (;;) {
                if (L - relC < (uint32_t)(Q - 1) && v3 + n3 - (relC ? rv[Q + (relC - 1) % Q] : 0u) <= (uint32_t)NT)
                  break;
                SPL_TW(1, mbar_wait_cl(&cfree[relC % Q], (relC / Q) & 1, 3, relC));
                relC++;
              }
              const uint32_t q = L % Q, p1 = v1 % NT;
              PairMeta m;
              m.p1 = (int)p1; m.h0 = t.x; m.c0 = t.y; m.c1 = comp ? t.z : t.y;
              m.o0 = t2.x; m.o1 = t2.y; m.nbo = t2.z - nb_base; m.v3 = v3;
              meta[q] = m;
              v1 += n1;
              v3 += n3;
              rv[q] = v1;
              rv[Q + q] = v3;
              mbar_expect_tx(&full[q], n1 * PXB);
              if (n1) {
                const uint32_t a1 = min(n1, (uint32_t)NT - p1);
                const T *src = Ug + (size_t)t.x * D2 * G;
                bulk_g2s(ring + (size_t)p1 * PXB, src, a1 * PXB, &full[q]);
                if (n1 > a1) bulk_g2s(ring, src + (size_t)a1 * D2 * G, (n1 - a1) * PXB, &full[q]);
              }
              L++;
            }
          }
          __syncwarp();
        }
        flush(1);
        return;
      }
      if (w == NB + 1) {
        // ----- forwarder: row L's U2 tiles are all in C -> C's full3 -----
        const uint32_t c_full3 = mapa_cl(smem_u32(full3), 1u);
        uint32_t L = 0;
        for (int item = pair; item < nitems; item += npairs) {
          int s, g, jb0, jb1;
          decode(item, s, g, jb0, jb1);
          const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
          for (int r = lo; r <= hi; r++, L++) {
            SPL_TW(0, mbar_wait_t(&full3[L % Q], (L / Q) & 1, 13, L));
            if (lane == 0) {
              if (relax & 2) mbar_arrive_cl_relaxed(c_full3 + 8u * (L % Q));
              else mbar_arrive_cl(c_full3 + 8u * (L % Q));
            }
            __syncwarp();
          }
        }
        flush(2);
        return;
      }
      if (w > NB + 1) return;
      // ----- B compute warps (K3d's B loop; U2 into C's ring over DSMEM) -----
      const uint32_t c_ring = mapa_cl(rbase, 1u) + lane_b;
      uint32_t Lbase = 0, it = 0;
      for (int item = pair; item < nitems; item += npairs, it++) {
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
            SPL_TW(0, mbar_wait_t(&full[L % Q], (L / Q) & 1, 4, L));
          }
        };
        auto tile1 = [&](const PairMeta &m, int pos) -> uint32_t {
          int sl = m.p1 + pos;
          if (sl >= NT) sl -= NT;
          return rbase + (uint32_t)sl * PXB + lane_b;
        };
        auto arrive3 = [&](int r) { mbar_arrive(&full3[seq(r) % Q]); };   // local; forwarded to C
        SPL_TW(2, mbar_wait_t(&nbf[it & 1], (it / 2) & 1, 5, it));
        int j = u2lo, rel_next = lo, cum = 0;
        for (int r = u2lo - 1; r <= u2lo + 1; r++) wait_row(r);
        __syncwarp();
        if (lane == 0)
          for (int r = lo; r < u2lo; r++) arrive3(r);   // halo row above: no U2
        PairMeta mc = meta[seq(j) % Q];
        PairMeta mN = j + 1 <= hi ? meta[seq(j + 1) % Q] : mc, mS = j - 1 >= lo ? meta[seq(j - 1) % Q] : mc;
        for (int f = w;; f += NB) {
          while (f >= cum + (mc.c1 - mc.c0)) {
            cum += mc.c1 - mc.c0;
            __syncwarp();
            if (lane == 0) arrive3(j);                    // this warp's U2 tiles of row j are in C
            if (++j > u2hi) break;
            if (rel_next <= j - 2) {
              if (lane == 0)
                for (int r = rel_next; r <= j - 2; r++) mbar_arrive(&empty[seq(r) % Q]);
              rel_next = j - 1;
            }
            wait_row(j + 1);
            mS = mc;
            mc = mN;
            mN = j + 1 <= hi ? meta[seq(j + 1) % Q] : mc;
          }
          if (j > u2hi) break;
          const int k = f - cum;
          const int a = mc.c0 + k;
          const int nbw = nbi[mc.nbo + k];
          const int code = nbw & 15, pos = a - mc.h0;
          const uint32_t xs_a = tile1(mc, pos);
          const uint32_t sl3 = (mc.v3 + (uint32_t)k) % (uint32_t)NT;
          SPL_TW(1, pair_pixel<T, NV, P, true>(xs_a, tile1(mc, pos + 1), tile1(mc, pos - 1 < 0 ? 0 : pos - 1),
                                               (code & 4) ? tile1(mN, (nbw >> 4) & 15) : xs_a,
                                               (code & 8) ? tile1(mS, (nbw >> 8) & 15) : xs_a, code,
                                               U0l + (size_t)a * D2 * G, nullptr, c_ring + sl3 * PXB, a2, c2,
                                               nullptr));
        }
        __syncwarp();
        if (lane == 0) {
          for (int r = u2hi + 1; r <= hi; r++) arrive3(r);   // halo row below: no U2
          for (int r = rel_next; r <= hi; r++) mbar_arrive(&empty[seq(r) % Q]);
          mbar_arrive(&nbe[it & 1]);
        }
        Lbase += (uint32_t)(hi - lo + 1);
      }
      flush(0);
      return;
    }

    // ================================= C CTA ================================
    if (w == NC) {
      // ----- meta warp: row descriptors (C ring slots as B computes them) -----
      uint32_t L = 0, v3 = 0, it = 0;
      for (int item = pair; item < nitems; item += npairs, it++) {
        int s, g, jb0, jb1;
        decode(item, s, g, jb0, jb1);
        const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
        const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
        const int ib = (int)(it & 1);
        if (lane == 0 && it >= 2) SPL_TW(2, mbar_wait_t(&nbe[ib], ((it / 2) - 1) & 1, 7, it));
        load_rt(s, lo, hi);
        if (lane == 0) {
          const int nb_base = copy_nb(lo, u2lo, u2hi, ib);
          for (int r = lo; r <= hi; r++, L++) {
            const int4 t = rt[2 * (r - lo)], t2 = rt[2 * (r - lo) + 1];
            const bool comp = r >= u2lo && r <= u2hi;
            const uint32_t q = L % Q;
            if (L >= (uint32_t)Q) SPL_TW(0, mbar_wait_t(&empty[q], ((L / Q) - 1) & 1, 8, L));   // C warps left row L-Q
            PairMeta m;
            m.p1 = 0; m.h0 = t.x; m.c0 = t.y; m.c1 = comp ? t.z : t.y;
            m.o0 = t2.x; m.o1 = t2.y; m.nbo = t2.z - nb_base; m.v3 = v3;
            meta[q] = m;
            v3 += comp ? (uint32_t)(t.z - t.y) : 0u;
            mbar_arrive(&full[q]);
          }
        }
        __syncwarp();
      }
      flush(2);
      return;
    }
    if (w == NC + 1) {
      // ----- forwarder: every C warp is done with row L -> B's cfree -----
      const uint32_t b_cfree = mapa_cl(smem_u32(cfree), 0u);
      uint32_t L = 0;
      for (int item = pair; item < nitems; item += npairs) {
        int s, g, jb0, jb1;
        decode(item, s, g, jb0, jb1);
        const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
        for (int r = lo; r <= hi; r++, L++) {
          SPL_TW(1, mbar_wait_t(&empty[L % Q], (L / Q) & 1, 14, L));
          if (lane == 0) mbar_arrive_cl(b_cfree + 8u * (L % Q));
          __syncwarp();
        }
      }
      return;
    }
    if (w > NC + 1) return;
    // ----- C compute warps: u' from the U2 ring (K3d's C loop) -----
    uint32_t Lbase = 0, it = 0;
    for (int item = pair; item < nitems; item += npairs, it++) {
      int s_, g, jb0, jb1;
      decode(item, s_, g, jb0, jb1);
      const int lo = max(0, jb0 - 2), hi = min(ny - 1, jb1 + 1);
      const int u2lo = max(0, jb0 - 1), u2hi = min(ny - 1, jb1);
      const T *U0l = U0 + g * gstride + lane * NV;
      T *Uog = Uout + g * gstride + lane * NV;
      const uint16_t *nbi = nbuf + (it & 1) * PAIR_NBUF;
      auto seq = [&](int r) { return Lbase + (uint32_t)(r - lo); };
      auto wait_meta = [&](int r) {
        const uint32_t L = seq(r);
        SPL_TW(2, mbar_wait_t(&full[L % Q], (L / Q) & 1, 9, L));
      };
      auto wait3 = [&](int r) {
        if (r >= u2lo && r <= u2hi) {
          const uint32_t L = seq(r);
          SPL_TW(0, mbar_wait_cl(&full3[L % Q], (L / Q) & 1, 10, L));
        }
      };
      auto tile3 = [&](const PairMeta &m, int pos) -> uint32_t {
        const uint32_t sl = (m.v3 + (uint32_t)(pos - (m.c0 - m.h0))) % (uint32_t)NT;
        return rbase + sl * PXB + lane_b;
      };
      auto release3 = [&](int r) {   // lane 0: this warp is done with row r
        const uint32_t L = seq(r);
        wait_meta(r);
        mbar_wait_cl(&full3[L % Q], (L / Q) & 1, 11, L);   // the row's full3 phase is complete (halo rows too)
        mbar_arrive(&empty[L % Q]);
      };
      SPL_TW(2, mbar_wait_t(&nbf[it & 1], (it / 2) & 1, 12, it));
      int j = jb0, rel_next = lo, cum = 0;
      for (int r = jb0 - 1; r <= jb0 + 1; r++) {
        if (r >= lo && r <= hi) wait_meta(r);
        wait3(r);
      }
      PairMeta mc = meta[seq(j) % Q];
      PairMeta mN = meta[seq(j + 1) % Q], mS = meta[seq(j - 1 >= lo ? j - 1 : j) % Q];
      for (int f = w;; f += NC) {
        while (f >= cum + (mc.o1 - mc.o0)) {
          cum += mc.o1 - mc.o0;
          if (++j >= jb1) break;
          if (rel_next <= j - 2) {
            __syncwarp();
            if (lane == 0)
              for (int r = rel_next; r <= j - 2; r++) release3(r);
            rel_next = j - 1;
          }
          if (j + 1 <= hi) wait_meta(j + 1);   // (j + 1 == ny: no row, no N face)
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
        SPL_TW(1, pair_pixel<T, NV, P>(xs_a, tile3(mc, pos + 1), tile3(mc, pos - 1),
                                       (code & 4) ? tile3(mN, (nbw >> 4) & 15) : xs_a,
                                       (code & 8) ? tile3(mS, (nbw >> 8) & 15) : xs_a, code,
                                       U0l + (size_t)a * D2 * G, Uog + (size_t)a * D2 * G, 0u, a3, c3, nullptr));
      }
      __syncwarp();
      if (lane == 0) {
        for (int r = rel_next; r <= hi; r++) release3(r);
        mbar_arrive(&nbe[it & 1]);
      }
      Lbase += (uint32_t)(hi - lo + 1);
    }
    flush(3);
  }();
  __syncwarp();
  cluster_sync_all();   // no CTA leaves while the other may still touch its shared memory
}

// one step's stages 2 + 3 on clusters of two CTAs; a.Uin = U1, a.U0 = u,
// a.Uout = u' (not u), a.rowtab / a.nbs as K3d, a.split_pairs = clusters
template <typename T, int NV, int P>
cudaError_t launch_pair_split(const dgl::StageArgs &a) {
  using Gm = SplitGeom<T, NV, P>;
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!(attr_set.load() >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_stage_pair_split<T, NV, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Gm::SMEM);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(uint64_t(1) << dev);
  }
  const int per_band = a.nstrips * a.ngroups;
  int nbands = std::max(1, std::min(a.ny, (4 * a.nsm + per_band - 1) / per_band));
  int band_rows = (a.ny + nbands - 1) / nbands;
  if (band_rows > PAIR_MAXBAND) band_rows = PAIR_MAXBAND;
  nbands = (a.ny + band_rows - 1) / band_rows;
  const int nitems = per_band * nbands;
  const int npairs = std::max(1, std::min(nitems, a.split_pairs));
  const double c = a.cs;
  int relax = 0;
#ifdef DGDIFF_TUNING
  if (const char *e = tune_env("DGDIFF_SPLIT_RELAX")) relax = atoi(e);
  const bool dbg = tune_env("DGDIFF_SPLIT_DBG") != nullptr;
  if (dbg) {
    unsigned long long z[4][4] = {};
    cudaMemcpyToSymbolAsync(g_split_dbg, z, sizeof(z), 0, cudaMemcpyHostToDevice, a.st);
  }
#endif
  k_stage_pair_split<T, NV, P><<<2 * npairs, Gm::THREADS, Gm::SMEM, a.st>>>(
      (const T *)a.Uin, (const T *)a.U0, (T *)a.Uout, a.nbs, a.rowtab, a.nact, a.ny, a.nstrips, a.ngroups, band_rows,
      nitems, (T)0.75, (T)(0.25 * c), (T)(1.0 / 3.0), (T)((2.0 / 3.0) * c), relax);
#ifdef DGDIFF_TUNING
  if (dbg) {
    unsigned long long z[4][4];
    cudaMemcpyFromSymbolAsync(z, g_split_dbg, sizeof(z), 0, cudaMemcpyDeviceToHost, a.st);
    cudaStreamSynchronize(a.st);
    const double nw[4] = {(double)SPL_NB, 1, 2, (double)SPL_NC};
    const char *nm[4] = {"Bcomp", "Bprod", "Bfwd|Cmeta", "Ccomp"};
    fprintf(stderr, "K3e dbg (Mcycles per warp; slots 0-2 / total):");
    for (int k = 0; k < 4; k++) {
      fprintf(stderr, " %s", nm[k]);
      for (int i = 0; i < 4; i++) fprintf(stderr, " %.2f", z[k][i] / nw[k] / npairs / 1e6);
      fprintf(stderr, ";");
    }
    fprintf(stderr, " pairs %d items %d\n", npairs, nitems);
  }
#endif
  return cudaGetLastError();
}
// clusters of the kernel that fit on the device at once (the launch's pair count)
template <typename T, int NV, int P>
int pair_split_clusters() {
  using Gm = SplitGeom<T, NV, P>;
  if (cudaFuncSetAttribute(k_stage_pair_split<T, NV, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM) !=
      cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2, 1, 1);
  cfg.blockDim = dim3(Gm::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Gm::SMEM;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_stage_pair_split<T, NV, P>, &cfg) != cudaSuccess) return 0;
  return n;
}

}  // namespace dgk
