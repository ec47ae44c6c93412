// stage_wave.cuh -- K3c: one whole SSP-RK3 step per launch as an L2-resident
// WAVEFRONT of K2 items (temporal_steps = 4; P1/P2 triangles, REFLECT).
//
// The ring kernel's work item (strip s of W columns, group g, band b of rows)
// gets a stage k in {0, 1, 2}; items are numbered in the order
//     for g: for wavefront w: for k: (b = w - k valid): for s
// and item (k, g, b, s) may start once the items (k-1, g, b-1..b+1, s-1..s+1)
// that write its input rows (band and strip halo of one pixel) are complete
// (per-item completion counters in global memory, release / acquire).
// Every dependency has a smaller number, and a CTA takes its items in
// increasing order, so the smallest unfinished item can always run.
//
// Stage k of band b sits in wavefront b + 2k, so an item's inputs were all
// written in earlier wavefronts.  Stage k runs 2k bands behind stage 0: the U1 / U2 rows a
// stage reads were written a few hundred items earlier and are still in L2,
// and so are the u rows of the alpha terms: HBM sees u read once, u written
// once, U1 and U2 written once (their dirty lines are evicted) -- 4 state
// passes per step instead of K2's 8, with no halo recompute (the arithmetic
// per pixel is K2's, so the result is bitwise K2's).
//
// In-place stage 3 (u' into u) is safe: the readers of u(band b) in this step
// are stage 0 of bands b-1..b+1 and stage 1 of band b, all transitive
// dependencies of stage 2 of band b.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include "kernels.cuh"
#include "stage_imm.cuh"
#include "stage_ring.cuh"
#include "launch.h"

namespace dgk {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr int WAVE_WQ = 8;   // item completion slots per CTA
#ifndef DGDIFF_WAVE_NC
#define DGDIFF_WAVE_NC 8     // consumer warps (the ring kernel's NC for P1 fp64)
#endif
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// item number -> (stage k, group g, band b, strip s).  Groups are taken in
// blocks of gblk: for block: for wavefront w: for k (b = w - k valid): for g
// in block: for s.  wtab[i] = {k, b} of the i-th (stage, band) pair.
__device__ __forceinline__ void wave_item(int item, int nstrips, int ngroups, int gblk, int nkb,
                                          const int2 *__restrict__ wtab, int &k, int &g, int &b, int &s) {
  const int full = nkb * gblk * nstrips;
  const int blk = item / full;
  const int rem = item - blk * full;
  const int gb = min(gblk, ngroups - blk * gblk);
  const int i = rem / (gb * nstrips);
  const int r2 = rem - i * gb * nstrips;
  g = blk * gblk + r2 / nstrips;
  s = r2 - (r2 / nstrips) * nstrips;
  const int2 kb = __ldg(&wtab[i]);
  k = kb.x;
  b = kb.y;
}

template <typename T, int NV, int P>
__global__ void __launch_bounds__((DGDIFF_WAVE_NC + 2) * 32, 1)
    k_step_wave(T *u, T *U1, T *U2, const int4 *__restrict__ nbr, const int4 *__restrict__ rowtab, int nact, int ny,
                int nstrips, int sblk, int ngroups, int gblk, int band_rows, int nbands, const int2 *__restrict__ wtab, int nitems,
                T c1, T c2, T c3, T a2, T a3, unsigned *cnt, unsigned epoch, int max_ahead, int n1_use,
                int n2_use, int diag) {
  using Gm = RingGeom<T, NV, P, true>;
  static_assert(!is_quad<P>() && P <= 2, "wavefront step: P1 / P2 triangles");
  static_assert(Gm::SMEM + 2 * WAVE_WQ * 8 <= Gm::SMEM_MAX, "no room for the completion slots");
  constexpr int G = Gm::G, D2 = Gm::D2, PXB = Gm::PXB, Q = RING_Q, NC = DGDIFF_WAVE_NC;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char *ring1 = smem;
  int4 *nbr_ring = reinterpret_cast<int4 *>(smem + Gm::OFF_NB);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Gm::OFF_BAR);
  uint64_t *empty = full + Q;
  RowMeta *meta = reinterpret_cast<RowMeta *>(smem + Gm::OFF_META);
  int4 *rt = reinterpret_cast<int4 *>(smem + Gm::OFF_RT);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // item completion inside the CTA: consumers arrive on done[i % WQ] (count
  // NC) after their stores; the publisher warp turns that into one gpu-scope
  // release per item and frees the slot through pubd[i % WQ]
  __shared__ uint64_t done[WAVE_WQ], pubd[WAVE_WQ];
  if (tid == 0) {
    for (int q = 0; q < Q; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NC);
    }
    for (int q = 0; q < WAVE_WQ; q++) {
      mbar_init(&done[q], NC);
      mbar_init(&pubd[q], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t gstride = (size_t)nact * D2 * G;
  const unsigned target = epoch;                  // one count per item per step
  const int nsb = (nstrips + sblk - 1) / sblk;      // strip blocks
  // completion counter of item (k, g, b, s)
  auto cidx = [&](int k, int g, int b, int s) { return (((size_t)g * 3 + k) * nbands + b) * nsb + s; };

  if (w == NC + 1) {
    // =========================== publisher warp ===========================
    uint32_t it = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, it++) {
      int k, g, b, sb;
      wave_item(item, nsb, ngroups, gblk, 3 * nbands, wtab, k, g, b, sb);
      mbar_wait(&done[it % WAVE_WQ], (it / WAVE_WQ) & 1);
      if (lane == 0) {
        __threadfence();
        red_release_add(cnt + cidx(k, g, b, sb), 1u);
        mbar_arrive(&pubd[it % WAVE_WQ]);
      }
      __syncwarp();
    }
    return;
  }
  if (w == NC) {
    // =========================== producer warp ===========================
    uint32_t *rv = reinterpret_cast<uint32_t *>(rt + RING_MAXBAND + 4);
    uint32_t L = 0, v1 = 0, v2 = 0, rel = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int k, g, b, sb;
      wave_item(item, nsb, ngroups, gblk, 3 * nbands, wtab, k, g, b, sb);
      const int jb0 = b * band_rows, jb1 = min(ny, jb0 + band_rows);
      const int lo = max(0, jb0 - 1), hi = min(ny - 1, jb1);
      // first strip's row table, loaded before the dependency wait (read-only;
      // prefetching it one item ahead measured no better)
      int4 pre = make_int4(0, 0, 0, 0);
      if (hi - lo < 32 && lo + lane <= hi) pre = __ldg(&rowtab[(size_t)(sb * sblk) * ny + lo + lane]);
      if (k > 0) {
        // wait for the 3 x 3 items of stage k-1 that write this item's input
        // (bands b-1..b+1, strip blocks sb-1..sb+1)
        const int db = lane / 3 - 1, ds = lane % 3 - 1;
        const bool mine = lane < 9 && b + db >= 0 && b + db < nbands && sb + ds >= 0 && sb + ds < nsb;
        const unsigned *cp = mine ? cnt + cidx(k - 1, g, b + db, sb + ds) : nullptr;
        const long long t0 = clock64();
        while (!__all_sync(0xffffffffu, !mine || ld_acquire_u32(cp) >= target)) {
          if (clock64() - t0 > (1LL << 34)) __trap();
        }
        fence_proxy_async_global();
      }
      const T *Ug = (k == 0 ? u : k == 1 ? U1 : U2) + g * gstride;
      for (int s = sb * sblk; s < min(nstrips, sb * sblk + sblk); s++) {
      __syncwarp();
      if (s == sb * sblk && hi - lo < 32) {
        if (lo + lane <= hi) rt[lane] = pre;
      } else {
        for (int r = lo + lane; r <= hi; r += 32) rt[r - lo] = __ldg(&rowtab[(size_t)s * ny + r]);
      }
      __syncwarp();
      for (int r0 = lo; r0 <= hi;) {
        const int r = r0 + lane;
        const bool valid = r <= hi;
        int4 t = make_int4(0, 0, 0, 0);
        if (valid) t = rt[r - lo];
        const bool comp = valid && r >= jb0 && r < jb1;
        const uint32_t n1 = valid ? (uint32_t)(t.w - t.x) : 0u;
        const uint32_t n2 = comp ? (uint32_t)(t.z - t.y) : 0u;
        uint32_t e1 = n1, e2 = n2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y1 = __shfl_up_sync(0xffffffffu, e1, o), y2 = __shfl_up_sync(0xffffffffu, e2, o);
          if (lane >= o) { e1 += y1; e2 += y2; }
        }
        const uint32_t nvalid = (uint32_t)min(32, hi - r0 + 1);
        uint32_t take;
        for (;;) {
          const uint32_t s1 = rel ? rv[(rel - 1) % Q] : 0u, s2 = rel ? rv[Q + (rel - 1) % Q] : 0u;
          const bool fits = valid && (L + lane - rel < (uint32_t)max_ahead) && (v1 + e1 - s1 <= (uint32_t)n1_use) &&
                            (v2 + e2 - s2 <= (uint32_t)n2_use);
          const uint32_t ok = __ballot_sync(0xffffffffu, fits);
          take = __ffs(~ok) - 1;
          if (ok == 0xffffffffu) take = 32;
          if (take > nvalid) take = nvalid;
          if (take > 0 || rel == L) break;
          mbar_wait(&empty[rel % Q], (rel / Q) & 1);
          rel++;
        }
        if (take == 0) take = 1;
        if ((uint32_t)lane < take) {
          const uint32_t Lr = L + lane, q = Lr % Q;
          const uint32_t bb1 = v1 + e1 - n1, bb2 = v2 + e2 - n2;
          const uint32_t p1 = bb1 % Gm::N1, p2 = bb2 % Gm::N2;
          RowMeta m;
          m.p1 = (int)p1; m.h0 = t.x; m.c0 = t.y; m.c1 = comp ? t.z : t.y; m.p2 = (int)p2;
          m.pad0 = m.pad1 = m.pad2 = 0;
          meta[q] = m;
          rv[q] = v1 + e1;
          rv[Q + q] = v2 + e2;
          mbar_expect_tx(&full[q], n1 * PXB + n2 * 16u);
          if (n1) {
            const uint32_t x1 = min(n1, (uint32_t)Gm::N1 - p1);
            const T *src = Ug + (size_t)t.x * D2 * G;
            bulk_g2s(ring1 + (size_t)p1 * PXB, src, x1 * PXB, &full[q]);
            if (n1 > x1) bulk_g2s(ring1, src + (size_t)x1 * D2 * G, (n1 - x1) * PXB, &full[q]);
          }
          if (n2) {
            const uint32_t x2 = min(n2, (uint32_t)Gm::N2 - p2);
            bulk_g2s(nbr_ring + p2, nbr + t.y, x2 * 16u, &full[q]);
            if (n2 > x2) bulk_g2s(nbr_ring, nbr + t.y + x2, (n2 - x2) * 16u, &full[q]);
          }
        }
        v1 += __shfl_sync(0xffffffffu, e1, take - 1);
        v2 += __shfl_sync(0xffffffffu, e2, take - 1);
        L += take;
        r0 += (int)take;
        __syncwarp();
      }
      }   // strips of the block
    }
    return;
  }

  // ============================= consumer warps ============================
  uint32_t Lbase = 0, it = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, it++) {
    int k, g, b, sb;
    wave_item(item, nsb, ngroups, gblk, 3 * nbands, wtab, k, g, b, sb);
    const int jb0 = b * band_rows, jb1 = min(ny, jb0 + band_rows);
    const int lo = max(0, jb0 - 1), hi = min(ny - 1, jb1);
    T *Uog = (k == 0 ? U1 : k == 1 ? U2 : u) + g * gstride + lane * NV;
    const T *U0l = u + g * gstride + lane * NV;
    const T cs = k == 0 ? c1 : k == 1 ? c2 : c3;
    const T alpha = k == 1 ? a2 : a3;
    for (int s_ = sb * sblk; s_ < min(nstrips, sb * sblk + sblk); s_++) {
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
    for (int r = jb0 - 1; r <= jb0 + 1; r++) wait_row(r);
    RowMeta mc = meta[seq(j) % Q];
    for (int f = w;; f += NC) {
      while (f >= cum + (mc.c1 - mc.c0)) {
        cum += mc.c1 - mc.c0;
        if (++j >= jb1) break;
        if (rel_next <= j - 2) {
          __syncwarp();
          if (lane == 0)
            for (int r = rel_next; r <= j - 2; r++) mbar_arrive(&empty[seq(r) % Q]);
          rel_next = j - 1;
        }
        wait_row(j + 1);
        mc = meta[seq(j) % Q];
      }
      if (j >= jb1) break;
      if (diag) continue;   // diagnostic: stream through the ring without computing
      const int a = mc.c0 + (f - cum);
      int sl2 = mc.p2 + (a - mc.c0);
      if (sl2 >= Gm::N2) sl2 -= Gm::N2;
      const int4 nb = nbr_ring[sl2];
      const T *ps = tile1(mc, a);
      T xs[D2][NV], acc[D2][NV], xn[D2][NV], z[D2][NV];
      if (k > 0) {
#pragma unroll
        for (int kk = 0; kk < D2; kk++) ldvc<T, NV>(U0l + ((size_t)a * D2 + kk) * G, z[kk]);
      }
#pragma unroll
      for (int kk = 0; kk < D2; kk++) lds<T, NV>(ps + kk * G, xs[kk]);
#pragma unroll
      for (int kk = 0; kk < D2; kk++)
#pragma unroll
        for (int e = 0; e < NV; e++) acc[kk][e] = (T)0;
      mv_self<T, NV, P>(open_code(nb), acc, xs);
      if (nb.x >= 0) {
        const T *pn = tile1(mc, nb.x);
#pragma unroll
        for (int kk = 0; kk < D2; kk++) lds<T, NV>(pn + kk * G, xn[kk]);
        mv_imm<T, NV, P, 5>(acc, xn);
      }
      if (nb.y >= 0) {
        const T *pn = tile1(mc, nb.y);
#pragma unroll
        for (int kk = 0; kk < D2; kk++) lds<T, NV>(pn + kk * G, xn[kk]);
        mv_imm<T, NV, P, 6>(acc, xn);
      }
      if (nb.z >= 0) {
        const T *pn = tile1(meta[seq(j + 1) % Q], nb.z);
#pragma unroll
        for (int kk = 0; kk < D2; kk++) lds<T, NV>(pn + kk * G, xn[kk]);
        mv_imm<T, NV, P, 7>(acc, xn);
      }
      if (nb.w >= 0) {
        const T *pn = tile1(meta[seq(j - 1) % Q], nb.w);
#pragma unroll
        for (int kk = 0; kk < D2; kk++) lds<T, NV>(pn + kk * G, xn[kk]);
        mv_imm<T, NV, P, 8>(acc, xn);
      }
      T *out = Uog + (size_t)a * D2 * G;
      if (k > 0) {
#pragma unroll
        for (int kk = 0; kk < D2; kk++) {
          T y[NV];
#pragma unroll
          for (int e = 0; e < NV; e++) y[e] = xs[kk][e] + alpha * (z[kk][e] - xs[kk][e]) + cs * acc[kk][e];
          stv<T, NV>(out + (size_t)kk * G, y);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < D2; kk++) {
          T y[NV];
#pragma unroll
          for (int e = 0; e < NV; e++) y[e] = xs[kk][e] + cs * acc[kk][e];
          stv<T, NV>(out + (size_t)kk * G, y);
        }
      }
    }
    __syncwarp();
    if (lane == 0)
      for (int r = rel_next; r <= hi; r++) mbar_arrive(&empty[seq(r) % Q]);
    Lbase += (uint32_t)(hi - lo + 1);
    }   // strips of the block
    // hand the item to the publisher (slot reuse waits for its release)
    fence_proxy_async_global();
    __syncwarp();
    if (lane == 0) {
      if (it >= WAVE_WQ) mbar_wait(&pubd[it % WAVE_WQ], ((it / WAVE_WQ) - 1) & 1);
      mbar_arrive(&done[it % WAVE_WQ]);
    }
  }
}

// rows per band of the wavefront; DGDIFF_WAVE_BAND overrides.  Bands of 2-4
// rows keep the live rows of u, U1, U2 in L2 (c4: DRAM 107 GB per step vs
// K2's 165 GB) but the per-item pipeline then runs at ~1.3 us per row and
// ~1 us per item (43 / 33 ms per c4 step); 32-row bands amortise the item
// cost and lose most L2 hits (28.3 ms, K2 28.0 ms) -- DESIGN.md section 6
inline int wave_band_rows() {
  static const int v = [] {
    const char *e = tune_env("DGDIFF_WAVE_BAND");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? std::min(x, RING_MAXBAND - 2) : 32;
  }();
  return v;
}
// strips per item (DGDIFF_WAVE_SBLK)
inline int wave_sblk() {
  static const int v = [] {
    const char *e = tune_env("DGDIFF_WAVE_SBLK");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? x : 4;
  }();
  return v;
}
// ring-1 pixel slots in use (DGDIFF_WAVE_N1; 0 = the whole ring): the
// wavefront reads from L2, so it wants as many rows in flight as fit
inline int wave_n1() {
  static const int v = [] {
    const char *e = tune_env("DGDIFF_WAVE_N1");
    return e ? atoi(e) : 0;
  }();
  return v;
}
// diagnostic (DGDIFF_WAVE_NODEP=1): skip the dependency waits -- WRONG results,
// timing only (how much the wavefront's dependency chain costs)
inline bool wave_nodep() {
  static const bool v = tune_env("DGDIFF_WAVE_NODEP") && atoi(tune_env("DGDIFF_WAVE_NODEP")) == 1;
  return v;
}
// source groups per wavefront block (DGDIFF_WAVE_GBLK; 0 = all groups)
inline int wave_gblk(int ngroups) {
  static const int v = [] {
    const char *e = tune_env("DGDIFF_WAVE_GBLK");
    return e ? atoi(e) : 1;
  }();
  return v <= 0 ? ngroups : std::min(v, ngroups);
}

// one SSP-RK3 step: a.Uin = u (in/out), a.U0 = U1 scratch, a.Uout = U2 scratch,
// a.cs = dt D / h^2, a.band_rows, a.wave_cnt (zeroed per chunk), a.wave_tab,
// a.wave_epoch = 1-based step index within the chunk
template <typename T, int NV, int P>
cudaError_t launch_wave(const dgl::StageArgs &a) {
  using Gm = RingGeom<T, NV, P, true>;
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (!(attr_set.load() >> dev & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_step_wave<T, NV, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(uint64_t(1) << dev);
  }
  const int band_rows = a.band_rows;
  const int nbands = (a.ny + band_rows - 1) / band_rows;
  const int sblk = wave_sblk();
  const int nitems = 3 * nbands * ((a.nstrips + sblk - 1) / sblk) * a.ngroups;
  const int grid = std::min(nitems, a.nsm);
  const double c = a.cs;
  // CTAs wait on items owned by other CTAs, so they must all be resident at
  // once: a cooperative launch guarantees that (or fails cleanly, e.g. under
  // an MPS SM limit) instead of a spin-wait that could never be satisfied
  T *pu = (T *)a.Uin, *pU1 = (T *)a.U0, *pU2 = (T *)a.Uout;
  const int4 *pnbr = a.nbr, *prt = a.rowtab;
  int nact = a.nact, ny = a.ny, nstrips = a.nstrips, ngroups = a.ngroups, gblk = wave_gblk(a.ngroups);
  int band = band_rows, nb = nbands, ni = nitems;
  const int2 *wt = a.wave_tab;
  T c1 = (T)c, c2 = (T)(0.25 * c), c3 = (T)((2.0 / 3.0) * c), a2 = (T)0.75, a3 = (T)(1.0 / 3.0);
  unsigned *cnt = a.wave_cnt;
  unsigned ep = wave_nodep() ? 0u : a.wave_epoch;
  int max_ahead = std::max(Gm::ROWS_MIN, std::min(RING_Q - 1, alpha_max_ahead(a, true)));
  int n1u = std::max(Gm::ROWS_MIN * (Gm::W + 2 * Gm::HALO), std::min(Gm::N1, wave_n1() > 0 ? wave_n1() : Gm::N1));
  int n2u = std::max(Gm::ROWS_MIN * Gm::W, std::min(Gm::N2, a.n2_use > 0 ? a.n2_use : Gm::N2));
  int diag = (tune_env("DGDIFF_WAVE_DIAG") && atoi(tune_env("DGDIFF_WAVE_DIAG")) == 1) ? 1 : 0;
  int sb = sblk;
  void *args[] = {&pu, &pU1, &pU2, &pnbr, &prt, &nact, &ny, &nstrips, &sb, &ngroups, &gblk, &band, &nb, &wt, &ni,
                  &c1, &c2, &c3, &a2, &a3, &cnt, &ep, &max_ahead, &n1u, &n2u, &diag};
  cudaError_t e = cudaLaunchCooperativeKernel((const void *)k_step_wave<T, NV, P>, dim3(grid),
                                              dim3((DGDIFF_WAVE_NC + 2) * 32), args, Gm::SMEM, a.st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dgk
