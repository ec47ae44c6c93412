// kernels.cuh -- shared device helpers of the hot path.
//
// State layout: source-minor, extracellular pixels only,
//   U[g][a][k][G]    g = source group, a = active-pixel index (raster order),
//                    k = dof slot 0..2d-1 (triangle-major, canonical node
//                    order), G = 32 lanes x NV sources
// so one warp owns one pixel x G sources: the open-face code, the operator
// variant and the masked-pixel skip are warp-uniform, and every access is a
// coalesced 8- or 16-byte-per-lane load or store.  Axon pixels hold u = 0
// exactly ("the contribution to the solution is null") and are not
// stored.  NV = lane bytes / sizeof(T): 16-byte lanes for the global-load
// kernels (v1, v2), 8-byte lanes for the row-ring kernel (v3), so that a
// P1 pixel is 1.5 KB and four full row tiles fit in shared memory.
#pragma once
#include <type_traits>
#include <cstdint>
#include <cstdlib>
#include <atomic>
#include <cuda_runtime.h>

namespace dgk {

// Tuning / diagnostic knobs of the experiments (DGDIFF_RING, DGDIFF_WAVE_*,
// ...) are read from the environment ONLY in builds compiled with
// -DDGDIFF_TUNING (python -m paper_1907_06191_b200.build --tuning); the
// product library ignores the environment, so no variable can change a
// result or a schedule behind the caller's back.  Every knob that a tuning
// build finds set is counted (dgdiff_stats_t.env_overrides).
inline std::atomic<int> &tune_overrides() {
  static std::atomic<int> n{0};
  return n;
}
inline const char *tune_env(const char *name) {
#ifdef DGDIFF_TUNING
  const char *v = getenv(name);
  if (v && v[0]) {
    tune_overrides().fetch_add(1);
    return v;
  }
  return nullptr;
#else
  (void)name;
  return nullptr;
#endif
}

template <typename T, int NV> struct VT;
template <> struct VT<double, 1> { typedef double type; };
template <> struct VT<double, 2> { typedef double2 type; };
template <> struct VT<float, 1> { typedef float type; };
template <> struct VT<float, 2> { typedef float2 type; };
template <> struct VT<float, 4> { typedef float4 type; };

template <typename V, typename T, int NV>
__device__ __forceinline__ void unpack(const V &v, T (&x)[NV]) {
  if constexpr (NV == 1) x[0] = v;
  else if constexpr (NV == 2) { x[0] = v.x; x[1] = v.y; }
  else { x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w; }
}
template <typename V, typename T, int NV>
__device__ __forceinline__ V pack(const T (&x)[NV]) {
  V v;
  if constexpr (NV == 1) v = x[0];
  else if constexpr (NV == 2) { v.x = x[0]; v.y = x[1]; }
  else { v.x = x[0]; v.y = x[1]; v.z = x[2]; v.w = x[3]; }
  return v;
}

// acc[e] += a * x[e] for the NV sources of one lane.  fp32 pairs go through
// packed FFMA2 (fma.rn.f32x2 with a broadcast coefficient: two independent
// round-to-nearest FMAs, bit-identical to scalar fmaf, half the issue slots).
template <typename T, int NV>
__device__ __forceinline__ void fma_bc(T a, const T (&x)[NV], T (&acc)[NV]) {
  if constexpr (std::is_same<T, float>::value && NV % 2 == 0) {
#pragma unroll
    for (int e = 0; e < NV; e += 2) {
      const float2 r = __ffma2_rn(make_float2(a, a), make_float2(x[e], x[e + 1]), make_float2(acc[e], acc[e + 1]));
      acc[e] = r.x;
      acc[e + 1] = r.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < NV; e++) acc[e] = fma(a, x[e], acc[e]);
  }
}

// read-only-path load (state of the previous stage, never written in-kernel)
template <typename T, int NV>
__device__ __forceinline__ void ldv(const T *p, T (&x)[NV]) {
  typedef typename VT<T, NV>::type V;
  unpack<V, T, NV>(__ldg(reinterpret_cast<const V *>(p)), x);
}
// coherent load: u0 may alias the output (stage 3 writes u in place; each
// element is read and then written by the same thread)
template <typename T, int NV>
__device__ __forceinline__ void ldvc(const T *p, T (&x)[NV]) {
  typedef typename VT<T, NV>::type V;
  unpack<V, T, NV>(*reinterpret_cast<const V *>(p), x);
}
template <typename T, int NV>
__device__ __forceinline__ void stv(T *p, const T (&x)[NV]) {
  typedef typename VT<T, NV>::type V;
  *reinterpret_cast<V *>(p) = pack<V, T, NV>(x);
}
// shared-memory load (generic pointer into smem)
template <typename T, int NV>
__device__ __forceinline__ void lds(const T *p, T (&x)[NV]) {
  typedef typename VT<T, NV>::type V;
  unpack<V, T, NV>(*reinterpret_cast<const V *>(p), x);
}

__device__ __forceinline__ int open_code(int4 nb) {
  return (nb.x >= 0) | ((nb.y >= 0) << 1) | ((nb.z >= 0) << 2) | ((nb.w >= 0) << 3);
}

// ---- mbarrier + 1-D bulk TMA (cp.async.bulk) ---------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// wait for the phase of parity `parity`; a watchdog traps after ~2^34 cycles
// (~10 s) so that a pipeline bug fails loudly instead of hanging the device
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(a, parity)) {
    if (clock64() - t0 > (1LL << 34)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (no shared-memory destination)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

}  // namespace dgk
