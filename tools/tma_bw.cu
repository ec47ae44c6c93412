// tma_bw.cu -- how fast can one CTA per SM stream HBM into shared memory with
// 1-D bulk copies (cp.async.bulk, the ring kernels' producer path), as a
// function of the copy size and the number of copies in flight?  Also the
// same bytes with 16-byte ld.global by 8 warps (the direct-load path).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const char *src, size_t per_cta, int bytes, int inflight, unsigned long long *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
  unsigned char *buf = sm + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight; i++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const char *base = src + (size_t)blockIdx.x * per_cta;
  const size_t n = per_cta / bytes;
  for (size_t k = 0; k < n; k++) {
    const int s = (int)(k % inflight);
    if (k >= (size_t)inflight) {
      const uint32_t par = (uint32_t)(((k / inflight) - 1) & 1);
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(&bar[s])), "r"(par) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(buf + (size_t)s * bytes)), "l"(base + k * bytes), "r"(bytes), "r"(su32(&bar[s])) : "memory");
  }
  for (size_t k = n > (size_t)inflight ? n - inflight : 0; k < n; k++) {
    const int s = (int)(k % inflight);
    const uint32_t par = (uint32_t)((k / inflight) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(su32(&bar[s])), "r"(par) : "memory");
  }
  if (buf[0] == 123 && buf[1] == 45) sink[0] = 1;
}

// the ring kernels' pattern: CTA b streams "rows" of `bytes` bytes spaced
// `stride` bytes apart (one strip of consecutive grid rows), neighbouring CTAs
// on neighbouring strips (offset 2/3 of a row tile: strips overlap by halos)
__global__ void k_bulk_rows(const char *src, size_t nrows, size_t stride, int bytes, int inflight,
                            unsigned long long *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
  unsigned char *buf = sm + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight; i++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const char *base = src + (size_t)blockIdx.x * (bytes / 3 * 2 / 16 * 16);
  for (size_t k = 0; k < nrows; k++) {
    const int s = (int)(k % inflight);
    if (k >= (size_t)inflight) {
      const uint32_t par = (uint32_t)(((k / inflight) - 1) & 1);
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(&bar[s])), "r"(par) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(buf + (size_t)s * bytes)), "l"(base + k * stride), "r"(bytes), "r"(su32(&bar[s])) : "memory");
  }
  for (size_t k = nrows > (size_t)inflight ? nrows - inflight : 0; k < nrows; k++) {
    const int s = (int)(k % inflight);
    const uint32_t par = (uint32_t)((k / inflight) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(su32(&bar[s])), "r"(par) : "memory");
  }
  if (buf[0] == 123 && buf[1] == 45) sink[0] = 1;
}

__global__ void k_ldg(const int4 *src, size_t per_cta16, unsigned long long *sink) {
  const int4 *base = src + (size_t)blockIdx.x * per_cta16;
  int acc = 0;
  for (size_t i = threadIdx.x; i < per_cta16; i += blockDim.x * 4) {
    int4 a = __ldcs(base + i), b = i + blockDim.x < per_cta16 ? __ldcs(base + i + blockDim.x) : make_int4(0, 0, 0, 0);
    int4 c = i + 2 * blockDim.x < per_cta16 ? __ldcs(base + i + 2 * blockDim.x) : make_int4(0, 0, 0, 0);
    int4 d = i + 3 * blockDim.x < per_cta16 ? __ldcs(base + i + 3 * blockDim.x) : make_int4(0, 0, 0, 0);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t total = (size_t)16 << 30;          // 16 GB >> L2
  const size_t per_cta = total / nsm / 65536 * 65536;
  char *src;
  unsigned long long *sink;
  CK(cudaMalloc(&src, per_cta * nsm));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(src, 1, per_cta * nsm));
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(k_bulk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("{\"copies\": [\n");
  const int sizes[] = {3072, 6144, 12288, 24576, 49152};
  const int flights[] = {1, 2, 4, 8, 16};
  bool first = true;
  for (int bytes : sizes)
    for (int f : flights) {
      if ((size_t)bytes * f > 200 * 1024) continue;
      k_bulk<<<nsm, 32, 1024 + bytes * f>>>(src, per_cta, bytes, f, sink);
      CK(cudaEventRecord(e0));
      k_bulk<<<nsm, 32, 1024 + bytes * f>>>(src, per_cta, bytes, f, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double gbs = (double)per_cta * nsm / (ms * 1e-3) / 1e9;
      printf("%s  {\"bytes\": %d, \"inflight\": %d, \"kb_in_flight\": %.0f, \"gbs\": %.0f, \"per_sm_gbs\": %.1f, "
             "\"latency_us\": %.2f}", first ? "" : ",\n", bytes, f, bytes * f / 1024.0, gbs, gbs / nsm,
             bytes * f / (gbs / nsm * 1e3));
      first = false;
    }
  printf("\n], \"rows\": [\n");
  first = true;
  for (int bytes : {12288, 14336, 21504})
    for (int f : {2, 4, 6, 8, 12}) {
      if ((size_t)bytes * f > 200 * 1024) continue;
      const size_t stride = 2516992;                  // one grid row of a c4 group (~820 pixels x 3 KB)
      const size_t nrows = (per_cta * nsm - (size_t)nsm * bytes) / stride;
      k_bulk_rows<<<nsm, 32, 1024 + bytes * f>>>(src, nrows, stride, bytes, f, sink);
      CK(cudaEventRecord(e0));
      k_bulk_rows<<<nsm, 32, 1024 + bytes * f>>>(src, nrows, stride, bytes, f, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double gbs = (double)nrows * bytes * nsm / (ms * 1e-3) / 1e9;
      printf("%s  {\"bytes\": %d, \"inflight\": %d, \"gbs\": %.0f, \"per_sm_gbs\": %.1f, \"us_per_row\": %.3f, "
             "\"latency_us\": %.2f}", first ? "" : ",\n", bytes, f, gbs, gbs / nsm, ms * 1e3 / nrows,
             ms * 1e3 / nrows * f);
      first = false;
    }
  k_ldg<<<nsm, 256>>>((const int4 *)src, per_cta / 16, sink);
  CK(cudaEventRecord(e0));
  printf("\n], \"rows\": [\n");
  first = true;
  for (int bytes : {12288, 14336, 21504})
    for (int f : {2, 4, 6, 8, 12}) {
      if ((size_t)bytes * f > 200 * 1024) continue;
      const size_t stride = 2516992;                  // one grid row of a c4 group (~820 pixels x 3 KB)
      const size_t nrows = (per_cta * nsm - (size_t)nsm * bytes) / stride;
      k_bulk_rows<<<nsm, 32, 1024 + bytes * f>>>(src, nrows, stride, bytes, f, sink);
      CK(cudaEventRecord(e0));
      k_bulk_rows<<<nsm, 32, 1024 + bytes * f>>>(src, nrows, stride, bytes, f, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double gbs = (double)nrows * bytes * nsm / (ms * 1e-3) / 1e9;
      printf("%s  {\"bytes\": %d, \"inflight\": %d, \"gbs\": %.0f, \"per_sm_gbs\": %.1f, \"us_per_row\": %.3f, "
             "\"latency_us\": %.2f}", first ? "" : ",\n", bytes, f, gbs, gbs / nsm, ms * 1e3 / nrows,
             ms * 1e3 / nrows * f);
      first = false;
    }
  k_ldg<<<nsm, 256>>>((const int4 *)src, per_cta / 16, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("\n], \"ldg_one_cta_per_sm_256_threads_gbs\": %.0f}\n", (double)per_cta * nsm / (ms * 1e-3) / 1e9);
  CK(cudaGetLastError());
  return 0;
}
