// pixel_bench.cu -- compute ceiling of the K3d per-pixel body (pair_pixel) on
// one SM with no pipeline around it: NW warps per CTA, one CTA per SM, each
// warp runs `iters` pixel tasks on shared-memory tiles with face codes drawn
// like the c4 substrate (45 % four open faces, 32 % three, 19 % two, 4 %
// fewer), alpha terms from a small L2-resident global array (or none), output
// to shared memory.  Reports tasks / s / SM and the FP64 pipe share.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_1907_06191_b200/csrc -o pixel_bench tools/pixel_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "stage_pair.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_pix(const double *z, int iters, int use_z, unsigned long long *sink) {
  using namespace dgk;
  constexpr int NV = 2, P = 1, PXB = 6 * 64 * 8, NT = 64;
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NT * PXB / 8; i += blockDim.x) reinterpret_cast<double *>(sm)[i] = 1e-3 * (i % 97);
  __syncthreads();
  const uint32_t base = smem_u32(sm), lane_b = lane * NV * 8;
  uint32_t h = 2654435761u * (w + 1 + blockIdx.x * 64);
  for (int t = 0; t < iters; t++) {
    h = h * 1664525u + 1013904223u;
    const int r = (h >> 24) % 100;
    const int code = r < 45 ? 15 : r < 77 ? (15 & ~(1 << ((h >> 8) & 3))) : r < 96 ? ((h >> 10) & 1 ? 5 : 10) : 1;
    const int p = (h >> 12) % (NT - 8) + 2;
    auto ta = [&](int q) { return base + (uint32_t)q * PXB + lane_b; };
    const double *zs = z + ((size_t)((h >> 4) % 4096) * 6 * 64) + lane * NV;
    pair_pixel<double, NV, P>(ta(p), ta(p + 1), ta(p - 1), ta((p + 17) % NT), ta((p + 41) % NT), code, zs, nullptr,
                              ta((p + 29) % NT), 0.75, 0.01, nullptr);
  }
  if (sm[7] == 123 && lane == 99) sink[0] = 1;
}

template <int NW>
void run(const double *z, unsigned long long *sink, int nsm, int use_z) {
  const int iters = 4000;
  const int smem = 64 * 6 * 64 * 8;
  CK(cudaFuncSetAttribute(k_pix<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_pix<NW><<<nsm, NW * 32, smem>>>(z, iters, use_z, sink);
  CK(cudaEventRecord(e0));
  k_pix<NW><<<nsm, NW * 32, smem>>>(z, iters, use_z, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double tasks = (double)NW * iters;            // per SM
  const double ns = ms * 1e6 / tasks;
  // mean structural DFMAs per task (P1, NV = 2): 2 x (36 + 20 x open faces) with the code mix above
  const double open = 0.45 * 4 + 0.32 * 3 + 0.19 * 2 + 0.04 * 1;
  const double dfma = 2 * (36 + 20 * open) + 2 * 6 * 2;
  printf("{\"warps\": %d, \"alpha_loads\": %d, \"ns_per_task_per_sm\": %.1f, \"cycles_per_task_at_1965\": %.0f, "
         "\"fp64_pipe_share\": %.2f}\n", NW, use_z, ns, ns * 1.965, dfma / 2.0 / (ns * 1.965));
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  double *z;
  unsigned long long *sink;
  CK(cudaMalloc(&z, (size_t)4096 * 6 * 64 * 8));
  CK(cudaMemset(z, 0, (size_t)4096 * 6 * 64 * 8));
  CK(cudaMalloc(&sink, 64));
  for (int uz = 1; uz < 2; uz++) {
    run<8>(z, sink, nsm, uz);
    run<12>(z, sink, nsm, uz);
    run<14>(z, sink, nsm, uz);
    run<16>(z, sink, nsm, uz);
    run<20>(z, sink, nsm, uz);
  }
  return 0;
}
