// fma_peak.cu -- measured FP64 / FP32 arithmetic peaks of this B200 (SURVEY §6
// "builder task 0"): the roofline denominators of the FP64-bound kernels (P2,
// P3, the temporal-blocked steps), which MEASURED_PEAKS.json does not carry.
//
//   DFMA     fma.rn.f64, 8 independent chains per thread
//   FFMA     fma.rn.f32
//   FFMA2    fma.rn.f32x2 (packed pair, one issue slot for two FMAs)
//   DMMA     mma.sync.aligned.m8n8k4.row.col.f64 (FP64 tensor core path)
//
// Each kernel runs a fixed count of dependent-free FMAs per thread on a grid
// of 148 x 8 CTAs x 256 threads (enough warps to cover the pipe latency),
// timed with CUDA events after a warm-up, best of 5.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak fma_peak.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define ITERS 4096
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_dfma(double *out, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_ffma(float *out, float a, float b) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; k++) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = fmaf(x[k], a, b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; k++) s += x[k];
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_ffma2(float *out, float a, float b) {
  float2 x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = __ffma2_rn(x[k], A, B);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k].x + x[k].y;
  if (s == 12345.678f) out[0] = s;
}

// D (8x8) += A (8x4) * B (4x8), fp64; per thread one A, one B, two C/D values
__global__ void k_dmma(double *out, double a, double b) {
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; k++) { c[k][0] = threadIdx.x * 1e-3 + k; c[k][1] = k; }
  const double av = a, bv = b;
  for (int i = 0; i < ITERS / 4; i++) {
#pragma unroll
    for (int k = 0; k < 4; k++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
static double best_ms(F launch) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  launch();
  CK(cudaDeviceSynchronize());
  double best = 1e30;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  const double nthreads = (double)blocks * threads;
  double *dout;
  CK(cudaMalloc(&dout, 64));
  const double t_dfma = best_ms([&] { k_dfma<<<blocks, threads>>>(dout, 0.999999, 1e-7); });
  const double t_ffma = best_ms([&] { k_ffma<<<blocks, threads>>>((float *)dout, 0.9999f, 1e-7f); });
  const double t_ffma2 = best_ms([&] { k_ffma2<<<blocks, threads>>>((float *)dout, 0.9999f, 1e-7f); });
  const double t_dmma = best_ms([&] { k_dmma<<<blocks, threads>>>(dout, 0.5, 1e-3); });
  CK(cudaGetLastError());
  // flops: an FMA is 2 flops; one m8n8k4 MMA is 2*8*8*4 = 512 flops per warp
  const double f_dfma = nthreads * ITERS * 8 * 2, f_ffma = nthreads * ITERS * 16 * 2;
  const double f_ffma2 = nthreads * ITERS * 8 * 2 * 2, f_dmma = nthreads / 32 * (ITERS / 4) * 4 * 512.0;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_attr_mhz\": %.0f, "
         "\"dfma_tflops\": %.2f, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"dmma_tflops\": %.2f, "
         "\"dfma_per_clk_per_sm_at_attr_clock\": %.1f, "
         "\"how\": \"%d CTAs x %d threads, %d iterations of independent FMA chains (DFMA 8, FFMA 16, FFMA2 8 pairs, DMMA m8n8k4 4 per warp), CUDA events, best of 5\"}\n",
         p.name, p.multiProcessorCount, clk_khz / 1e3, f_dfma / t_dfma / 1e9, f_ffma / t_ffma / 1e9,
         f_ffma2 / t_ffma2 / 1e9, f_dmma / t_dmma / 1e9,
         f_dfma / 2 / (t_dfma * 1e-3) / (clk_khz * 1e3) / p.multiProcessorCount, blocks, threads, ITERS);
  return 0;
}
