// fp64 throughput probes for the roofline denominator (MEASURED_PEAKS.json has
// only bf16 and HBM).  Two kernels: scalar DFMA chains and warp-level DMMA
// (mma.sync.aligned.m8n8k4.row.col.f64, the only fp64 tensor path on sm_100a;
// tcgen05 has no kind::f64).  Launched persistent (one wave, 148 x occupancy).
#include "common.cuh"

namespace ttb {

__global__ void __launch_bounds__(256) peak_dfma_kernel(double* out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) peak_dmma_kernel(double* out, int iters, double seed) {
  double acc[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = 0.0;
  double a = seed * (threadIdx.x + 1), b = seed - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma_884(acc[k], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace ttb

using namespace ttb;

extern "C" int ttb_fp64_peak(void* stream_, double* dfma_tflops, double* dmma_tflops) {
  TTB_TRY_BEGIN
  cudaStream_t st = (cudaStream_t)stream_;
  int dev = 0, sms = 0;
  TTB_CUDA(cudaGetDevice(&dev));
  TTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* sink = nullptr;
  TTB_CUDA(cudaMallocAsync(&sink, 64, st));
  cudaEvent_t e0, e1;
  TTB_CUDA(cudaEventCreate(&e0));
  TTB_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256;
  float ms = 0.f;
  // DFMA: 8 chains x 16 unroll x iters per thread, 2 flops each
  int it1 = 4096;
  peak_dfma_kernel<<<blocks, threads, 0, st>>>(sink, 64, 1.0);
  TTB_CUDA(cudaEventRecord(e0, st));
  peak_dfma_kernel<<<blocks, threads, 0, st>>>(sink, it1, 1.0);
  TTB_CUDA(cudaEventRecord(e1, st));
  TTB_CUDA(cudaEventSynchronize(e1));
  TTB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *dfma_tflops = 2.0 * 8 * 16 * (double)it1 * blocks * threads / (ms * 1e-3) / 1e12;
  // DMMA: each mma = 8*8*4 FMAs per warp
  int it2 = 2048;
  peak_dmma_kernel<<<blocks, threads, 0, st>>>(sink, 64, 1.0);
  TTB_CUDA(cudaEventRecord(e0, st));
  peak_dmma_kernel<<<blocks, threads, 0, st>>>(sink, it2, 1.0);
  TTB_CUDA(cudaEventRecord(e1, st));
  TTB_CUDA(cudaEventSynchronize(e1));
  TTB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  double warps = (double)blocks * threads / 32;
  *dmma_tflops = 2.0 * 256 * 4 * 8 * (double)it2 * warps / (ms * 1e-3) / 1e12;
  TTB_CUDA(cudaFreeAsync(sink, st));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  TTB_TRY_END
}
