// Same-run compute ceilings for the roofline (SURVEY.md §8(d) "fp64 FMA peak ... measure it in the
// same run with a dependent-FMA loop kernel (and an mma.sync f64 loop if K5 uses DMMA)").
//
// k_fma_peak: every thread runs FMA_CHAINS independent dependent chains of fp64 FMAs (enough
// independent work per warp to cover the FMA latency), a grid of 8 CTAs x 256 threads per SM.
// k_dmma_peak: every warp issues back-to-back mma.sync.m8n8k4 f64 (DMMA) on register fragments
// with DMMA_CHAINS independent accumulators.  Both write one value per thread so nothing is
// eliminated.  Flops: FMA = 2, one m8n8k4 = 2·8·8·4 = 512 per warp.
#include "common.cuh"
#include "internal.h"

#define FMA_CHAINS 8
#define DMMA_CHAINS 4

__global__ void __launch_bounds__(256) k_fma_peak(double* out, int iters, double seed) {
  double a[FMA_CHAINS];
#pragma unroll
  for (int c = 0; c < FMA_CHAINS; ++c) a[c] = seed + 1e-3 * (threadIdx.x + c);
  const double m = 0.999999999, s = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < FMA_CHAINS; ++c) a[c] = fma(a[c], m, s);
  }
  double r = 0.0;
#pragma unroll
  for (int c = 0; c < FMA_CHAINS; ++c) r += a[c];
  out[blockIdx.x * (size_t)blockDim.x + threadIdx.x] = r;
}

__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters, double seed) {
  double acc[DMMA_CHAINS][2];
  const double a = seed + 1e-3 * (threadIdx.x & 31), b = 1e-9 * (threadIdx.x & 7);
#pragma unroll
  for (int c = 0; c < DMMA_CHAINS; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < DMMA_CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(a), "d"(b));
  }
  double r = 0.0;
#pragma unroll
  for (int c = 0; c < DMMA_CHAINS; ++c) r += acc[c][0] + acc[c][1];
  out[blockIdx.x * (size_t)blockDim.x + threadIdx.x] = r;
}

extern "C" cnpint_status cnpint_peak_kernel(int kind, double* d_out, int iters, void* stream, double* flops) {
  if (!d_out || iters < 1 || (kind != 0 && kind != 1)) return CNPINT_EINVAL;
  int dev = 0, sms = CNP_NUM_SMS_DEFAULT;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = 8 * sms, threads = 256;
  if (kind == 0) {
    k_fma_peak<<<blocks, threads, 0, (cudaStream_t)stream>>>(d_out, iters, 1.0);
    if (flops) *flops = 2.0 * FMA_CHAINS * (double)iters * blocks * threads;
  } else {
    k_dmma_peak<<<blocks, threads, 0, (cudaStream_t)stream>>>(d_out, iters, 1.0);
    if (flops) *flops = 512.0 * DMMA_CHAINS * (double)iters * blocks * (threads / 32);
  }
  return cudaGetLastError() == cudaSuccess ? CNPINT_OK : CNPINT_ECUDA;
}
