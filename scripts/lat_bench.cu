// Dependent-chain latencies on B200 (one warp, clock64): DFMA, DMUL, MUFU.RCP64H (rcp.approx.ftz.f64),
// crecip_nr as used in K3, LDS.128, SHFL (double), and a 128-thread bar.sync round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat scripts/lat_bench.cu && /tmp/lat
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, double seed) {
  __shared__ double2 sh[256];
  const int t = threadIdx.x;
  sh[t] = make_double2(seed + t, seed - t);
  __syncthreads();
  double x = seed + t * 1e-3, y = 1.0000001;
  long long c0, c1;
  const int R = 512;
  // DFMA chain
  c0 = clock64();
  for (int i = 0; i < R; ++i) x = fma(x, y, 1e-9);
  c1 = clock64(); if (t == 0) cyc[0] = (c1 - c0);
  // DMUL chain
  c0 = clock64();
  for (int i = 0; i < R; ++i) x = x * y;
  c1 = clock64(); if (t == 0) cyc[1] = (c1 - c0);
  // MUFU rcp.approx.ftz.f64 chain
  c0 = clock64();
  for (int i = 0; i < R; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  c1 = clock64(); if (t == 0) cyc[2] = (c1 - c0);
  // full-precision reciprocal with two NR steps
  c0 = clock64();
  for (int i = 0; i < R; ++i) {
    double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); r = fma(r, e, r); x = r + 1.0;
  }
  c1 = clock64(); if (t == 0) cyc[3] = (c1 - c0);
  // LDS.128 chain (address depends on previous value)
  int idx = t;
  double2 v = make_double2(0, 0);
  c0 = clock64();
  for (int i = 0; i < R; ++i) { v = sh[idx]; idx = ((int)v.x & 127) + (t & 1); }
  c1 = clock64(); if (t == 0) cyc[4] = (c1 - c0);
  // SHFL double chain
  double s = x;
  c0 = clock64();
  for (int i = 0; i < R; ++i) s = __shfl_down_sync(0xffffffffu, s, 1) + 1.0;
  c1 = clock64(); if (t == 0) cyc[5] = (c1 - c0);
  // barrier rounds (128 threads)
  c0 = clock64();
  for (int i = 0; i < R; ++i) __syncthreads();
  c1 = clock64(); if (t == 0) cyc[6] = (c1 - c0);
  // DADD chain
  c0 = clock64();
  for (int i = 0; i < R; ++i) x = x + y;
  c1 = clock64(); if (t == 0) cyc[7] = (c1 - c0);
  out[t] = x + s + v.x + idx;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64 * 8);
  long long h[8];
  for (int rep = 0; rep < 3; ++rep) {
    k_lat<<<1, 128>>>(out, cyc, 1.5);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  }
  const char* nm[8] = {"DFMA", "DMUL", "MUFU.RCP64H", "rcp+2NR(+DADD)", "LDS.128 (+cvt)", "SHFL.f64(+DADD)", "bar.sync 128", "DADD"};
  for (int i = 0; i < 8; ++i) printf("%-18s %6.1f cycles per dependent op\n", nm[i], h[i] / 512.0);
  return 0;
}
