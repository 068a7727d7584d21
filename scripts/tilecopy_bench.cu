// Micro-benchmark (not product code): achievable HBM bandwidth of the time-FFT access pattern.
// A CTA copies a tile of X adjacent fp64 columns × R rows (row pitch W doubles) through shared
// memory (cp.async in, coalesced stores out), for several X / R / CTA sizes, vs a flat copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tilecopy scripts/tilecopy_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g) : "memory");
}

extern __shared__ double2 sm[];

// tile = X columns (X/2 double2) × R rows; grid covers W/X column tiles × (N/R) row blocks
__global__ void tilecopy(const double* in, double* out, long W, int N, int X, int R) {
  const int nc = X / 2;
  const long col0 = (long)blockIdx.x * X;
  const int row0 = blockIdx.y * R;
  for (int q = threadIdx.x; q < R * nc; q += blockDim.x) {
    const int r = q / nc, c = q - r * nc;
    cp16(sm + q, in + (long)(row0 + r) * W + col0 + 2 * c);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int q = threadIdx.x; q < R * nc; q += blockDim.x) {
    const int r = q / nc, c = q - r * nc;
    double2 v = sm[q];
    __stcs(reinterpret_cast<double2*>(out + (long)(row0 + r) * W + col0 + 2 * c), v);
  }
}

__global__ void flatcopy(const double2* in, double2* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

int main2();
int main() {
  main2();
  const long W = 4096, N = 4096;  // c2: 16.8 M doubles = 134 MB
  const size_t n = (size_t)W * N;
  double *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 3; ++rep) flatcopy<<<148 * 8, 256>>>((double2*)a, (double2*)b, n / 2);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 10; ++rep) flatcopy<<<148 * 8, 256>>>((double2*)a, (double2*)b, n / 2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("flat copy: %.1f GB/s\n", 2.0 * n * 8 * 10 / (ms * 1e-3) / 1e9);
  int Xs[] = {2, 4, 8, 16, 32, 64, 128};
  int Rs[] = {4096, 2048, 512, 128, 32};
  for (int X : Xs)
    for (int R : Rs) {
      const size_t smem = (size_t)X * R * 8;
      if (smem > 200 * 1024) continue;
      cudaFuncSetAttribute(tilecopy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      dim3 grid((unsigned)(W / X), (unsigned)(N / R));
      tilecopy<<<grid, 256, smem>>>(a, b, W, (int)N, X, R);
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) tilecopy<<<grid, 256, smem>>>(a, b, W, (int)N, X, R);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      printf("tile X=%3d R=%5d smem=%6zu KB: %.1f GB/s %s\n", X, R, smem / 1024,
             2.0 * n * 8 * 5 / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  return 0;
}

// ---- K2 load-phase mimic: persistent CTAs, each "tile" = NC column pairs × R rows with row stride
// RS (rows t = n·RS + rank), cp.async into padded columns, barrier; nothing computed or stored.
__global__ void loadonly(const double* in, long W, int ntiles, int R, int RS, int NC, int CSs) {
  const int rank = blockIdx.x % RS;
  const int cl = blockIdx.x / RS, ncl = gridDim.x / RS;
  for (int tile = cl; tile < ntiles; tile += ncl) {
    const long col0 = (long)tile * 2 * NC;
    for (int q = threadIdx.x; q < R * NC; q += blockDim.x) {
      const int n = q / NC, c = q - n * NC;
      cp16(sm + c * CSs + n + (n >> 3), in + (long)(n * RS + rank) * W + col0 + 2 * c);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
}

int main2() {
  const long W = 4096, N = 4096;
  const size_t n = (size_t)W * N;
  double* a;
  cudaMalloc(&a, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  cudaFuncSetAttribute(loadonly, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int NC, RS, per_sm; };
  Cfg cfgs[] = {{2, 2, 2}, {2, 2, 3}, {2, 1, 2}, {4, 2, 2}, {8, 8, 2}, {8, 8, 3}, {2, 2, 1}};
  for (Cfg g : cfgs) {
    const int R = (int)N / g.RS;
    const int CSs = R + R / 8 + 1;
    const size_t smem = (size_t)g.NC * CSs * 16;
    const int ntiles = (int)(W / (2 * g.NC));
    int grid = 148 * g.per_sm;
    grid -= grid % g.RS;
    for (int rep = 0; rep < 2; ++rep) loadonly<<<grid, 256, smem>>>(a, W, ntiles, R, g.RS, g.NC, CSs);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) loadonly<<<grid, 256, smem>>>(a, W, ntiles, R, g.RS, g.NC, CSs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("loadonly NC=%d rowstride=%d per_sm=%d smem=%zu KB: %.1f us, read %.1f GB/s %s\n", g.NC, g.RS, g.per_sm,
           smem / 1024, ms * 1e3 / 5, n * 8.0 * 5 / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
