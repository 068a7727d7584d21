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

// same, but a CTA keeps NB tiles in flight (multi-buffered prefetch)
__global__ void loadonly_nb(const double* in, long W, int ntiles, int R, int RS, int NC, int CSs, int NB) {
  const int rank = blockIdx.x % RS;
  const int cl = blockIdx.x / RS, ncl = gridDim.x / RS;
  const int bufsz = NC * CSs;
  auto issue = [&](int tile, int b) {
    if (tile < ntiles) {
      const long col0 = (long)tile * 2 * NC;
      for (int q = threadIdx.x; q < R * NC; q += blockDim.x) {
        const int n = q / NC, c = q - n * NC;
        cp16(sm + b * bufsz + c * CSs + n + (n >> 3), in + (long)(n * RS + rank) * W + col0 + 2 * c);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int it = 0;
  for (int k = 0; k < NB - 1; ++k) issue(cl + k * ncl, k);
  for (int tile = cl; tile < ntiles; tile += ncl, ++it) {
    issue(tile + (NB - 1) * ncl, (it + NB - 1) % NB);
    if (NB == 2) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else if (NB == 3) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
}

// one CTA per tile (non-persistent), load only
__global__ void loadonly_np(const double* in, long W, int R, int RS, int NC, int CSs) {
  const int rank = blockIdx.x % RS;
  const int tile = blockIdx.x / RS;
  const long col0 = (long)tile * 2 * NC;
  for (int q = threadIdx.x; q < R * NC; q += blockDim.x) {
    const int n = q / NC, c = q - n * NC;
    cp16(sm + c * CSs + n + (n >> 3), in + (long)(n * RS + rank) * W + col0 + 2 * c);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
}

int main3(long W);
__global__ void readtile(const double* in, long W, int X, int R, double* sink) {
  // read-only tile: X columns x R rows (grid: W/X column tiles x N/R row blocks), cp.async into smem
  const long col0 = (long)blockIdx.x * X;
  const int row0 = blockIdx.y * R;
  const int nc = X / 2;
  for (int q = threadIdx.x; q < R * nc; q += blockDim.x) {
    const int r = q / nc, c = q - r * nc;
    cp16(sm + q, in + (long)(row0 + r) * W + col0 + 2 * c);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && sm[0].x == 12345.0) sink[0] = sm[1].y;
}
__global__ void readflat(const double2* in, size_t n2, double* sink) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(in + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.0) sink[0] = acc;
}
// persistent load-only on a column-block-tiled layout [W/16][N][16]: tile = NC column pairs of one block
__global__ void loadonly_tiled(const double* in, int N, int ntiles, int R, int RS, int NC, int CSs) {
  const int rank = blockIdx.x % RS;
  const int cl = blockIdx.x / RS, ncl = gridDim.x / RS;
  for (int tile = cl; tile < ntiles; tile += ncl) {
    const long col0 = (long)tile * 2 * NC;
    const double* blk = in + (col0 >> 4) * (long)N * 16 + (col0 & 15);
    for (int q = threadIdx.x; q < R * NC; q += blockDim.x) {
      const int n = q / NC, c = q - n * NC;
      cp16(sm + c * CSs + n + (n >> 3), blk + (long)(n * RS + rank) * 16 + 2 * c);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
}
int main2() {
  {
    const long W = 4096, N = 4096;
    double* a;
    cudaMalloc(&a, W * N * 8);
    cudaMemset(a, 0, W * N * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    cudaFuncSetAttribute(loadonly_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int cf[][3] = {{2, 2, 2}, {8, 8, 2}, {8, 2, 1}, {4, 4, 2}, {2, 1, 1}};
    for (auto& g : cf) {
      const int NC = g[0], RS = g[1], per_sm = g[2];
      const int R = (int)N / RS, CSs = R + R / 8 + 1;
      const size_t smem = (size_t)NC * CSs * 16;
      const int ntiles = (int)(W / (2 * NC));
      int grid = 148 * per_sm;
      grid -= grid % RS;
      for (int rep = 0; rep < 2; ++rep) loadonly_tiled<<<grid, 256, smem>>>(a, (int)N, ntiles, R, RS, NC, CSs);
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) loadonly_tiled<<<grid, 256, smem>>>(a, (int)N, ntiles, R, RS, NC, CSs);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      printf("loadonly TILED NC=%d rowstride=%d per_sm=%d smem=%zu KB: %.1f us, read %.1f GB/s %s\n", NC, RS, per_sm,
             smem / 1024, ms * 1e3 / 5, W * N * 8.0 * 5 / (ms * 1e-3) / 1e9,
             err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
    cudaFree(a);
  }
  {
    const long W = 4096, N = 4096;
    const size_t n = (size_t)W * N;
    double *a, *sink;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&sink, 64);
    cudaMemset(a, 0, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 2; ++rep) readflat<<<148 * 8, 256>>>((double2*)a, n / 2, sink);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) readflat<<<148 * 8, 256>>>((double2*)a, n / 2, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read flat: %.1f GB/s\n", n * 8.0 * 5 / (ms * 1e-3) / 1e9);
    cudaFuncSetAttribute(readtile, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int XR[][2] = {{16, 512}, {16, 128}, {16, 2048}, {4, 2048}, {32, 128}, {64, 64}, {128, 32}, {8, 512}};
    for (auto& g : XR) {
      const int X = g[0], R = g[1];
      const size_t smem = (size_t)X * R * 8;
      dim3 grid((unsigned)(W / X), (unsigned)(N / R));
      for (int rep = 0; rep < 2; ++rep) readtile<<<grid, 256, smem>>>(a, W, X, R, sink);
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) readtile<<<grid, 256, smem>>>(a, W, X, R, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("read tile X=%d R=%d (smem %zu KB): %.1f GB/s\n", X, R, smem / 1024, n * 8.0 * 5 / (ms * 1e-3) / 1e9);
    }
    cudaFree(a);
  }
  return 0;
}
int main3(long W) {
  const long N = 4096;
  printf("--- row pitch W = %ld doubles\n", W);
  const size_t n = (size_t)W * N;
  double* a;
  cudaMalloc(&a, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const long Wtiles = 4096;  // columns actually processed (pitch W may be larger)
  cudaFuncSetAttribute(loadonly, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int NC, RS, per_sm; };
  Cfg cfgs[] = {{2, 2, 2}, {2, 2, 3}, {2, 1, 2}, {4, 2, 2}, {8, 8, 2}, {8, 8, 3}, {2, 2, 1}};
  for (Cfg g : cfgs) {
    const int R = (int)N / g.RS;
    const int CSs = R + R / 8 + 1;
    const size_t smem = (size_t)g.NC * CSs * 16;
    const int ntiles = (int)(Wtiles / (2 * g.NC));
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
           smem / 1024, ms * 1e3 / 5, Wtiles * N * 8.0 * 5 / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  cudaFree(a);
  return 0;
  cudaFuncSetAttribute(loadonly_nb, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(loadonly_np, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg2 { int NC, RS, NB, per_sm; };
  Cfg2 c2s[] = {{2, 2, 2, 1}, {2, 2, 3, 1}, {1, 2, 2, 2}, {1, 2, 3, 2}, {8, 8, 2, 1}, {8, 8, 3, 1}, {4, 4, 2, 1}, {2, 2, 1, 3}};
  for (Cfg2 g : c2s) {
    const int R = (int)N / g.RS;
    const int CSs = R + R / 8 + 1;
    const size_t smem = (size_t)g.NB * g.NC * CSs * 16;
    const int ntiles = (int)(Wtiles / (2 * g.NC));
    int grid = 148 * g.per_sm;
    grid -= grid % g.RS;
    for (int rep = 0; rep < 2; ++rep) loadonly_nb<<<grid, 256, smem>>>(a, W, ntiles, R, g.RS, g.NC, CSs, g.NB);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) loadonly_nb<<<grid, 256, smem>>>(a, W, ntiles, R, g.RS, g.NC, CSs, g.NB);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("loadonly_nb NC=%d rowstride=%d NB=%d per_sm=%d smem=%zu KB: %.1f us, read %.1f GB/s %s\n", g.NC, g.RS, g.NB,
           g.per_sm, smem / 1024, ms * 1e3 / 5, Wtiles * N * 8.0 * 5 / (ms * 1e-3) / 1e9,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  int nps[][2] = {{2, 2}, {8, 8}, {8, 1}, {1, 2}};
  for (auto& g : nps) {
    const int NC = g[0], RS = g[1];
    const int R = (int)N / RS;
    const int CSs = R + R / 8 + 1;
    const size_t smem = (size_t)NC * CSs * 16;
    if (smem > 220 * 1024) continue;
    const int grid = (int)(Wtiles / (2 * NC)) * RS;
    for (int rep = 0; rep < 2; ++rep) loadonly_np<<<grid, 256, smem>>>(a, W, R, RS, NC, CSs);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) loadonly_np<<<grid, 256, smem>>>(a, W, R, RS, NC, CSs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("loadonly_np NC=%d rowstride=%d smem=%zu KB: %.1f us, read %.1f GB/s %s\n", NC, RS, smem / 1024,
           ms * 1e3 / 5, Wtiles * N * 8.0 * 5 / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
