// Common device helpers for cnpint (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define CNP_DEV __device__ __forceinline__

// ------------------------------------------------------------------ complex (double2) helpers
CNP_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
CNP_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
CNP_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
CNP_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
CNP_DEV double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
CNP_DEV double2 cmul_conj(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// a - b*c  (complex)
CNP_DEV double2 cfms(double2 a, double2 b, double2 c) {
  return make_double2(a.x - fma(b.x, c.x, -b.y * c.y), a.y - fma(b.x, c.y, b.y * c.x));
}
// a - r*c  (r real)
CNP_DEV double2 crfms(double2 a, double r, double2 c) { return make_double2(fma(-r, c.x, a.x), fma(-r, c.y, a.y)); }
CNP_DEV double2 crecip(double2 a) {
  double d = 1.0 / fma(a.x, a.x, a.y * a.y);
  return make_double2(a.x * d, -a.y * d);
}
// 1/a with a Newton-refined hardware reciprocal of |a|² (two steps: within an ulp of the IEEE
// quotient, no slow-path branch); zero or non-finite |a|² gives NaN (caught by cfinite).  Used on the
// critical path of K3's variable-row sweeps and merges.
CNP_DEV double2 crecip_nr(double2 a) {
  const double d = fma(a.x, a.x, a.y * a.y);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  return make_double2(a.x * r, -a.y * r);
}
// 1/d for real d > 0: hardware reciprocal + two Newton steps (within an ulp, no slow path)
CNP_DEV double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
// multiply by -i (forward) or +i (inverse)
template <bool INV>
CNP_DEV double2 cmul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
CNP_DEV bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }

// Programmatic dependent launch: a kernel launched with the PDL attribute (cnp_launch) may become
// resident while its predecessor drains; griddepcontrol.wait blocks until the predecessor grid has
// completed and its writes are visible (a no-op for a plain launch).  Every kernel calls this before its
// first access to data another kernel wrote, so the memory semantics are those of plain stream order.
// The dependents' launch is triggered implicitly as each CTA exits: an explicit
// griddepcontrol.launch_dependents right after the wait (round 1) let the next grid's CTAs become
// resident for the whole life of the current one and cost 12 % at c5 n511 N1024 (49.4 vs 43.4 ms per
// solve) and 10 % at c3 (2.83 vs 2.51 ms), while the exit trigger is as fast as or faster than both
// that and plain launches at every BASELINE size (profiles/r02_pdl_trigger_ab.txt).
// -DCNPINT_PDL_EARLY_TRIGGER restores the early trigger (A/B only).
CNP_DEV void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef CNPINT_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// ------------------------------------------------------------------ reductions
CNP_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block reduction of NV per-thread accumulators (any block shape, ≤ 32 warps): fixed warp trees and a
// fixed-order sum over warps; writes part[block_linear * stride + i], i < NV.
template <int NV>
CNP_DEV void block_reduce_nv(double (&acc)[NV], double* part, int stride) {
  __shared__ double red[32][NV];
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = (blockDim.x * blockDim.y) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double v = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][i] = v;
  }
  __syncthreads();
  if (tid < NV) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += red[w][tid];
    part[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * (size_t)blockIdx.z)) * stride + tid] = v;
  }
}

// Deterministic grid-level fold.  Every block has written its partial sums part[b*stride + col]
// (col < ncols); the last block to arrive (atomic ticket) adds them up in block order — lane l sums
// b = l, l+32, ... in order, then a fixed shuffle tree — and writes out[col], so the result does not
// depend on which block finishes last (bitwise reproducible).  Partials are read with ld.global.cg
// (L2) since other blocks wrote them.  The counter is reset for the next launch.  Returns true in
// the block that folded.
template <int MAXC = 10>  // columns folded at most
CNP_DEV bool grid_fold(const double* part, int nparts, int stride, int ncols, double* out, unsigned* counter) {
  __shared__ bool amlast;
  __shared__ double red[32][MAXC];
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = atomicAdd(counter, 1u) == (unsigned)(nparts - 1);
  __syncthreads();
  if (!amlast) return false;
  __threadfence();
  // every thread sums a fixed strided subset of the partials for all columns (independent L2 loads),
  // then warp trees and a fixed-order sum over warps
  const int nthr = blockDim.x * blockDim.y, lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
  double acc[MAXC];
#pragma unroll
  for (int col = 0; col < MAXC; ++col) acc[col] = 0.0;
  for (int b = tid; b < nparts; b += nthr) {
    const double* pb = part + (size_t)b * stride;
#pragma unroll
    for (int col = 0; col < MAXC; ++col)
      if (col < ncols) acc[col] += __ldcg(pb + col);
  }
#pragma unroll
  for (int col = 0; col < MAXC; ++col) {
    if (col < ncols) {
      double v = acc[col];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][col] = v;
    }
  }
  __syncthreads();
  if (tid < ncols) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += red[w][tid];
    out[tid] = v;
  }
  if (tid == 0) *counter = 0u;
  return true;  // this block did the fold (its thread tid < ncols wrote out[tid])
}

// Padded shared-memory index for complex FFT buffers: one pad entry every 16 elements breaks the
// power-of-two strides of the Stockham stages into bank-conflict-free patterns.
CNP_DEV int padi(int i) { return i + (i >> 4); }
static inline int padi_host(int i) { return i + (i >> 4); }

// Vector-stream loads use the default (L2-allocating) policy: measured on B200 (profiles/
// r01_l2_policy.txt) the GMRES update finds part of the Krylov vectors the previous kernels left in
// the 126-MB L2 (c2: K7 86.5 -> 84.6 us, c4: 182.8 -> 177.7 us); evict-first (.cs) loads were no
// faster anywhere.  CNP_L2_STREAM_LOADS restores evict-first loads.  Stores stay evict-first
// (CNP_L2_KEEP_STORES: default policy; measured no gain).
#ifdef CNP_L2_STREAM_LOADS
CNP_DEV double2 ldg_cs2(const double2* p) { return __ldcs(p); }
CNP_DEV double ldg_cs(const double* p) { return __ldcs(p); }
#else
CNP_DEV double2 ldg_cs2(const double2* p) { return __ldg(p); }
CNP_DEV double ldg_cs(const double* p) { return __ldg(p); }
#endif
#ifdef CNP_L2_KEEP_STORES
CNP_DEV void stg_cs2(double2* p, double2 v) { *p = v; }
CNP_DEV void stg_cs(double* p, double v) { *p = v; }
#else
CNP_DEV void stg_cs2(double2* p, double2 v) { __stcs(p, v); }
CNP_DEV void stg_cs(double* p, double v) { __stcs(p, v); }
#endif

// Asynchronous 16-byte global→shared copies (cp.async, LDGSTS): no register staging, any number
// in flight; completion per thread by commit/wait groups, then a barrier for visibility.
CNP_DEV void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
CNP_DEV void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
CNP_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
CNP_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// Bulk prefetch of [p, p + bytes) into L2 (TMA unit; p 16-B aligned, bytes a multiple of 16): no
// registers, no shared memory, no completion to wait for — the later loads of that range hit L2.
CNP_DEV void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// Named barrier over `count` threads (multiple of 32); id 1..15 (0 is __syncthreads).
CNP_DEV void named_sync(int id, int count) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory"); }

template <typename T>
CNP_DEV T shfl_down(T v, int d);
template <>
CNP_DEV double2 shfl_down<double2>(double2 v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}
CNP_DEV double2 shfl_up2(double2 v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
CNP_DEV double2 cneg(double2 a) { return make_double2(-a.x, -a.y); }
CNP_DEV double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
CNP_DEV double2 crfma(double r, double2 b, double2 c) { return make_double2(fma(r, b.x, c.x), fma(r, b.y, c.y)); }
