// K0 stream copy, K1 AaO matvec y = 𝓜u (1D / 2D), K10 P_α matvec, GMRES residual r = b − 𝓜u.
//
// PAPER.md:337-343 (§3.2): 𝓜 = block-bidiagonal with Q1 = I − ½Ã on the diagonal and −Q2 =
// −(I + ½Ã) below it, Ã = τ L_h.  Row t:  y_t = Q1 u_t − Q2 u_{t−1} = (u_t − u_{t−1}) − ½τ L_h (u_t + u_{t−1}),
// u_{−1} = 0.  PAPER.md:344-350: P_α adds −αQ2 u_{N−1} to row 0, i.e. the same formula with
// u_{−1} := α u_{N−1}.  One HBM pass: each thread walks a chunk of time rows keeping u_{t−1} in
// registers; x-neighbours come from warp shuffles, y-neighbours (2D) from L1 re-reads (register kernel,
// k_matvec2d: the launches with side vectors) or from the cp.async shared-memory ring of the staged
// kernel (k_matvec2d_s: the plain 𝓜u / P_αu).  16 B/unknown of compulsory traffic (read u, write y).
#include "common.cuh"
#include "internal.h"
#include "post_op.cuh"

#include <algorithm>
#include <cstdlib>

// ------------------------------------------------------------------------------- K0 stream copy
__global__ void __launch_bounds__(256) k_stream_copy(const double2* __restrict__ src, double2* __restrict__ dst,
                                                     size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 4
  for (; i < n2; i += stride) stg_cs2(dst + i, ldg_cs2(src + i));
}

__global__ void k_copy_tail(const double* __restrict__ src, double* __restrict__ dst, size_t n) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && (n & 1)) dst[n - 1] = src[n - 1];
}

cudaError_t launch_stream_copy(const double* src, double* dst, size_t n, cudaStream_t s) {
  size_t n2 = n / 2;
  int dev = 0, sms = CNP_NUM_SMS_DEFAULT;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t blocks = std::min<size_t>((n2 + 255) / 256, (size_t)sms * 8);
  if (blocks == 0) blocks = 1;
  if (((uintptr_t)src | (uintptr_t)dst) & 15) return cudaErrorMisalignedAddress;
  k_stream_copy<<<(unsigned)blocks, 256, 0, s>>>((const double2*)src, (double2*)dst, n2);
  if (n & 1) k_copy_tail<<<1, 32, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- host-layout repack (host API)
// dir 0: packed [rows][nx] → padded [rows][ld] (padding written as 0); dir 1: padded → packed.
__global__ void __launch_bounds__(256) k_repack(const double* __restrict__ src, double* __restrict__ dst, size_t rows,
                                                int nx, int64_t ld, int dir) {
  for (size_t r = blockIdx.x; r < rows; r += gridDim.x) {
    if (dir == 0) {
      for (int x = threadIdx.x; x < ld; x += blockDim.x) dst[r * ld + x] = x < nx ? src[r * nx + x] : 0.0;
    } else {
      for (int x = threadIdx.x; x < nx; x += blockDim.x) dst[r * nx + x] = src[r * ld + x];
    }
  }
}

cudaError_t launch_repack(cnpint_ctx* c, const double* src, double* dst, int dir) {
  const size_t rows = (size_t)c->N * c->ny;
  const unsigned grid = (unsigned)(rows < 65535 * 4 ? rows : 65535 * 4);
  k_repack<<<grid, 256, 0, c->stream>>>(src, dst, rows, c->nx, c->ld, dir);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------ block-level sum helper
template <int NT>
CNP_DEV void block_partial(double v, double* part, double* out = nullptr, unsigned* counter = nullptr,
                           const PostOp& post = PostOp{}) {
  __shared__ double red[NT / 32];
  v = warp_sum(v);
  int w = threadIdx.x / 32 + threadIdx.y * (blockDim.x / 32);
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    double s = 0.0;
    for (int i = 0; i < NT / 32; ++i) s += red[i];
    part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * (size_t)blockIdx.z)] = s;
  }
  if (out && grid_fold(part, gridDim.x * gridDim.y * gridDim.z, 1, 1, out, counter)) run_post(post);
}

#ifndef MV_REVERSE
#define MV_REVERSE 1
#endif
// rows of the time chunk a 1D block walks (CNPINT_MV_TCHUNK: tuning override, 8/16/32/64)
static int mv_tchunk(const cnpint_ctx* c) {
  static const int v = [] {  // read once (thread-safe static initialisation)
    const char* e = getenv("CNPINT_MV_TCHUNK");
    const int t = e ? atoi(e) : 0;
    return (t == 8 || t == 16 || t == 32 || t == 64) ? t : 0;
  }();
  return v ? v : (c->N >= 4096 ? 32 : 16);
}

// rows of the time chunk a 2D block walks (CNPINT_MV2_TCHUNK: tuning override)
static bool mv2d_staged(const cnpint_ctx* c, int ns);
// ns = vectors read beside u (b of the residual modes, the Ṽ_i of the fused dots).  The staged kernel takes
// longer chunks (its ring fills and drains once per block): 64 rows alone, 128 with side vectors (one or two
// CTAs per SM), halved while the grid would have fewer than four waves of resident blocks.
static int mv2_tchunk(const cnpint_ctx* c, int ns) {
  static const int v = [] {
    const char* e = getenv("CNPINT_MV2_TCHUNK");
    const int t = e ? atoi(e) : 0;
    return (t == 8 || t == 16 || t == 32 || t == 64 || t == 128) ? t : 0;
  }();
  if (v) return v;
  // the register kernel (two CTAs per SM) also gains from long chunks — the rows of t0 − 1 are a dependent
  // round trip before the first batch: 16 → 64 rows, K1 class of a c5 n511 N1024 solve 1557 → 1410 µs
  // (profiles/r02_mvs_ab.txt)
  const bool st = mv2d_staged(c, ns);
  int t = (!st || ns == 0) ? 64 : 128;
  const int64_t tiles = ((c->ld + 63) / 64) * (int64_t)((c->ny + 7) / 8);
  const int64_t want = 4LL * c->num_sms * (!st ? 2 : ns == 0 ? 3 : ns == 1 ? 2 : 1);
  while (t > 16 && tiles * ((c->N + t - 1) / t) < want) t /= 2;
  return t;
}

// ------------------------------------------------------------------------------- K1 1D
// MODE 0: y = 𝓜u.  MODE 1: y = P_α u.  MODE 2: y = b − 𝓜u.  MODE 3: as 2 without storing y (norm
// only).  NORM: per-block Σ y².
// WW (with NVD > 0): also ww = yᵀy as column NVD of the folded dots, and the pending post-fold step run by
// the folding block (the derived-norm probe of cnpint_gmres, post op 5).
template <int MODE, bool NORM, int NVD = 0, bool WW = false>
__global__ void __launch_bounds__(128) k_matvec1d(const double* __restrict__ u, double* __restrict__ y,
                                                  const double* __restrict__ b, const double* __restrict__ lo,
                                                  const double* __restrict__ di, const double* __restrict__ up,
                                                  int N, int64_t ld, double htau, double alpha, int tchunk,
                                                  double* __restrict__ part, double* __restrict__ out,
                                                  unsigned* counter, DotPtrs vd = DotPtrs{},
                                                  const double* __restrict__ dt = nullptr, PostOp post = PostOp{}) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  double dacc[NVD > 0 ? NVD + (WW ? 1 : 0) : 1];
#pragma unroll
  for (int i = 0; i < (NVD > 0 ? NVD + (WW ? 1 : 0) : 1); ++i) dacc[i] = 0.0;
  const int lane = threadIdx.x & 31;
  const int64_t gx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // column pair
  const bool active = 2 * gx < ld;
  const int64_t x0 = active ? 2 * gx : 0;
  // residual (MODE >= 2, right after the combine wrote u front to back): time chunks back to front,
  // so u's tail still in L2 is read first (see k_update's GDOTS walk)
  const int t0 = ((MODE >= 2 && MV_REVERSE) ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y) * tchunk;
  const int t1 = min(N, t0 + tchunk);
  const bool hasL = active && lane == 0 && x0 > 0;
  const bool hasR = lane == 31 && active && x0 + 2 < ld;
  const int64_t xl = x0 - 1, xr = x0 + 2;

  double lo0 = 0, lo1 = 0, di0 = 0, di1 = 0, up0 = 0, up1 = 0;
  if (active) {
    lo0 = lo[x0]; lo1 = lo[x0 + 1]; di0 = di[x0]; di1 = di[x0 + 1]; up0 = up[x0]; up1 = up[x0 + 1];
  }
  // previous row (u_{t0-1}) incl. halo
  double2 pv = make_double2(0.0, 0.0);
  double pl = 0.0, pr = 0.0;
  if (t0 > 0) {
    const double* r = u + (int64_t)(t0 - 1) * ld;
    if (active) pv = *reinterpret_cast<const double2*>(r + x0);
    if (hasL) pl = r[xl];
    if (hasR) pr = r[xr];
  } else if (MODE == 1) {
    const double* r = u + (int64_t)(N - 1) * ld;
    if (active) { pv = *reinterpret_cast<const double2*>(r + x0); pv.x *= alpha; pv.y *= alpha; }
    if (hasL) pl = alpha * r[xl];
    if (hasR) pr = alpha * r[xr];
  }
  double acc = 0.0;
  // rows in batches of TB: all loads of a batch are issued before any is used (memory-level
  // parallelism; a row-at-a-time loop leaves one load per warp in flight and stalls on it)
  constexpr int TB = NVD <= 1 ? 4 : NVD <= 3 ? 2 : 1;  // rows per batch (the dot vectors add loads per row)
  for (int tb = t0; tb < t1; tb += TB) {
    double2 cvb[TB], bvb[TB], vvb[TB][NVD > 0 ? NVD : 1];
    double clb[TB], crb[TB];
#pragma unroll
    for (int q = 0; q < TB; ++q) {
      const int t = tb + q;
      cvb[q] = bvb[q] = make_double2(0.0, 0.0);
      clb[q] = crb[q] = 0.0;
#pragma unroll
      for (int i = 0; i < (NVD > 0 ? NVD : 1); ++i) vvb[q][i] = make_double2(0.0, 0.0);
      if (t < t1) {
        const double* r = u + (int64_t)t * ld;
        if (active) cvb[q] = ldg_cs2(reinterpret_cast<const double2*>(r + x0));
        if (hasL) clb[q] = r[xl];
        if (hasR) crb[q] = r[xr];
        if (MODE >= 2 && active) bvb[q] = ldg_cs2(reinterpret_cast<const double2*>(b + (int64_t)t * ld + x0));
        if (NVD > 0 && active) {
#pragma unroll
          for (int i = 0; i < NVD; ++i)
            vvb[q][i] = ldg_cs2(reinterpret_cast<const double2*>(vd.p[i] + (int64_t)t * ld + x0));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < TB; ++q) {
      const int t = tb + q;
      if (t >= t1) break;
      const double2 cv = cvb[q];
      const double cl = clb[q], cr = crb[q];
      const double s0 = cv.x + pv.x, s1 = cv.y + pv.y;
      const double d0 = cv.x - pv.x, d1 = cv.y - pv.y;
      double sl = __shfl_up_sync(0xffffffffu, s1, 1);
      double sr = __shfl_down_sync(0xffffffffu, s0, 1);
      if (lane == 0) sl = hasL ? cl + pl : 0.0;
      if (lane == 31) sr = hasR ? cr + pr : 0.0;
      const double ht = dt ? htau * dt[t] : htau;  // row t of D̃B2 (Eq. 5.8)
      double y0 = d0 - ht * fma(lo0, sl, fma(di0, s0, up0 * s1));
      double y1 = d1 - ht * fma(lo1, s0, fma(di1, s1, up1 * sr));
      if (MODE >= 2) {
        y0 = bvb[q].x - y0;
        y1 = bvb[q].y - y1;
      }
      if (active && MODE != 3) stg_cs2(reinterpret_cast<double2*>(y + (int64_t)t * ld + x0), make_double2(y0, y1));
      if (NVD > 0 && active) {  // fused first CGS pass: partial dots Ṽ_iᵀ y
#pragma unroll
        for (int i = 0; i < NVD; ++i) dacc[i] = fma(vvb[q][i].x, y0, fma(vvb[q][i].y, y1, dacc[i]));
        if constexpr (WW) dacc[NVD] = fma(y0, y0, fma(y1, y1, dacc[NVD]));
      }
      if (NORM) acc = fma(y0, y0, fma(y1, y1, acc));
      pv = cv; pl = cl; pr = cr;
    }
  }
  if (NORM) block_partial<128>(acc, part, out, counter, post);
  if constexpr (NVD > 0) {
    constexpr int NC = NVD + (WW ? 1 : 0);
    block_reduce_nv<NC>(dacc, part, CNP_MAX_DOT + 1);
    const bool folded = grid_fold(part, gridDim.x * gridDim.y * gridDim.z, CNP_MAX_DOT + 1, NC, out, counter);
    if constexpr (WW) {
      if (folded) run_post(post);
    }
  }
}

// ------------------------------------------------------------------------------- K1 2D
// Register kernel.  Block: 32 lanes along x (2 columns each = 64 columns) x 8 warps along y.  Each thread
// walks a chunk of t in batches of TB rows whose loads (own row, rows y−1 and y+1 through L1, side
// vectors) are all issued before the first is used.
// WW (with NVD > 0): also ww = yᵀy as column NVD of the folded dots, and the pending post-fold step
// (the derived-norm probe of cnpint_gmres, post op 5) run by the folding block.
template <int MODE, bool NORM, int NVD = 0, bool WW = false>
__global__ void __launch_bounds__(256) k_matvec2d(const double* __restrict__ u, double* __restrict__ y,
                                                  const double* __restrict__ b, int N, int nx, int ny, int64_t ld,
                                                  double htau, double alpha, double cxs, double cxu, double cys,
                                                  double cyu, double cdiag, int tchunk, double* __restrict__ part,
                                                  double* __restrict__ out, unsigned* counter,
                                                  DotPtrs vd = DotPtrs{}, const double* __restrict__ dt = nullptr,
                                                  PostOp post = PostOp{}) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  // Warp wy of the block owns y row ybase + wy; its y−1 / y+1 neighbours are read straight from
  // global memory through L1 (the block's other warps load the same rows, so most of those reads
  // hit L1) — no shared-memory exchange and no barrier per time row.  x-neighbours by __shfl.
  double dacc[NVD > 0 ? NVD + (WW ? 1 : 0) : 1];
#pragma unroll
  for (int i = 0; i < (NVD > 0 ? NVD + (WW ? 1 : 0) : 1); ++i) dacc[i] = 0.0;
  const int lane = threadIdx.x, wy = threadIdx.y;
  const int64_t x0 = (int64_t)blockIdx.x * 64 + 2 * lane;
  const int yrow = blockIdx.y * 8 + wy;
  const int t0 = ((MODE >= 2 && MV_REVERSE) ? (int)(gridDim.z - 1 - blockIdx.z) : (int)blockIdx.z) * tchunk;
  const int t1 = min(N, t0 + tchunk);
  const bool colok = x0 < ld;
  const bool rowok = yrow < ny;
  const bool act = colok && rowok;
  const bool hasL = act && lane == 0 && x0 > 0;
  const bool hasR = act && lane == 31 && x0 + 2 < ld;
  const bool hasD = act && yrow > 0;
  const bool hasU = act && yrow + 1 < ny;
  const int64_t slice = (int64_t)ny * ld;
  const int64_t off = (int64_t)yrow * ld + x0;

  auto ld2 = [&](const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); };
  double2 pv = make_double2(0, 0), pd = pv, pu = pv;
  double pl = 0, pr = 0;
  if (t0 > 0 || MODE == 1) {
    const double sc = (t0 > 0) ? 1.0 : alpha;
    const double* r = u + (int64_t)((t0 > 0) ? t0 - 1 : N - 1) * slice + off;
    if (act) pv = ld2(r);
    if (hasD) pd = ld2(r - ld);
    if (hasU) pu = ld2(r + ld);
    if (hasL) pl = r[-1];
    if (hasR) pr = r[2];
    pv.x *= sc; pv.y *= sc; pd.x *= sc; pd.y *= sc; pu.x *= sc; pu.y *= sc; pl *= sc; pr *= sc;
  }
  double acc = 0.0;
  // rows in batches whose loads are all issued before use (see k_matvec1d)
#ifndef MV2D_TB0
#define MV2D_TB0 4
#endif
  constexpr int TB = NVD == 0 ? MV2D_TB0 : NVD <= 1 ? 4 : NVD <= 3 ? 2 : 1;
  for (int tb = t0; tb < t1; tb += TB) {
    double2 cvb[TB], cdb[TB], cub[TB], bvb[TB], vvb[TB][NVD > 0 ? NVD : 1];
    double clb[TB], crb[TB];
#pragma unroll
    for (int q = 0; q < TB; ++q) {
      const int t = tb + q;
      cvb[q] = cdb[q] = cub[q] = bvb[q] = make_double2(0, 0);
      clb[q] = crb[q] = 0.0;
#pragma unroll
      for (int i = 0; i < (NVD > 0 ? NVD : 1); ++i) vvb[q][i] = make_double2(0, 0);
      if (t < t1) {
        const double* r = u + (int64_t)t * slice + off;
        if (act) cvb[q] = ld2(r);
        if (hasD) cdb[q] = ld2(r - ld);
        if (hasU) cub[q] = ld2(r + ld);
        if (hasL) clb[q] = r[-1];
        if (hasR) crb[q] = r[2];
        if (MODE >= 2 && act) bvb[q] = ldg_cs2(reinterpret_cast<const double2*>(b + (int64_t)t * slice + off));
        if (NVD > 0 && act) {
#pragma unroll
          for (int i = 0; i < NVD; ++i)
            vvb[q][i] = ldg_cs2(reinterpret_cast<const double2*>(vd.p[i] + (int64_t)t * slice + off));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < TB; ++q) {
      const int t = tb + q;
      if (t >= t1) break;
      const double2 cv = cvb[q];
      const double2 s = make_double2(cv.x + pv.x, cv.y + pv.y);
      const double2 sd = make_double2(cdb[q].x + pd.x, cdb[q].y + pd.y);  // row y−1
      const double2 su = make_double2(cub[q].x + pu.x, cub[q].y + pu.y);  // row y+1
      double sl = __shfl_up_sync(0xffffffffu, s.y, 1);
      double sr = __shfl_down_sync(0xffffffffu, s.x, 1);
      if (lane == 0) sl = hasL ? clb[q] + pl : 0.0;
      if (lane == 31) sr = hasR ? crb[q] + pr : 0.0;
      const double ht = dt ? htau * dt[t] : htau;  // row t of D̃B2 (Eq. 5.8)
      double y0 = (cv.x - pv.x) - ht * (cxs * sl + cxu * s.y + cys * sd.x + cyu * su.x + cdiag * s.x);
      double y1 = (cv.y - pv.y) - ht * (cxs * s.x + cxu * sr + cys * sd.y + cyu * su.y + cdiag * s.y);
      if (x0 >= nx) y0 = 0.0;
      if (x0 + 1 >= nx) y1 = 0.0;
      if (MODE >= 2 && act) {
        y0 = bvb[q].x - y0;
        y1 = bvb[q].y - y1;
      }
      if (act) {
        if (MODE != 3) stg_cs2(reinterpret_cast<double2*>(y + (int64_t)t * slice + off), make_double2(y0, y1));
        if constexpr (NVD > 0) {  // fused first CGS pass: partial dots Ṽ_iᵀ y
#pragma unroll
          for (int i = 0; i < NVD; ++i) dacc[i] = fma(vvb[q][i].x, y0, fma(vvb[q][i].y, y1, dacc[i]));
          if constexpr (WW) dacc[NVD] = fma(y0, y0, fma(y1, y1, dacc[NVD]));
        }
        if (NORM) acc = fma(y0, y0, fma(y1, y1, acc));
      }
      pv = cv; pd = cdb[q]; pu = cub[q]; pl = clb[q]; pr = crb[q];
    }
  }
  if (NORM) block_partial<256>(acc, part, out, counter, post);
  if constexpr (NVD > 0) {
    constexpr int NC = NVD + (WW ? 1 : 0);
    block_reduce_nv<NC>(dacc, part, CNP_MAX_DOT + 1);
    const bool folded = grid_fold(part, gridDim.x * gridDim.y * gridDim.z, CNP_MAX_DOT + 1, NC, out, counter);
    if constexpr (WW) {
      if (folded) run_post(post);
    }
  }
}


// ------------------------------------------------------------------------------- K1 2D, staged (round 2)
// The same block tile (64 columns × 8 rows, one warp per y row, a chunk of time rows), but every vector
// arrives through a shared-memory ring filled by cp.async: MVS_NG groups of MVS_G time rows; a slot holds
// the 10 × 66 patch of u (rows y0−1 … y0+8, columns x0−1 … x0+64) of one time row and the 8 × 64 tile of
// each of the NS vectors read alongside it (b for the residual modes, the Ṽ_i of the fused dots).  A thread
// keeps no load in registers, so two groups (8 time rows of every stream) stay in flight per CTA while a
// third is computed — k_matvec2d holds one batch of ≤ 4 rows in registers (own row and both y neighbours)
// and waits for it (a plain 𝓜u ran at 0.67 of HBM, latency-bound; this one 0.80-0.82).  The y neighbours
// come from the ring instead of L1 re-reads; one CTA barrier per group.  Positions outside the domain
// are never written and stay 0.  NS ≤ 3 (65 / 114 / 164 / 213 KB of ring: 3 / 2 / 1 / 1 CTAs per SM);
// more dot vectors go through k_matvec2d.
constexpr int MVS_G = 4, MVS_NG = 3, MVS_ROWS = 10, MVS_RW = 68;  // row: [1] = x0−1, [2..65] = the tile, [66] = x0+64
constexpr int MVS_MAXNVD = 3;
constexpr int mvs_slot(int ns) { return MVS_ROWS * MVS_RW + ns * 512; }  // doubles per slot
constexpr size_t mvs_bytes(int ns) { return (size_t)MVS_G * MVS_NG * mvs_slot(ns) * sizeof(double); }

template <int MODE, bool NORM, int NVD = 0>
__global__ void __launch_bounds__(256, (NVD + (MODE >= 2)) == 0 ? 3 : (NVD + (MODE >= 2)) == 1 ? 2 : 1)
    k_matvec2d_s(const double* __restrict__ u, double* __restrict__ y, const double* __restrict__ b, int N, int nx,
                 int ny, int64_t ld, double htau, double alpha, double cxs, double cxu, double cys, double cyu,
                 double cdiag, int tchunk, double* __restrict__ part, double* __restrict__ out, unsigned* counter,
                 DotPtrs vd = DotPtrs{}, const double* __restrict__ dt = nullptr, PostOp post = PostOp{}) {
  constexpr int NS = NVD + (MODE >= 2 ? 1 : 0), SLOT = mvs_slot(NS);
  static_assert(MODE < 2 || NVD == 0, "the residual modes carry no fused dots");
  extern __shared__ __align__(16) double mvs_ring[];
  const int lane = threadIdx.x, wy = threadIdx.y;
  for (int i = wy * 32 + lane; i < MVS_G * MVS_NG * SLOT; i += 256) mvs_ring[i] = 0.0;
  __syncthreads();
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  double dacc[NVD > 0 ? NVD : 1];
#pragma unroll
  for (int i = 0; i < (NVD > 0 ? NVD : 1); ++i) dacc[i] = 0.0;
  const int64_t x0 = (int64_t)blockIdx.x * 64 + 2 * lane;
  const int yrow = blockIdx.y * 8 + wy;
  const int t0 = ((MODE >= 2 && MV_REVERSE) ? (int)(gridDim.z - 1 - blockIdx.z) : (int)blockIdx.z) * tchunk;
  const int t1 = min(N, t0 + tchunk);
  const bool act = x0 < ld && yrow < ny;
  const bool hasL = act && lane == 0 && x0 > 0;
  const bool hasR = act && lane == 31 && x0 + 2 < ld;
  const bool hasD = act && yrow > 0;
  const bool hasU = act && yrow + 1 < ny;
  const int64_t slice = (int64_t)ny * ld;
  const int64_t off = (int64_t)yrow * ld + x0;
  double* const mine = mvs_ring + (wy + 1) * MVS_RW + 2 + 2 * lane;         // this thread's pair of u in slot 0
  double* const minev = mvs_ring + MVS_ROWS * MVS_RW + wy * 64 + 2 * lane;  // … of the first side vector

  auto issue_group = [&](int g) {
#pragma unroll
    for (int q = 0; q < MVS_G; ++q) {
      const int t = t0 + g * MVS_G + q;
      if (t < t1) {
        const int so = ((g % MVS_NG) * MVS_G + q) * SLOT;
        double* const d = mine + so;
        const int64_t go = (int64_t)t * slice + off;
        const double* const r = u + go;
        if (act) cp_async16(d, r);
        if (hasL) cp_async8(d - 1, r - 1);
        if (hasR) cp_async8(d + 2, r + 2);
        if (wy == 0 && hasD) cp_async16(d - MVS_RW, r - ld);
        if (wy == 7 && hasU) cp_async16(d + MVS_RW, r + ld);
        if (act) {
          if (MODE >= 2) cp_async16(minev + so, b + go);
#pragma unroll
          for (int i = 0; i < NVD; ++i) cp_async16(minev + so + i * 512, vd.p[i] + go);
        }
      }
    }
    cp_async_commit();
  };
  const int ngroups = (t1 - t0 + MVS_G - 1) / MVS_G;
#pragma unroll
  for (int g = 0; g < MVS_NG - 1; ++g) issue_group(g);  // rows past t1 issue nothing; the group is still committed

  auto ld2 = [&](const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); };
  double2 pv = make_double2(0, 0), pd = pv, pu = pv;
  double pl = 0, pr = 0;
  if (t0 > 0 || MODE == 1) {
    const double sc = (t0 > 0) ? 1.0 : alpha;
    const double* r = u + (int64_t)((t0 > 0) ? t0 - 1 : N - 1) * slice + off;
    if (act) pv = ld2(r);
    if (hasD) pd = ld2(r - ld);
    if (hasU) pu = ld2(r + ld);
    if (hasL) pl = r[-1];
    if (hasR) pr = r[2];
    pv.x *= sc; pv.y *= sc; pd.x *= sc; pd.y *= sc; pu.x *= sc; pu.y *= sc; pl *= sc; pr *= sc;
  }
  double acc = 0.0;
  for (int g = 0; g < ngroups; ++g) {
    cp_async_wait<MVS_NG - 2>();  // this thread's copies of group g have landed
    __syncthreads();              // … everyone's; and group g − 1 is computed: its slots are free
    issue_group(g + MVS_NG - 1);
    const int go = (g % MVS_NG) * MVS_G * SLOT;
#pragma unroll
    for (int q = 0; q < MVS_G; ++q) {
      const int t = t0 + g * MVS_G + q;
      if (t >= t1) break;
      const double* const d = mine + go + q * SLOT;
      const double2 cv = *reinterpret_cast<const double2*>(d);
      const double2 cd = *reinterpret_cast<const double2*>(d - MVS_RW);
      const double2 cu = *reinterpret_cast<const double2*>(d + MVS_RW);
      const double cl = lane == 0 ? d[-1] : 0.0, cr = lane == 31 ? d[2] : 0.0;
      const double2 s = make_double2(cv.x + pv.x, cv.y + pv.y);
      const double2 sd = make_double2(cd.x + pd.x, cd.y + pd.y);  // row y−1
      const double2 su = make_double2(cu.x + pu.x, cu.y + pu.y);  // row y+1
      double sl = __shfl_up_sync(0xffffffffu, s.y, 1);
      double sr = __shfl_down_sync(0xffffffffu, s.x, 1);
      if (lane == 0) sl = cl + pl;
      if (lane == 31) sr = cr + pr;
      const double ht = dt ? htau * dt[t] : htau;  // row t of D̃B2 (Eq. 5.8)
      double y0 = (cv.x - pv.x) - ht * (cxs * sl + cxu * s.y + cys * sd.x + cyu * su.x + cdiag * s.x);
      double y1 = (cv.y - pv.y) - ht * (cxs * s.x + cxu * sr + cys * sd.y + cyu * su.y + cdiag * s.y);
      if (x0 >= nx) y0 = 0.0;
      if (x0 + 1 >= nx) y1 = 0.0;
      if (act) {
        const double* const dv = minev + go + q * SLOT;
        if (MODE >= 2) {
          const double2 bv = *reinterpret_cast<const double2*>(dv);
          y0 = bv.x - y0;
          y1 = bv.y - y1;
        }
        if (MODE != 3) stg_cs2(reinterpret_cast<double2*>(y + (int64_t)t * slice + off), make_double2(y0, y1));
        if constexpr (NVD > 0) {  // fused first CGS pass: partial dots Ṽ_iᵀ y
#pragma unroll
          for (int i = 0; i < NVD; ++i) {
            const double2 vv = *reinterpret_cast<const double2*>(dv + i * 512);
            dacc[i] = fma(vv.x, y0, fma(vv.y, y1, dacc[i]));
          }
        }
        if (NORM) acc = fma(y0, y0, fma(y1, y1, acc));
      }
      pv = cv; pd = cd; pu = cu; pl = cl; pr = cr;
    }
  }
  cp_async_wait<0>();
  if (NORM) block_partial<256>(acc, part, out, counter, post);
  if constexpr (NVD > 0) {
    block_reduce_nv<NVD>(dacc, part, CNP_MAX_DOT + 1);
    grid_fold(part, gridDim.x * gridDim.y * gridDim.z, CNP_MAX_DOT + 1, NVD, out, counter);
  }
}

// 2D launch: the staged kernel by default (≤ MVS_MAXNVD dot vectors), k_matvec2d behind
// cnpint_set_debug(1048576) (A/B, parity) and for more dot vectors
// (CNPINT_MVS_MAXNS: the largest number of side vectors that still takes the staged kernel; A/B)
static bool mv2d_staged(const cnpint_ctx* c, int ns) {
  static const int maxns = [] {
    const char* e = getenv("CNPINT_MVS_MAXNS");
    return e ? atoi(e) : 0;
  }();
  return !(c->debug & 1048576) && ns <= maxns && ns <= MVS_MAXNVD;
}

template <int MODE, bool NORM, int NVD, typename... Args>
static cudaError_t launch_mv2d(cnpint_ctx* c, dim3 grid, Args... args) {
  dim3 block(32, 8);
  if constexpr (NVD <= MVS_MAXNVD) {
    if (mv2d_staged(c, NVD + (MODE >= 2 ? 1 : 0))) {
      constexpr size_t bytes = mvs_bytes(NVD + (MODE >= 2 ? 1 : 0));
      auto kern = k_matvec2d_s<MODE, NORM, NVD>;
      int done = 0;
      cudaError_t ce = cnp_dev_cached((const void*)kern, &done, [&](int* v) {
        *v = 1;
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      });
      if (ce != cudaSuccess) return ce;
      return cnp_launch(c, kern, grid, block, bytes, args...);
    }
  }
  return cnp_launch(c, k_matvec2d<MODE, NORM, NVD>, grid, block, 0, args...);
}

// ----------------------------------------------------------------------------------- launcher
template <int MODE, bool NORM>
static cudaError_t run_matvec(cnpint_ctx* c, const double* u, double* y, const double* b, double* part,
                              double* out) {
  // 𝓜 (modes 0, 2, 3) weights row t by d(t_{t+½}); P_α (mode 1) uses d̄
  const double htau = 0.5 * (MODE == 1 ? c->tau_p : c->tau);
  const double* dt = MODE == 1 ? nullptr : c->d_dt;
  const PostOp post = NORM ? c->post : PostOp{};  // pending post-fold step (cycle start)
  if (NORM) c->post = PostOp{};
  cnp_prof_begin(c, KID_MATVEC);
  if (c->dim == 1) {
    const int tchunk = mv_tchunk(c);
    dim3 block(128);
    dim3 grid((unsigned)((c->ld / 2 + 127) / 128), (unsigned)((c->N + tchunk - 1) / tchunk));
    const cudaError_t e = cnp_launch(c, k_matvec1d<MODE, NORM>, grid, block, 0, u, y, b, c->d_lo, c->d_di, c->d_up,
                                     c->N, c->ld, htau, c->alpha, tchunk, part, out, c->d_counter, DotPtrs{}, dt, post);
    if (e != cudaSuccess) return e;
  } else {
    const int tchunk = mv2_tchunk(c, MODE >= 2 ? 1 : 0);
    dim3 grid((unsigned)((c->ld + 63) / 64), (unsigned)((c->ny + 7) / 8), (unsigned)((c->N + tchunk - 1) / tchunk));
    const cudaError_t e = launch_mv2d<MODE, NORM, 0>(c, grid, u, y, b, c->N, c->nx, c->ny, c->ld, htau, c->alpha, c->xs,
                                                     c->xu, c->ys, c->yu, c->xd + c->yd + c->shift, tchunk, part, out,
                                                     c->d_counter, DotPtrs{}, dt, post);
    if (e != cudaSuccess) return e;
  }
  cnp_prof_end(c, KID_MATVEC, (MODE == 2 ? 24.0 : 16.0) * cnp_units(c));  // mode 3: 2 reads
  return cudaGetLastError();
}

template <int NVD>
static cudaError_t run_matvec_dots(cnpint_ctx* c, const double* u, double* y, const DotPtrs& vd, double* part,
                                   double* out, int ww) {
  const double htau = 0.5 * c->tau;
  cnp_prof_begin(c, KID_MATVEC);
  if (c->dim == 1) {
    const int tchunk = mv_tchunk(c);
    dim3 block(128);
    dim3 grid((unsigned)((c->ld / 2 + 127) / 128), (unsigned)((c->N + tchunk - 1) / tchunk));
    cudaError_t e;
    if (ww) {  // + ww = yᵀy and the pending post-fold step (the derived-norm probe of cnpint_gmres)
      const PostOp post = c->post;
      c->post = PostOp{};
      e = cnp_launch(c, k_matvec1d<0, false, NVD, true>, grid, block, 0, u, y, (const double*)nullptr, c->d_lo, c->d_di,
                     c->d_up, c->N, c->ld, htau, c->alpha, tchunk, part, out, c->d_counter, vd, c->d_dt, post);
    } else {
      e = cnp_launch(c, k_matvec1d<0, false, NVD>, grid, block, 0, u, y, (const double*)nullptr, c->d_lo, c->d_di,
                     c->d_up, c->N, c->ld, htau, c->alpha, tchunk, part, out, c->d_counter, vd, c->d_dt, PostOp{});
    }
    if (e != cudaSuccess) return e;
  } else {
    const int tchunk = ww ? mv2_tchunk(c, MVS_MAXNVD + 1) : mv2_tchunk(c, NVD);  // ww: always the register kernel
    dim3 grid((unsigned)((c->ld + 63) / 64), (unsigned)((c->ny + 7) / 8), (unsigned)((c->N + tchunk - 1) / tchunk));
    cudaError_t e;
    if (ww) {  // + ww = yᵀy and the pending post-fold step (the derived-norm probe of cnpint_gmres)
      const PostOp post = c->post;
      c->post = PostOp{};
      e = cnp_launch(c, k_matvec2d<0, false, NVD, true>, grid, dim3(32, 8), 0, u, y, (const double*)nullptr, c->N,
                     c->nx, c->ny, c->ld, htau, c->alpha, c->xs, c->xu, c->ys, c->yu, c->xd + c->yd + c->shift, tchunk,
                     part, out, c->d_counter, vd, (const double*)c->d_dt, post);
    } else {
      e = launch_mv2d<0, false, NVD>(c, grid, u, y, (const double*)nullptr, c->N, c->nx, c->ny, c->ld, htau, c->alpha,
                                     c->xs, c->xu, c->ys, c->yu, c->xd + c->yd + c->shift, tchunk, part, out,
                                     c->d_counter, vd, (const double*)c->d_dt, PostOp{});
    }
    if (e != cudaSuccess) return e;
  }
  cnp_prof_end(c, KID_MATVEC, (16.0 + 8.0 * NVD) * cnp_units(c));
  return cudaGetLastError();
}

// ww: also out[nv] = yᵀy, and c->post runs in the folding block
cudaError_t launch_matvec_dots(cnpint_ctx* c, const double* u, double* y, double* const* V, int nv, double* part,
                               double* out, int ww) {
  DotPtrs vd{};
  for (int i = 0; i < nv && i < CNP_MAX_DOT; ++i) vd.p[i] = V[i];
  switch (nv) {
    case 1: return run_matvec_dots<1>(c, u, y, vd, part, out, ww);
    case 2: return run_matvec_dots<2>(c, u, y, vd, part, out, ww);
    case 3: return run_matvec_dots<3>(c, u, y, vd, part, out, ww);
    case 4: return run_matvec_dots<4>(c, u, y, vd, part, out, ww);
    case 5: return run_matvec_dots<5>(c, u, y, vd, part, out, ww);
    case 6: return run_matvec_dots<6>(c, u, y, vd, part, out, ww);
    case 7: return run_matvec_dots<7>(c, u, y, vd, part, out, ww);
    case 8: return run_matvec_dots<8>(c, u, y, vd, part, out, ww);
    default: return cudaErrorInvalidValue;
  }
}

int matvec_partial_blocks(const cnpint_ctx* c) {
  if (c->dim == 1) {
    const int tchunk = mv_tchunk(c);
    return (int)(((c->ld / 2 + 127) / 128) * ((c->N + tchunk - 1) / tchunk));
  }
  return (int)(((c->ld + 63) / 64) * ((c->ny + 7) / 8) * ((c->N + 7) / 8));  // the smallest 2D time chunk
}

cudaError_t launch_matvec(cnpint_ctx* c, const double* u, double* y, int mode, const double* b, double* part,
                          double* out) {
  switch (mode) {
    case 0: return run_matvec<0, false>(c, u, y, nullptr, nullptr, nullptr);
    case 1: return run_matvec<1, false>(c, u, y, nullptr, nullptr, nullptr);
    case 2: return part ? run_matvec<2, true>(c, u, y, b, part, out) : run_matvec<2, false>(c, u, y, b, nullptr, nullptr);
    case 3: return run_matvec<3, true>(c, u, y, b, part, out);
    default: return cudaErrorInvalidValue;
  }
}
