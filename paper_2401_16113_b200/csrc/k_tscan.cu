// K6, recurrence form (round 2): the 2D time pass of P_α⁻¹ without a transform.
//
// After W⁻¹ has diagonalised L_h in space, P_α = C1^(α)⊗I − C2^(α)⊗τL_h
// is, per spatial mode μ' = τ(e_x + e_y + shift), the N×N α-circulant matrix
//     T_μ = C1^(α) − μ' C2^(α) = (1 − μ'/2) I − (1 + μ'/2) S_α,   (S_α z)_t = z_{t−1},  (S_α z)_0 = α z_{N−1},
// because C1^(α) = I − S_α and C2^(α) = ½(I + S_α) (their symbols are the λ1_k = 1 − a e^{−iθ_k},
// λ2_k = ½(1 + a e^{−iθ_k}) of Eq. 3.2 after the Γ_α scaling).  Steps (a)–(c) of Eq. 3.2
// invert T_μ by Γ_α·FFT → ÷(λ1_k − λ2_k μ') → iFFT·Γ_α⁻¹ (k_tpass2.cu, k_tpass.cu, k_tfft.cu MODE 2,
// k_fstep.cu); the same z = s·T_μ⁻¹ v is the first-order recurrence
//     z_t = ρ z_{t−1} + c v_t,   ρ = (1 + μ'/2)/(1 − μ'/2),  c = s/(1 − μ'/2),   z_{−1} = α z_{N−1}
// (s the GMRES basis scale), stable forwards because μ' < 0 ⇒ |ρ| < 1 (checked at create for every mode,
// cnpint_ctx::mu_max; otherwise the transform kernels run).  It is still parallel in time: the time axis
// is cut into J = CS·NW chunks of L rows, every chunk is scanned from a zero state by its own thread,
// the chunk ends are combined (z at a chunk end is affine in the state entering it: e + ρ^L·carry) first
// over the NW warps of a CTA through shared memory, then over the CS CTAs of a thread-block cluster
// through distributed shared memory, the cyclic closure z_{N−1} = G/(1 − αρ^N) is taken, and every
// thread adds ρ^{i+1}·carry to its rows.  A thread owns 2 adjacent columns (16-B accesses; a warp row
// access is one 512-B segment) and keeps its L rows in registers: one HBM read and one write of the
// vector, 3 fp64 instructions per unknown instead of the ≈ 100 of FFT + divide + iFFT, no shared-memory
// exchange of the data.  Measured: profiles/r02_tscan_ab.txt.
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace {

// Every power of ρ is carried as ρ^k − 1: for the smooth modes ρ = 1 + d with d = 2h/(1 − h) ≈ −4e-5, and
// a rounded ρ keeps d only to ε/|d| ≈ 3e-12 — the recurrence would then solve a slightly different mode
// (forward error 1.8e-12 for P₁ at N = 1024, or, with an exact closure denominator beside the rounded
// powers, a residual spike at t = 0: backward error 1.5e-12 at N = 2048).  With d exact to ε,
// ρx = x + dx and (1 + a)(1 + b) − 1 = a + b + ab keep every product accurate to a few ε.
CNP_DEV double2 fma2(double2 a, double2 b, double2 c) { return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y)); }
CNP_DEV double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
CNP_DEV double2 mul2(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
// (1 + a)x + y
CNP_DEV double2 rmul_add(double2 a, double2 x, double2 y) { return fma2(a, x, add2(x, y)); }
// (1 + a)² − 1
CNP_DEV double2 sq_m1(double2 a) { return make_double2(a.x * (a.x + 2.0), a.y * (a.y + 2.0)); }
// (1 + a)^n − 1, n ≥ 0, by binary exponentiation
CNP_DEV double2 pow_m1(double2 a, int n) {
  double2 r = make_double2(0.0, 0.0);
  while (n) {
    if (n & 1) r = fma2(r, a, add2(r, a));
    a = sq_m1(a);
    n >>= 1;
  }
  return r;
}

}  // namespace

// grid = ntiles·CS CTAs in clusters of CS; CTA rank r, warp w own rows [(r·NW + w)·L, +L) of the tile's
// 64 columns.  N = CS·NW·L.
template <int L, int NW, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB)
    k_tscan(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ vscale, int64_t W,
            int ld, int nx, const double* __restrict__ ex, const double* __restrict__ ey, double tau, double tau_shift,
            double alpha, int CS) {
  __shared__ double2 E1[NW][32];   // chunk ends of this CTA
  __shared__ double2 X[8][32];     // CTA aggregates of the cluster (CS ≤ 8)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  // a CTA's shared memory may be written by its peers only once it runs: arrive now, wait before the
  // remote stores of level 2
  if (CS > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const int tile = blockIdx.x / CS;
  const int col = 2 * (tile * 32 + lane);  // W = ld·ny < 2^21
  const bool ok = col < (int)W;
  const int xin = col % ld, yy = col / ld;
  const bool padA = !ok || xin >= nx, padB = !ok || xin + 1 >= nx;
  // per-column recurrence coefficients (create-time tables: before the PDL wait): d = ρ − 1 = 2h/(1 − h),
  // c = 1/(1 − h), h = μ'/2; padding columns (input and output exactly 0) take ρ = c = 0
  double2 d = make_double2(-1.0, -1.0), cc = make_double2(0.0, 0.0);
  if (!padA) {
    const double h = 0.5 * (tau * (ex[xin] + ey[yy]) + tau_shift);
    cc.x = 1.0 / (1.0 - h);
    d.x = 2.0 * h * cc.x;
  }
  if (!padB) {
    const double h = 0.5 * (tau * (ex[xin + 1] + ey[yy]) + tau_shift);
    cc.y = 1.0 / (1.0 - h);
    d.y = 2.0 * h * cc.y;
  }
  pdl_enter();  // the input and the basis scale come from earlier kernels
  const double s = vscale ? *vscale : 1.0;
  cc.x *= s;
  cc.y *= s;
  const int64_t t0 = (int64_t)(r * NW + w) * L;
  const double* const src = in + t0 * W + col;
  double2 v[L];
#pragma unroll
  for (int i = 0; i < L; ++i) v[i] = ok ? ldg_cs2(reinterpret_cast<const double2*>(src + (int64_t)i * W)) : make_double2(0.0, 0.0);
  // chunk scan from a zero state (unscaled: c is applied with the carry): s_i = ρ s_{i−1} + v_i
#pragma unroll
  for (int i = 1; i < L; ++i) v[i] = rmul_add(d, v[i - 1], v[i]);
  // level 1: the NW chunk ends of the CTA → state entering warp w's chunk relative to the CTA's (pre)
  // and the CTA's aggregate g = Σ_i P^{NW−1−i} e_i
  E1[w][lane] = v[L - 1];
  double2 dP = d;  // ρ^L − 1
#pragma unroll
  for (int q = 1; q < L; q *= 2) dP = sq_m1(dP);
  double2 dQ = dP;  // ρ^{L·NW} − 1
#pragma unroll
  for (int q = 1; q < NW; q *= 2) dQ = sq_m1(dQ);
  __syncthreads();
  double2 g = make_double2(0.0, 0.0), pre = g;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    if (i == w) pre = g;
    g = rmul_add(dP, g, E1[i][lane]);
  }
  // level 2: the CS aggregates of the cluster, the cyclic closure, the state entering CTA r
  if (CS > 1) {
    cg::cluster_group cl = cg::this_cluster();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (w == 0) {
      for (int p = 0; p < CS; ++p) {
        double2* xr = cl.map_shared_rank(&X[0][0], p);
        xr[r * 32 + lane] = g;
      }
      // only this warp wrote peer memory: it arrives with release, the others relaxed (ncu: 17 % of the
      // stall samples were every warp's release fence)
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    } else {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    if (w == 0) X[0][lane] = g;
    __syncthreads();
  }
  double2 G = make_double2(0.0, 0.0), preC = G;
  for (int i = 0; i < CS; ++i) {
    if (i == r) preC = G;
    G = rmul_add(dQ, G, X[i][lane]);
  }
  // z_{N−1} = G + αρ^N z_{N−1}, 1 − αρ^N = (1 − α) − α(ρ^N − 1); state entering CTA r: Q^r αz_{N−1} + preC;
  // entering warp w's chunk: P^w · that + pre
  const double2 dN = pow_m1(dQ, CS);
  const double2 zl = make_double2(alpha * G.x / ((1.0 - alpha) - alpha * dN.x), alpha * G.y / ((1.0 - alpha) - alpha * dN.y));
  const double2 cr = rmul_add(pow_m1(dQ, r), zl, preC);
  const double2 cin = rmul_add(pow_m1(dP, w), cr, pre);
  // z_i = c (s_i + ρ^{i+1} carry)
  double2 q = mul2(cc, cin);
  if (ok) {
    double* const dst = out + t0 * W + col;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      q = fma2(d, q, q);
      const double2 z = fma2(cc, v[i], q);
      stg_cs2(reinterpret_cast<double2*>(dst + (int64_t)i * W), z);
    }
  }
}

template <int L, int NW, int MINB>
static cudaError_t run_tscan(cnpint_ctx* c, const double* in, double* out, const double* vscale, int CS) {
  auto kern = k_tscan<L, NW, MINB>;
  const int64_t W = c->slice;
  const int ntiles = (int)((W / 2 + 31) / 32);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ntiles * CS));
  cfg.blockDim = dim3(32 * NW);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (CS > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = CS;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (c->pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, in, out, vscale, W, (int)c->ld, c->nx, (const double*)c->d_ex,
                            (const double*)c->d_ey, c->tau_p, c->tau_p * c->shift, c->alpha, CS);
}

// The recurrence form applies when every mode is stable (μ' < 0) and N = CS·NW·L has a supported
// factorisation: powers of two 8 ≤ N ≤ 2048.  CNPINT_TSCAN_CFG = "L,NW,MINB" overrides the rows per thread,
// the warps per CTA and the CTAs per SM the registers are capped for (A/B); debug bit 524288 keeps the
// transform kernels.
bool tscan_ok(const cnpint_ctx* c) {
  // any bit that selects a transform kernel (8, 16, 64, 16384, 262144), the transform's negative controls
  // (1, 2) and 524288 keep the transform path
  if (c->dim != 2 || (c->debug & (1 | 2 | 8 | 16 | 64 | 16384 | 262144 | 524288))) return false;
  if (!(c->mu_max < 0.0)) return false;
  const int N = c->N;
  return N >= 8 && N <= 2048 && (N & (N - 1)) == 0 && (c->ld % 2) == 0;
}

cudaError_t launch_tscan_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  const int N = c->N;
  int L = N >= 128 ? 16 : N / 8, NW = N >= 2048 ? 16 : 8, MB = NW == 8 ? 2 : 1;
  if (const char* e = getenv("CNPINT_TSCAN_CFG")) {
    int l = 0, nw = 0, mb = 0;
    if (sscanf(e, "%d,%d,%d", &l, &nw, &mb) == 3 && N % (l * nw) == 0 && N / (l * nw) <= 8) {
      L = l;
      NW = nw;
      MB = mb;
    }
  }
  const int CS = N / (L * NW);
  if (CS < 1 || CS > 8 || CS * L * NW != N) return cudaErrorNotSupported;
  cnp_prof_begin(c, KID_TIMEPASS2D);
  cudaError_t e = cudaErrorNotSupported;
#define TS_CASE(LL, WW, MM) \
  if (L == LL && NW == WW && MB == MM) e = run_tscan<LL, WW, MM>(c, in, out, vscale, CS);
  TS_CASE(1, 8, 2) TS_CASE(2, 8, 2) TS_CASE(4, 8, 2) TS_CASE(8, 8, 2) TS_CASE(16, 8, 2) TS_CASE(16, 16, 1)
  TS_CASE(8, 16, 2) TS_CASE(8, 16, 1) TS_CASE(16, 8, 3) TS_CASE(4, 16, 2) TS_CASE(8, 8, 4)
#undef TS_CASE
  cnp_prof_end(c, KID_TIMEPASS2D, 16.0 * cnp_units(c));
  return e;
}
