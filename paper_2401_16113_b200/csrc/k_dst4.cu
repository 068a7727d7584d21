// K5, lean x pass (round 2): one axis of W⁻¹ / W (the diagonal-similarity reading of
// k_dst.cu) on rows, as a half-length sine transform with a low instruction count per sample.
//
// Why another kernel: ncu's SASS counts (profiles/r02_dst_lean.txt) show the Stockham x pass executing
// ≈ 234 thread-instructions per sample (47 IMAD + 22 LEA of index arithmetic, 38 DADD of the odd-extension
// FFT, 17 LDS + 8 STS) and keeping 86 % of its time with every HBM access removed: it is bound by issue
// and shared-memory latency, not by HBM.  This kernel does the same transform with ≈ 30-40:
//   * half-length DST-I (see k_dst2.cu): y_j = A_j f_j + B_j f_{M−j} with A_j = (sin(jπ/M) + ½) g_j,
//     B_j = (sin(jπ/M) − ½) g_{M−j} (the pre-scale g = ρ^{−j} folded in: 2 FMAs per line and sample),
//     z = y^a + i y^b, one M-point complex FFT for two rows, F_{2k} = −Im Y_k, F_{2k+1} a prefix sum;
//   * a line pair is owned by TP = M/8 threads for its whole life (64 at M = 512): samples are loaded
//     from HBM straight into registers (coalesced rows, the mirrored sample f_{M−j} from L1), the FFT is
//     three radix-8 register passes whose exchanges stay in the pair's 8-KB shared region behind
//     named barriers of the pair alone (no CTA-wide barrier), the prefix sum is a warp-shuffle scan,
//     results leave as 16-B stores;
//   * all index arithmetic is compile time except the pair's row; tables (ω_M, A/B, post-scale) are
//     built once per persistent CTA; 4 CTAs × 256 threads per SM (64 registers, 32 warps) hide latency.
#include "common.cuh"
#include "internal.h"

#include "fft_device.cuh"
#include "post_op.cuh"

namespace {

CNP_DEV int zpos4(int k) { return k ^ ((k >> 3) & 7); }

CNP_DEV void pair_sync(int id, int nthreads) {
  if (nthreads >= 64) asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
  else __syncwarp();
}

}  // namespace

template <int LOGM>
struct D4Plan {
  static constexpr int M = 1 << LOGM, H = M / 2, n = M - 1;
  static constexpr int R1 = 8;
  static constexpr int R2 = LOGM == 7 ? 4 : 8;
  static constexpr int R3 = M / (R1 * R2);   // 8, 4, 4, 1 for LOGM = 9, 8, 7, 6
  static constexpr int TP = M / 8;           // threads per line pair
  static constexpr int NT = 256;
  static constexpr int P = NT / TP;          // line pairs per CTA
  static constexpr int I1 = (M / R1) / TP, I2 = (M / R2) / TP, I3 = (M / R3) / TP;
  // tables laid out so that a warp's reads hit distinct banks (ncu: the plain ω_M table and a
  // post-scale read at stride 16 doubles cost 2-8× the ideal shared wavefronts)
  static constexpr size_t off_tw = (size_t)P * M * 16;          // pair regions: P × M complex
  static constexpr size_t off_t2 = off_tw + (size_t)M * 16;     // T1[k1][m] = ω_M^{m k1}
  static constexpr size_t off_ab = off_t2 + (size_t)(M / R1) * 16;  // T2[k2][m3] = ω_M^{R1 m3 k2}
  static constexpr size_t off_post = off_ab + (size_t)M * 16;   // (A_j, B_j)
  static constexpr size_t bytes = off_post + (size_t)M * 8;     // post pairs [i][q]
};

#ifndef DST4_MINB
#define DST4_MINB 4
#endif

template <int LOGM>
__global__ void __launch_bounds__(256, DST4_MINB)
    k_dst4(const double* __restrict__ in, double* __restrict__ out, int nlines, int64_t ld,
           const double* __restrict__ pre, const double* __restrict__ post, const double2* __restrict__ tw2M,
           int accumulate, int debug_sign, int l2pf) {
  using PL = D4Plan<LOGM>;
  constexpr int M = PL::M, H = PL::H, n = PL::n, TP = PL::TP, P = PL::P;
  constexpr int R1 = PL::R1, R2 = PL::R2, R3 = PL::R3;
  char* const smem = reinterpret_cast<char*>(fft_smem);
  double2* const T1 = reinterpret_cast<double2*>(smem + PL::off_tw);
  double2* const T2 = reinterpret_cast<double2*>(smem + PL::off_t2);
  double2* const ab = reinterpret_cast<double2*>(smem + PL::off_ab);
  double2* const post2 = reinterpret_cast<double2*>(smem + PL::off_post);
  const int tid = threadIdx.x, pr = tid / TP, r = tid % TP;
  double2* const A = reinterpret_cast<double2*>(smem) + pr * M;  // this pair's exchange region
  // ---- tables (create-time constants): ω_M^q = ω_{2M}^{2q}; A_j, B_j; post-scale
  const double sg = debug_sign ? -1.0 : 1.0;
  // ω_M^q = ω_{2M}^{2q} (q < M, exact table); T1[k1·(M/R1) + m] = ω_M^{(m k1) mod M},
  // T2[k2·R3 + m3] = ω_M^{R1 m3 k2}; post2[i·(TP/2) + q] = (post[16q + 2i], post[16q + 2i + 1])
  auto omega = [&](int e) {
    double2 w = tw2M[2 * (e & (M - 1))];
    w.y *= sg;
    return w;
  };
  for (int q = tid; q < M; q += PL::NT) {
    const int k1 = q / (M / R1), m = q % (M / R1);
    T1[q] = omega(m * k1);
    if (q < M / R1) T2[q] = omega(R1 * (q % R3) * (q / R3));
    if (q < M / 2) {
      const int i = q / (TP / 2), l = q % (TP / 2), x = 16 * l + 2 * i;
      post2[q] = make_double2(x < n ? (post ? post[x] : 1.0) : 0.0, x + 1 < n ? (post ? post[x + 1] : 1.0) : 0.0);
    }
    double a = 0.0, b = 0.0;
    if (q > 0) {
      const double s = -tw2M[q].y;  // sin(qπ/M)
      const double gj = pre ? pre[q - 1] : 1.0, gm = pre ? pre[M - q - 1] : 1.0;
      a = (s + 0.5) * gj;
      b = (s - 0.5) * gm;
    }
    ab[q] = make_double2(a, b);
  }
  __syncthreads();
  pdl_enter();  // PDL: the rows below come from the previous kernel
  const int npairs = nlines / 2;  // N·ny is even
  const int stride = gridDim.x * P;
  const int first = blockIdx.x * P;
  const int iters = first < npairs ? (npairs - first + stride - 1) / stride : 0;  // uniform per CTA
  const int bar = 1 + pr;
  for (int it = 0; it < iters; ++it) {
    const int g = first + pr + it * stride;
    const bool act = g < npairs;
    const double* ra = in + (int64_t)(2 * g) * ld;  // rows 2g (line a) and 2g + 1 (line b)
    const double* rb = ra + ld;
    // ---- step 1: z_j = y^a_j + i y^b_j for j = m + (M/R1) n1, loaded straight from HBM
#pragma unroll
    for (int i1 = 0; i1 < PL::I1; ++i1) {
      const int m = r + i1 * TP;
      double2 v[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int j = m + (M / R1) * n1;
        double2 z = make_double2(0.0, 0.0);
        if (j > 0 && act) {
          const double2 c = ab[j];
          const double fa = __ldg(ra + j - 1), fam = __ldg(ra + M - j - 1);
          const double fb = __ldg(rb + j - 1), fbm = __ldg(rb + M - j - 1);
          z = make_double2(fma(c.x, fa, c.y * fam), fma(c.x, fb, c.y * fbm));
        }
        v[n1] = z;
      }
      dftR<R1, false>(v);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) A[k1 * (M / R1) + m] = k1 ? cmul(v[k1], T1[k1 * (M / R1) + m]) : v[0];
    }
    // the pair's next two rows (2·ld contiguous doubles; with accumulate also the output rows) into L2
    // while this pair computes: its step-1 loads then hit L2 (ncu: 21 % of the stall samples)
    if (l2pf && r < (accumulate ? 2 : 1) && g + stride < npairs)
      prefetch_l2((r == 0 ? ra : out + (ra - in)) + 2 * (int64_t)stride * ld, (unsigned)(2 * ld * 8));
    pair_sync(bar, TP);
    // ---- step 2: item (k1, m3): B[k1][m3 + R3 m2] → DFT_R2 → ω_M^{R1 m3 k2} → C (in place, swizzled)
    double2 u[PL::I2][R2];
#pragma unroll
    for (int i2 = 0; i2 < PL::I2; ++i2) {
      const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
      for (int m2 = 0; m2 < R2; ++m2) u[i2][m2] = A[k1 * (M / R1) + m3 + R3 * m2];
      dftR<R2, false>(u[i2]);
    }
    pair_sync(bar, TP);
#pragma unroll
    for (int i2 = 0; i2 < PL::I2; ++i2) {
      const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2)
        A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))] = (k2 && m3) ? cmul(u[i2][k2], T2[k2 * R3 + m3]) : u[i2][k2];
    }
    pair_sync(bar, TP);
    // ---- step 3: item (k1, k2): C → DFT_R3 → Z_k, k = k1 + R1 k2 + R1 R2 k3 (in place, swizzled)
    double2 w3[PL::I3][R3];
#pragma unroll
    for (int i3 = 0; i3 < PL::I3; ++i3) {
      const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
      for (int m3 = 0; m3 < R3; ++m3) w3[i3][m3] = A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))];
      if constexpr (R3 > 1) dftR<R3, false>(w3[i3]);
    }
    pair_sync(bar, TP);
#pragma unroll
    for (int i3 = 0; i3 < PL::I3; ++i3) {
      const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
      for (int k3 = 0; k3 < R3; ++k3) A[zpos4(k1 + R1 * k2 + R1 * R2 * k3)] = w3[i3][k3];
    }
    pair_sync(bar, TP);
    // ---- post: line ℓ (lanes [0, TP/2) → a, [TP/2, TP) → b); lane q owns k ∈ [8q, 8q+8]
    {
      const int ln = r / (TP / 2), q = r % (TP / 2);
      double Rk[8], Ik[8];
      double loc = 0.0;
#pragma unroll
      for (int i = 0; i <= 8; ++i) {
        const int k = 8 * q + i;
        const double2 Zk = A[zpos4(k & (M - 1))];
        const double2 Zm = A[zpos4((M - k) & (M - 1))];
        // Y^a = (Z_k + conj Z_{M−k})/2, Y^b = (Z_k − conj Z_{M−k})/(2i)
        const double re = ln == 0 ? 0.5 * (Zk.x + Zm.x) : 0.5 * (Zk.y + Zm.y);
        const double im = ln == 0 ? 0.5 * (Zk.y - Zm.y) : 0.5 * (Zm.x - Zk.x);
        if (i < 8) {
          Rk[i] = (k == 0) ? 0.5 * re : re;
          loc += Rk[i];
        }
        if (i > 0) Ik[i - 1] = (k < H) ? -im : 0.0;  // F_{2k} at x = 2k − 1 (F_M: the padding column)
      }
      constexpr int W = TP / 2 < 32 ? TP / 2 : 32;
      double incl = loc;
#pragma unroll
      for (int o = 1; o < W; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o, W);
        if (q % W >= o) incl += t;
      }
      double run = incl - loc;
      pair_sync(bar, TP);  // every Z read: the region takes the two staged output lines
      double* sl = reinterpret_cast<double*>(A) + ln * M;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        run += Rk[i];
        // outputs x = 16q + 2i (F_{2k+1}) and x + 1 (F_{2k+2}), k = 8q + i; x = n is the padding column
        const double2 ps = post2[i * (TP / 2) + q];
        const int x = 16 * q + 2 * i;
        sl[x ^ ((x >> 4) & 15)] = run * ps.x;           // XOR swizzle: 16 lanes → distinct banks
        sl[(x + 1) ^ ((x >> 4) & 15)] = Ik[i] * ps.y;
      }
    }
    pair_sync(bar, TP);
    if (act) {  // the two rows leave as consecutive 16-B stores (512 B per warp instruction)
      const double* sr = reinterpret_cast<const double*>(A);
#pragma unroll
      for (int e = r; e < M; e += TP) {  // e: double2 index over the 2 rows × M/2
        const int ln = e / (M / 2), x = 2 * (e - ln * (M / 2));
        const int p0 = x ^ ((x >> 4) & 15);       // x even: the pair (x, x+1) stays adjacent, maybe swapped
        const double2 s2 = *reinterpret_cast<const double2*>(sr + ln * M + (p0 & ~1));
        double2 o2 = (p0 & 1) ? make_double2(s2.y, s2.x) : s2;
        double2* dst = reinterpret_cast<double2*>(out + (int64_t)(2 * g + ln) * ld + x);
        if (accumulate) {
          const double2 pv = *dst;
          o2.x += pv.x;
          o2.y += pv.y;
        }
        stg_cs2(dst, o2);
      }
    }
    pair_sync(bar, TP);  // the region is free for the next pair's step 1
  }
}

template <int LOGM>
static cudaError_t run_dst4(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                            int accumulate) {
  using PL = D4Plan<LOGM>;
  auto kern = k_dst4<LOGM>;
  int grid_max = 0;
  cudaError_t ce = cnp_dev_cached((const void*)kern, &grid_max, [&](int* v) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PL::bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PL::NT, PL::bytes);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    *v = per_sm * c->num_sms;
    return cudaSuccess;
  });
  if (ce != cudaSuccess) return ce;
  const int nlines = c->N * c->ny;
  const int ntiles = (nlines / 2 + PL::P - 1) / PL::P;
  const int grid = ntiles < grid_max ? ntiles : grid_max;
  return cnp_launch(c, kern, dim3(grid), dim3(PL::NT), PL::bytes, in, out, nlines, c->ld, pre, post,
                    (const double2*)c->d_twx, accumulate, c->debug & 1, c->l2pf);
}

// x pass (rows) through the lean kernel when nx + 1 ∈ {64, …, 512} and ld = nx + 1; else NotSupported
cudaError_t launch_dst4_x(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                          int accumulate) {
  if (c->ld != c->nx + 1) return cudaErrorNotSupported;
  switch (c->nx + 1) {
    case 64: return run_dst4<6>(c, in, out, pre, post, accumulate);
    case 128: return run_dst4<7>(c, in, out, pre, post, accumulate);
    case 256: return run_dst4<8>(c, in, out, pre, post, accumulate);
    case 512: return run_dst4<9>(c, in, out, pre, post, accumulate);
    default: return cudaErrorNotSupported;
  }
}

// ================================================================================================
// K7 + K5 fusion (round 2; 2D right GMRES, Gram CGS2): the update of Arnoldi step j
//   Ṽ_{j+1} = w − Σ_i (c1_i + c2_i) s_i² Ṽ_i,  c2 = c1 − G̃ S² c1   (exactly k_update<NV,0,false,true,false,true>)
// with ‖Ṽ_{j+1}‖² and the Gram row Ṽ_iᵀṼ_{j+1} folded into out (post op 4: the Arnoldi finalize), fused
// with the FIRST pass of the next P_α⁻¹ — the x sine pass of W⁻¹ (D_x⁻¹ pre-scale, half-length DST-I,
// PAPER.md:315-316) of Ṽ_{j+1} — written to dout.  P_α⁻¹ is linear, so the pass may run on the
// unnormalised Ṽ_{j+1} (the basis scale s_{j+1} is folded into the time pass as before).
// Why: the update streams j + 2 vectors with the SMs idle (ncu: issue 11 %, 95 % long-scoreboard),
// the sine pass is bound on chip (issue 39 %, DRAM 42 %); in one kernel the warps of a CTA alternate
// between the two, so the pass's on-chip work hides under the update's HBM time and the pass's read
// of Ṽ_{j+1} disappears.  Each line pair is updated by the TP threads that then transform it: thread r
// forms elements r + TP·q of both rows (coalesced), stores them, accumulates the reductions, and stages
// them in the pair's region, from which step 1 reads f_j and the mirrored f_{M−j}.  The rest is k_dst4.
// The host launches it only when the next Arnoldi step is expected to run (cnpint_gmres); P_α⁻¹ then
// skips its first pass (cnpint_ctx::xdst_src).
struct VPtrsD {
  const double* p[CNP_MAX_DOT];
};

template <int LOGM, int NV>
__global__ void __launch_bounds__(256, DST4_MINB)
    k_upd_dst4(VPtrsD V, const double* __restrict__ cd, const double* __restrict__ scl, double* w,
               double* __restrict__ dout, int nlines, int64_t ld, const double* __restrict__ pre,
               const double2* __restrict__ tw2M, int debug_sign, double* __restrict__ part, int stride,
               double* __restrict__ out, unsigned* counter, PostOp post) {
  using PL = D4Plan<LOGM>;
  constexpr int M = PL::M, H = PL::H, n = PL::n, TP = PL::TP, P = PL::P;
  constexpr int R1 = PL::R1, R2 = PL::R2, R3 = PL::R3;
  char* const smem = reinterpret_cast<char*>(fft_smem);
  double2* const T1 = reinterpret_cast<double2*>(smem + PL::off_tw);
  double2* const T2 = reinterpret_cast<double2*>(smem + PL::off_t2);
  double2* const ab = reinterpret_cast<double2*>(smem + PL::off_ab);
  double2* const post2 = reinterpret_cast<double2*>(smem + PL::off_post);
  const int tid = threadIdx.x, pr = tid / TP, r = tid % TP;
  double2* const A = reinterpret_cast<double2*>(smem) + pr * M;  // this pair's region (staging, then exchanges)
  const double sg = debug_sign ? -1.0 : 1.0;
  auto omega = [&](int e) {
    double2 wv = tw2M[2 * (e & (M - 1))];
    wv.y *= sg;
    return wv;
  };
  for (int q = tid; q < M; q += PL::NT) {  // tables as k_dst4 (forward pass: no post-scale)
    const int k1 = q / (M / R1), m = q % (M / R1);
    T1[q] = omega(m * k1);
    if (q < M / R1) T2[q] = omega(R1 * (q % R3) * (q / R3));
    if (q < M / 2) {
      const int i = q / (TP / 2), l = q % (TP / 2), x = 16 * l + 2 * i;
      post2[q] = make_double2(x < n ? 1.0 : 0.0, x + 1 < n ? 1.0 : 0.0);
    }
    double a = 0.0, b = 0.0;
    if (q > 0) {
      const double s = -tw2M[q].y;  // sin(qπ/M)
      a = (s + 0.5) * pre[q - 1];
      b = (s - 0.5) * pre[M - q - 1];
    }
    ab[q] = make_double2(a, b);
  }
  __syncthreads();
  pdl_enter();  // PDL: c1, G̃, the scales and the vectors come from earlier kernels
  // the update's coefficients, as k_update's Gram form: (c1 + c2) s², c2 = c1 − G̃ S² c1
  double coef[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double c2 = cd[i];
#pragma unroll
    for (int k = 0; k < NV; ++k) c2 -= post.G[(size_t)i * post.ldh + k] * (scl[k] * scl[k] * cd[k]);
    coef[i] = (cd[i] + c2) * scl[i] * scl[i];
  }
  double acc[NV + 1];
#pragma unroll
  for (int i = 0; i <= NV; ++i) acc[i] = 0.0;
  const int npairs = nlines / 2;
  const int stride_p = gridDim.x * P;
  const int first = blockIdx.x * P;
  const int iters = first < npairs ? (npairs - first + stride_p - 1) / stride_p : 0;  // uniform per CTA
  const int bar = 1 + pr;
  for (int it = 0; it < iters; ++it) {
    const int gl = first + pr + it * stride_p;
    const bool act = gl < npairs;
    const int g = npairs - 1 - gl;  // back to front: the tail of w the matvec left in L2 is read first
    // ---- update of rows 2g, 2g+1: thread r forms the element pairs (e, e + 1), e = 2r + 2TP·q (16-B
    // accesses), staged as (row a, row b) complex samples
    const int64_t o = act ? (int64_t)(2 * g) * ld : 0;
    constexpr int UQ = NV <= 3 ? 2 : 1;  // element pairs in flight per thread (registers: 64)
#pragma unroll UQ
    for (int q = 0; q < M / (2 * TP); ++q) {
      const int e = 2 * r + 2 * TP * q;
      double2 xa = make_double2(0.0, 0.0), xb = xa;
      if (act) {
        xa = *reinterpret_cast<const double2*>(w + o + e);
        xb = *reinterpret_cast<const double2*>(w + o + ld + e);
        double2 va[NV], vb[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          va[i] = __ldcs(reinterpret_cast<const double2*>(V.p[i] + o + e));
          vb[i] = __ldcs(reinterpret_cast<const double2*>(V.p[i] + o + ld + e));
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          xa.x = fma(-coef[i], va[i].x, xa.x); xa.y = fma(-coef[i], va[i].y, xa.y);
          xb.x = fma(-coef[i], vb[i].x, xb.x); xb.y = fma(-coef[i], vb[i].y, xb.y);
        }
        *reinterpret_cast<double2*>(w + o + e) = xa;
        *reinterpret_cast<double2*>(w + o + ld + e) = xb;
        acc[0] = fma(xa.x, xa.x, fma(xa.y, xa.y, fma(xb.x, xb.x, fma(xb.y, xb.y, acc[0]))));
#pragma unroll
        for (int i = 0; i < NV; ++i)
          acc[1 + i] = fma(va[i].x, xa.x, fma(va[i].y, xa.y, fma(vb[i].x, xb.x, fma(vb[i].y, xb.y, acc[1 + i]))));
      }
      A[e] = make_double2(xa.x, xb.x);
      A[e + 1] = make_double2(xa.y, xb.y);
    }
    pair_sync(bar, TP);
    // ---- step 1 from the staged rows: z_j = y^a_j + i y^b_j, y_j = A_j f_j + B_j f_{M−j}, f_j = row[j − 1]
    double2 v1[PL::I1][R1];
#pragma unroll
    for (int i1 = 0; i1 < PL::I1; ++i1) {
      const int m = r + i1 * TP;
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int j = m + (M / R1) * n1;
        double2 z = make_double2(0.0, 0.0);
        if (j > 0) {
          const double2 c = ab[j];
          const double2 f = A[j - 1], fm = A[M - j - 1];
          z = make_double2(fma(c.x, f.x, c.y * fm.x), fma(c.x, f.y, c.y * fm.y));
        }
        v1[i1][n1] = z;
      }
    }
    pair_sync(bar, TP);  // every staged sample read: the region takes the exchanges
#pragma unroll
    for (int i1 = 0; i1 < PL::I1; ++i1) {
      const int m = r + i1 * TP;
      dftR<R1, false>(v1[i1]);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) A[k1 * (M / R1) + m] = k1 ? cmul(v1[i1][k1], T1[k1 * (M / R1) + m]) : v1[i1][0];
    }
    pair_sync(bar, TP);
    // ---- steps 2, 3, the post-processing and the store: k_dst4
    double2 u[PL::I2][R2];
#pragma unroll
    for (int i2 = 0; i2 < PL::I2; ++i2) {
      const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
      for (int m2 = 0; m2 < R2; ++m2) u[i2][m2] = A[k1 * (M / R1) + m3 + R3 * m2];
      dftR<R2, false>(u[i2]);
    }
    pair_sync(bar, TP);
#pragma unroll
    for (int i2 = 0; i2 < PL::I2; ++i2) {
      const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2)
        A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))] = (k2 && m3) ? cmul(u[i2][k2], T2[k2 * R3 + m3]) : u[i2][k2];
    }
    pair_sync(bar, TP);
    double2 w3[PL::I3][R3];
#pragma unroll
    for (int i3 = 0; i3 < PL::I3; ++i3) {
      const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
      for (int m3 = 0; m3 < R3; ++m3) w3[i3][m3] = A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))];
      if constexpr (R3 > 1) dftR<R3, false>(w3[i3]);
    }
    pair_sync(bar, TP);
#pragma unroll
    for (int i3 = 0; i3 < PL::I3; ++i3) {
      const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
      for (int k3 = 0; k3 < R3; ++k3) A[zpos4(k1 + R1 * k2 + R1 * R2 * k3)] = w3[i3][k3];
    }
    pair_sync(bar, TP);
    {
      const int ln = r / (TP / 2), q = r % (TP / 2);
      double Rk[8], Ik[8];
      double loc = 0.0;
#pragma unroll
      for (int i = 0; i <= 8; ++i) {
        const int k = 8 * q + i;
        const double2 Zk = A[zpos4(k & (M - 1))];
        const double2 Zm = A[zpos4((M - k) & (M - 1))];
        const double re = ln == 0 ? 0.5 * (Zk.x + Zm.x) : 0.5 * (Zk.y + Zm.y);
        const double im = ln == 0 ? 0.5 * (Zk.y - Zm.y) : 0.5 * (Zm.x - Zk.x);
        if (i < 8) {
          Rk[i] = (k == 0) ? 0.5 * re : re;
          loc += Rk[i];
        }
        if (i > 0) Ik[i - 1] = (k < H) ? -im : 0.0;
      }
      constexpr int WW = TP / 2 < 32 ? TP / 2 : 32;
      double incl = loc;
#pragma unroll
      for (int ofs = 1; ofs < WW; ofs <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, ofs, WW);
        if (q % WW >= ofs) incl += t;
      }
      double run = incl - loc;
      pair_sync(bar, TP);
      double* sl = reinterpret_cast<double*>(A) + ln * M;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        run += Rk[i];
        const double2 ps = post2[i * (TP / 2) + q];
        const int x = 16 * q + 2 * i;
        sl[x ^ ((x >> 4) & 15)] = run * ps.x;
        sl[(x + 1) ^ ((x >> 4) & 15)] = Ik[i] * ps.y;
      }
    }
    pair_sync(bar, TP);
    if (act) {
      const double* sr = reinterpret_cast<const double*>(A);
#pragma unroll
      for (int e = r; e < M; e += TP) {
        const int ln = e / (M / 2), x = 2 * (e - ln * (M / 2));
        const int p0 = x ^ ((x >> 4) & 15);
        const double2 s2 = *reinterpret_cast<const double2*>(sr + ln * M + (p0 & ~1));
        const double2 o2 = (p0 & 1) ? make_double2(s2.y, s2.x) : s2;
        stg_cs2(reinterpret_cast<double2*>(dout + (int64_t)(2 * g + ln) * ld + x), o2);
      }
    }
    pair_sync(bar, TP);
  }
  // block partials in the (now free) pair regions — a static array here would cost the fourth CTA per SM
  // — with block_reduce_nv's fixed order (warp trees, then warps in order), then the deterministic fold
  {
    __syncthreads();
    double* red = reinterpret_cast<double*>(smem);  // [8 warps][NV + 1]
    const int lane = tid & 31, wp = tid >> 5;
#pragma unroll
    for (int i = 0; i <= NV; ++i) {
      double v = acc[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[wp * (NV + 1) + i] = v;
    }
    __syncthreads();
    if (tid <= NV) {
      double v = 0.0;
      for (int k = 0; k < PL::NT / 32; ++k) v += red[k * (NV + 1) + tid];
      part[(size_t)blockIdx.x * stride + tid] = v;
    }
  }
  // the last block folds the partials (grid_fold's order: thread t sums blocks t, t + NT, …; warp trees;
  // warps in order), again with the pair regions as scratch
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  {
    double* red = reinterpret_cast<double*>(smem) + 8 * (NV + 1);  // [8 warps][NV + 1]
    const int lane = tid & 31, wp = tid >> 5;
    double a[NV + 1];
#pragma unroll
    for (int i = 0; i <= NV; ++i) a[i] = 0.0;
    for (int b = tid; b < (int)gridDim.x; b += PL::NT)
#pragma unroll
      for (int i = 0; i <= NV; ++i) a[i] += __ldcg(part + (size_t)b * stride + i);
#pragma unroll
    for (int i = 0; i <= NV; ++i) {
      double v = a[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[wp * (NV + 1) + i] = v;
    }
    __syncthreads();
    if (tid <= NV) {
      double v = 0.0;
      for (int k = 0; k < PL::NT / 32; ++k) v += red[k * (NV + 1) + tid];
      out[tid] = v;
    }
    if (tid == 0) *counter = 0u;
  }
  run_post(post);
}

template <int LOGM, int NV>
static cudaError_t run_upd_dst4(cnpint_ctx* c, const VPtrsD& V, const double* c1, double* w, double* dout,
                                double* part, double* out, const PostOp& post) {
  using PL = D4Plan<LOGM>;
  auto kern = k_upd_dst4<LOGM, NV>;
  int grid_max = 0;
  cudaError_t ce = cnp_dev_cached((const void*)kern, &grid_max, [&](int* v) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PL::bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PL::NT, PL::bytes);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    *v = per_sm * c->num_sms;
    return cudaSuccess;
  });
  if (ce != cudaSuccess) return ce;
  const int nlines = c->N * c->ny;
  const int ntiles = (nlines / 2 + PL::P - 1) / PL::P;
  int grid = ntiles < grid_max ? ntiles : grid_max;
  if (grid > CNP_RED_BLOCKS) grid = CNP_RED_BLOCKS;  // partial-sum rows of the fold
  return cnp_launch(c, kern, dim3(grid), dim3(PL::NT), PL::bytes, V, c1, (const double*)c->d_scl, w, dout, nlines,
                    c->ld, (const double*)c->d_dxi, (const double2*)c->d_twx, c->debug & 1, part, CNP_MAX_DOT + 1,
                    out, c->d_counter, post);
}

template <int LOGM>
static cudaError_t run_upd_dst4_nv(cnpint_ctx* c, const VPtrsD& V, int nv, const double* c1, double* w,
                                   double* dout, double* part, double* out, const PostOp& post) {
  switch (nv) {
    case 1: return run_upd_dst4<LOGM, 1>(c, V, c1, w, dout, part, out, post);
    case 2: return run_upd_dst4<LOGM, 2>(c, V, c1, w, dout, part, out, post);
    case 3: return run_upd_dst4<LOGM, 3>(c, V, c1, w, dout, part, out, post);
    case 4: return run_upd_dst4<LOGM, 4>(c, V, c1, w, dout, part, out, post);
    case 5: return run_upd_dst4<LOGM, 5>(c, V, c1, w, dout, part, out, post);
    case 6: return run_upd_dst4<LOGM, 6>(c, V, c1, w, dout, part, out, post);
    case 7: return run_upd_dst4<LOGM, 7>(c, V, c1, w, dout, part, out, post);
    case 8: return run_upd_dst4<LOGM, 8>(c, V, c1, w, dout, part, out, post);
    default: return cudaErrorInvalidValue;
  }
}

// Can the Gram update of this handle carry the next x sine pass (the lean x pass applies and no debug
// bit selects another x-pass kernel)?  debug 131072 turns the fusion off (A/B).
bool upd_dst_ok(const cnpint_ctx* c) {
  if (c->dim != 2 || c->ld != c->nx + 1) return false;
  if (c->debug & (32 | 256 | 4096 | 32768 | 131072)) return false;
  return c->nx + 1 == 64 || c->nx + 1 == 128 || c->nx + 1 == 256 || c->nx + 1 == 512;
}

// The Gram CGS2 update of Arnoldi step nv − 1 (as launch_cgs2_pass phase 2) fused with the x sine pass of
// the new vector into dout; consumes the pending post op (Arnoldi finalize).
cudaError_t launch_cgs2_pass_dst(cnpint_ctx* c, double* const* Vp, int nv, const double* c1, double* w,
                                 double* part, double* out, double* dout) {
  if (nv < 1 || nv > CNP_MAX_DOT || !upd_dst_ok(c)) return cudaErrorInvalidValue;
  VPtrsD V;
  for (int i = 0; i < CNP_MAX_DOT; ++i) V.p[i] = i < nv ? Vp[i] : nullptr;
  const PostOp post = c->post;
  c->post = PostOp{};
  cnp_prof_begin(c, KID_UPD_DST);
  cudaError_t e;
  switch (c->nx + 1) {
    case 64: e = run_upd_dst4_nv<6>(c, V, nv, c1, w, dout, part, out, post); break;
    case 128: e = run_upd_dst4_nv<7>(c, V, nv, c1, w, dout, part, out, post); break;
    case 256: e = run_upd_dst4_nv<8>(c, V, nv, c1, w, dout, part, out, post); break;
    default: e = run_upd_dst4_nv<9>(c, V, nv, c1, w, dout, part, out, post); break;
  }
  cnp_prof_end(c, KID_UPD_DST, 8.0 * cnp_units(c) * (nv + 2) + 8.0 * cnp_units(c));  // update + the pass's write
  return e;
}
