// Four-step time FFTs of P_α⁻¹ (Eq. 3.2 steps (a)-(c), Remark 3.1), same
// definitions as k_tfft.cu:
//   K2  (MODE 0, 1D)  ŵ_k[x] = Σ_t e^{−2πikt/N} · γ_t · s · v_t[x],  k = 0..N/2
//   K4  (MODE 1, 1D)  z_t[x] = 1/(N γ_t) · Σ_{k<N} e^{+2πikt/N} ẑ_k[x],  ẑ_{N−k} = conj ẑ_k
//   K6  (MODE 2, 2D)  z_t = 1/(N γ_t) · iFFT_k[ FFT_t(γ s v)_k / (λ1_k − λ2_k μ) ]  per spatial mode
//                     column (μ = τ(e_x + e_y) + τ·shift)
//
// Why another decomposition.  The cluster kernel keeps all N rows of a column tile on chip, so at
// N = 4096 a tile is only 8 real columns wide (64-B row segments) and its loads run at ~2 TB/s
// (profiles/r01_tilecopy_pattern.txt, r01_tfft_phases.txt).  Here N = N1·N2, t = t1 + N1 t2,
// k = k2 + N2 k1 and
//   pass A  Y[t1][k2] = ω_N^{t1 k2} · FFT_{N2}( γ_t s v_{t1 + N1 t2} )[k2]            (per t1)
//   pass B  X[k2 + N2 k1] = FFT_{N1}( Y[·][k2] )[k1]                                 (per k2)
// (inverse: the same two passes backwards with conjugate twiddles; MODE 2 runs forward pass B, the
// spectral divide and inverse pass A' in one family item, so the 2D time pass is three phases).
// Each pass moves tiles of 2·NC real columns.  The intermediate Y of a column block goes through L2
// only: all phases run in ONE persistent kernel whose work items are handed out in ticket order —
// phase-0 items of block b, phase-1 items of block b − L, phase-2 items of block b − 2L — and an
// item of a later phase waits on its block's counter until the earlier phases of the block have
// landed.  The last reader of a Y row drops it from L2 (discard.global.L2), so Y is never written
// back to HBM: HBM traffic is one read of the input and one write of the output.  Deadlock
// freedom: an item only waits for items with smaller tickets, which were taken by CTAs that are
// already running and whose phase-0 items never wait.
// Two real columns (a, b) are packed as one complex column z_t = v_t[a] + i v_t[b]; the Hermitian
// separation X_a[k] = (Z_k + conj Z_{N−k})/2, X_b[k] = (Z_k − conj Z_{N−k})/(2i) pairs k2 with
// N2 − k2, so the pass-B items are frequency families {k2, N2 − k2}, k2 = 0..N2/2.
#include "common.cuh"
#include "internal.h"

#include <cstdlib>

#include "fft_tile.cuh"

#ifndef FS_NC6
#define FS_NC6 16  // pair columns per block when N1, N2 = 64 (8 threads per column; 32 measured slower)
#endif
#ifndef FS_NC5
#define FS_NC5 32  // pair columns per block when max(N1, N2) <= 32 (2D time pass, N <= 1024)
#endif
#ifndef FS_TT6
#define FS_TT6 1  // t1 values per t1 item when N1, N2 = 64 (2 measured slower: 166 registers, fewer CTAs)
#endif
#ifndef FS_NC7
#define FS_NC7 16  // pair columns per block when max(N1, N2) >= 128 (16 threads per column)
#endif
#ifndef FS_MINB6
#define FS_MINB6 0  // CTAs per SM for N1, N2 <= 64 (0: 768 threads per SM)
#endif
#ifndef FS_MINB7
#define FS_MINB7 2
#endif

// timing-experiment knob (CNPINT_FS_SKIP): compiled out of product builds
#ifdef CNPINT_EXPERIMENTS
#define FS_SKIP(b) (a.skip & (b))
#else
#define FS_SKIP(b) 0
#endif

namespace {

CNP_DEV void fs_separate(double2 zk, double2 zm, double2& xa, double2& xb) {
  xa = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
  xb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
}
CNP_DEV double2 fs_pack(double2 xa, double2 xb) { return make_double2(xa.x - xb.y, xa.y + xb.x); }

CNP_DEV unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CNP_DEV void discard_l2(const void* p) { asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory"); }
template <bool INV>
CNP_DEV double2 twm(double2 a, double2 w) {  // a·w (forward) or a·conj(w) (inverse)
  return INV ? cmul_conj(a, w) : cmul(a, w);
}

// Register FFT of length L = R1·R2 over one column, two thread roles (Cooley–Tukey, n = n2 + R2 n1,
// k = k1 + R1 k2):  step 1 — thread n2 holds x[n2 + R2 n1] (n1 < R1), R1-point DFT in registers,
// twiddle ω_L^{n2 k1}, write A[k1][n2] to the column's exchange area; step 2 — thread k1 reads
// A[k1][·], R2-point DFT → X[k1 + R1 k2] (k2 < R2).  One shared-memory round trip per pass
// (the Stockham version of fft_tile.cuh makes one per radix stage).  The transposed plan (R2, R1)
// takes its input exactly as the plan (R1, R2) leaves its output in the threads, which MODE 2
// uses to go from the forward to the inverse transform without an exchange.
template <int A_, int B_>
struct RP {
  static constexpr int R1 = A_, R2 = B_, L = A_ * B_;
  static constexpr int SK = R2 + 1;          // exchange layout A[k1][n2] at k1·SK + n2
  static constexpr int G1 = R1 + 1;          // gather layout x[n2 + R2 n1] at n2·G1 + n1
  static constexpr int S1 = R1 * SK, S2 = R2 * G1;
  static constexpr int SC = (S1 > S2 ? S1 : S2) | 1;  // odd per-column stride: lanes = columns, conflict free
};
__host__ __device__ constexpr int rf_r1(int logl) { return logl >= 8 ? 16 : logl >= 6 ? 8 : 4; }
template <int LOGL>
using RF = RP<rf_r1(LOGL), (1 << LOGL) / rf_r1(LOGL)>;
template <int LOGL>
using RFT = RP<(1 << LOGL) / rf_r1(LOGL), rf_r1(LOGL)>;

template <class F, bool INV>
CNP_DEV void rf_step1(double2 (&v)[F::R1], double2* col, const double2* twL, int n2) {
  dftR<F::R1, INV>(v);
#pragma unroll
  for (int k1 = 1; k1 < F::R1; ++k1) v[k1] = twm<INV>(v[k1], twL[n2 * k1]);
#pragma unroll
  for (int k1 = 0; k1 < F::R1; ++k1) col[k1 * F::SK + n2] = v[k1];
}
template <class F, bool INV>
CNP_DEV void rf_step2(double2 (&u)[F::R2], const double2* col, int k1) {
#pragma unroll
  for (int n2 = 0; n2 < F::R2; ++n2) u[n2] = col[k1 * F::SK + n2];
  dftR<F::R2, INV>(u);
}

// compile-time geometry: blocks of NC pair columns; t1 items hold NC columns, family items NC
// columns = 2 members × NF pairs (half of the block's pairs)
template <int MODE, int LOG1, int LOG2>
struct FsGeo {
  static constexpr int N1 = 1 << LOG1, N2 = 1 << LOG2, N = N1 * N2, H = N / 2;
  static constexpr int MX = LOG1 > LOG2 ? LOG1 : LOG2;
  static constexpr int NC = MX <= 5 ? FS_NC5 : MX == 6 ? FS_NC6 : FS_NC7;
  static constexpr int NF = NC / 2;
  // t1 items take TT consecutive t1 values (independent FFTs interleaved in every thread: more
  // memory- and instruction-level parallelism per item, fewer items)
  static constexpr int TT = MX == 6 ? FS_TT6 : 1;
  static constexpr int AREA_T = TT * NC * RF<LOG2>::SC, AREA_F = NC * RF<LOG1>::SC;
  static constexpr int off_tw1 = AREA_T > AREA_F ? AREA_T : AREA_F;  // ω_{N1}^j, j < N1
  static constexpr int off_tw2 = off_tw1 + N1;       // ω_{N2}^j
  static constexpr int off_twn = off_tw2 + N2;       // per-item ω_N table [2·max(N1, N2)]
  static constexpr int NTW = 2 * (N1 > N2 ? N1 : N2);
  static constexpr int off_lam = off_twn + NTW;      // MODE 2: λ1[H+1], λ2[H+1]
  static constexpr int NLAM = MODE == 2 ? 2 * (H + 1) : 0;
  static constexpr int HI = N / 64;
  static constexpr int off_g = off_lam + NLAM;       // doubles: ghi[HI] glo[64] ihi[HI] ilo[64]
  static constexpr size_t bytes = (size_t)(off_g + (2 * (HI + 64)) / 2 + 1) * 16;
  static constexpr int TP1 = RF<LOG1>::R1 > RF<LOG1>::R2 ? RF<LOG1>::R1 : RF<LOG1>::R2;
  static constexpr int TP2 = RF<LOG2>::R1 > RF<LOG2>::R2 ? RF<LOG2>::R1 : RF<LOG2>::R2;
  static constexpr int NT = NC * (TP1 > TP2 ? TP1 : TP2);  // threads: tid = col + NC·j
  static constexpr int MINB = (MX <= 6 && MODE != 2) ? (FS_MINB6 > 0 ? FS_MINB6 : NT <= 384 ? 768 / NT / TT : 1)
                                                   : MODE == 2 ? 2 : FS_MINB7;
  // items per block and phase (see k_fstep); PER = slots per schedule step
  static constexpr int NFAM = 2 * (N2 / 2 + 1);
  static constexpr int NP0 = MODE == 1 ? NFAM : N1 / TT, NP1 = MODE == 2 ? NFAM : 0, NP2 = MODE == 0 ? NFAM : N1 / TT;
  static constexpr int PER = NP0 + NP1 + NP2;
};

}  // namespace

// Work-item order.  Step s (0 ≤ s < nxb + lag_2) lists n[0] slots for phase 0 of block s, n[1] slots
// for phase 1 of block s − lag_1 and n[2] slots for phase 2 of block s − lag_2 (lag_0 = 0 ≤ lag_1 ≤
// lag_2; n[1] = 0 for the two-phase 1D transforms); a slot whose block is out of range is empty
// (its ticket is skipped), which keeps the ticket → item map a division and a few compares.
struct FsSched {
  int nxb, n[3], lag[3];
  unsigned total;
};

template <class G>
CNP_DEV bool fs_item(const FsSched& S, unsigned T, int& ph, int& xb, int& idx) {
  const int st = (int)(T / (unsigned)G::PER);  // constant divisor
  const int r = (int)(T - (unsigned)st * G::PER);
  ph = r < G::NP0 ? 0 : r < G::NP0 + G::NP1 ? 1 : 2;
  idx = ph == 0 ? r : ph == 1 ? r - G::NP0 : r - G::NP0 - G::NP1;
  xb = st - (ph == 0 ? 0 : ph == 1 ? S.lag[1] : S.lag[2]);
  return xb >= 0 && xb < S.nxb;
}

CNP_DEV void fs_wait(const unsigned* cnt, unsigned target) {
  if (threadIdx.x == 0)
    while ((int)(ld_acquire(cnt) - target) < 0) __nanosleep(32);
  __syncthreads();
}
CNP_DEV void fs_signal(unsigned* cnt) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // cumulative over the CTA's stores ordered before it by the barrier
    atomicAdd(cnt, 1u);
  }
}

struct FsArgs {
  const double* vin;
  const double2* spin;
  double* vout;
  double2* spout;
  double2* Y;
  const double* vscale;
  const double* gam;
  const double* igam;
  const double2* twN;  // ω_N^q, q < N (host long-double table, debug sign applied)
  const double2* lam1;
  const double2* lam2;
  const double* ex;
  const double* ey;
  double tau, tau_shift;
  int W, ld, nx, accumulate, debug_sign, no_discard;
  int skip;  // timing experiments only (CNPINT_FS_SKIP): 1 no input loads, 2 no spectrum stores, 4 no Y traffic
  unsigned* cnt;
  unsigned* ticket;
  unsigned tick_base, base;
};

// Item kinds by mode and phase:
//   MODE 0: phase 0 forward t1 items (input → Y), phase 2 forward family items (Y → spectrum)
//   MODE 1: phase 0 inverse family items (spectrum → Y), phase 2 inverse t1 items (Y → output)
//   MODE 2: phase 0 forward t1 items, phase 1 fused family items (Y → forward, divide, inverse → Y),
//           phase 2 inverse t1 items
// Family item index = 2·k2 + h (h: which half of the block's pair columns).  Threads:
// tid = col + NC·j, j = the role index of the register FFT.
template <int MODE, int LOG1, int LOG2>
__global__ void __launch_bounds__(FsGeo<MODE, LOG1, LOG2>::NT, FsGeo<MODE, LOG1, LOG2>::MINB)
    k_fstep(FsArgs a, FsSched S) {
  using G = FsGeo<MODE, LOG1, LOG2>;
  using F1 = RF<LOG1>;   // family items: length N1
  using F1T = RFT<LOG1>; // MODE 2: the inverse over k1, transposed plan
  using F2 = RF<LOG2>;   // t1 items: length N2
  constexpr int NT = G::NT;
  constexpr int N1 = G::N1, N2 = G::N2, N = G::N, H = G::H, NC = G::NC, NF = G::NF;
  constexpr int X = 2 * NC;  // real columns per block
  const int tid = threadIdx.x;
  const int col = tid % NC, j = tid / NC;
  const int W = a.W;
  double2* const buf = tf_smem;
  double2* const tw1 = tf_smem + G::off_tw1;
  double2* const tw2 = tf_smem + G::off_tw2;
  double2* const twn = tf_smem + G::off_twn;
  double2* const l1s = tf_smem + G::off_lam;
  double2* const l2s = l1s + (H + 1);
  double* const ghi = reinterpret_cast<double*>(tf_smem + G::off_g);
  double* const glo = ghi + G::HI;
  double* const ihi = glo + 64;
  double* const ilo = ihi + G::HI;
  __shared__ unsigned s_tk[2];  // ticket of item i in s_tk[i & 1]

  // ---- per-CTA tables once: ω_{N1}, ω_{N2}; Γ_α and 1/(NΓ_α) as two-level tables
  //      g_t = ghi[t >> 6]·glo[t & 63], 1/(Nγ_t) = ihi[t >> 6]·ilo[t & 63] (ilo carries the N back)
  const double sg = a.debug_sign ? -1.0 : 1.0;
  for (int q = tid; q < N1; q += NT) { double2 w = expi_neg(q, N1); w.y *= sg; tw1[q] = w; }
  for (int q = tid; q < N2; q += NT) { double2 w = expi_neg(q, N2); w.y *= sg; tw2[q] = w; }
  if (MODE != 1) {
    for (int q = tid; q < G::HI; q += NT) ghi[q] = __ldg(a.gam + q * 64);
    for (int q = tid; q < 64; q += NT) glo[q] = __ldg(a.gam + q);
  }
  if (MODE != 0) {
    for (int q = tid; q < G::HI; q += NT) ihi[q] = __ldg(a.igam + q * 64);
    for (int q = tid; q < 64; q += NT) ilo[q] = (double)N * __ldg(a.igam + q);
  }
  if (MODE == 2)
    for (int q = tid; q <= H; q += NT) { l1s[q] = a.lam1[q]; l2s[q] = a.lam2[q]; }
  // PDL: the tables above come from create-time constants; everything below may read what the previous
  // kernel on the stream wrote (the basis scale, the input, the shared ticket counters)
  pdl_enter();
  const double s = (MODE != 1 && a.vscale) ? *a.vscale : 1.0;
  if (tid == 0) s_tk[0] = atomicAdd(a.ticket, 1u) - a.tick_base;

  for (int it = 0;; ++it) {
    __syncthreads();  // previous item done with buf / twn; s_tk[it & 1] published
    const unsigned T = s_tk[it & 1];
    if (T >= S.total) break;
    unsigned nxt = 0;  // next ticket requested now, published in the other slot at the end
    if (tid == 0) nxt = atomicAdd(a.ticket, 1u);
    int ph, xb, idx;
    if (!fs_item<G>(S, T, ph, xb, idx)) {  // empty slot (schedule edge)
      if (tid == 0) s_tk[(it + 1) & 1] = nxt - a.tick_base;
      continue;
    }
    const int col0 = xb * X;
    double2* const Yb = a.Y + (size_t)xb * N * NC;  // block's Y: [t1][k2][c], c < NC
    const bool fwd_t1 = MODE != 1 && ph == 0;
    const bool inv_t1 = MODE != 0 && ph == 2;
    if (ph > 0) fs_wait(a.cnt + xb, a.base + (unsigned)(ph == 1 ? G::NP0 : G::NP0 + G::NP1));

    if (fwd_t1 || inv_t1) {
      // ================= t1 items (length N2): forward pass A or inverse pass B' for the TT rows
      //                   t1 = idx·TT + tt (TT interleaved transforms per thread)
      constexpr int TT = G::TT;
      const int t1b = idx * TT;
      const int mycol = col0 + 2 * col;
      const int xin = MODE == 2 ? mycol % a.ld : mycol;  // 1D: W = ld
      const bool padA = xin >= a.nx, padB = xin + 1 >= a.nx, colok = mycol < W;
      if (fwd_t1)
        for (int q = tid; q < TT * N2; q += NT) {  // ω_N^{t1 k2} for each t1 of the item
          const int tt = q / N2, k2 = q - tt * N2;
          twn[q] = __ldg(a.twN + (((t1b + tt) * k2) & (N - 1)));
        }
      if (j < F2::R2) {
        const int n2 = j;
        double2 v[TT][F2::R1];
        if (fwd_t1) {
#pragma unroll
          for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int n1 = 0; n1 < F2::R1; ++n1) {
              const int t = t1b + tt + N1 * (n2 + F2::R2 * n1);
              v[tt][n1] = (colok && !FS_SKIP(1)) ? ldg_cs2(reinterpret_cast<const double2*>(a.vin + (int64_t)t * W + mycol))
                                                   : make_double2(0.0, 0.0);
            }
          double gls[TT];
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) gls[tt] = glo[(t1b + tt) & 63] * s;
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
            for (int n1 = 0; n1 < F2::R1; ++n1) {
              const int t = t1b + tt + N1 * (n2 + F2::R2 * n1);
              // g_t: for N1 ≥ 64, t & 63 = t1 & 63 and t >> 6 = (t1 >> 6) + (N1/64)(n2 + R2 n1)
              const double g = N1 >= 64 ? ghi[((t1b + tt) >> 6) + (N1 >> 6) * (n2 + F2::R2 * n1)] * gls[tt]
                                        : ghi[t >> 6] * glo[t & 63] * s;
              v[tt][n1] = cscale(v[tt][n1], g);
            }
            rf_step1<F2, false>(v[tt], buf + (tt * NC + col) * F2::SC, tw2, n2);
          }
        } else {
#pragma unroll
          for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int n1 = 0; n1 < F2::R1; ++n1)
              v[tt][n1] = __ldcg(Yb + ((size_t)(t1b + tt) * N2 + n2 + F2::R2 * n1) * NC + col);
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) rf_step1<F2, true>(v[tt], buf + (tt * NC + col) * F2::SC, tw2, n2);
        }
      }
      __syncthreads();
      if (inv_t1 && !a.no_discard) {  // these t1's Y rows: TT·N2·NC·16 B, contiguous, last reader
        const char* src = reinterpret_cast<const char*>(Yb + (size_t)t1b * N2 * NC);
        for (int q = tid; q < TT * N2 * NC * 16 / 128; q += NT) discard_l2(src + q * 128);
      }
      if (j < F2::R1) {
        const int k1 = j;
        double2 u[TT][F2::R2];
        if (fwd_t1) {
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) rf_step2<F2, false>(u[tt], buf + (tt * NC + col) * F2::SC, k1);
        } else {
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) rf_step2<F2, true>(u[tt], buf + (tt * NC + col) * F2::SC, k1);
        }
        if (fwd_t1) {
#pragma unroll
          for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int k2 = 0; k2 < F2::R2; ++k2) {
              const int kk = k1 + F2::R1 * k2;  // pass frequency k2' of the four-step
              if (!FS_SKIP(4))
                Yb[((size_t)(t1b + tt) * N2 + kk) * NC + col] = cmul(u[tt][k2], twn[tt * N2 + kk]);
            }
        } else if (colok) {
#pragma unroll
          for (int tt = 0; tt < TT; ++tt)
#pragma unroll
            for (int k2 = 0; k2 < F2::R2; ++k2) {
              const int t = t1b + tt + N1 * (k1 + F2::R1 * k2);
              const double g = N1 >= 64 ? ihi[((t1b + tt) >> 6) + (N1 >> 6) * (k1 + F2::R1 * k2)] * ilo[(t1b + tt) & 63]
                                        : ihi[t >> 6] * ilo[t & 63];
              double2 val = make_double2(padA ? 0.0 : u[tt][k2].x * g, padB ? 0.0 : u[tt][k2].y * g);
              double2* dst = reinterpret_cast<double2*>(a.vout + (int64_t)t * W + mycol);
              if (a.accumulate) {
                const double2 o = *dst;
                val.x += o.x;
                val.y += o.y;
              }
              stg_cs2(dst, val);
            }
        }
      }
      if (fwd_t1) fs_signal(a.cnt + xb);
    } else {
      // ================= family items {k2, N2 − k2} × half block h (length N1).  Column
      //                   col = m·NF + p: member m, pair h·NF + p.
      const int k2 = idx >> 1, h = idx & 1;
      const int k2m = (N2 - k2) & (N2 - 1);
      const bool two = k2m != k2;
      const int m = col / NF, p = col - m * NF;
      const int km = m ? k2m : k2;
      const bool active = m == 0 || two;
      const int gp = h * NF + p;
      const int mycol = col0 + 2 * gp;
      const int xin = MODE == 2 ? mycol % a.ld : mycol;  // 1D: W = ld
      const bool padA = xin >= a.nx, padB = xin + 1 >= a.nx, colok = mycol < W;
      double2* const fb = buf + col * F1::SC;
      // partner of frequency index ko of this column (Hermitian pairing k ↔ N − k)
      auto partner = [&](int ko, int& pcol, int& pko) {
        if (m == 1) { pcol = col - NF; pko = N1 - 1 - ko; }
        else if (k2 == 0) { pcol = col; pko = (N1 - ko) & (N1 - 1); }
        else if (!two) { pcol = col; pko = N1 - 1 - ko; }
        else { pcol = col + NF; pko = N1 - 1 - ko; }
      };
      if (MODE == 0 || MODE == 2) {
        // ---- forward pass B over t1: Y rows (t1, km) of this half block
        if (j < F1::R2) {
          const int n2 = j;
          double2 v[F1::R1];
#pragma unroll
          for (int n1 = 0; n1 < F1::R1; ++n1)
            v[n1] = (active && !FS_SKIP(4)) ? __ldcg(Yb + ((size_t)(n2 + F1::R2 * n1) * N2 + km) * NC + gp)
                                              : make_double2(0.0, 0.0);
          rf_step1<F1, false>(v, fb, tw1, n2);
        }
        __syncthreads();
        if (MODE == 0 && !a.no_discard) {  // rows (t1, km): NF·16 B at each of N1 rows, 2 members
          constexpr int LPR = NF * 16 / 128;
          for (int q = tid; q < 2 * N1 * LPR; q += NT) {
            const int mm = q / (N1 * LPR), r = q - mm * N1 * LPR;
            const int t1 = r / LPR, l = r - t1 * LPR;
            if (mm == 1 && !two) continue;
            const char* ad = reinterpret_cast<const char*>(Yb + ((size_t)t1 * N2 + (mm ? k2m : k2)) * NC + h * NF);
            discard_l2(ad + l * 128);
          }
        }
        double2 u[F1::R2];
        if (j < F1::R1) rf_step2<F1, false>(u, fb, j);
        __syncthreads();  // every thread has read its exchange row: the areas now take X
        if (j < F1::R1) {
#pragma unroll
          for (int k2i = 0; k2i < F1::R2; ++k2i) fb[j * F1::SK + k2i] = u[k2i];  // X[k1 + R1 k2] at k1·SK + k2
        }
        if (MODE == 2)
          for (int q = tid; q < N1; q += NT) {  // ω_N^{k2 t1}, ω_N^{k2m t1} (conjugated at use)
            twn[q] = __ldg(a.twN + ((k2 * q) & (N - 1)));
            twn[N1 + q] = __ldg(a.twN + ((k2m * q) & (N - 1)));
          }
        __syncthreads();
        if (MODE == 0) {
          if (j < F1::R1 && active && colok) {
            const int k1 = j;
#pragma unroll
            for (int k2i = 0; k2i < F1::R2; ++k2i) {
              const int ko = k1 + F1::R1 * k2i;  // outer frequency: spectrum row km + N2·ko
              const int k = km + N2 * ko;
              if (k > H) continue;
              int pcol, pko;
              partner(ko, pcol, pko);
              const double2 zm = buf[pcol * F1::SC + (pko % F1::R1) * F1::SK + pko / F1::R1];
              double2 xa, xbv;
              fs_separate(u[k2i], zm, xa, xbv);
              if (padA) xa = make_double2(0.0, 0.0);
              if (padB) xbv = make_double2(0.0, 0.0);
              double2* o = a.spout + (int64_t)k * W + mycol;
              if (!FS_SKIP(2)) {
                stg_cs2(o, xa);
                stg_cs2(o + 1, xbv);
              }
            }
          }
        } else {
          // ---- MODE 2: divide every frequency of the member by (λ1_k − λ2_k μ) per real column,
          //      repack, inverse over k1 with the transposed plan (input = this thread's values)
          double2 z[F1::R2];
          if (j < F1::R1) {
            const int k1 = j;
            double mua = 1.0, mub = 1.0;  // padding columns: μ = 1 (α = 1 has λ1_0 = 0; see k_tpass2.cu)
            if (colok && !padA) {
              const int yy = mycol / a.ld;
              mua = a.tau * (a.ex[xin] + a.ey[yy]) + a.tau_shift;
              if (!padB) mub = a.tau * (a.ex[xin + 1] + a.ey[yy]) + a.tau_shift;
            }
#pragma unroll
            for (int k2i = 0; k2i < F1::R2; ++k2i) {
              const int ko = k1 + F1::R1 * k2i;
              const int k = km + N2 * ko;
              int pcol, pko;
              partner(ko, pcol, pko);
              const double2 zm = buf[pcol * F1::SC + (pko % F1::R1) * F1::SK + pko / F1::R1];
              double2 xa, xbv;
              fs_separate(u[k2i], zm, xa, xbv);
              const double2 l1 = k <= H ? l1s[k] : cconj(l1s[N - k]);
              const double2 l2 = k <= H ? l2s[k] : cconj(l2s[N - k]);
              xa = cmul(xa, crecip(csub(l1, cscale(l2, mua))));
              xbv = cmul(xbv, crecip(csub(l1, cscale(l2, mub))));
              z[k2i] = (k == 0 || k == H) ? make_double2(xa.x, xbv.x) : fs_pack(xa, xbv);
            }
          }
          __syncthreads();  // all partner reads of X done: the areas take the inverse exchange
          if (j < F1T::R2) rf_step1<F1T, true>(z, fb, tw1, j);
          __syncthreads();
          if (j < F1T::R1 && active) {
            const int k1 = j;
            double2 w2[F1T::R2];
            rf_step2<F1T, true>(w2, fb, k1);
#pragma unroll
            for (int k2i = 0; k2i < F1T::R2; ++k2i) {
              const int t1 = k1 + F1T::R1 * k2i;
              Yb[((size_t)t1 * N2 + km) * NC + gp] = cmul_conj(w2[k2i], twn[m * N1 + t1]);
            }
          }
          fs_signal(a.cnt + xb);
        }
      } else {
        // ---- MODE 1 pass A': every step-1 thread loads the Z values of its own column straight from
        //      the stored half spectrum: Z_k for k = km + N2 j ≤ H from row k, else the conjugate of
        //      row N − k (the partner member's row, or the own member's for the self-paired
        //      families) — each row is read by both member columns (the second read hits L2/L1)
        for (int q = tid; q < N1; q += NT) {  // ω_N^{k2 t1}, ω_N^{k2m t1} (conjugated at use)
          twn[q] = __ldg(a.twN + ((k2 * q) & (N - 1)));
          twn[N1 + q] = __ldg(a.twN + ((k2m * q) & (N - 1)));
        }
        double2 v[F1::R1];
        if (j < F1::R2) {
          const int n2 = j;
          double2 ga[F1::R1], gb[F1::R1];
#pragma unroll
          for (int n1 = 0; n1 < F1::R1; ++n1) {  // all loads first
            const int jj = n2 + F1::R2 * n1;
            const int k = km + N2 * jj;
            const int kr = k <= H ? k : N - k;
            ga[n1] = gb[n1] = make_double2(0.0, 0.0);
            if (active && colok) {
              const double2* src = a.spin + (int64_t)kr * W + mycol;
              ga[n1] = ldg_cs2(src);
              gb[n1] = ldg_cs2(src + 1);
            }
          }
#pragma unroll
          for (int n1 = 0; n1 < F1::R1; ++n1) {
            const int k = km + N2 * (n2 + F1::R2 * n1);
            const double2 xa = ga[n1], xbv = gb[n1];
            v[n1] = (k == 0 || k == H) ? make_double2(xa.x, xbv.x)
                    : k < H ? fs_pack(xa, xbv) : fs_pack(cconj(xa), cconj(xbv));
          }
        }
        __syncthreads();  // twn ready; the previous users of the areas are done
        if (j < F1::R2) rf_step1<F1, true>(v, fb, tw1, j);
        __syncthreads();
        if (j < F1::R1 && active) {
          const int k1 = j;
          double2 u[F1::R2];
          rf_step2<F1, true>(u, fb, k1);
#pragma unroll
          for (int k2i = 0; k2i < F1::R2; ++k2i) {
            const int t1 = k1 + F1::R1 * k2i;
            Yb[((size_t)t1 * N2 + km) * NC + gp] = cmul_conj(u[k2i], twn[m * N1 + t1]);
          }
        }
        fs_signal(a.cnt + xb);
      }
    }
    // publish the next ticket in the other slot (its readers passed this item's first barrier; the
    // loop-top barrier publishes it)
    if (tid == 0) s_tk[(it + 1) & 1] = nxt - a.tick_base;
  }
}

// ------------------------------------------------------------------------------------ host side
static void fs_logs(int N, int& l1, int& l2) {
  int logN = 0;
  while ((1 << logN) < N) ++logN;
  l1 = (logN + 1) / 2;
  l2 = logN - l1;
}

// 2D: from N = 2048 on (the cluster kernel's own range ends in C = 8 clusters there); at N ≤ 1024 the
// items of the three-phase pass are 8–16 KB and the cluster kernel measured faster (c4: 326 vs 781
// µs, profiles/r01_k6_sweep.txt)
static int fs_min2d() {  // CNPINT_FS_2D_MIN: tuning experiments only
  static const int v = getenv("CNPINT_FS_2D_MIN") ? atoi(getenv("CNPINT_FS_2D_MIN")) : 2048;
  return v;
}
static bool fs_shape_ok(int dim, int N) {
  return dim == 1 ? (N >= 2048 && N <= 65536) : (N >= fs_min2d() && N >= 256 && N <= 16384);
}
bool fstep_ok(const cnpint_ctx* c) { return fs_shape_ok(c->dim, c->N) && c->d_fsY; }

static int fs_nc(int N) {
  int l1, l2;
  fs_logs(N, l1, l2);
  const int mx = l1 > l2 ? l1 : l2;
  return mx <= 5 ? FS_NC5 : mx == 6 ? FS_NC6 : FS_NC7;
}
// W = real columns of a time row (1D: ld; 2D: ny·ld)
int fstep_nxb(int N, int64_t W) { return (int)((W + 2 * fs_nc(N) - 1) / (2 * fs_nc(N))); }
// Y: nxb blocks of N × NC complex (the last block padded to whole pairs of NC columns)
size_t fstep_y_bytes(int dim, int N, int64_t W) {
  return fs_shape_ok(dim, N) ? (size_t)fstep_nxb(N, W) * N * fs_nc(N) * 16 : 0;
}

template <int MODE, int LOG1, int LOG2>
static cudaError_t fs_launch(cnpint_ctx* c, const double* vin, const double2* spin, double* vout, double2* spout,
                             const double* vscale, int accumulate) {
  using G = FsGeo<MODE, LOG1, LOG2>;
  auto kern = k_fstep<MODE, LOG1, LOG2>;
  int per_sm = 0;
  cudaError_t ce = cnp_dev_cached((const void*)kern, &per_sm, [&](int* v) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::bytes);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(v, kern, G::NT, G::bytes);
    if (e != cudaSuccess || *v < 1) *v = 1;
    return cudaSuccess;
  });
  if (ce != cudaSuccess) return ce;
  const int W = (int)c->slice;  // real columns per time row
  FsSched S;
  S.nxb = (W + 2 * G::NC - 1) / (2 * G::NC);
  S.n[0] = G::NP0;
  S.n[1] = G::NP1;
  S.n[2] = G::NP2;
  const int per = G::PER;
  const int grid_max = per_sm * c->num_sms;
  // lag: enough steps between a block's phases that the CTAs in flight (≈ grid) finish the earlier
  // phase first
  // (measured, profiles/r01_fs_sweep.txt: c2 (c = 7) best near 21, c3 (c = 2) at 5)
  const int cpl = (grid_max + per - 1) / per;  // schedule steps the resident CTAs span
  int L = cpl <= 2 ? 2 * cpl + 1 : (3 * cpl < 21 ? 3 * cpl : 21);
  if (const char* e = getenv("CNPINT_FS_LAG")) L = atoi(e) > 0 ? atoi(e) : L;
  S.lag[0] = 0;
  S.lag[1] = L;
  S.lag[2] = MODE == 2 ? 2 * L : L;
  S.total = (unsigned)(S.nxb + S.lag[2]) * (unsigned)per;  // including the empty edge slots
  const int grid = (int)(S.total < (unsigned)grid_max ? S.total : (unsigned)grid_max);
  static const int no_discard = getenv("CNPINT_FS_NODISCARD") ? 1 : 0;  // tuning knob, read once
  FsArgs a;
  a.vin = vin; a.spin = spin; a.vout = vout; a.spout = spout; a.Y = (double2*)c->d_fsY; a.vscale = vscale;
  a.gam = c->d_gam; a.igam = c->d_igam; a.twN = c->d_tw; a.lam1 = c->d_lam1; a.lam2 = c->d_lam2; a.ex = c->d_ex; a.ey = c->d_ey;
  a.tau = c->tau_p; a.tau_shift = c->tau_p * c->shift;
  a.W = W; a.ld = (int)c->ld; a.nx = c->nx; a.accumulate = accumulate; a.debug_sign = c->debug & 1;
  a.no_discard = no_discard;
#ifdef CNPINT_EXPERIMENTS  // result-corrupting timing knob: only in experiment builds
  static const int skip = getenv("CNPINT_FS_SKIP") ? atoi(getenv("CNPINT_FS_SKIP")) : 0;
  a.skip = skip;
#else
  a.skip = 0;
#endif
  a.cnt = c->d_fscnt; a.ticket = c->d_fscnt + S.nxb; a.tick_base = c->fs_tick; a.base = c->fs_cnt;
  cudaError_t le = cnp_launch(c, kern, dim3(grid), dim3(G::NT), G::bytes, a, S);
  if (le != cudaSuccess) return le;
  c->fs_cnt += (unsigned)(S.n[0] + S.n[1]);  // phases 0 and 1 count per block
  c->fs_tick += S.total + (unsigned)grid;    // every CTA also takes one ticket past the end
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t fs_dispatch(cnpint_ctx* c, const double* vin, const double2* spin, double* vout, double2* spout,
                               const double* vscale, int accumulate) {
  int l1, l2;
  fs_logs(c->N, l1, l2);
#define FS_CASE(A, B) \
  if (l1 == A && l2 == B) return fs_launch<MODE, A, B>(c, vin, spin, vout, spout, vscale, accumulate);
  if constexpr (MODE == 2) {
    FS_CASE(4, 4) FS_CASE(5, 4) FS_CASE(5, 5) FS_CASE(6, 5) FS_CASE(6, 6) FS_CASE(7, 6) FS_CASE(7, 7)
  } else {
    FS_CASE(6, 5) FS_CASE(6, 6) FS_CASE(7, 6) FS_CASE(7, 7) FS_CASE(8, 7) FS_CASE(8, 8)
  }
#undef FS_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_fstep_fwd(cnpint_ctx* c, const double* v, const double* vscale, double2* what) {
  cnp_prof_begin(c, KID_FFT_FWD);
  cudaError_t e = fs_dispatch<0>(c, v, nullptr, nullptr, what, vscale, 0);
  cnp_prof_end(c, KID_FFT_FWD, 8.0 * cnp_units(c) + 16.0 * cnp_spec_units(c));
  return e;
}
cudaError_t launch_fstep_inv(cnpint_ctx* c, const double2* zhat, double* z, int accumulate) {
  cnp_prof_begin(c, KID_FFT_INV);
  cudaError_t e = fs_dispatch<1>(c, nullptr, zhat, z, nullptr, nullptr, accumulate);
  cnp_prof_end(c, KID_FFT_INV, 8.0 * cnp_units(c) * (accumulate ? 2.0 : 1.0) + 16.0 * cnp_spec_units(c));
  return e;
}
cudaError_t launch_fstep_pass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  cnp_prof_begin(c, KID_TIMEPASS2D);
  cudaError_t e = fs_dispatch<2>(c, in, nullptr, out, nullptr, vscale, 0);
  cnp_prof_end(c, KID_TIMEPASS2D, 16.0 * cnp_units(c));
  return e;
}
