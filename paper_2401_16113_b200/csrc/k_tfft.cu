// Time-axis transforms of P_α⁻¹ (Eq. 3.2 steps (a) and (c), Remark 3.1).
//
//   K2  (MODE 0)  ŵ_k[x] = Σ_t e^{−2πikt/N} · γ_t · s · v_t[x],  k = 0..N/2        (step (a) × √N)
//   K4  (MODE 1)  z_t[x] = 1/(N γ_t) · Σ_{k<N} e^{+2πikt/N} ẑ_k[x],  ẑ_{N−k} = conj ẑ_k  (step (c))
//   K6  (MODE 2)  2D fused time pass: K2, divide by (λ1_k − λ2_k τ μ_x), K4, all on chip.
//
// γ_t = α^{t/N} (Λ_α); s is an optional device scalar (GMRES basis scale).
//
// B200 design: thread-block-cluster FFT.  The time axis is strided in HBM (row pitch W doubles),
// so a tile is X adjacent columns × all N rows and every row access is an X·8-byte segment
// (X = 16: a full 128-B line).  A whole tile (N·X·8 B, 512 KB at N = 4096) does not fit one SM,
// so it is spread over a cluster of C CTAs: CTA r holds the time-residue class t ≡ r (mod C)
// (N2 = N/C rows), i.e. the decimation-in-time split
//     X[k2 + N2 k1] = Σ_r ω_C^{r k1} · ω_N^{r k2} · F_r[k2],   F_r = FFT_{N2}(z_{nC+r}),
// F_r is a local shared-memory FFT, and the radix-C stage across CTAs reads the other CTAs'
// F_r through distributed shared memory (DSMEM).  Each CTA owns the frequencies of a set of k2
// "families" {k2, N2−k2} that is closed under k → N−k, so the Hermitian separation below is local.
// The inverse runs the same steps backwards: the radix-C stage pushes T_r[k2] into CTA r's shared
// memory, then CTA r runs its local inverse FFT and writes its residue rows.
// Two real columns (a, b) are packed as one complex column z_t = v_t[a] + i v_t[b]:
//   X_a[k] = (Z_k + conj Z_{N−k})/2,  X_b[k] = (Z_k − conj Z_{N−k})/(2i),  k = 0..N/2,
// and back Z_k = X_a[k] + i X_b[k].  Rows come in with cp.async (LDGSTS) straight into the shared
// column buffers; Γ_α·s is applied inside the first butterfly stage; the local FFT is a Stockham
// autosort (radix 8/4/2) with its twiddles ω_{N2}^q staged in shared memory.
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

#include <cstdlib>

namespace cg = cooperative_groups;

namespace {

extern __shared__ double2 tf_smem[];

// Shared column layout: one pad slot every 8 complex entries (8 × 16 B = one bank sweep), so the
// strided butterfly writes (stride R entries) and the per-column reads are conflict free.
CNP_DEV int pd(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int tf_cs(int logN2) { return (1 << logN2) + ((1 << logN2) >> 3) + 1; }
// Per-stage twiddle table sizes: stage with NS > 1 and radix R stores ω_{NS R}^{r k} at [(r−1) NS + k].
__host__ __device__ constexpr int tf_stage_tw(int logN2, int logNs = 0) {
  return logNs >= logN2 ? 0
                        : ((logNs > 0 ? ((1 << (logN2 - logNs >= 3 ? 3 : logN2 - logNs)) - 1) << logNs : 0) +
                           tf_stage_tw(logN2, logNs + (logN2 - logNs >= 3 ? 3 : logN2 - logNs)));
}

template <bool INV>
CNP_DEV void dft4r(double2& v0, double2& v1, double2& v2, double2& v3) {
  double2 t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = cmul_mi<INV>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

#define TF_C8 0.70710678118654752440

template <bool INV>
CNP_DEV double2 tw8_1(double2 a) {  // a · e^{∓iπ/4}
  return INV ? make_double2(TF_C8 * (a.x - a.y), TF_C8 * (a.x + a.y))
             : make_double2(TF_C8 * (a.x + a.y), TF_C8 * (a.y - a.x));
}
template <bool INV>
CNP_DEV double2 tw8_3(double2 a) {  // a · e^{∓3iπ/4}
  return INV ? make_double2(-TF_C8 * (a.x + a.y), TF_C8 * (a.x - a.y))
             : make_double2(TF_C8 * (a.y - a.x), -TF_C8 * (a.x + a.y));
}

// v[k] ← Σ_r v[r] e^{∓2πi r k / R}  (forward −, inverse +)
template <int R, bool INV>
CNP_DEV void dftR(double2* v) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    const double2 t = v[0];
    v[0] = cadd(t, v[1]);
    v[1] = csub(t, v[1]);
  } else if constexpr (R == 4) {
    dft4r<INV>(v[0], v[1], v[2], v[3]);
  } else {
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4r<INV>(e0, e1, e2, e3);
    dft4r<INV>(o0, o1, o2, o3);
    o1 = tw8_1<INV>(o1);
    o2 = cmul_mi<INV>(o2);
    o3 = tw8_3<INV>(o3);
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
  }
}

// One Stockham stage over all NC complex columns of length N2 = 2^LOGN2 (all sizes compile time):
// column c at buf[c*CS + pd(i)].  Work item (c, j), j < N2/R: reads i = j + r N2/R, twiddles by
// ω_{Ns R}^{r (j mod Ns)} (from this stage's table, laid out [r−1][k] so a warp reads it
// contiguously), radix-R DFT, writes i = (j − j mod Ns) R + (j mod Ns) + r Ns.  All of a thread's
// items are read before one barrier and written after it.  SCALE (first stage only): input i is
// multiplied by gm[i]·s (gm = this CTA's residue slice of Γ_α, s = GMRES basis scale).
template <int LOGR, bool INV, bool SCALE, int LOGN2, int NC, int LOGNS, int NT>
CNP_DEV void stage(double2* buf, const double2* stw, const double* gm, double s) {
  constexpr int R = 1 << LOGR;
  constexpr int LOGPER = LOGN2 - LOGR;
  constexpr int PER = 1 << LOGPER;
  constexpr int NS = 1 << LOGNS;
  constexpr int TOTAL = NC * PER;
  constexpr int ITER = (TOTAL + NT - 1) / NT;
  constexpr int CS = tf_cs(LOGN2);
  double2 v[ITER][R];
  int colj[ITER], jj[ITER];
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int q = it * NT + (int)threadIdx.x;
    const bool on = (TOTAL % NT == 0) || q < TOTAL;
    const int c = q >> LOGPER;
    const int j = q & (PER - 1);
    jj[it] = j;
    colj[it] = c * CS;
    if (on) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        v[it][r] = buf[c * CS + pd(j + r * PER)];
        if (SCALE) v[it][r] = cscale(v[it][r], gm[j + r * PER] * s);
      }
      if (NS > 1) {
        const int k = j & (NS - 1);
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = stw[(r - 1) * NS + k];
          if (INV) w.y = -w.y;
          v[it][r] = cmul(v[it][r], w);
        }
      }
      dftR<R, INV>(v[it]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int q = it * NT + (int)threadIdx.x;
    const bool on = (TOTAL % NT == 0) || q < TOTAL;
    if (on) {
      const int j = jj[it];
      const int k = j & (NS - 1);
      const int base = ((j - k) << LOGR) + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[colj[it] + pd(base + r * NS)] = v[it][r];
    }
  }
  __syncthreads();
}

template <bool INV, bool SCALE, int LOGN2, int NC, int NT, int LOGNS = 0>
CNP_DEV void local_fft(double2* buf, const double2* stw, const double* gm, double s) {
  if constexpr (LOGNS < LOGN2) {
    constexpr int REM = LOGN2 - LOGNS;
    constexpr int LOGR = REM >= 3 ? 3 : REM;
    stage<LOGR, INV, SCALE && LOGNS == 0, LOGN2, NC, LOGNS, NT>(buf, stw, gm, s);
    local_fft<INV, SCALE, LOGN2, NC, NT, LOGNS + LOGR>(buf, stw + (LOGNS > 0 ? ((1 << LOGR) - 1) << LOGNS : 0), gm,
                                                        s);
  }
}

// e^{−2πi num/den}, exact argument reduction by sincospi (den a power of two)
CNP_DEV double2 expi_neg(int num, int den) {
  double sn, cs;
  sincospi(2.0 * (double)num / (double)den, &sn, &cs);
  return make_double2(cs, -sn);
}

// Hermitian separation of one packed pair: (Z_k, Z_{N−k}) → (X_a[k], X_b[k])
CNP_DEV void separate(double2 zk, double2 zm, double2& xa, double2& xb) {
  xa = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
  xb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
}
// (X_a, X_b) → Z_k = X_a + i X_b
CNP_DEV double2 pack(double2 xa, double2 xb) { return make_double2(xa.x - xb.y, xa.y + xb.x); }

CNP_DEV double2 lam_at(const double2* __restrict__ lam, int k, int N) {  // λ_k for k in [0, N)
  return k <= N / 2 ? lam[k] : cconj(lam[N - k]);
}

template <int C>
CNP_DEV double2* rank_buf(double2* buf, int r) {
  if constexpr (C > 1) return cg::this_cluster().map_shared_rank(buf, r);
  else return buf;
}

template <int C>
CNP_DEV void cluster_barrier() {
  if constexpr (C > 1) cg::this_cluster().sync();
  else __syncthreads();
}

}  // namespace

// Shared memory (complex entries): data[NC·CS] | twl[N2] (ω_{N2}^q) | stw[stage tables] | wc[C]
// (ω_N^j, j < C) | gm[N2], ig[N2] (doubles: Γ_α and 1/(NΓ_α) of this CTA's residue class) |
// l1[N/2+1], l2[N/2+1] (λ tables, MODE 2 only).  Everything but data is loaded once per CTA.
template <int MODE, int C, int LOGN2, int NC>
struct TfLayout {
  static constexpr int N2 = 1 << LOGN2;
  static constexpr int CS = tf_cs(LOGN2);
  static constexpr int off_twl = NC * CS;
  static constexpr int off_stw = off_twl + N2;
  static constexpr int off_wc = off_stw + tf_stage_tw(LOGN2);
  static constexpr int off_gm = off_wc + C;
  static constexpr int off_lam = off_gm + N2;
  static constexpr int nlam = MODE == 2 ? N2 * C / 2 + 1 : 0;
  static constexpr size_t bytes = (size_t)(off_lam + 2 * nlam) * 16;
};

template <int MODE, int C, int LOGN2, int NC>
__global__ void __launch_bounds__(256, 2)
    k_tfft(const double* __restrict__ vin, const double2* __restrict__ spin, double* __restrict__ vout,
           double2* __restrict__ spout, const double* __restrict__ vscale, int64_t W,
           const double* __restrict__ gam, const double* __restrict__ igam, int accumulate,
           const double2* __restrict__ lam1, const double2* __restrict__ lam2, const double* __restrict__ ex,
           const double* __restrict__ ey, double tau_shift, double tau, int64_t ld, int nx, int debug_sign,
           int ntiles) {
  using LY = TfLayout<MODE, C, LOGN2, NC>;
  constexpr int NT = 256;
  constexpr int X = 2 * NC;
  constexpr int N2 = LY::N2;
  constexpr int N = N2 * C;
  constexpr int H = N / 2;
  constexpr int CS = LY::CS;
  const int tid = threadIdx.x;
  int rank = 0;
  if constexpr (C > 1) rank = (int)cg::this_cluster().block_rank();
  const int cl = blockIdx.x / C, ncl = gridDim.x / C;
  const int Wi = (int)W, ldi = (int)ld;
  double2* const buf = tf_smem;
  double2* const twl = tf_smem + LY::off_twl;
  double2* const stw = tf_smem + LY::off_stw;
  double2* const wc = tf_smem + LY::off_wc;
  double* const gm = reinterpret_cast<double*>(tf_smem + LY::off_gm);
  double* const ig = gm + N2;
  double2* const l1s = tf_smem + LY::off_lam;
  double2* const l2s = l1s + LY::nlam;
  // families {k2, N2−k2} owned by this rank: k2 = rank + C·i, k2 <= N2/2
  const int nfam = rank <= N2 / 2 ? (N2 / 2 - rank) / C + 1 : 0;

  // ---- per-CTA tables, once: Γ_α slices and λ by cp.async, twiddles on chip (sincospi)
  if (MODE != 1)
    for (int q = tid; q < N2; q += NT) cp_async8(gm + q, gam + q * C + rank);
  if (MODE != 0)
    for (int q = tid; q < N2; q += NT) cp_async8(ig + q, igam + q * C + rank);
  if (MODE == 2)
    for (int q = tid; q < LY::nlam; q += NT) {
      cp_async16(l1s + q, lam1 + q);
      cp_async16(l2s + q, lam2 + q);
    }
  cp_async_commit();
  const double sg = debug_sign ? -1.0 : 1.0;  // sign flip = negative-control debug hook
  for (int q = tid; q < N2; q += NT) {
    double2 w = expi_neg(q, N2);
    w.y *= sg;
    twl[q] = w;
  }
  if (tid < C) {
    double2 w = expi_neg(tid, N);
    w.y *= sg;
    wc[tid] = w;
  }
  {
    int off = 0;
    for (int logNs = 0; logNs < LOGN2;) {
      const int lr = LOGN2 - logNs >= 3 ? 3 : LOGN2 - logNs;
      if (logNs > 0) {
        const int ns = 1 << logNs, cnt = ((1 << lr) - 1) << logNs;
        for (int q = tid; q < cnt; q += NT) {
          const int r = q / ns + 1, k = q - (r - 1) * ns;
          double2 w = expi_neg(r * k, ns << lr);
          w.y *= sg;
          stw[off + q] = w;
        }
        off += cnt;
      }
      logNs += lr;
    }
  }
  auto wN = [&](int j) { return cmul(wc[j & (C - 1)], twl[j / C]); };  // ω_N^j, j < N
  auto lam_s = [&](const double2* l, int k) { return k <= H ? l[k] : cconj(l[N - k]); };
  const double s = (MODE != 1 && vscale) ? *vscale : 1.0;

  // ---- persistent loop over this cluster's tiles
  for (int tile = cl; tile < ntiles; tile += ncl) {
  const int col0 = tile * X;
  // this thread's column pair is fixed in every loop below (NC divides the block size)
  const int cpair = tid % NC;
  const int mycol = col0 + 2 * cpair;
  const bool padA = mycol < Wi ? (mycol % ldi) >= nx : true;
  const bool padB = mycol < Wi ? ((mycol + 1) % ldi) >= nx : true;
  if (MODE == 0 || MODE == 2) {
    for (int q = tid; q < N2 * NC; q += NT) {
      const int n = q / NC, c = q - n * NC;
      const int col = col0 + 2 * c;
      double2* dst = buf + c * CS + pd(n);
      if (col < Wi) cp_async16(dst, vin + (int64_t)(n * C + rank) * W + col);
      else *dst = make_double2(0.0, 0.0);
    }
    cp_async_commit();
  } else {
    // MODE 1: other CTAs push into this buffer below; they must not start before this CTA has
    // finished reading it for the previous tile
    cluster_barrier<C>();
  }
  cp_async_wait<0>();
  __syncthreads();

  if (MODE == 0 || MODE == 2) {
    local_fft<false, true, LOGN2, NC, NT>(buf, stw, gm, s);
    cluster_barrier<C>();
    // ---- radix-C stage across the cluster for the owned families, then separation / divide
    const int items = nfam * NC;
    for (int q = tid; q < items; q += NT) {
      const int fi = q / NC, c = q - fi * NC;
      const int k2 = rank + C * fi;
      const int k2m = (N2 - k2) & (N2 - 1);
      double2 A[C], B[C];
#pragma unroll
      for (int r = 0; r < C; ++r) {
        const double2* rb = rank_buf<C>(buf, r);
        double2 a = rb[c * CS + pd(k2)];
        double2 bb = rb[c * CS + pd(k2m)];
        if (r > 0) {
          a = cmul(a, wN(r * k2));
          bb = cmul(bb, wN(r * k2m));
        }
        A[r] = a;
        B[r] = bb;
      }
      dftR<C, false>(A);
      dftR<C, false>(B);
      // A[k1] = Z[k2 + N2 k1], B[k1] = Z[k2m + N2 k1]; the partner of k = k2 + N2 k1 is
      // N − k = k2m + N2 (C−1−k1) (k2 ≠ 0) or N2 ((C − k1) mod C) (k2 = 0).
      if (MODE == 0) {
#pragma unroll
        for (int k1 = 0; k1 < C; ++k1) {
          const int k = k2 + N2 * k1;
          if (k <= H && mycol < Wi) {
            const double2 zm = (k2 == 0) ? A[(C - k1) & (C - 1)] : B[C - 1 - k1];
            double2 xa, xb;
            separate(A[k1], zm, xa, xb);
            if (padA) xa = make_double2(0.0, 0.0);
            if (padB) xb = make_double2(0.0, 0.0);
            double2* o = spout + (int64_t)k * W + mycol;
            stg_cs2(o, xa);
            stg_cs2(o + 1, xb);
          }
          const int km = k2m + N2 * k1;
          if (k2m != k2 && km <= H && mycol < Wi) {
            double2 xa, xb;
            separate(B[k1], A[C - 1 - k1], xa, xb);
            if (padA) xa = make_double2(0.0, 0.0);
            if (padB) xb = make_double2(0.0, 0.0);
            double2* o = spout + (int64_t)km * W + mycol;
            stg_cs2(o, xa);
            stg_cs2(o + 1, xb);
          }
        }
      } else {
        // MODE 2: divide every frequency by (λ1_k − λ2_k μ) per real column, repack, then the
        // inverse radix-C stage pushes T_r[k2] back to CTA r (positions k2/k2m of every CTA's
        // buffer are read and written only by this item).
        double2 A2[C], B2[C];
        double mua = 0.0, mub = 0.0;
        if (mycol < Wi) {
          const int ya = mycol / ldi, xa_ = mycol - ya * ldi;
          const int yb = (mycol + 1) / ldi, xb_ = (mycol + 1) - yb * ldi;
          mua = tau * (ex[xa_] + ey[ya]) + tau_shift;
          mub = tau * (ex[xb_] + ey[yb]) + tau_shift;
        }
#pragma unroll
        for (int k1 = 0; k1 < C; ++k1) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            const int kk = (side == 0 ? k2 : k2m) + N2 * k1;
            const double2 zk = side == 0 ? A[k1] : B[k1];
            const double2 zm = side == 0 ? ((k2 == 0) ? A[(C - k1) & (C - 1)] : B[C - 1 - k1]) : A[C - 1 - k1];
            double2 xa, xb;
            separate(zk, zm, xa, xb);
            const double2 l1 = lam_s(l1s, kk), l2 = lam_s(l2s, kk);
            xa = cmul(xa, crecip(csub(l1, cscale(l2, mua))));
            xb = cmul(xb, crecip(csub(l1, cscale(l2, mub))));
            double2 z = pack(xa, xb);
            if (kk == 0 || kk == H) z = make_double2(xa.x, xb.x);  // Hermitian endpoints: real parts
            if (side == 0) A2[k1] = z;
            else B2[k1] = z;
          }
        }
#pragma unroll
        for (int k1 = 0; k1 < C; ++k1) {
          A[k1] = A2[k1];
          B[k1] = (k2m == k2) ? A2[k1] : B2[k1];
        }
        dftR<C, true>(A);
        dftR<C, true>(B);
#pragma unroll
        for (int r = 0; r < C; ++r) {
          double2* rb = rank_buf<C>(buf, r);
          double2 a = A[r], bb = B[r];
          if (r > 0) {
            a = cmul_conj(a, wN(r * k2));
            bb = cmul_conj(bb, wN(r * k2m));
          }
          rb[c * CS + pd(k2)] = a;
          if (k2m != k2) rb[c * CS + pd(k2m)] = bb;
        }
      }
    }
    if (MODE == 0) {
      cluster_barrier<C>();  // keep F_r alive until every reader is done, then refill
      continue;
    }
  } else {
    // ---- MODE 1: half-spectrum rows of the owned families → Z → inverse radix-C stage (push)
    const int items = nfam * NC;
    for (int q = tid; q < items; q += NT) {
      const int fi = q / NC, c = q - fi * NC;
      const int k2 = rank + C * fi;
      const int k2m = (N2 - k2) & (N2 - 1);
      const int col = col0 + 2 * c;
      double2 ra[C], rb2[C];
#pragma unroll
      for (int k1 = 0; k1 < C; ++k1) {  // issue every row load first (memory-level parallelism)
        const int k = k2 + N2 * k1;
        const int kr = k <= H ? k : N - k;
        ra[k1] = rb2[k1] = make_double2(0.0, 0.0);
        if (col < Wi) {
          const double2* src = spin + (int64_t)kr * W + col;
          ra[k1] = ldg_cs2(src);
          rb2[k1] = ldg_cs2(src + 1);
        }
      }
      double2 A[C], B[C];
#pragma unroll
      for (int k1 = 0; k1 < C; ++k1) {
        const int k = k2 + N2 * k1;
        const double2 xa = ra[k1], xb = rb2[k1];
        // Z_k and its partner Z_{N−k} from the one stored row min(k, N−k)
        double2 zk, zp;
        if (k == 0 || k == H) {
          zk = zp = make_double2(xa.x, xb.x);
        } else if (k < H) {
          zk = pack(xa, xb);
          zp = pack(cconj(xa), cconj(xb));
        } else {
          zk = pack(cconj(xa), cconj(xb));
          zp = pack(xa, xb);
        }
        A[k1] = zk;
        B[C - 1 - k1] = zp;
      }
      if (k2 == 0 || k2m == k2) {
#pragma unroll
        for (int k1 = 0; k1 < C; ++k1) B[k1] = A[k1];
      }
      dftR<C, true>(A);
      dftR<C, true>(B);
#pragma unroll
      for (int r = 0; r < C; ++r) {
        double2* rbuf = rank_buf<C>(buf, r);
        double2 a = A[r], bb = B[r];
        if (r > 0) {
          a = cmul_conj(a, wN(r * k2));
          bb = cmul_conj(bb, wN(r * k2m));
        }
        rbuf[c * CS + pd(k2)] = a;
        if (k2m != k2) rbuf[c * CS + pd(k2m)] = bb;
      }
    }
  }
  // ---- every T_r[k2] has arrived: local inverse FFT, then residue rows with 1/(N γ_t)
  cluster_barrier<C>();
  local_fft<true, false, LOGN2, NC, NT>(buf, stw, gm, 1.0);
  for (int q = tid; q < N2 * NC; q += NT) {
    const int n = q / NC, c = q - n * NC;
    const int col = col0 + 2 * c;
    if (col >= Wi) continue;
    const int t = n * C + rank;
    const double g = ig[n];
    const double2 z = buf[c * CS + pd(n)];
    double2 val = make_double2(padA ? 0.0 : z.x * g, padB ? 0.0 : z.y * g);
    double2* dst = reinterpret_cast<double2*>(vout + (int64_t)t * W + col);
    if (accumulate) {
      const double2 o = *dst;
      val.x += o.x;
      val.y += o.y;
    }
    stg_cs2(dst, val);
  }
  __syncthreads();  // this tile's reads of buf are done before the next tile refills it
  }  // tile loop
  if constexpr (C > 1) cg::this_cluster().sync();  // no CTA leaves while others may access its smem
}

TfftCfg tfft_cfg(int N) {
  TfftCfg f;
  int logN = 0;
  while ((1 << logN) < N) ++logN;
  // default: local FFTs of N2 = 512 rows (C = N/512 CTAs per cluster) up to N = 4096, C = 8 beyond;
  // tiles of 16 columns (128-B row segments) while N2 <= 512, 8 at N2 = 1024, 4 at N2 = 2048.
  f.C = N >= 8192 ? 8 : N >= 1024 ? N / 512 : 1;
  if (const char* e = getenv("CNPINT_TFFT_C")) {  // tuning override (experiments only)
    const int v = atoi(e);
    if ((v == 1 || v == 2 || v == 4 || v == 8) && N / v >= 2 && N / v <= 2048) f.C = v;
  }
  f.logN2 = logN - (f.C == 1 ? 0 : f.C == 2 ? 1 : f.C == 4 ? 2 : 3);
  const int NC = f.logN2 <= 9 ? 8 : f.logN2 == 10 ? 4 : 2;
  f.X = 2 * NC;
  f.CS = tf_cs(f.logN2);
  f.smem = 0;
  f.T = 256;
  f.ok = N >= 2 && N <= 16384 && f.logN2 >= 1 && f.logN2 <= 11;
  return f;
}

template <int MODE, int C, int LOGN2>
static cudaError_t launch_c(cnpint_ctx* c, const TfftCfg& f, const double* vin, const double2* spin, double* vout,
                            double2* spout, const double* vscale, int accumulate) {
  constexpr int NC = LOGN2 <= 9 ? 8 : LOGN2 == 10 ? 4 : 2;
  using LY = TfLayout<MODE, C, LOGN2, NC>;
  auto kern = k_tfft<MODE, C, LOGN2, NC>;
  static int max_clusters = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = LY::bytes;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!max_clusters) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LY::bytes);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3(C * c->num_sms);
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    if (e != cudaSuccess || n < 1) n = c->num_sms / C;
    max_clusters = n < 1 ? 1 : n;
  }
  const int64_t W = c->slice;  // 1D: ld; 2D: ny*ld
  const int ntiles = (int)((W + 2 * NC - 1) / (2 * NC));
  const int ncl = ntiles < max_clusters ? ntiles : max_clusters;
  cfg.gridDim = dim3(ncl * C);
  return cudaLaunchKernelEx(&cfg, kern, vin, spin, vout, spout, vscale, W, (const double*)c->d_gam,
                            (const double*)c->d_igam, accumulate, (const double2*)c->d_lam1, (const double2*)c->d_lam2,
                            (const double*)c->d_ex, (const double*)c->d_ey, c->tau * c->shift, c->tau, (int64_t)c->ld,
                            c->nx, c->debug & 1, ntiles);
}

template <int MODE>
static cudaError_t dispatch(cnpint_ctx* c, const TfftCfg& f, const double* vin, const double2* spin, double* vout,
                            double2* spout, const double* vscale, int accumulate) {
#define TF_CASE(CC, LL) \
  if (f.C == CC && f.logN2 == LL) return launch_c<MODE, CC, LL>(c, f, vin, spin, vout, spout, vscale, accumulate);
  TF_CASE(1, 1) TF_CASE(1, 2) TF_CASE(1, 3) TF_CASE(1, 4) TF_CASE(1, 5) TF_CASE(1, 6) TF_CASE(1, 7)
  TF_CASE(1, 8) TF_CASE(1, 9) TF_CASE(1, 10) TF_CASE(1, 11)
  TF_CASE(2, 9) TF_CASE(2, 10) TF_CASE(2, 11)
  TF_CASE(4, 9) TF_CASE(4, 10) TF_CASE(4, 11)
  TF_CASE(8, 9) TF_CASE(8, 10) TF_CASE(8, 11)
#undef TF_CASE
  return cudaErrorInvalidValue;
}

template <int MODE>
static cudaError_t run_tfft(cnpint_ctx* c, const double* vin, const double2* spin, double* vout, double2* spout,
                            const double* vscale, int accumulate) {
  const TfftCfg f = tfft_cfg(c->N);
  const int kid = MODE == 0 ? KID_FFT_FWD : MODE == 1 ? KID_FFT_INV : KID_TIMEPASS2D;
  const double bytes = MODE == 2 ? 16.0 * cnp_units(c)
                                 : 8.0 * cnp_units(c) * (accumulate ? 2.0 : 1.0) + 16.0 * cnp_spec_units(c);
  cnp_prof_begin(c, kid);
  cudaError_t e = dispatch<MODE>(c, f, vin, spin, vout, spout, vscale, accumulate);
  cnp_prof_end(c, kid, bytes);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_tfft_fwd(cnpint_ctx* c, const double* v, const double* vscale, double2* what) {
  return run_tfft<0>(c, v, nullptr, nullptr, what, vscale, 0);
}
cudaError_t launch_tfft_inv(cnpint_ctx* c, const double2* zhat, double* z, int accumulate) {
  return run_tfft<1>(c, nullptr, zhat, z, nullptr, nullptr, accumulate);
}
cudaError_t launch_tfft_pass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  return run_tfft<2>(c, in, nullptr, out, nullptr, vscale, 0);
}
