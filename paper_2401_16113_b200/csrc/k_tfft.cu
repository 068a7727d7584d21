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

#include "fft_tile.cuh"

// threads per CTA of the time-FFT kernels (two CTAs per SM)
#ifndef TF_NT
#define TF_NT 256
#endif

namespace {

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

// Shared memory (complex entries): data[NC·CS] | stw[stage tables] | whi[N/64], wlo[64] (ω_N^j =
// whi[j >> 6]·wlo[j & 63]) | ghi, glo, ihi, ilo (doubles: Γ_α and 1/(NΓ_α) as two-level tables,
// γ_t = ghi[t >> 6]·glo[t & 63]) | l1[N/2+1], l2[N/2+1] (λ tables, MODE 2 only).  Everything but
// data is built once per CTA; the two-level tables keep it small (a few KB at any N).
template <int MODE, int C, int LOGN2, int NC>
struct TfLayout {
  static constexpr int N2 = 1 << LOGN2;
  static constexpr int N = N2 * C;
  static constexpr int LO = N < 64 ? N : 64;
  static constexpr int HI = N / LO;
  static constexpr int CS = tf_cs(LOGN2);
  static constexpr int off_stw = NC * CS;
  static constexpr int off_whi = off_stw + tf_stage_tw(LOGN2);
  static constexpr int off_wlo = off_whi + HI;
  static constexpr int off_g = off_wlo + 64;  // doubles: ghi[HI] glo[64] ihi[HI] ilo[64] → (2HI+128)/2 slots
  static constexpr int off_lam = off_g + HI + 64;
  static constexpr int nlam = MODE == 2 ? N / 2 + 1 : 0;
  static constexpr size_t bytes = (size_t)(off_lam + 2 * nlam) * 16;
};

template <int MODE, int C, int LOGN2, int NC>
__global__ void __launch_bounds__(TF_NT, 2)
    k_tfft(const double* __restrict__ vin, const double2* __restrict__ spin, double* __restrict__ vout,
           double2* __restrict__ spout, const double* __restrict__ vscale, int64_t W,
           const double* __restrict__ gam, const double* __restrict__ igam, int accumulate,
           const double2* __restrict__ lam1, const double2* __restrict__ lam2, const double* __restrict__ ex,
           const double* __restrict__ ey, double tau_shift, double tau, int64_t ld, int nx, int debug_sign,
           int ntiles) {
  using LY = TfLayout<MODE, C, LOGN2, NC>;
  constexpr int NT = TF_NT;
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
  double2* const stw = tf_smem + LY::off_stw;
  double2* const whi = tf_smem + LY::off_whi;
  double2* const wlo = tf_smem + LY::off_wlo;
  double* const ghi = reinterpret_cast<double*>(tf_smem + LY::off_g);
  double* const glo = ghi + LY::HI;
  double* const ihi = glo + 64;
  double* const ilo = ihi + LY::HI;
  double2* const l1s = tf_smem + LY::off_lam;
  double2* const l2s = l1s + LY::nlam;
  // families {k2, N2−k2} owned by this rank: k2 = rank + C·i, k2 <= N2/2
  const int nfam = rank <= N2 / 2 ? (N2 / 2 - rank) / C + 1 : 0;

  // ---- per-CTA tables, once: Γ_α two-level tables (exact host values: γ_{64i}, γ_i; N is a power
  //      of two so N·(1/(Nγ_i)) is exact), λ by cp.async; twiddles on chip (sincospi)
  for (int q = tid; q < LY::HI; q += NT) {
    cp_async8(ghi + q, gam + q * LY::LO);
    cp_async8(ihi + q, igam + q * LY::LO);
  }
  if (MODE == 2)
    for (int q = tid; q < LY::nlam; q += NT) {
      cp_async16(l1s + q, lam1 + q);
      cp_async16(l2s + q, lam2 + q);
    }
  cp_async_commit();
  for (int q = tid; q < LY::LO; q += NT) {
    glo[q] = __ldg(gam + q);
    ilo[q] = (double)N * __ldg(igam + q);
  }
  const double sg = debug_sign ? -1.0 : 1.0;  // sign flip = negative-control debug hook
  for (int q = tid; q < LY::HI; q += NT) {
    double2 w = expi_neg(q * LY::LO, N);
    w.y *= sg;
    whi[q] = w;
  }
  for (int q = tid; q < LY::LO; q += NT) {
    double2 w = expi_neg(q, N);
    w.y *= sg;
    wlo[q] = w;
  }
  fill_stage_twiddles(stw, LOGN2, sg, tid, NT);
  auto wN = [&](int j) { return cmul(whi[j >> 6], wlo[j & 63]); };  // ω_N^j, j < N
  auto lam_s = [&](const double2* l, int k) { return k <= H ? l[k] : cconj(l[N - k]); };
  const double s = (MODE != 1 && vscale) ? *vscale : 1.0;
  const TfScale sc{ghi, glo, C, rank, s};

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
    local_fft<false, TF_SCALE, LOGN2, NC, NT>(buf, stw, sc);
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
  local_fft<true, TF_PLAIN, LOGN2, NC, NT>(buf, stw, sc);
  for (int q = tid; q < N2 * NC; q += NT) {
    const int n = q / NC, c = q - n * NC;
    const int col = col0 + 2 * c;
    if (col >= Wi) continue;
    const int t = n * C + rank;
    const double g = ihi[t >> 6] * ilo[t & 63];
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

TfftCfg tfft_cfg(int N, int mode) {
  TfftCfg f;
  int logN = 0;
  while ((1 << logN) < N) ++logN;
  // default (measured, profiles/r01_tfft_sweep.txt): a pair of CTAs (C = 2) for 1024 <= N <= 4096,
  // C = 8 beyond; tiles of 16 columns (128-B row segments) while N2 <= 512, 8 at N2 = 1024, 4 at
  // N2 = 2048.  The 2D time pass at N = 1024 (c5 N1024) runs one CTA per tile (C = 1): 200 → 187 µs
  // at n = 127, 759 → 714 µs at n = 255 (profiles/r01_k6_sweep.txt).
  f.C = N >= 8192 ? 8 : (N >= 1024 && !(mode == 2 && N == 1024)) ? 2 : 1;
  if (const char* e = getenv("CNPINT_TFFT_C")) {  // tuning override (experiments only)
    const int v = atoi(e);
    if ((v == 1 || v == 2 || v == 4 || v == 8) && N / v >= 2 && N / v <= 2048) f.C = v;
  }
  f.logN2 = logN - (f.C == 1 ? 0 : f.C == 2 ? 1 : f.C == 4 ? 2 : 3);
  const int NC = f.logN2 <= 9 ? 8 : f.logN2 == 10 ? 4 : 2;
  f.X = 2 * NC;
  f.CS = tf_cs(f.logN2);
  f.smem = 0;
  f.T = TF_NT;
  f.ok = N >= 2 && N <= 16384 && f.logN2 >= 1 && f.logN2 <= 11;
  return f;
}

template <int MODE, int C, int LOGN2>
static cudaError_t launch_c(cnpint_ctx* c, const TfftCfg& f, const double* vin, const double2* spin, double* vout,
                            double2* spout, const double* vscale, int accumulate) {
  constexpr int NC = LOGN2 <= 9 ? 8 : LOGN2 == 10 ? 4 : 2;
  using LY = TfLayout<MODE, C, LOGN2, NC>;
  auto kern = k_tfft<MODE, C, LOGN2, NC>;
  int max_clusters = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(TF_NT);
  cfg.dynamicSmemBytes = LY::bytes;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  {
    cudaError_t ce = cnp_dev_cached((const void*)kern, &max_clusters, [&](int* v) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LY::bytes);
      if (e != cudaSuccess) return e;
      cfg.gridDim = dim3(C * c->num_sms);
      int n = 0;
      e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
      if (e != cudaSuccess || n < 1) n = c->num_sms / C;
      *v = n < 1 ? 1 : n;
      return cudaSuccess;
    });
    if (ce != cudaSuccess) return ce;
  }
  const int64_t W = c->slice;  // 1D: ld; 2D: ny*ld
  const int ntiles = (int)((W + 2 * NC - 1) / (2 * NC));
  const int ncl = ntiles < max_clusters ? ntiles : max_clusters;
  cfg.gridDim = dim3(ncl * C);
  return cudaLaunchKernelEx(&cfg, kern, vin, spin, vout, spout, vscale, W, (const double*)c->d_gam,
                            (const double*)c->d_igam, accumulate, (const double2*)c->d_lam1, (const double2*)c->d_lam2,
                            (const double*)c->d_ex, (const double*)c->d_ey, c->tau_p * c->shift, c->tau_p, (int64_t)c->ld,
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
  const TfftCfg f = tfft_cfg(c->N, MODE);
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
