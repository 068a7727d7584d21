// Time-axis transforms of P_α⁻¹ (Eq. 3.2 steps (a) and (c), Remark 3.1).
//
//   K2  (MODE 0)  ŵ_k[x] = Σ_t e^{−2πikt/N} · γ_t · s · v_t[x],  k = 0..N/2        (step (a) × √N)
//   K4  (MODE 1)  z_t[x] = 1/(N γ_t) · Σ_{k<N} e^{+2πikt/N} ẑ_k[x],  ẑ_{N−k} = conj ẑ_k  (step (c))
//   K6  (MODE 2)  2D fused time pass: K2, divide by (λ1_k − λ2_k τ μ_x), K4, all on chip.
//
// γ_t = α^{t/N} (Λ_α); s is an optional device scalar (GMRES basis scale).
// Layout: the time axis is strided (row pitch W doubles, x fastest).  A CTA owns a tile of X
// adjacent columns × all N rows: rows are read/written coalesced (X·8 contiguous bytes per row),
// staged in shared memory as X independent columns, and transformed there.  The real length-N
// transform is a complex length-H = N/2 FFT of z_t = w_{2t} + i w_{2t+1} plus the standard
// split/merge post-processing (Hermitian half spectrum, Remark 3.1).  The FFT is a Stockham
// autosort with radix-16 register butterflies (radix 2/4/8 for the remainder), twiddles from an
// fp64 table (never recurrences), and a padded shared-memory index (one pad per 16 entries) that
// keeps the power-of-two strides bank-conflict free.
#include "common.cuh"
#include "internal.h"

#include "fft_device.cuh"

// ---------------------------------------------------------------- the kernel
// MODE 0: real rows (v) -> half spectrum (what).  MODE 1: half spectrum -> real rows (+accumulate).
// MODE 2: real rows -> real rows with the 2D per-mode divide in between.
template <int MODE>
__global__ void __launch_bounds__(512) k_time_fft(const double* __restrict__ vin, const double2* __restrict__ spin,
                                                  double* __restrict__ vout, double2* __restrict__ spout,
                                                  const double* __restrict__ vscale, int N, int logH, int64_t W,
                                                  int X, int CS, const double2* __restrict__ tw,
                                                  const double* __restrict__ gam, const double* __restrict__ igam,
                                                  int accumulate, const double2* __restrict__ lam1,
                                                  const double2* __restrict__ lam2, const double* __restrict__ ex,
                                                  const double* __restrict__ ey, double tau_shift, double tau,
                                                  int64_t ld) {
  double2* const sbuf = fft_smem;
  const int tid = threadIdx.x, T = blockDim.x;
  const int H = 1 << logH;
  const int64_t col0 = (int64_t)blockIdx.x * X;
  double* sd = reinterpret_cast<double*>(sbuf);

  if (MODE == 0 || MODE == 2) {
    // ---- load real rows (coalesced), scale by γ_t · s, scatter into complex columns
    const double s = vscale ? *vscale : 1.0;
    if (X >= 2) {
      const int hx = X >> 1;
      const int total = N * hx;
      for (int q = tid; q < total; q += T) {
        const int t = q / hx, p = q - t * hx;
        const int64_t col = col0 + 2 * p;
        double2 val = make_double2(0.0, 0.0);
        if (col < W) val = ldg_cs2(reinterpret_cast<const double2*>(vin + (int64_t)t * W + col));
        const double g = gam[t] * s;
        const int ci = 2 * p;
        const int zi = padi(t >> 1);
        sd[2 * (ci * CS + zi) + (t & 1)] = val.x * g;
        sd[2 * ((ci + 1) * CS + zi) + (t & 1)] = val.y * g;
      }
    } else {
      for (int t = tid; t < N; t += T) {
        double val = (col0 < W) ? ldg_cs(vin + (int64_t)t * W + col0) : 0.0;
        sd[2 * padi(t >> 1) + (t & 1)] = val * gam[t] * s;
      }
    }
    __syncthreads();
    fft_columns<false>(CS, X, logH, tw, tid, T);

    if (MODE == 0) {
      // ---- split into the half spectrum, write rows k = 0..H (coalesced along x)
      const int total = (H + 1) * X;
      for (int q = tid; q < total; q += T) {
        const int k = q / X, c = q - k * X;
        const int64_t col = col0 + c;
        if (col >= W) continue;
        const double2* cb = sbuf + c * CS;
        const double2 zk = cb[padi(k & (H - 1))];
        const double2 zm = cb[padi((H - k) & (H - 1))];
        spout[(int64_t)k * W + col] = split_fwd(zk, zm, tw[k]);
      }
      return;
    }
    // ---- MODE 2: split in place (pairs k, H−k), divide, merge in place
    const int halfp = (H >> 1) + 1;  // pairs k = 0..H/2
    const int total = halfp * X;
    for (int q = tid; q < total; q += T) {
      const int c = q / halfp, k = q - c * halfp;
      const int64_t col = col0 + c;
      double2* cb = sbuf + c * CS;
      const int km = (H - k) & (H - 1);
      const double2 zk = cb[padi(k & (H - 1))];
      const double2 zm = cb[padi(km)];
      // mode eigenvalue μ for this column (transformed coordinates y = col / ld, x = col % ld)
      double mu = 0.0;
      if (col < W) {
        const int64_t yy = col / ld, xx = col - yy * ld;
        mu = tau * (ex[xx] + ey[yy]) + tau_shift;
      }
      const double2 Xk = split_fwd(zk, zm, tw[k]);
      const double2 Xm = split_fwd(zm, zk, tw[H - k]);  // X_{H−k}
      const double2 dk = crecip(csub(lam1[k], cscale(lam2[k], mu)));
      const double2 dm = crecip(csub(lam1[H - k], cscale(lam2[H - k], mu)));
      const double2 Yk = cmul(Xk, dk);
      const double2 Ym = cmul(Xm, dm);
      const double2 Zk = merge_inv(Yk, Ym, tw[k]);
      if (k == 0) {
        cb[padi(0)] = Zk;  // Z'_0 from (Y_0, Y_H)
      } else if (2 * k == H) {
        cb[padi(k)] = Zk;
      } else {
        cb[padi(k)] = Zk;
        cb[padi(km)] = merge_inv(Ym, Yk, tw[H - k]);
      }
    }
    __syncthreads();
  } else {
    // ---- MODE 1: load half-spectrum rows k = 0..H, then merge pairs in place
    const int total = (H + 1) * X;
    for (int q = tid; q < total; q += T) {
      const int k = q / X, c = q - k * X;
      const int64_t col = col0 + c;
      double2 val = make_double2(0.0, 0.0);
      if (col < W) val = ldg_cs2(spin + (int64_t)k * W + col);
      sbuf[c * CS + padi(k)] = val;
    }
    __syncthreads();
    const int halfp = (H >> 1) + 1;
    const int tp = halfp * X;
    for (int q = tid; q < tp; q += T) {
      const int c = q / halfp, k = q - c * halfp;
      double2* cb = sbuf + c * CS;
      const double2 yk = cb[padi(k)];
      const double2 ym = cb[padi(H - k)];
      const double2 zk = merge_inv(yk, ym, tw[k]);
      if (k == 0 || 2 * k == H) {
        cb[padi(k)] = zk;
      } else {
        cb[padi(k)] = zk;
        cb[padi(H - k)] = merge_inv(ym, yk, tw[H - k]);
      }
    }
    __syncthreads();
  }
  // ---- inverse FFT (MODE 1, 2), then write rows with 1/(N γ_t)
  fft_columns<true>(CS, X, logH, tw, tid, T);
  if (X >= 2) {
    const int hx = X >> 1;
    const int total = N * hx;
    for (int q = tid; q < total; q += T) {
      const int t = q / hx, p = q - t * hx;
      const int64_t col = col0 + 2 * p;
      if (col >= W) continue;
      const int ci = 2 * p;
      const int zi = padi(t >> 1);
      const double g = igam[t];
      double2 val = make_double2(sd[2 * (ci * CS + zi) + (t & 1)] * g, sd[2 * ((ci + 1) * CS + zi) + (t & 1)] * g);
      double2* dst = reinterpret_cast<double2*>(vout + (int64_t)t * W + col);
      if (accumulate) {
        const double2 o = *dst;
        val.x += o.x;
        val.y += o.y;
      }
      stg_cs2(dst, val);
    }
  } else {
    for (int t = tid; t < N; t += T) {
      if (col0 >= W) break;
      double val = sd[2 * padi(t >> 1) + (t & 1)] * igam[t];
      double* dst = vout + (int64_t)t * W + col0;
      if (accumulate) val += *dst;
      stg_cs(dst, val);
    }
  }
}

// ---------------------------------------------------------------- launch configuration
struct FftCfg {
  int X, CS, T, logH;
  size_t smem;
};

static FftCfg fft_cfg(int N) {
  FftCfg f;
  int H = N / 2;
  f.logH = 0;
  while ((1 << f.logH) < H) ++f.logH;
  int X = 16384 / N;
  if (X < 1) X = 1;
  if (X > 16) X = 16;
  f.X = X;
  f.CS = padi_host(H + 1) + 1;
  int per = H >= 16 ? H / 16 : 1;
  f.T = X * per;
  if (f.T < 32) f.T = 32;
  f.smem = (size_t)X * f.CS * sizeof(double2);
  return f;
}

template <int MODE>
static cudaError_t run_fft(cnpint_ctx* c, const double* vin, const double2* spin, double* vout, double2* spout,
                           const double* vscale, int accumulate) {
  FftCfg f = fft_cfg(c->N);
  const int64_t W = c->slice;  // 1D: ld; 2D: ny*ld
  {
    int done = 0;
    cudaError_t ce = cnp_dev_cached((const void*)k_time_fft<MODE>, &done, [&](int* v) {
      *v = 1;
      return cudaFuncSetAttribute(k_time_fft<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    if (ce != cudaSuccess) return ce;
  }
  unsigned grid = (unsigned)((W + f.X - 1) / f.X);
  const int kid = MODE == 0 ? KID_FFT_FWD : MODE == 1 ? KID_FFT_INV : KID_TIMEPASS2D;
  const double bytes = MODE == 2 ? 16.0 * cnp_units(c)
                                 : 8.0 * cnp_units(c) * (accumulate ? 2.0 : 1.0) + 16.0 * cnp_spec_units(c);
  cnp_prof_begin(c, kid);
  k_time_fft<MODE><<<grid, f.T, f.smem, c->stream>>>(vin, spin, vout, spout, vscale, c->N, f.logH, W, f.X, f.CS,
                                                    c->d_tw, c->d_gam, c->d_igam, accumulate, c->d_lam1, c->d_lam2,
                                                    c->d_ex, c->d_ey, c->tau_p * c->shift, c->tau_p, c->ld);
  cnp_prof_end(c, kid, bytes);
  return cudaGetLastError();
}

// 1D with N >= 2048 and the 2D time pass with N >= 2048: four-step kernel of k_fstep.cu (debug bit 16
// opts out); other N <= 16384: the
// cluster kernels of k_tfft.cu; larger N (2D) stays here (one column per CTA, even/odd time
// packing).  debug bit 8 forces this path (cross-check in the parity tests).
cudaError_t launch_time_fft(cnpint_ctx* c, const double* v, const double* vscale, double2* what) {
  if (!(c->debug & 8) && !(c->debug & 16) && fstep_ok(c)) return launch_fstep_fwd(c, v, vscale, what);
  if (tfft_cfg(c->N).ok && !(c->debug & 8)) return launch_tfft_fwd(c, v, vscale, what);
  return run_fft<0>(c, v, nullptr, nullptr, what, vscale, 0);
}
cudaError_t launch_time_ifft(cnpint_ctx* c, const double2* zhat, double* z, int accumulate) {
  if (!(c->debug & 8) && !(c->debug & 16) && fstep_ok(c)) return launch_fstep_inv(c, zhat, z, accumulate);
  if (tfft_cfg(c->N).ok && !(c->debug & 8)) return launch_tfft_inv(c, zhat, z, accumulate);
  return run_fft<1>(c, nullptr, zhat, z, nullptr, nullptr, accumulate);
}
cudaError_t launch_tpass2(cnpint_ctx* c, const double* in, double* out, const double* vscale);

cudaError_t launch_time_pass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale) {
  // the recurrence form (k_tscan.cu: no transform, 3 fp64 instructions per unknown) when every mode is
  // stable; debug 524288 (or any transform-selecting bit) keeps the transform kernels below
  if (tscan_ok(c)) {
    const cudaError_t e = launch_tscan_2d(c, in, out, vscale);
    if (e != cudaErrorNotSupported) return e;
  }
  if (!(c->debug & 8) && !(c->debug & 16) && fstep_ok(c)) return launch_fstep_pass_2d(c, in, out, vscale);
  // the lean time pass (k_tpass2.cu) at N = 256 and 1024 (c5 n511 N1024 2758 → 1990 µs, N256 577 → 417 µs;
  // at N = 512 it ties k_tpass_r: 225 vs 222 µs, profiles/r02_tpass2_ab.txt); debug 16384 forces it at
  // N = 512 too, debug 64 keeps the cluster kernel (and k_tpass_r off)
  if (!(c->debug & (8 | 64)) && (c->N == 256 || c->N == 1024 || (c->debug & 16384))) {
    cnp_prof_begin(c, KID_TIMEPASS2D);
    const cudaError_t e = launch_tpass2(c, in, out, vscale);
    cnp_prof_end(c, KID_TIMEPASS2D, 16.0 * cnp_units(c));
    if (e != cudaErrorNotSupported) return e;
  }
  if (!(c->debug & 8) && tpass_ok(c)) return launch_tpass_2d(c, in, out, vscale);  // N = 256, 512 (bit 64 off)
  if (tfft_cfg(c->N, 2).ok && !(c->debug & 8)) return launch_tfft_pass_2d(c, in, out, vscale);
  return run_fft<2>(c, in, nullptr, out, nullptr, vscale, 0);
}
