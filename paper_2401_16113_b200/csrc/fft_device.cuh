// Shared-memory Stockham FFT machinery (device code) used by the time-axis kernels (K2/K4/K6)
// and the 2D sine transforms (K5).  See k_timefft.cu for the layout conventions.
#pragma once
#include "common.cuh"

// All FFT buffers live in the kernel's dynamic shared memory; indexing this array (rather than
// generic pointers) keeps every access a 32-bit shared-space LDS/STS.
extern __shared__ double2 fft_smem[];

// ---------------------------------------------------------------- in-register DFTs (sign by INV)
template <bool INV>
CNP_DEV void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
CNP_DEV void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  double2 t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = cmul_mi<INV>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

// e^{∓2πi e/16} constants
#define C16_1 0.92387953251128675613
#define S16_1 0.38268343236508977173
#define C16_2 0.70710678118654752440

__host__ __device__ constexpr double c16(int e) {
  return e == 0 ? 1.0 : e == 1 ? C16_1 : e == 2 ? C16_2 : e == 3 ? S16_1 : e == 4 ? 0.0 : e == 5 ? -S16_1
       : e == 6 ? -C16_2 : e == 7 ? -C16_1 : e == 8 ? -1.0 : e == 9 ? -C16_1 : e == 10 ? -C16_2
       : e == 11 ? -S16_1 : e == 12 ? 0.0 : e == 13 ? S16_1 : e == 14 ? C16_2 : C16_1;
}
__host__ __device__ constexpr double s16(int e) { return c16((e + 12) & 15); }  // sin(2πe/16) = cos(2π(e−4)/16)

template <int E, bool INV>
CNP_DEV double2 tw16(double2 a) {
  // multiply a by w^E, w = e^{-2πi/16} (forward) or e^{+2πi/16} (inverse); E in [0, 16)
  constexpr int e = E & 15;
  if constexpr (e == 0) return a;
  else if constexpr (e == 4) return cmul_mi<INV>(a);
  else if constexpr (e == 8) return make_double2(-a.x, -a.y);
  else if constexpr (e == 12) return cmul_mi<!INV>(a);
  else {
    constexpr double c = c16(e);
    constexpr double sf = -s16(e);  // forward: e^{-iθ} = cos θ − i sin θ
    const double s = INV ? -sf : sf;
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

template <bool INV>
CNP_DEV void dft8(double2* v) {
  // radix-2 DIT over two radix-4: E = dft4(v0,v2,v4,v6), O = dft4(v1,v3,v5,v7)
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = tw16<2, INV>(o1);
  o2 = tw16<4, INV>(o2);
  o3 = tw16<6, INV>(o3);
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

template <bool INV>
CNP_DEV void dft16(double2* v) {
  // four-step 4x4: A[r2][k1] = dft4_{r1}(v[4 r1 + r2]); A *= w16^{r2 k1}; out[k1 + 4 k2] = dft4_{r2}(A[r2][k1])
  double2 a[4][4];
#pragma unroll
  for (int r2 = 0; r2 < 4; ++r2) {
    a[r2][0] = v[r2]; a[r2][1] = v[r2 + 4]; a[r2][2] = v[r2 + 8]; a[r2][3] = v[r2 + 12];
    dft4<INV>(a[r2][0], a[r2][1], a[r2][2], a[r2][3]);
  }
  a[1][1] = tw16<1, INV>(a[1][1]); a[1][2] = tw16<2, INV>(a[1][2]); a[1][3] = tw16<3, INV>(a[1][3]);
  a[2][1] = tw16<2, INV>(a[2][1]); a[2][2] = tw16<4, INV>(a[2][2]); a[2][3] = tw16<6, INV>(a[2][3]);
  a[3][1] = tw16<3, INV>(a[3][1]); a[3][2] = tw16<6, INV>(a[3][2]); a[3][3] = tw16<9, INV>(a[3][3]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 b0 = a[0][k1], b1 = a[1][k1], b2 = a[2][k1], b3 = a[3][k1];
    dft4<INV>(b0, b1, b2, b3);
    v[k1] = b0; v[k1 + 4] = b1; v[k1 + 8] = b2; v[k1 + 12] = b3;
  }
}

template <int R, bool INV>
CNP_DEV void dftR(double2* v) {
  if constexpr (R == 2) dft2<INV>(v[0], v[1]);
  else if constexpr (R == 4) dft4<INV>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<INV>(v);
  else dft16<INV>(v);
}

// ---------------------------------------------------------------- one Stockham stage, all columns
// Not inlined on purpose: isolates each stage's register allocation (16 complex values live
// across the barrier) from the caller's live state, which otherwise forces spills.
// Column c occupies buf[c*CS + padi(i)], i < H.  Work item (c, j), j < H/R: reads i = j + r H/R,
// twiddles by ω_{Ns R}^{r (j mod Ns)}, radix-R DFT, writes i = (j − j mod Ns) R + (j mod Ns) + r Ns.
template <int R, bool INV>
__device__ __noinline__ void fft_stage(int CS, int X, int logH, int Ns, int logNs, const double2* __restrict__ tw, int tid, int T) {
  constexpr int IT = (16 / R) > 0 ? 16 / R : 1;
  constexpr int logR = (R == 2) ? 1 : (R == 4) ? 2 : (R == 8) ? 3 : 4;
  const int logPer = logH - logR;
  const int per = 1 << logPer;  // items per column
  const int total = X << logPer;
  double2 v[IT][R];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int q = tid + it * T;
    if (q < total) {
      const int c = q >> logPer, j = q & (per - 1);
      const int col = c * CS;
#pragma unroll
      for (int r = 0; r < R; ++r) v[it][r] = fft_smem[col + padi(j + r * per)];
      const int k = j & (Ns - 1);
      if (Ns > 1) {
        // angle index in units of 2π/N: 2 r k (H / (Ns R)) = r k 2^{logH + 1 − logNs − logR}
        const int sh = logH + 1 - logNs - logR;
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = tw[(r * k) << sh];
          if (INV) w.y = -w.y;
          v[it][r] = cmul(v[it][r], w);
        }
      }
      dftR<R, INV>(v[it]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int q = tid + it * T;
    if (q < total) {
      const int c = q >> logPer, j = q & (per - 1);
      const int k = j & (Ns - 1);
      const int col = c * CS;
      const int base = ((j - k) << logR) + k;
#pragma unroll
      for (int r = 0; r < R; ++r) fft_smem[col + padi(base + r * Ns)] = v[it][r];
    }
  }
  __syncthreads();
}

template <bool INV>
CNP_DEV void fft_columns(int CS, int X, int logH, const double2* __restrict__ tw, int tid, int T) {
  int logNs = 0;
  while (logNs < logH) {
    const int rem = logH - logNs;
    const int Ns = 1 << logNs;
    if (rem >= 4) { fft_stage<16, INV>(CS, X, logH, Ns, logNs, tw, tid, T); logNs += 4; }
    else if (rem == 3) { fft_stage<8, INV>(CS, X, logH, Ns, logNs, tw, tid, T); logNs += 3; }
    else if (rem == 2) { fft_stage<4, INV>(CS, X, logH, Ns, logNs, tw, tid, T); logNs += 2; }
    else { fft_stage<2, INV>(CS, X, logH, Ns, logNs, tw, tid, T); logNs += 1; }
  }
}

// ---------------------------------------------------------------- split / merge (real ↔ half)
// forward: X_k = ½[(Z_k + conj Z_{H−k}) − i ω_N^k (Z_k − conj Z_{H−k})], k = 0..H   (Z_H := Z_0)
CNP_DEV double2 split_fwd(double2 zk, double2 zmk, double2 wk) {
  const double2 zc = cconj(zmk);
  const double2 e = cadd(zk, zc);
  const double2 o = cmul(wk, csub(zk, zc));
  return make_double2(0.5 * (e.x + o.y), 0.5 * (e.y - o.x));  // e − i o
}
// inverse pre-processing: Z'_k = (Y_k + conj Y_{H−k}) + i ω_N^{−k} (Y_k − conj Y_{H−k})  (= 2 Z_k)
CNP_DEV double2 merge_inv(double2 yk, double2 ymk, double2 wk /* ω_N^k */) {
  const double2 yc = cconj(ymk);
  const double2 e = cadd(yk, yc);
  const double2 o = cmul_conj(csub(yk, yc), wk);
  return make_double2(e.x - o.y, e.y + o.x);  // e + i o
}

