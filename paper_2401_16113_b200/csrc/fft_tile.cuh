// Tile FFT machinery shared by the time-axis kernels (k_tfft.cu) and the 2D sine transforms
// (k_dst.cu): compile-time-sized Stockham FFTs (radix 8/4/2) over NC complex columns held in the
// kernel's dynamic shared memory, with per-stage twiddle tables laid out for conflict-free reads.
#pragma once
#include "common.cuh"

namespace {

extern __shared__ double2 tf_smem[];

// e^{−2πi num/den}, exact argument reduction by sincospi (den a power of two)
CNP_DEV double2 expi_neg(int num, int den) {
  double sn, cs;
  sincospi(2.0 * (double)num / (double)den, &sn, &cs);
  return make_double2(cs, -sn);
}

// Shared column layout: one pad slot every 8 complex entries (8 × 16 B = one bank sweep), so the
// strided butterfly writes (stride R entries) and the per-column reads are conflict free.
CNP_DEV int pd(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int tf_cs(int logN2) { return (1 << logN2) + ((1 << logN2) >> 3) + 1; }
// Stage plan of a length-2^L local FFT: s stages of radix 2^{⌈L/s⌉} / 2^{⌊L/s⌋} (larger radices first),
// s = ⌈L/4⌉ from L = 10 on (radix 16 where one work item per thread keeps it in registers: 16·8·8,
// 16·16·8) and ⌈L/3⌉ below (8·8·8, 8·8·4, ...): few shared-memory passes, no radix-2 tail.
__host__ __device__ constexpr int tf_nst(int L) { return L >= 10 ? (L + 3) / 4 : (L + 2) / 3; }
__host__ __device__ constexpr int tf_lr(int L, int logNs) {  // radix (log) of the stage starting at logNs
  int acc = 0;
  const int s = tf_nst(L), rem = L % s;
  for (int i = 0; i < s; ++i) {
    const int r = rem == 0 ? L / s : (i < rem ? L / s + 1 : L / s);
    if (acc == logNs) return r;
    acc += r;
  }
  return 0;
}
// Per-stage twiddle table sizes: stage with NS > 1 and radix R stores ω_{NS R}^{r k} at [(r−1) NS + k].
__host__ __device__ constexpr int tf_stage_tw(int logN2, int logNs = 0) {
  return logNs >= logN2 ? 0
                        : ((logNs > 0 ? ((1 << tf_lr(logN2, logNs)) - 1) << logNs : 0) +
                           tf_stage_tw(logN2, logNs + tf_lr(logN2, logNs)));
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

// a · e^{∓2πi E/16} for odd E (forward −, inverse +)
template <int E, bool INV>
CNP_DEV double2 tw16s(double2 a) {
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
  constexpr double c = (E == 1 || E == 15) ? C1 : (E == 3 || E == 13) ? S1 : (E == 5 || E == 11) ? -S1 : -C1;
  constexpr double sn = (E == 1 || E == 7) ? S1 : (E == 3 || E == 5) ? C1 : (E == 9 || E == 15) ? -S1 : -C1;
  const double s = INV ? sn : -sn;  // e^{∓iθ} = cos θ ∓ i sin θ
  return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
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
  } else if constexpr (R == 16) {
    // four-step 4×4: A[r2][k1] = dft4_{r1}(v[4 r1 + r2]); A *= w16^{r2 k1}; out[k1 + 4 k2] = dft4_{r2}
    double2 a[4][4];
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) {
      a[r2][0] = v[r2]; a[r2][1] = v[r2 + 4]; a[r2][2] = v[r2 + 8]; a[r2][3] = v[r2 + 12];
      dft4r<INV>(a[r2][0], a[r2][1], a[r2][2], a[r2][3]);
    }
    a[1][1] = tw16s<1, INV>(a[1][1]); a[1][2] = tw8_1<INV>(a[1][2]); a[1][3] = tw16s<3, INV>(a[1][3]);
    a[2][1] = tw8_1<INV>(a[2][1]); a[2][2] = cmul_mi<INV>(a[2][2]); a[2][3] = tw8_3<INV>(a[2][3]);
    a[3][1] = tw16s<3, INV>(a[3][1]); a[3][2] = tw8_3<INV>(a[3][2]); a[3][3] = tw16s<9, INV>(a[3][3]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 b0 = a[0][k1], b1 = a[1][k1], b2 = a[2][k1], b3 = a[3][k1];
      dft4r<INV>(b0, b1, b2, b3);
      v[k1] = b0; v[k1 + 4] = b1; v[k1 + 8] = b2; v[k1 + 12] = b3;
    }
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
// items are read before one barrier and written after it.  First-stage input modes (FIRST):
//   TF_SCALE  input i multiplied by gm[i]·s (gm = a CTA's residue slice of Γ_α, s = basis scale);
//   TF_ODDEXT odd extension of a sequence held in slots 1..N2/2−1: elements 0 and N2/2 are 0 and
//             element i > N2/2 is −element(N2 − i) (the DST-I embedding of K5); if sc.ghi is set,
//             slot j is first multiplied by sc.ghi[j] (K5's diagonal pre-scaling D⁻¹).
enum { TF_PLAIN = 0, TF_SCALE = 1, TF_ODDEXT = 2 };
// TF_SCALE's factor for element i is the time row t = i·cstride + crank:
//   γ_t · s = ghi[t >> 6] · glo[t & 63] · s   (two-level table of Γ_α, see k_tfft.cu).
struct TfScale {
  const double* ghi;
  const double* glo;
  int cstride, crank;
  double s;
};
template <int LOGR, bool INV, int FIRST, int LOGN2, int NC, int LOGNS, int NT>
CNP_DEV void stage(double2* buf, const double2* stw, const TfScale& sc) {
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
        const int i = j + r * PER;
        if (FIRST == TF_ODDEXT) {
          constexpr int HALF = 1 << (LOGN2 - 1);
          const int src = i <= HALF ? i : (1 << LOGN2) - i;
          double2 x = buf[c * CS + pd(src)];
          if (sc.ghi) x = cscale(x, sc.ghi[src]);  // optional pre-scale table (0 at 0 and HALF)
          if (i == 0 || i == HALF) x = make_double2(0.0, 0.0);
          v[it][r] = i > HALF ? make_double2(-x.x, -x.y) : x;
        } else {
          v[it][r] = buf[c * CS + pd(i)];
          if (FIRST == TF_SCALE) {
            const int t = i * sc.cstride + sc.crank;
            v[it][r] = cscale(v[it][r], sc.ghi[t >> 6] * sc.glo[t & 63] * sc.s);
          }
        }
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

template <bool INV, int FIRST, int LOGN2, int NC, int NT, int LOGNS = 0>
CNP_DEV void local_fft(double2* buf, const double2* stw, const TfScale& sc) {
  if constexpr (LOGNS < LOGN2) {
    constexpr int LOGR = tf_lr(LOGN2, LOGNS);
    stage<LOGR, INV, LOGNS == 0 ? FIRST : TF_PLAIN, LOGN2, NC, LOGNS, NT>(buf, stw, sc);
    local_fft<INV, FIRST, LOGN2, NC, NT, LOGNS + LOGR>(buf, stw + (LOGNS > 0 ? ((1 << LOGR) - 1) << LOGNS : 0), sc);
  }
}

// Per-stage twiddle tables of a length-2^logN2 local FFT into stw (sign flip: debug hook).
CNP_DEV void fill_stage_twiddles(double2* stw, int logN2, double sg, int tid, int nt) {
  int off = 0;
  for (int logNs = 0; logNs < logN2;) {
    const int lr = tf_lr(logN2, logNs);
    if (logNs > 0) {
      const int ns = 1 << logNs, cnt = ((1 << lr) - 1) << logNs;
      for (int q = tid; q < cnt; q += nt) {
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


}  // namespace
