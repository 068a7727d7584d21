// K5 fused (round 2): both axes of W⁻¹ or of W (the fast diagonalisation of step
// (b) of Eq. 3.2) in ONE pass over HBM, so the 2D P_α⁻¹ is three HBM passes (W⁻¹, the fused time pass,
// W) instead of five (48 B per unknown as structured).
//
// A persistent kernel runs two kinds of work items, handed out in ticket order (the k_fstep.cu scheme):
//   x-items  16 rows of time slice t: the x sine transform of k_dst4.cu (a line pair per 64 threads,
//            register radix passes, pair-local named barriers), rows written to the scratch vector Y;
//   y-items  16 columns of slice t: the y sine transform of k_dst5.cu (pair-fastest threads, 128-B
//            row segments) reading Y, written to the output; each Y line is dropped from L2 after
//            its last read (discard.global.L2), so Y never travels to HBM.
// Step s of the schedule lists the x-items of slice s and, `lag` steps later, the y-items of slice
// s − lag; a y-item waits (acquire) for its slice's counter, which every x-item bumps (release) after
// its rows are written.  The x-items a y-item waits for have smaller tickets and never wait, and the
// grid is the resident CTA count, so the wait always ends.  The window of slices between the phases
// (≈ lag + the CTAs in flight, ≈ 10-20 slices of 2 MB at n = 511) stays in the 126-MB L2.
// Both axes are x then y for W⁻¹ (pre-scales D_x⁻¹, D_y⁻¹) and for W (post-scales D_x·2/M, D_y·2/M):
// the axes commute (Kronecker product), only the scalings differ.
#include "common.cuh"
#include "internal.h"

#include "fft_device.cuh"

namespace {

CNP_DEV int zp(int k) { return k ^ ((k >> 3) & 7); }
CNP_DEV int op16(int x) { return x ^ ((x >> 4) & 15); }
CNP_DEV unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CNP_DEV void discard_line(const void* p) { asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory"); }
// barrier of one line pair's TP threads (a named barrier from two warps on; the warp below that)
CNP_DEV void pair_bar(int id, int tp) {
  if (tp >= 64) named_sync(id, tp);
  else __syncwarp();
}

}  // namespace

template <int LOGM>
struct XYPlan {
  static constexpr int M = 1 << LOGM, H = M / 2, n = M - 1;
  static constexpr int R1 = 8, R2 = LOGM == 7 ? 4 : 8, R3 = M / (R1 * R2);
  static constexpr int TP = M / 8;            // threads per line pair
  static constexpr int P = 8;                 // line pairs per item (16 rows / 16 columns)
  static constexpr int NT = P * TP;           // 512 at M = 512
  static constexpr int MINB = 1024 / NT;
  static constexpr int RS = M + 1;            // y regions: odd stride (x regions use M of them)
  static constexpr int I1 = (M / R1) / TP, I2 = (M / R2) / TP, I3 = (M / R3) / TP;
  static constexpr int XI = (n + 15) / 16;    // x-items per slice
  static constexpr int YI = M / 16;           // y-items per slice
  static constexpr int PER = XI + YI;         // schedule slots per step
  static constexpr size_t off_t1 = (size_t)P * RS * 16;
  static constexpr size_t off_t2 = off_t1 + (size_t)M * 16;
  static constexpr size_t off_abx = off_t2 + (size_t)(M / R1) * 16;
  static constexpr size_t off_aby = off_abx + (size_t)M * 16;
  static constexpr size_t off_px = off_aby + (size_t)M * 16;
  static constexpr size_t off_py = off_px + (size_t)M * 8;
  static constexpr size_t off_misc = off_py + (size_t)M * 8;
  static constexpr size_t bytes = off_misc + 16;
};

template <int LOGM>
__global__ void __launch_bounds__(XYPlan<LOGM>::NT, XYPlan<LOGM>::MINB)
    k_dstxy(const double* __restrict__ in, double* __restrict__ Y, double* __restrict__ out, int N, int64_t ld,
            const double* __restrict__ prex, const double* __restrict__ postx, const double* __restrict__ prey,
            const double* __restrict__ posty, const double2* __restrict__ tw2M, unsigned* __restrict__ cnt,
            unsigned* __restrict__ ticket, int lag, int accumulate, int debug_sign, int nx) {
  using PL = XYPlan<LOGM>;
  constexpr int M = PL::M, H = PL::H, n = PL::n, TP = PL::TP, P = PL::P, NT = PL::NT, RS = PL::RS;
  constexpr int R1 = PL::R1, R2 = PL::R2, R3 = PL::R3;
  char* const smem = reinterpret_cast<char*>(fft_smem);
  double2* const reg0 = reinterpret_cast<double2*>(smem);
  double2* const T1 = reinterpret_cast<double2*>(smem + PL::off_t1);
  double2* const T2 = reinterpret_cast<double2*>(smem + PL::off_t2);
  double2* const abx = reinterpret_cast<double2*>(smem + PL::off_abx);
  double2* const aby = reinterpret_cast<double2*>(smem + PL::off_aby);
  double2* const p2x = reinterpret_cast<double2*>(smem + PL::off_px);
  double2* const p2y = reinterpret_cast<double2*>(smem + PL::off_py);
  unsigned* const s_tick = reinterpret_cast<unsigned*>(smem + PL::off_misc);
  const int tid = threadIdx.x;
  const double sg = debug_sign ? -1.0 : 1.0;
  auto omega = [&](int e) {
    double2 w = tw2M[2 * (e & (M - 1))];
    w.y *= sg;
    return w;
  };
  for (int q = tid; q < M; q += NT) {
    const int k1 = q / (M / R1), m = q % (M / R1);
    T1[q] = omega(m * k1);
    if (q < M / R1) T2[q] = omega(R1 * (q % R3) * (q / R3));
    if (q < M / 2) {
      const int i = q / (TP / 2), l = q % (TP / 2), x = 16 * l + 2 * i;
      p2x[q] = make_double2(x < n ? (postx ? postx[x] : 1.0) : 0.0, x + 1 < n ? (postx ? postx[x + 1] : 1.0) : 0.0);
      p2y[q] = make_double2(x < n ? (posty ? posty[x] : 1.0) : 0.0, x + 1 < n ? (posty ? posty[x + 1] : 1.0) : 0.0);
    }
    double ax = 0.0, bx = 0.0, ay = 0.0, by = 0.0;
    if (q > 0) {
      const double s = -tw2M[q].y;  // sin(qπ/M)
      ax = (s + 0.5) * (prex ? prex[q - 1] : 1.0);
      bx = (s - 0.5) * (prex ? prex[M - q - 1] : 1.0);
      ay = (s + 0.5) * (prey ? prey[q - 1] : 1.0);
      by = (s - 0.5) * (prey ? prey[M - q - 1] : 1.0);
    }
    abx[q] = make_double2(ax, bx);
    aby[q] = make_double2(ay, by);
  }
  __syncthreads();
  pdl_enter();  // PDL: the input vector comes from the previous kernel
  const unsigned total = (unsigned)(N + lag) * PL::PER;
  const int64_t sl = (int64_t)n * ld;  // one time slice (ny = n rows of ld)
  while (true) {
    if (tid == 0) *s_tick = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned T = *s_tick;
    __syncthreads();
    if (T >= total) break;
    const int st = (int)(T / (unsigned)PL::PER), slot = (int)(T - (unsigned)st * PL::PER);
    const bool xitem = slot < PL::XI;
    const int t = xitem ? st : st - lag;
    if (t < 0 || t >= N) continue;
    if (xitem) {
      // ================= x-item: rows 16·slot .. +15 of slice t; pair pr = rows (2pr, 2pr + 1)
      const int pr = tid / TP, r = tid % TP, bar = 1 + pr;
      const int ya = 16 * slot + 2 * pr, yb = ya + 1;
      const bool actA = ya < n, actB = yb < n;
      const double* ra = in + (int64_t)t * sl + (int64_t)ya * ld;
      const double* rb = ra + ld;
      double2* const A = reg0 + pr * M;
#pragma unroll
      for (int i1 = 0; i1 < PL::I1; ++i1) {
        const int m = r + i1 * TP;
        double2 v[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) {
          const int j = m + (M / R1) * n1;
          double2 z = make_double2(0.0, 0.0);
          if (j > 0) {
            const double2 cf = abx[j];
            const double fa = actA ? __ldg(ra + j - 1) : 0.0, fam = actA ? __ldg(ra + M - j - 1) : 0.0;
            const double fb = actB ? __ldg(rb + j - 1) : 0.0, fbm = actB ? __ldg(rb + M - j - 1) : 0.0;
            z = make_double2(fma(cf.x, fa, cf.y * fam), fma(cf.x, fb, cf.y * fbm));
          }
          v[n1] = z;
        }
        dftR<R1, false>(v);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) A[k1 * (M / R1) + m] = k1 ? cmul(v[k1], T1[k1 * (M / R1) + m]) : v[0];
      }
      pair_bar(bar, TP);
      double2 u[PL::I2][R2];
#pragma unroll
      for (int i2 = 0; i2 < PL::I2; ++i2) {
        const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
        for (int m2 = 0; m2 < R2; ++m2) u[i2][m2] = A[k1 * (M / R1) + m3 + R3 * m2];
        dftR<R2, false>(u[i2]);
      }
      pair_bar(bar, TP);
#pragma unroll
      for (int i2 = 0; i2 < PL::I2; ++i2) {
        const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2)
          A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))] = (k2 && m3) ? cmul(u[i2][k2], T2[k2 * R3 + m3]) : u[i2][k2];
      }
      pair_bar(bar, TP);
      double2 w3[PL::I3][R3];
#pragma unroll
      for (int i3 = 0; i3 < PL::I3; ++i3) {
        const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
        for (int m3 = 0; m3 < R3; ++m3) w3[i3][m3] = A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))];
        if constexpr (R3 > 1) dftR<R3, false>(w3[i3]);
      }
      pair_bar(bar, TP);
#pragma unroll
      for (int i3 = 0; i3 < PL::I3; ++i3) {
        const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
        for (int k3 = 0; k3 < R3; ++k3) A[zp(k1 + R1 * k2 + R1 * R2 * k3)] = w3[i3][k3];
      }
      pair_bar(bar, TP);
      {
        const int ln = r / (TP / 2), q = r % (TP / 2);
        double Rk[8], Ik[8];
        double loc = 0.0;
#pragma unroll
        for (int i = 0; i <= 8; ++i) {
          const int k = 8 * q + i;
          const double2 Zk = A[zp(k & (M - 1))];
          const double2 Zm = A[zp((M - k) & (M - 1))];
          const double re = ln == 0 ? 0.5 * (Zk.x + Zm.x) : 0.5 * (Zk.y + Zm.y);
          const double im = ln == 0 ? 0.5 * (Zk.y - Zm.y) : 0.5 * (Zm.x - Zk.x);
          if (i < 8) {
            Rk[i] = (k == 0) ? 0.5 * re : re;
            loc += Rk[i];
          }
          if (i > 0) Ik[i - 1] = (k < H) ? -im : 0.0;
        }
        constexpr int W = TP / 2 < 32 ? TP / 2 : 32;
        double incl = loc;
#pragma unroll
        for (int o = 1; o < W; o <<= 1) {
          const double tt = __shfl_up_sync(0xffffffffu, incl, o, W);
          if (q % W >= o) incl += tt;
        }
        double run = incl - loc;
        pair_bar(bar, TP);
        double* so = reinterpret_cast<double*>(A) + ln * M;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          run += Rk[i];
          const double2 ps = p2x[i * (TP / 2) + q];
          const int x = 16 * q + 2 * i;
          so[op16(x)] = run * ps.x;
          so[op16(x + 1)] = Ik[i] * ps.y;
        }
      }
      pair_bar(bar, TP);
      {  // the two rows into Y (16-B stores, whole rows)
        const double* sr = reinterpret_cast<const double*>(A);
        double* ya_row = Y + (int64_t)t * sl + (int64_t)ya * ld;
#pragma unroll
        for (int e = r; e < M; e += TP) {
          const int ln = e / (M / 2), x = 2 * (e - ln * (M / 2));
          if (ln == 0 ? !actA : !actB) continue;
          const int p0 = op16(x);
          const double2 s2 = *reinterpret_cast<const double2*>(sr + ln * M + (p0 & ~1));
          *reinterpret_cast<double2*>(ya_row + (int64_t)ln * ld + x) = (p0 & 1) ? make_double2(s2.y, s2.x) : s2;
        }
      }
      __syncthreads();  // every pair's rows written (and its region free)
      if (tid == 0) {
        __threadfence();
        atomicAdd(cnt + t, 1u);
      }
    } else {
      // ================= y-item: columns 16·(slot − XI) .. +15 of slice t, after its x-items
      const int gy = slot - PL::XI, col0 = 16 * gy;
      if (tid == 0)
        while (ld_acq(cnt + t) < (unsigned)PL::XI) __nanosleep(64);
      __syncthreads();
      const int c = tid % P, r = tid / P;
      double2* const A = reg0 + c * RS;
      const double* slice = Y + (int64_t)t * sl + col0 + 2 * c;
#pragma unroll
      for (int i1 = 0; i1 < PL::I1; ++i1) {
        const int m = r + i1 * TP;
        double2 v[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) {
          const int j = m + (M / R1) * n1;
          double2 z = make_double2(0.0, 0.0);
          if (j > 0) {
            const double2 cf = aby[j];
            const double2 f = __ldcg(reinterpret_cast<const double2*>(slice + (int64_t)(j - 1) * ld));
            const double2 fm = __ldcg(reinterpret_cast<const double2*>(slice + (int64_t)(M - j - 1) * ld));
            z = make_double2(fma(cf.x, f.x, cf.y * fm.x), fma(cf.x, f.y, cf.y * fm.y));
          }
          v[n1] = z;
        }
        dftR<R1, false>(v);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) A[k1 * (M / R1) + m] = k1 ? cmul(v[k1], T1[k1 * (M / R1) + m]) : v[0];
      }
      __syncthreads();
      // the tile's Y lines are read: drop them from L2 (never written back to HBM)
      for (int q = tid; q < n; q += NT) discard_line(Y + (int64_t)t * sl + (int64_t)q * ld + col0);
      double2 u[PL::I2][R2];
#pragma unroll
      for (int i2 = 0; i2 < PL::I2; ++i2) {
        const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
        for (int m2 = 0; m2 < R2; ++m2) u[i2][m2] = A[k1 * (M / R1) + m3 + R3 * m2];
        dftR<R2, false>(u[i2]);
      }
      __syncthreads();
#pragma unroll
      for (int i2 = 0; i2 < PL::I2; ++i2) {
        const int q = r + i2 * TP, m3 = q % R3, k1 = q / R3;
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2)
          A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))] = (k2 && m3) ? cmul(u[i2][k2], T2[k2 * R3 + m3]) : u[i2][k2];
      }
      __syncthreads();
      double2 w3[PL::I3][R3];
#pragma unroll
      for (int i3 = 0; i3 < PL::I3; ++i3) {
        const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
        for (int m3 = 0; m3 < R3; ++m3) w3[i3][m3] = A[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))];
        if constexpr (R3 > 1) dftR<R3, false>(w3[i3]);
      }
      __syncthreads();
#pragma unroll
      for (int i3 = 0; i3 < PL::I3; ++i3) {
        const int q = r + i3 * TP, k1 = q % R1, k2 = q / R1;
#pragma unroll
        for (int k3 = 0; k3 < R3; ++k3) A[zp(k1 + R1 * k2 + R1 * R2 * k3)] = w3[i3][k3];
      }
      __syncthreads();
      const int cp = tid / TP, rr = tid % TP, ln = rr / (TP / 2), q = rr % (TP / 2);
      const double2* Z = reg0 + cp * RS;
      double Rk[8], Ik[8];
      double loc = 0.0;
#pragma unroll
      for (int i = 0; i <= 8; ++i) {
        const int k = 8 * q + i;
        const double2 Zk = Z[zp(k & (M - 1))];
        const double2 Zm = Z[zp((M - k) & (M - 1))];
        const double re = ln == 0 ? 0.5 * (Zk.x + Zm.x) : 0.5 * (Zk.y + Zm.y);
        const double im = ln == 0 ? 0.5 * (Zk.y - Zm.y) : 0.5 * (Zm.x - Zk.x);
        if (i < 8) {
          Rk[i] = (k == 0) ? 0.5 * re : re;
          loc += Rk[i];
        }
        if (i > 0) Ik[i - 1] = (k < H) ? -im : 0.0;
      }
      constexpr int W = TP / 2 < 32 ? TP / 2 : 32;
      double incl = loc;
#pragma unroll
      for (int o = 1; o < W; o <<= 1) {
        const double tt = __shfl_up_sync(0xffffffffu, incl, o, W);
        if (q % W >= o) incl += tt;
      }
      double run = incl - loc;
      __syncthreads();
      double* const stage = reinterpret_cast<double*>(smem);
      {
        double* so = stage + (2 * cp + ln) * RS;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          run += Rk[i];
          const double2 ps = p2y[i * (TP / 2) + q];
          const int x = 16 * q + 2 * i;
          so[op16(x)] = run * ps.x;
          so[op16(x + 1)] = Ik[i] * ps.y;
        }
      }
      __syncthreads();
      for (int e = tid; e < n * P; e += NT) {
        const int x = e / P, cc = e - x * P;
        const int px = op16(x);
        double2 v2 = make_double2(stage[(2 * cc) * RS + px], stage[(2 * cc + 1) * RS + px]);
        const int col = col0 + 2 * cc;
        if (col >= nx) v2.x = 0.0;  // padding columns stay exactly zero
        if (col + 1 >= nx) v2.y = 0.0;
        double2* o = reinterpret_cast<double2*>(out + (int64_t)t * sl + (int64_t)x * ld + col);
        if (accumulate) {
          const double2 pv = *o;
          v2.x += pv.x;
          v2.y += pv.y;
        }
        stg_cs2(o, v2);
      }
      __syncthreads();
    }
  }
}

template <int LOGM>
static cudaError_t run_dstxy(cnpint_ctx* c, const double* in, double* out, int inverse, int accumulate) {
  using PL = XYPlan<LOGM>;
  auto kern = k_dstxy<LOGM>;
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
  // schedule: the y-items of a slice `lag` steps after its x-items, lag ≥ the steps the resident CTAs
  // span (so the waits are short); the counters restart at 0 for every launch
  const int lag = (grid_max + PL::PER - 1) / PL::PER + 2;
  const unsigned total = (unsigned)(c->N + lag) * PL::PER;
  const int grid = (int)(total < (unsigned)grid_max ? total : (unsigned)grid_max);
  cudaError_t e = cudaMemsetAsync(c->d_xycnt, 0, (size_t)(c->N + 1) * sizeof(unsigned), c->stream);
  if (e != cudaSuccess) return e;
  const double* prex = inverse ? nullptr : c->d_dxi;
  const double* postx = inverse ? c->d_dx : nullptr;
  const double* prey = inverse ? nullptr : c->d_dyi;
  const double* posty = inverse ? c->d_dy : nullptr;
  return cnp_launch(c, kern, dim3(grid), dim3(PL::NT), PL::bytes, in, c->d_tmp3, out, c->N, c->ld, prex, postx,
                    prey, posty, (const double2*)c->d_twx, c->d_xycnt, c->d_xycnt + c->N, lag, accumulate,
                    c->debug & 1, c->nx);
}

// W⁻¹ (inverse = 0) or W (inverse = 1) on both axes in one pass (square grids, n + 1 ∈ {64, …, 512});
// NotSupported otherwise.  Uses the handle's scratch vector tmp3 as the L2-resident intermediate.
cudaError_t launch_dstxy(cnpint_ctx* c, const double* in, double* out, int inverse, int accumulate) {
  if (c->dim != 2 || c->ld != c->nx + 1 || c->ny != c->nx || !c->d_xycnt) return cudaErrorNotSupported;
  switch (c->nx + 1) {
    case 64: return run_dstxy<6>(c, in, out, inverse, accumulate);
    case 128: return run_dstxy<7>(c, in, out, inverse, accumulate);
    case 256: return run_dstxy<8>(c, in, out, inverse, accumulate);
    case 512: return run_dstxy<9>(c, in, out, inverse, accumulate);
    default: return cudaErrorNotSupported;
  }
}
