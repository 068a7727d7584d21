// K3: step (b) of Eq. 3.2 for a tridiagonal L_h — the N/2+1 complex
// shifted systems (λ1_k I − λ2_k Ã) ẑ_k = ŵ_k, k = 0..N/2 (Remark 3.1 halving).
//
// Each system is divided by λ2_k (Re λ2_k > 0) so that the off-diagonals stay
// real: rows  a_i x_{i−1} + b_i x_i + c_i x_{i+1} = d_i  with  a_i = −τ lo_i, c_i = −τ up_i (real),
// b_i = s_k − τ di_i, s_k = λ1_k/λ2_k, d_i = ŵ_i/λ2_k.  Every system is diagonally dominant
// (R22), so no pivoting is needed; a zero or non-finite pivot still sets the device
// status word (SPEC.md:298 SingularPreconditioner).
//
// Design (B200).  One system per G warps (P = 32G threads), NS systems per CTA, two or more CTAs
// per SM so that one CTA's HBM traffic overlaps another's arithmetic.  The system is brought into
// shared memory by cp.async (LDGSTS, no register staging) and written back coalesced.  Per system:
//   level 1   thread p owns a contiguous chunk of Lmin or Lmin+1 rows (long chunks first), held in
//             registers; a chunk-local elimination (forward sweep keeping the chunk's first unknown
//             as a spike, backward sweep keeping the last) leaves every interior unknown as
//             x_j = δ'_j − α'_j x_first − γ'_j x_last and two interface rows per chunk:
//               F: fa x_{first−1} + fb x_first + fc x_last = fd
//               G: ga x_first + gb x_last + gc x_{last+1} = gd
//   tree      adjacent segments are merged pairwise (log2 P levels: 5 by warp shuffles, the rest
//             through shared memory): merging A = [s, m] and B = [m+1, e] solves the 2×2 system of
//             A's G row and B's F row for (x_m, x_{m+1}) as affine functions of (x_s, x_e) and
//             substitutes them into A's F row and B's G row.  The root gives a 2×2 system for
//             (x_0, x_{m−1}); the stored affine maps then hand every chunk its two boundary values.
//   back-sub  x_j = δ'_j − α'_j x_first − γ'_j x_last in place, coalesced store.
// Three variants (template MODE):
//   MODE_VAR   variable rows (c3): everything computed per row.
//   MODE_TOEP  Toeplitz rows: the chunk coefficients (pivots, α', γ', F/G rows) depend only on k
//              and on the position in the chunk, so they are tabulated at cnpint_create (host, long
//              double); each thread only sweeps its right-hand side.
//   MODE_FAST  Toeplitz rows with equal chunks except the last (m = P·Ls − r, r ∈ {0, …}): every
//              merge's coefficient part is data independent and identical along a tree level
//              (two variants: with / without the last segment), so it is tabulated too and the tree
//              only carries the right-hand sides fd, gd (2 complex per merge instead of 8).
// Rows live in shared memory at sidx(i) = i ^ ((i >> padsh) & smask): an XOR swizzle inside each
// chunk-length block that keeps both the coalesced copies and the per-thread chunk reads
// bank-conflict free without padding.
#include "common.cuh"
#include "internal.h"

#include <cstdlib>
#include <cstring>

namespace {

struct Seg {
  double2 fa, fb, fc, fd, ga, gb, gc, gd;
};

CNP_DEV Seg shfl_seg(const Seg& s, int d) {
  Seg r;
  r.fa = shfl_down<double2>(s.fa, d); r.fb = shfl_down<double2>(s.fb, d);
  r.fc = shfl_down<double2>(s.fc, d); r.fd = shfl_down<double2>(s.fd, d);
  r.ga = shfl_down<double2>(s.ga, d); r.gb = shfl_down<double2>(s.gb, d);
  r.gc = shfl_down<double2>(s.gc, d); r.gd = shfl_down<double2>(s.gd, d);
  return r;
}

// Merge segment A (in place) with its right neighbour B; the affine maps
//   x_m = P0 + P1 x_s + P2 x_e,  x_{m+1} = R0 + R1 x_s + R2 x_e
// are written to cf[0..5].  Returns false on a zero / non-finite 2x2 determinant.
// "Singular to working precision": a pivot or 2×2 determinant that cancels to below 1e-13 of the
// magnitude of its terms (or is not finite).  An exactly singular system (e.g. P_1 at k = 0 with a
// singular Ã, Remark 3.2) rarely produces an exact zero in the partitioned elimination, so the zero
// test of the header is read relatively.  The shifted systems of P_α (α < 1) are diagonally dominant
// (R22): their pivots never come near this.
CNP_DEV bool cancels(double2 x, double ref2) {
  const double x2 = fma(x.x, x.x, x.y * x.y);
  return !(x2 > 1e-26 * ref2) || !isfinite(x2);
}
CNP_DEV double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

CNP_DEV bool merge(Seg& A, const Seg& B, double2* cf) {
  const double2 det = csub(cmul(A.gb, B.fb), cmul(A.gc, B.fa));
  const bool sing = cancels(det, cabs2(cmul(A.gb, B.fb)) + cabs2(cmul(A.gc, B.fa)));
  const double2 id = crecip_nr(det);
  const double2 P0 = cmul(csub(cmul(B.fb, A.gd), cmul(A.gc, B.fd)), id);
  const double2 P1 = cneg(cmul(cmul(B.fb, A.ga), id));
  const double2 P2 = cmul(cmul(A.gc, B.fc), id);
  const double2 R0 = cmul(csub(cmul(A.gb, B.fd), cmul(B.fa, A.gd)), id);
  const double2 R1 = cmul(cmul(B.fa, A.ga), id);
  const double2 R2 = cneg(cmul(cmul(A.gb, B.fc), id));
  cf[0] = P0; cf[1] = P1; cf[2] = P2; cf[3] = R0; cf[4] = R1; cf[5] = R2;
  A.fb = cfma(A.fc, P1, A.fb);
  A.fd = cfms(A.fd, A.fc, P0);
  A.fc = cmul(A.fc, P2);
  A.ga = cmul(B.ga, R1);
  A.gb = cfma(B.ga, R2, B.gb);
  A.gd = cfms(B.gd, B.ga, R0);
  A.gc = B.gc;
  return cfinite(id) && !sing;
}

CNP_DEV void unmerge(const double2* cf, double2 xs, double2 xe, double2& xm, double2& xm1) {
  xm = cfma(cf[2], xe, cfma(cf[1], xs, cf[0]));
  xm1 = cfma(cf[5], xe, cfma(cf[4], xs, cf[3]));
}

}  // namespace

enum { MODE_VAR = 0, MODE_TOEP = 1, MODE_FAST = 2 };

// Toeplitz table per frequency k (tri_cfg().tabstride complex entries):
//   [0, L)                   inv_j = 1/pivot_j of the chunk forward sweep (j = 1..L−1)
//   v = 0, 1 (chunk length Lmin + v), base L + v(2L+3):
//     +0 α_{len−1} (G row ga)   +1 F row fb   +2 F row fc   +3.. α'_j (j < L)   +3+L.. γ'_j (j < L)
//   fast tree, base 5L+6, level q = 0..NLV−1, variant v (0 standard, 1 merge with the last
//   segment), 10 entries: pa pb ra rb P1 P2 R1 R2 fcA gaB, with
//     P0 = pa gd_A + pb fd_B,  R0 = ra fd_B + rb gd_A,  fd ← fd_A − fcA P0,  gd ← gd_B − gaB R0,
//     x_m = P0 + P1 x_s + P2 x_e,  x_{m+1} = R0 + R1 x_s + R2 x_e;
//   root (4 entries): x_0 = c0 fd + c1 gd,  x_{m−1} = c2 fd + c3 gd.
// two CTAs per SM (measured: forcing three for the fast tree, 80 registers, is slower at c2)
template <int MODE, int L, int MAXT>
__global__ void __launch_bounds__(MAXT, 2)
    k_tridiag(const double2* __restrict__ what, double2* __restrict__ zhat, const double* __restrict__ lo,
              const double* __restrict__ di, const double* __restrict__ up, const double2* __restrict__ sk,
              const double2* __restrict__ il2, const double2* __restrict__ tab, int m, int64_t W, int K, int G,
              int logG, int NS, int padsh, int smask, int TS, double tau, int* __restrict__ status,
              const double2* __restrict__ lam1, int skip) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  constexpr bool TOEP = MODE != MODE_VAR;
  constexpr bool FAST = MODE == MODE_FAST;
  constexpr int NCF = FAST ? 2 : 6;  // stored coefficients per merge
  constexpr int L1S = 5 * L + 6;
  extern __shared__ double2 smem[];
  const int nwarp = NS * G, P = 32 * G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp / G, wg = warp - g * G, p = wg * 32 + lane;
  const int MP = tri_rows_alloc(m, padsh);
  const int per_sys = TOEP ? MP + TS : 3 * MP;
  double2* const D = smem + g * per_sys;
  double2* const T = D + MP;                 // Toeplitz table
  double2* const Ap = D + MP;                // variable rows: α'
  double2* const Gp = D + 2 * MP;            //                γ'
  double2* const coefw = smem + NS * per_sys;            // [nwarp][31][NCF]
  double2* const coefx = coefw + nwarp * 31 * NCF;       // [NS][15][NCF]
  double2* const segr = coefx + NS * 15 * NCF;           // [nwarp][8]
  double2* const bnd = segr + nwarp * 8;                 // [nwarp][2]
  auto sidx = [&](int i) { return i ^ ((i >> padsh) & smask); };
  const int k = blockIdx.x * NS + g;
  const bool act = k < K;  // uniform over the system's warps
  // per-frequency scalars first: their latency overlaps the copy issue below
  double2 il = make_double2(0.0, 0.0), skk = il;
  if (act) { il = __ldg(il2 + k); skk = __ldg(sk + k); }
  // ---------------- asynchronous load of the system (and its table) into shared memory
  if (act) {
    const double2* src = what + (int64_t)k * W;
    if (!(skip & 1))
      for (int i = p; i < m; i += P) cp_async16(D + sidx(i), src + i);
    if (TOEP)
      for (int i = p; i < TS; i += P) cp_async16(T + i, tab + (size_t)k * TS + i);
  }
  cp_async_commit();
  const int Lmin = m / P, nlong = m - P * Lmin;
  const int len = p < nlong ? Lmin + 1 : Lmin;
  const int i0 = p < nlong ? p * (Lmin + 1) : nlong * (Lmin + 1) + (p - nlong) * Lmin;
  const int i1 = i0 + len;
  bool ok = true;
  cp_async_wait<0>();
  __syncthreads();
  Seg sg;
  // α = 1, k = N/2: λ2 = 0 (il2 = 0 from the host tables) — the system is λ1 z = w; uniform per system
  const bool diag_only = act && il.x == 0.0 && il.y == 0.0;
  if (diag_only) {
    const double2 r = crecip(lam1[k]);
    for (int i = p; i < m; i += P) D[sidx(i)] = cmul(D[sidx(i)], r);
  }
  double2 dl[L];  // the chunk's right-hand side; for Toeplitz rows δ' stays here until the back-substitution
  if (act && !diag_only && !(skip & 2)) {
#pragma unroll
    for (int j = 0; j < L; ++j) dl[j] = (j < len) ? cmul(D[sidx(i0 + j)], il) : make_double2(0.0, 0.0);
    if (TOEP) {
      const double2* tv = T + L + (len - Lmin) * (2 * L + 3);
      const double a = -tau * lo[1], c = -tau * up[1];
      // forward: δ_1 = d_1 inv_1, δ_j = (d_j − a δ_{j−1}) inv_j
      double2 last = dl[0];
#pragma unroll
      for (int j = 1; j < L; ++j) {
        if (j < len) {
          last = cmul(j == 1 ? dl[1] : crfms(dl[j], a, last), T[j]);
          dl[j] = last;
        }
      }
      sg.gd = last;
      if (!FAST) {
        sg.ga = tv[0];
        sg.gb = make_double2(1.0, 0.0);
        sg.gc = cscale(T[len - 1], c);
      }
      // backward: δ'_j = δ_j − γ_j δ'_{j+1}, γ_j = c inv_j  (δ'_{len−2} = δ_{len−2})
#pragma unroll
      for (int j = L - 3; j >= 1; --j)
        if (j <= len - 3) dl[j] = cfms(dl[j], cscale(T[j], c), dl[j + 1]);
      if (!FAST) {
        sg.fa = make_double2(i0 == 0 ? 0.0 : a, 0.0);
        sg.fb = tv[1];
        sg.fc = tv[2];
      }
      sg.fd = len >= 3 ? crfms(dl[0], c, dl[1]) : dl[0];
      if (!FAST) {  // the fast tree keeps δ' in registers through the merges (enough registers there)
#pragma unroll
        for (int j = 1; j < L - 1; ++j)
          if (j <= len - 2) D[sidx(i0 + j)] = dl[j];
      }
    } else {
      double2 ap[L], gp[L];
      double2 alp = make_double2(0.0, 0.0), gam = alp, last = dl[0];
#pragma unroll
      for (int j = 1; j < L; ++j) {
        if (j < len) {
          const int i = i0 + j;
          const double a = -tau * lo[i], c = -tau * up[i];
          const double2 bb = make_double2(skk.x - tau * di[i], skk.y);
          const double2 piv = (j == 1) ? bb : crfms(bb, a, gam);
          const double2 inv = crecip_nr(piv);
          ok &= cfinite(inv) && !cancels(piv, cabs2(bb) + (j == 1 ? 0.0 : a * a * cabs2(gam)));
          alp = (j == 1) ? cscale(inv, a) : cscale(cmul(alp, inv), -a);
          gam = cscale(inv, c);
          last = (j == 1) ? cmul(dl[1], inv) : cmul(crfms(dl[j], a, last), inv);
          dl[j] = last;
          ap[j] = alp;
          gp[j] = gam;
        }
      }
      sg.ga = alp;
      sg.gb = make_double2(1.0, 0.0);
      sg.gc = gam;
      sg.gd = last;
#pragma unroll
      for (int j = L - 3; j >= 1; --j) {
        if (j <= len - 3) {
          const double2 gj = gp[j];
          dl[j] = cfms(dl[j], gj, dl[j + 1]);
          ap[j] = cfms(ap[j], gj, ap[j + 1]);
          gp[j] = cneg(cmul(gj, gp[j + 1]));
        }
      }
      const double a0 = -tau * lo[i0], c0 = -tau * up[i0];
      const double2 b0 = make_double2(skk.x - tau * di[i0], skk.y);
      sg.fa = make_double2(a0, 0.0);
      if (len >= 3) {
        sg.fb = crfms(b0, c0, ap[1]);
        sg.fc = cscale(gp[1], -c0);
        sg.fd = crfms(dl[0], c0, dl[1]);
      } else {
        sg.fb = b0;
        sg.fc = make_double2(c0, 0.0);
        sg.fd = dl[0];
      }
#pragma unroll
      for (int j = 1; j < L - 1; ++j) {
        if (j <= len - 2) {
          const int q = sidx(i0 + j);
          D[q] = dl[j];
          Ap[q] = ap[j];
          Gp[q] = gp[j];
        }
      }
    }
  }
  // ---------------- tree up: 5 warp levels
  double2* cw = coefw + warp * 31 * NCF;
  const double2* TT = T + L1S;  // fast-tree table
  if (act && !diag_only) {
#pragma unroll
    for (int lv = 1; lv <= 5; ++lv) {
      const int sft = 1 << (lv - 1);
      const bool left = (lane & ((1 << lv) - 1)) == 0;
      double2* slot = cw + (32 - (64 >> lv) + (lane >> lv)) * NCF;
      if (FAST) {
        const double2 fdB = shfl_down<double2>(sg.fd, sft), gdB = shfl_down<double2>(sg.gd, sft);
        if (left) {
          const int v = (wg == G - 1 && lane + 2 * sft == 32) ? 1 : 0;
          const double2* cf = TT + ((lv - 1) * 2 + v) * 10;
          const double2 P0 = cfma(cf[0], sg.gd, cmul(cf[1], fdB));
          const double2 R0 = cfma(cf[2], fdB, cmul(cf[3], sg.gd));
          slot[0] = P0;
          slot[1] = R0;
          sg.fd = cfms(sg.fd, cf[8], P0);
          sg.gd = cfms(gdB, cf[9], R0);
        }
      } else {
        const Seg B = shfl_seg(sg, sft);
        if (left) ok &= merge(sg, B, slot);
      }
    }
  }
  double2 xs = make_double2(0.0, 0.0), xe = make_double2(0.0, 0.0);
  auto root = [&](const Seg& t) {
    if (FAST) {
      const double2* r = TT + (5 + logG) * 20;
      xs = cfma(r[0], t.fd, cmul(r[1], t.gd));
      xe = cfma(r[2], t.fd, cmul(r[3], t.gd));
      return;
    }
    // fb x_0 + fc x_{m−1} = fd ; ga x_0 + gb x_{m−1} = gd  (x_{−1} = x_m = 0)
    const double2 det = csub(cmul(t.fb, t.gb), cmul(t.fc, t.ga));
    const double2 id = crecip(det);
    ok &= cfinite(id) && !cancels(det, cabs2(cmul(t.fb, t.gb)) + cabs2(cmul(t.fc, t.ga)));
    xs = cmul(csub(cmul(t.fd, t.gb), cmul(t.fc, t.gd)), id);
    xe = cmul(csub(cmul(t.fb, t.gd), cmul(t.ga, t.fd)), id);
  };
  if (G == 1) {
    if (act && !diag_only && lane == 0) root(sg);
  } else {
    // ---------------- cross-warp levels (warp 0 of the system, lanes 0..G−1)
    if (lane == 0) {
      double2* r = segr + warp * 8;
      r[3] = sg.fd; r[7] = sg.gd;
      if (!FAST) { r[0] = sg.fa; r[1] = sg.fb; r[2] = sg.fc; r[4] = sg.ga; r[5] = sg.gb; r[6] = sg.gc; }
    }
    named_sync(1 + g, 32 * G);
    if (wg == 0 && act && !diag_only) {
      Seg t = sg;
      if (lane < G) {
        const double2* r = segr + (g * G + lane) * 8;
        t.fd = r[3]; t.gd = r[7];
        if (!FAST) { t.fa = r[0]; t.fb = r[1]; t.fc = r[2]; t.ga = r[4]; t.gb = r[5]; t.gc = r[6]; }
      }
      double2* cx = coefx + g * 15 * NCF;
      for (int lv = 1; lv <= logG; ++lv) {
        const int sft = 1 << (lv - 1);
        const bool left = (lane & ((1 << lv) - 1)) == 0 && lane < G;
        double2* slot = cx + (G - (2 * G >> lv) + (lane >> lv)) * NCF;
        if (FAST) {
          const double2 fdB = shfl_down<double2>(t.fd, sft), gdB = shfl_down<double2>(t.gd, sft);
          if (left) {
            const int v = (lane + 2 * sft == G) ? 1 : 0;
            const double2* cf = TT + ((5 + lv - 1) * 2 + v) * 10;
            const double2 P0 = cfma(cf[0], t.gd, cmul(cf[1], fdB));
            const double2 R0 = cfma(cf[2], fdB, cmul(cf[3], t.gd));
            slot[0] = P0;
            slot[1] = R0;
            t.fd = cfms(t.fd, cf[8], P0);
            t.gd = cfms(gdB, cf[9], R0);
          }
        } else {
          const Seg B = shfl_seg(t, sft);
          if (left) ok &= merge(t, B, slot);
        }
      }
      if (lane == 0) root(t);
      for (int lv = logG; lv >= 1; --lv) {
        const int sft = 1 << (lv - 1);
        const bool left = (lane & ((1 << lv) - 1)) == 0 && lane < G;
        const bool right = (lane & ((1 << lv) - 1)) == sft && lane < G;
        double2 xm = make_double2(0.0, 0.0), xm1 = xm;
        if (left) {
          const double2* slot = cx + (G - (2 * G >> lv) + (lane >> lv)) * NCF;
          if (FAST) {
            const int v = (lane + 2 * sft == G) ? 1 : 0;
            const double2* cf = TT + ((5 + lv - 1) * 2 + v) * 10;
            xm = cfma(cf[5], xe, cfma(cf[4], xs, slot[0]));
            xm1 = cfma(cf[7], xe, cfma(cf[6], xs, slot[1]));
          } else {
            unmerge(slot, xs, xe, xm, xm1);
          }
        }
        const double2 rs = shfl_up2(xm1, sft), re = shfl_up2(xe, sft);
        if (left) xe = xm;
        if (right) { xs = rs; xe = re; }
      }
      if (lane < G) {
        bnd[(g * G + lane) * 2] = xs;
        bnd[(g * G + lane) * 2 + 1] = xe;
      }
    }
    named_sync(1 + g, 32 * G);
    if (lane == 0) {
      xs = bnd[warp * 2];
      xe = bnd[warp * 2 + 1];
    }
  }
  if (act && !diag_only) {
    // ---------------- tree down: 5 warp levels
#pragma unroll
    for (int lv = 5; lv >= 1; --lv) {
      const int sft = 1 << (lv - 1);
      const bool left = (lane & ((1 << lv) - 1)) == 0;
      const bool right = (lane & ((1 << lv) - 1)) == sft;
      double2 xm = make_double2(0.0, 0.0), xm1 = xm;
      if (left) {
        const double2* slot = cw + (32 - (64 >> lv) + (lane >> lv)) * NCF;
        if (FAST) {
          const int v = (wg == G - 1 && lane + 2 * sft == 32) ? 1 : 0;
          const double2* cf = TT + ((lv - 1) * 2 + v) * 10;
          xm = cfma(cf[5], xe, cfma(cf[4], xs, slot[0]));
          xm1 = cfma(cf[7], xe, cfma(cf[6], xs, slot[1]));
        } else {
          unmerge(slot, xs, xe, xm, xm1);
        }
      }
      const double2 rs = shfl_up2(xm1, sft), re = shfl_up2(xe, sft);
      if (left) xe = xm;
      if (right) { xs = rs; xe = re; }
    }
    // ---------------- back-substitution in place
    D[sidx(i0)] = xs;
    D[sidx(i1 - 1)] = xe;
    if (TOEP) {
      const double2* tv = T + L + (len - Lmin) * (2 * L + 3);
#pragma unroll
      for (int j = 1; j < L - 1; ++j) {
        if (j <= len - 2) {
          const int q = sidx(i0 + j);
          D[q] = cfms(cfms(FAST ? dl[j] : D[q], tv[3 + j], xs), tv[3 + L + j], xe);
        }
      }
    } else {
#pragma unroll
      for (int j = 1; j < L - 1; ++j) {
        if (j <= len - 2) {
          const int q = sidx(i0 + j);
          D[q] = cfms(cfms(D[q], Ap[q], xs), Gp[q], xe);
        }
      }
    }
    if (!ok) atomicOr(status, 1);
  }
  __syncthreads();
  if (act) {
    double2* dst = zhat + (int64_t)k * W;
    if (!(skip & 4))
      for (int i = p; i < m; i += P) stg_cs2(dst + i, D[sidx(i)]);
    for (int i = m + p; i < W; i += P) dst[i] = make_double2(0.0, 0.0);
  }
}

// Variable rows, second generation (round 2; c3).  MODE_VAR above measured (r01 ncu: 210 µs at c3, DRAM
// 12 %, 18 % warps active, fp64 pipe 31 %): its merge tree runs levels 1–5 in every warp on all 32 lanes
// while 16, 8, …, 1 of them merge, so a merge (≈ 115 fp64 instructions) is paid per warp per level, and
// α', γ', δ' go through shared memory (3·MP complex per system).  Phase traces (scripts/trivar_trace.py,
// clock64 per CTA, c3, cycles per system) of the intermediate designs: a dense shared-memory tree — load
// 1.9 k, sweeps 5.3 k, tree 8.3 k (≈ 860 cycles per level), back-substitution and store 1.5 k; warp-shuffle
// levels in each warp plus the upper levels in warp 0 — sweeps 2.4 k, tree 10.3 k.  A tree level is bound
// by one warp issuing the merge's ≈ 115 fp64 instructions (the fp64 pipe takes a warp instruction every
// other cycle per SM sub-partition) behind its ≈ 130-cycle dependency chain (DFMA 8 cycles, rcp + two
// Newton steps 47 cycles: scripts/lat_bench.cu), and the upper levels are a serial chain of them.
// But everything in a merge except the right-hand-side parts (fd, gd) depends only on the frequency k
// and the rows, which are fixed for the handle.  So:
//   * build (once per handle, k_trivar<…, BUILD>: at cnpint_create and whenever the tables change): the
//     coefficient part of every merge of the upper levels S+1 … log2 P (S = max(2, log2 G) levels stay in
//     the warps) and of the root is written to a per-frequency table vtab (MODE_FAST's layout: pa pb ra rb
//     P1 P2 R1 R2 fcA gaB per merge, 4 root entries; ≈ 5 KB per frequency at c3), and every
//     coefficient-only test of reading R29 (chunk pivots, merge and root determinants) runs there; a
//     frequency that fails it is flagged in its table row, and every solve reports it in the status word;
//   * solve: the chunk sweeps (α', γ', δ' stay in registers until the back-substitution; the rows lo, di,
//     up are fetched while the system copy is in flight), tree levels 1 … S by warp shuffles inside each
//     warp with the generic merge, one shared-memory hand-over of the P/2^S ≤ 32 segments' (fd, gd) to
//     warp 0, whose lanes run the upper levels from the table (2 complex per merge through the shuffles,
//     four complex FMAs), the root and the upper down levels, then the down levels 1 … S in each warp and
//     the back-substitution.  The table row is staged into shared memory with the system (cp.async).
// UNI: every chunk holds L − 1 or L rows (m ∈ (P(L−1), PL], c3), so only a chunk's last row is conditional.
#ifndef CNPINT_TRIVAR_MINB
#define CNPINT_TRIVAR_MINB 3  // resident CTAs per SM for P = 128 (c3): 168 registers, no spills
#endif
#ifdef CNPINT_TRIVAR_TRACE
// experiment builds only: per-CTA clock64 stamps at the phase boundaries of k_trivar (scripts/trivar_trace.py)
__device__ long long g_trv_trace[16384 * 10];
#define TRV_STAMP(q) \
  if (!BUILD && threadIdx.x == 0 && blockIdx.x < 16384) { \
    long long t_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)); g_trv_trace[blockIdx.x * 10 + (q)] = t_; \
    if ((q) == 0) { unsigned s_; asm volatile("mov.u32 %0, %%smid;" : "=r"(s_)); g_trv_trace[blockIdx.x * 10 + 9] = s_; } }
extern "C" int cnpint_trivar_trace(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trv_trace, sizeof(long long) * (size_t)n);
}
#else
#define TRV_STAMP(q)
#endif

namespace {
// build-time merge: as merge(), plus the coefficient part of the merge in MODE_FAST's layout
// (P0 = pa gd_A + pb fd_B, R0 = ra fd_B + rb gd_A, fd ← fd_A − fcA P0, gd ← gd_B − gaB R0), field f at tb[f·st]
CNP_DEV bool merge_tab(Seg& A, const Seg& B, double2* tb, int st) {
  const double2 det = csub(cmul(A.gb, B.fb), cmul(A.gc, B.fa));
  const bool sing = cancels(det, cabs2(cmul(A.gb, B.fb)) + cabs2(cmul(A.gc, B.fa)));
  const double2 id = crecip_nr(det);
  const double2 P1 = cneg(cmul(cmul(B.fb, A.ga), id));
  const double2 P2 = cmul(cmul(A.gc, B.fc), id);
  const double2 R1 = cmul(cmul(B.fa, A.ga), id);
  const double2 R2 = cneg(cmul(cmul(A.gb, B.fc), id));
  tb[0] = cmul(B.fb, id); tb[st] = cneg(cmul(A.gc, id)); tb[2 * st] = cmul(A.gb, id); tb[3 * st] = cneg(cmul(B.fa, id));
  tb[4 * st] = P1; tb[5 * st] = P2; tb[6 * st] = R1; tb[7 * st] = R2; tb[8 * st] = A.fc; tb[9 * st] = B.ga;
  A.fb = cfma(A.fc, P1, A.fb);
  A.fc = cmul(A.fc, P2);
  A.ga = cmul(B.ga, R1);
  A.gb = cfma(B.ga, R2, B.gb);
  A.gc = B.gc;
  return cfinite(id) && !sing;
}
}  // namespace

// table row per frequency (complex): upper level h = 1 … LOGP − S with n_h = NX >> h merges at
// 10(NX − 2n_h) + f·n_h + q (f = 0..9), the root (c0 c1 c2 c3: x_0 = c0 fd + c1 gd, x_{m−1} = c2 fd + c3 gd)
// at 10(NX − 1), the build's verdict at 10(NX − 1) + 4 (.x = 1: a coefficient-only test failed)
__host__ __device__ constexpr int trv_nx(int P) { return P >> ((P / 32) > 4 ? ((P / 32) == 8 ? 3 : 4) : 2); }
__host__ __device__ constexpr int trv_ts(int P) { return 10 * (trv_nx(P) - 1) + 5; }

template <int L, int MAXT, bool UNI, bool BUILD, bool APS>
__global__ void __launch_bounds__(MAXT, ((APS ? CNPINT_TRIVAR_MINB + 1 : CNPINT_TRIVAR_MINB) * 128 / MAXT) > 0
                                            ? (APS ? CNPINT_TRIVAR_MINB + 1 : CNPINT_TRIVAR_MINB) * 128 / MAXT : 1)
    k_trivar(const double2* __restrict__ what, double2* __restrict__ zhat, const double* __restrict__ lo,
             const double* __restrict__ di, const double* __restrict__ up, const double2* __restrict__ sk,
             const double2* __restrict__ il2, double2* __restrict__ vtab, int m, int64_t W, int padsh, int smask,
             double tau, int* __restrict__ status, const double2* __restrict__ lam1) {
  constexpr int P = MAXT, G = MAXT / 32;
  constexpr int LOGG = G == 1 ? 0 : G == 2 ? 1 : G == 4 ? 2 : G == 8 ? 3 : 4;
  constexpr int S = LOGG > 2 ? LOGG : 2;  // tree levels inside each warp
  constexpr int NX = P >> S;              // segments handed to warp 0 (<= 32)
  constexpr int LOGP = 5 + LOGG;
  constexpr int TS = trv_ts(P);
  static_assert(NX == trv_nx(P) && NX <= 32, "hand-over to one warp");
  TRV_STAMP(0);
  extern __shared__ double2 smem[];
  const int p = threadIdx.x, lane = p & 31, warp = p >> 5, k = blockIdx.x;
  const int MP = tri_rows_alloc(m, padsh);
  // APS: α' of the chunk rows goes to D (where its right-hand side was) and γ' to GP after the sweeps
  // (fewer registers: four CTAs per SM), else both stay in registers
  double2* const D = smem;          // [MP] rows; α' (APS) or the hand-over to warp 0 while the rows are dead
  double2* const CF = D + MP;       // [6P] levels 1..S: 6 coefficients per merge; then upper levels: P0, R0
  double2* const BX = CF + 6 * P;   // [2·NX] boundary values handed back by warp 0
  double2* const T = BX + 2 * NX;   // [TS] this frequency's table row (solve)
  double2* const GP = T + TS;       // APS: [MP] γ'
  double2* const HO = APS ? GP + MP : D;  // hand-over of the segments to warp 0 ([8·NX] build, [2·NX] solve)
  auto sidx = [&](int i) { return i ^ ((i >> padsh) & smask); };
  // create-time constants first (the frequency's scalars, the chunk's rows, the table row): with PDL
  // their latency overlaps the previous kernel's tail; the system itself only after griddepcontrol.wait
  const double2 il = __ldg(il2 + k), skk = __ldg(sk + k);
  const int Lmin = m / P, nlong = m - P * Lmin;
  const int len = p < nlong ? Lmin + 1 : Lmin;
  const int i0 = p < nlong ? p * (Lmin + 1) : nlong * (Lmin + 1) + (p - nlong) * Lmin;
  const int i1 = i0 + len;
  auto has = [&](int j) { return UNI ? (j < L - 1 || len == L) : j < len; };  // row j of the chunk exists
  double ra[L], rc[L], rd[L];  // lo, di, up are zero padded to ld >= m
#pragma unroll
  for (int j = 0; j < L; ++j) {
    const int i = has(j) ? i0 + j : i0;
    ra[j] = __ldg(lo + i);
    rc[j] = __ldg(up + i);
    rd[j] = __ldg(di + i);
  }
  if (!BUILD) {
    const double2* tr = vtab + (size_t)k * TS;
    for (int i = p; i < TS; i += P) cp_async16(T + i, tr + i);
    pdl_enter();
    const double2* src = what + (int64_t)k * W;
    for (int i = p; i < m; i += P) cp_async16(D + sidx(i), src + i);
  }
  cp_async_commit();
  bool ok = true;
  cp_async_wait<0>();
  __syncthreads();
  TRV_STAMP(1);
  double2* const dst = zhat + (int64_t)k * W;
  if (il.x == 0.0 && il.y == 0.0) {  // α = 1, k = N/2: λ2 = 0, the system is λ1 z = w (uniform per CTA)
    if (!BUILD) {
      const double2 r = crecip(lam1[k]);
      for (int i = p; i < m; i += P) stg_cs2(dst + i, cmul(D[sidx(i)], r));
      for (int i = m + p; i < W; i += P) dst[i] = make_double2(0.0, 0.0);
    } else if (p == 0) {
      vtab[(size_t)k * TS + TS - 1] = make_double2(0.0, 0.0);
    }
    return;
  }
  double2 dl[L], ap[L], gp[L];
  Seg sg;
#pragma unroll
  for (int j = 0; j < L; ++j) dl[j] = (!BUILD && has(j)) ? cmul(D[sidx(i0 + j)], il) : make_double2(0.0, 0.0);
  {
    double2 alp = make_double2(0.0, 0.0), gam = alp, last = dl[0];
#pragma unroll
    for (int j = 1; j < L; ++j) {
      if (has(j)) {
        const double a = -tau * ra[j], c = -tau * rc[j];
        const double2 bb = make_double2(skk.x - tau * rd[j], skk.y);
        const double2 piv = (j == 1) ? bb : crfms(bb, a, gam);
        const double2 inv = crecip_nr(piv);
        if (BUILD) ok &= cfinite(inv) && !cancels(piv, cabs2(bb) + (j == 1 ? 0.0 : a * a * cabs2(gam)));
        alp = (j == 1) ? cscale(inv, a) : cscale(cmul(alp, inv), -a);
        gam = cscale(inv, c);
        if (!BUILD) {
          last = (j == 1) ? cmul(dl[1], inv) : cmul(crfms(dl[j], a, last), inv);
          dl[j] = last;
        }
        ap[j] = alp;
        gp[j] = gam;
      }
    }
    sg.ga = alp;
    sg.gb = make_double2(1.0, 0.0);
    sg.gc = gam;
    sg.gd = last;
#pragma unroll
    for (int j = L - 3; j >= 1; --j) {
      if (UNI ? (j < L - 3 || len == L) : j <= len - 3) {
        const double2 gj = gp[j];
        if (!BUILD) dl[j] = cfms(dl[j], gj, dl[j + 1]);
        ap[j] = cfms(ap[j], gj, ap[j + 1]);
        gp[j] = cneg(cmul(gj, gp[j + 1]));
      }
    }
    const double a0 = -tau * ra[0], c0 = -tau * rc[0];
    const double2 b0 = make_double2(skk.x - tau * rd[0], skk.y);
    sg.fa = make_double2(a0, 0.0);
    if (len >= 3) {
      sg.fb = crfms(b0, c0, ap[1]);
      sg.fc = cscale(gp[1], -c0);
      sg.fd = crfms(dl[0], c0, dl[1]);
    } else {
      sg.fb = b0;
      sg.fc = make_double2(c0, 0.0);
      sg.fd = dl[0];
    }
  }
  if (APS && !BUILD) {
    __syncthreads();  // every row read from D before α' overwrites it
#pragma unroll
    for (int j = 1; j < L - 1; ++j)
      if (UNI ? (j < L - 2 || len == L) : j <= len - 2) {
        D[sidx(i0 + j)] = ap[j];
        GP[sidx(i0 + j)] = gp[j];
      }
  }
  TRV_STAMP(2);
  auto put_cf = [&](int l, int q, const double2* cf) {
    const int n = P >> l;
    double2* c = CF + 6 * (P - 2 * n) + q;
#pragma unroll
    for (int f = 0; f < 6; ++f) c[f * n] = cf[f];
  };
  auto get_cf = [&](int l, int q, double2* cf) {
    const int n = P >> l;
    const double2* c = CF + 6 * (P - 2 * n) + q;
#pragma unroll
    for (int f = 0; f < 6; ++f) cf[f] = c[f * n];
  };
  // ---------------- tree levels 1..S inside each warp (lane ≡ chunk within the warp), generic merges
#pragma unroll
  for (int l = 1; l <= S; ++l) {
    const Seg B = shfl_seg(sg, 1 << (l - 1));
    if ((lane & ((1 << l) - 1)) == 0) {
      double2 cf[6];
      const bool mok = merge(sg, B, cf);
      if (BUILD) ok &= mok;
      else put_cf(l, p >> l, cf);
    }
  }
  if (!APS) __syncthreads();  // every row read from D: the hand-over area may overwrite it
  if ((lane & ((1 << S) - 1)) == 0) {
    const int t = p >> S;
    if (BUILD) {
      HO[t] = sg.fa; HO[NX + t] = sg.fb; HO[2 * NX + t] = sg.fc;
      HO[4 * NX + t] = sg.ga; HO[5 * NX + t] = sg.gb; HO[6 * NX + t] = sg.gc;
    } else {
      HO[t] = sg.fd; HO[NX + t] = sg.gd;
    }
  }
  if (BUILD) {
    // ---------------- build: upper merges and the root into the table; the verdict of every test
    const bool bad = __syncthreads_or(!ok);
    if (warp == 0) {
      Seg t;
      const int u = lane < NX ? lane : 0;
      t.fa = HO[u]; t.fb = HO[NX + u]; t.fc = HO[2 * NX + u]; t.fd = make_double2(0.0, 0.0);
      t.ga = HO[4 * NX + u]; t.gb = HO[5 * NX + u]; t.gc = HO[6 * NX + u]; t.gd = t.fd;
      double2* const tr = vtab + (size_t)k * TS;
      bool wok = true;
#pragma unroll
      for (int h = 1; h <= LOGP - S; ++h) {
        const Seg B = shfl_seg(t, 1 << (h - 1));
        const int n = NX >> h;
        if (lane < NX && (lane & ((1 << h) - 1)) == 0) wok &= merge_tab(t, B, tr + 10 * (NX - 2 * n) + (lane >> h), n);
      }
      if (lane == 0) {
        const double2 det = csub(cmul(t.fb, t.gb), cmul(t.fc, t.ga));
        const double2 id = crecip(det);
        wok &= cfinite(id) && !cancels(det, cabs2(cmul(t.fb, t.gb)) + cabs2(cmul(t.fc, t.ga)));
        double2* r = tr + 10 * (NX - 1);
        r[0] = cmul(t.gb, id); r[1] = cneg(cmul(t.fc, id)); r[2] = cneg(cmul(t.ga, id)); r[3] = cmul(t.fb, id);
      }
      wok = !__any_sync(0xffffffffu, !wok);
      if (lane == 0) tr[TS - 1] = make_double2((bad || !wok) ? 1.0 : 0.0, 0.0);
    }
    return;
  }
  __syncthreads();
  TRV_STAMP(7);
  // ---------------- levels S+1..LOGP, the root and the upper down levels in warp 0 (lane ≡ segment) from
  // the table: the tree carries only (fd, gd) up and (x_s, x_e) down
  if (warp == 0) {
    const int u = lane < NX ? lane : 0;
    double2 fd = HO[u], gd = HO[NX + u];
    // every lane runs the arithmetic (lanes that do not merge at a level read a valid table slot and
    // discard the result): no divergent branches on the serial chain of levels
#pragma unroll
    for (int h = 1; h <= LOGP - S; ++h) {
      const int sft = 1 << (h - 1), n = NX >> h, q = u >> h;
      const bool left = lane < NX && (lane & ((1 << h) - 1)) == 0;
      const double2 fdB = shfl_down<double2>(fd, sft), gdB = shfl_down<double2>(gd, sft);
      const double2* cf = T + 10 * (NX - 2 * n) + q;
      const double2 P0 = cfma(cf[0], gd, cmul(cf[n], fdB));
      const double2 R0 = cfma(cf[2 * n], fdB, cmul(cf[3 * n], gd));
      if (left) {
        double2* cu = CF + 6 * (P - NX) + 2 * (NX - 2 * n) + q;
        cu[0] = P0;
        cu[n] = R0;
      }
      const double2 fdn = cfms(fd, cf[8 * n], P0), gdn = cfms(gdB, cf[9 * n], R0);
      fd = left ? fdn : fd;
      gd = left ? gdn : gd;
    }
    double2 xs = make_double2(0.0, 0.0), xe = xs;
    if (lane == 0) {
      const double2* r = T + 10 * (NX - 1);
      xs = cfma(r[0], fd, cmul(r[1], gd));
      xe = cfma(r[2], fd, cmul(r[3], gd));
    }
#pragma unroll
    for (int h = LOGP - S; h >= 1; --h) {
      const int sft = 1 << (h - 1), n = NX >> h, q = u >> h;
      const bool left = lane < NX && (lane & ((1 << h) - 1)) == 0;
      const bool right = lane < NX && (lane & ((1 << h) - 1)) == sft;
      const double2* cf = T + 10 * (NX - 2 * n) + q;
      const double2* cu = CF + 6 * (P - NX) + 2 * (NX - 2 * n) + q;
      const double2 xm = cfma(cf[5 * n], xe, cfma(cf[4 * n], xs, cu[0]));
      const double2 xm1 = cfma(cf[7 * n], xe, cfma(cf[6 * n], xs, cu[n]));
      const double2 rs = shfl_up2(xm1, sft), re = shfl_up2(xe, sft);
      if (left) xe = xm;
      if (right) { xs = rs; xe = re; }
    }
    if (lane < NX) { BX[lane] = xs; BX[NX + lane] = xe; }
  }
  __syncthreads();
  TRV_STAMP(3);
  // ---------------- down levels S..1 inside each warp
  double2 xs = make_double2(0.0, 0.0), xe = xs;
  if ((lane & ((1 << S) - 1)) == 0) { xs = BX[p >> S]; xe = BX[NX + (p >> S)]; }
#pragma unroll
  for (int l = S; l >= 1; --l) {
    const int sft = 1 << (l - 1);
    const bool left = (lane & ((1 << l) - 1)) == 0;
    const bool right = (lane & ((1 << l) - 1)) == sft;
    double2 xm = make_double2(0.0, 0.0), xm1 = xm;
    if (left) {
      double2 cf[6];
      get_cf(l, p >> l, cf);
      unmerge(cf, xs, xe, xm, xm1);
    }
    const double2 rs = shfl_up2(xm1, sft), re = shfl_up2(xe, sft);
    if (left) xe = xm;
    if (right) { xs = rs; xe = re; }
  }
  TRV_STAMP(4);
  // ---------------- back-substitution into D (the hand-over area there is dead)
  D[sidx(i0)] = xs;
  D[sidx(i1 - 1)] = xe;
#pragma unroll
  for (int j = 1; j < L - 1; ++j)
    if (UNI ? (j < L - 2 || len == L) : j <= len - 2) {
      const int q = sidx(i0 + j);
      D[q] = APS ? cfms(cfms(dl[j], D[q], xs), GP[q], xe) : cfms(cfms(dl[j], ap[j], xs), gp[j], xe);
    }
  if (p == 0 && T[TS - 1].x != 0.0) atomicOr(status, 1);  // the build flagged this frequency (R29)
  __syncthreads();
  TRV_STAMP(5);
  for (int i = p; i < m; i += P) stg_cs2(dst + i, D[sidx(i)]);
  for (int i = m + p; i < W; i += P) dst[i] = make_double2(0.0, 0.0);
  TRV_STAMP(6);
}

// Small-m path (m < 64): one thread per frequency, plain Thomas on the scaled system.
__global__ void k_tridiag_small(const double2* __restrict__ what, double2* __restrict__ zhat,
                                const double* __restrict__ lo, const double* __restrict__ di,
                                const double* __restrict__ up, const double2* __restrict__ sk,
                                const double2* __restrict__ il2, int m, int64_t W, double tau, int K,
                                int* __restrict__ status, const double2* __restrict__ lam1) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double2 s = sk[k], il = il2[k];
  double2 cp[64], dp[64];
  const double2* src = what + (int64_t)k * W;
  double2* dst = zhat + (int64_t)k * W;
  bool ok = true;
  if (il.x == 0.0 && il.y == 0.0) {  // α = 1, k = N/2: λ1 z = w
    const double2 r = crecip(lam1[k]);
    for (int i = 0; i < m; ++i) dst[i] = cmul(src[i], r);
    for (int i = m; i < W; ++i) dst[i] = make_double2(0.0, 0.0);
    return;
  }
  for (int i = 0; i < m; ++i) {
    const double a = -tau * lo[i], c = -tau * up[i];
    const double2 b = make_double2(s.x - tau * di[i], s.y);
    const double2 d = cmul(src[i], il);
    const double2 piv = (i == 0) ? b : crfms(b, a, cp[i - 1]);
    const double2 inv = crecip(piv);
    ok &= cfinite(inv) && !cancels(piv, cabs2(b) + (i == 0 ? 0.0 : a * a * cabs2(cp[i - 1])));
    cp[i] = cscale(inv, c);
    dp[i] = (i == 0) ? cmul(d, inv) : cmul(crfms(d, a, dp[i - 1]), inv);
  }
  double2 x = dp[m - 1];
  dst[m - 1] = x;
  for (int i = m - 2; i >= 0; --i) {
    x = cfms(dp[i], cp[i], x);
    dst[i] = x;
  }
  for (int i = m; i < W; ++i) dst[i] = make_double2(0.0, 0.0);
  if (!ok) atomicOr(status, 1);
}

TriCfg tri_cfg(int m, int toeplitz) {
  TriCfg t;
  std::memset(&t, 0, sizeof(t));
  t.small = m < 64;
  // chunks of <= Lcap rows: Lcap = 16 (Toeplitz: only the right-hand side lives in registers) or 8
  // (variable rows also carry α', γ'; measured: 8 / 512 threads at c2 and 4 at c3 are slower);
  // G = warps per system, NS = systems per CTA (<= 8 warps when G < 8).  Tuning overrides:
  // CNPINT_TRI_LCAP_T / CNPINT_TRI_LCAP_V (4, 8 or 16).
  static const int lcap_t = [] {  // tuning knobs, read once (thread-safe static initialisation)
    const char* e = getenv("CNPINT_TRI_LCAP_T");
    return e && (atoi(e) == 4 || atoi(e) == 8 || atoi(e) == 16) ? atoi(e) : 16;
  }();
  static const int lcap_v = [] {
    const char* e = getenv("CNPINT_TRI_LCAP_V");
    return e && (atoi(e) == 4 || atoi(e) == 8) ? atoi(e) : 8;
  }();
  const int Lcap = toeplitz ? lcap_t : lcap_v;
  int G = 1;
  while (G < 16 && 32 * G * Lcap < m) G <<= 1;
  t.G = G;
  t.logG = 0;
  while ((1 << t.logG) < G) ++t.logG;
  const int P = 32 * G;
  const int need = (m + P - 1) / P;
  t.L = need <= 4 ? 4 : need <= 8 ? 8 : need <= 16 ? 16 : -1;
  if (!toeplitz && t.L > 8) t.L = -1;
  t.Lmin = m / P;
  const int nlong = m - P * t.Lmin;
  t.fast = toeplitz && (nlong == 0 || nlong == P - 1);
  const int Ls = nlong ? t.Lmin + 1 : t.Lmin;  // swizzle block = the standard chunk length
  t.padsh = 0;
  while ((1 << (t.padsh + 1)) <= Ls) ++t.padsh;
  t.smask = (1 << t.padsh) - 1;
  if (t.smask > 7) t.smask = 7;
  t.nlv = 5 + t.logG;
  t.tabstride = toeplitz && t.L > 0 ? 5 * t.L + 6 + t.nlv * 20 + 4 : 0;
  t.NS = G >= 8 ? 1 : 8 / G;
  const int MP = tri_rows_alloc(m, t.padsh);
  const int per_sys = toeplitz ? MP + t.tabstride : 3 * MP;
  const int ncf = t.fast ? 2 : 6;
  auto smem_of = [&](int ns) {
    const int nw = ns * G;
    return (size_t)(ns * per_sys + nw * 31 * ncf + ns * 15 * ncf + nw * 8 + nw * 2) * sizeof(double2);
  };
  while (t.NS > 1 && smem_of(t.NS) > 110 * 1024) t.NS >>= 1;
  t.smem = smem_of(t.NS);
  return t;
}

// timing experiments only (results wrong): CNPINT_TRI_SKIP bit 1 = no load, 2 = no chunk sweeps,
// 4 = no store
// (read only in builds with -DCNPINT_EXPERIMENTS; the product build always runs every phase)
static int tri_skip() {
#ifdef CNPINT_EXPERIMENTS
  static const int v = getenv("CNPINT_TRI_SKIP") ? atoi(getenv("CNPINT_TRI_SKIP")) : 0;
  return v;
#else
  return 0;
#endif
}

template <int MODE, int L, int MAXT>
static cudaError_t run_tri_t(cnpint_ctx* c, const TriCfg& t, const double2* what, double2* zhat) {
  {
    int done = 0;
    cudaError_t ce = cnp_dev_cached((const void*)k_tridiag<MODE, L, MAXT>, &done, [&](int* v) {
      *v = 1;
      return cudaFuncSetAttribute(k_tridiag<MODE, L, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    if (ce != cudaSuccess) return ce;
  }
  const int K = c->H + 1;
  const int grid = (K + t.NS - 1) / t.NS;
  // shared memory of this variant (the generic trees store 6 coefficients per merge, the fast one 2)
  const int ncf = MODE == MODE_FAST ? 2 : 6, nw = t.NS * t.G;
  const int MP = tri_rows_alloc(c->nx, t.padsh);
  const size_t smem = (size_t)(t.NS * (MODE == MODE_VAR ? 3 * MP : MP + t.tabstride) + nw * 31 * ncf +
                               t.NS * 15 * ncf + nw * 8 + nw * 2) * sizeof(double2);
  return cnp_launch(c, k_tridiag<MODE, L, MAXT>, dim3(grid), dim3(32 * t.G * t.NS), smem, what, zhat, c->d_lo,
                    c->d_di, c->d_up, c->d_sk, c->d_il2, c->d_tritab, c->nx, c->ld, K, t.G, t.logG, t.NS, t.padsh,
                    t.smask, t.tabstride, c->tau_p, c->d_status, c->d_lam1, tri_skip());
}

template <int MODE, int L>
static cudaError_t run_tri(cnpint_ctx* c, const TriCfg& t, const double2* what, double2* zhat) {
  const int nt = 32 * t.G * t.NS;
  if (nt <= 256) return run_tri_t<MODE, L, 256>(c, t, what, zhat);
  if (nt <= 512) return run_tri_t<MODE, L, 512>(c, t, what, zhat);
  return cudaErrorInvalidValue;
}

template <int L, int MAXT, bool UNI, bool BUILD, bool APS>
static cudaError_t run_trivar_t(cnpint_ctx* c, const TriCfg& t, const double2* what, double2* zhat) {
  {
    int done = 0;
    cudaError_t ce = cnp_dev_cached((const void*)k_trivar<L, MAXT, UNI, BUILD, APS>, &done, [&](int* v) {
      *v = 1;
      return cudaFuncSetAttribute(k_trivar<L, MAXT, UNI, BUILD, APS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024);
    });
    if (ce != cudaSuccess) return ce;
  }
  constexpr int P = MAXT, NX = trv_nx(P), TS = trv_ts(P);
  const int MP = tri_rows_alloc(c->nx, t.padsh);
  const size_t smem = (size_t)(MP + 6 * P + 2 * NX + TS + (APS ? MP + 2 * NX : 0)) * sizeof(double2);
  if (BUILD) {  // plain launch: not part of a PDL chain
    k_trivar<L, MAXT, UNI, BUILD, APS><<<c->H + 1, P, smem, c->stream>>>(
        what, zhat, c->d_lo, c->d_di, c->d_up, c->d_sk, c->d_il2, c->d_vtab, c->nx, c->ld, t.padsh, t.smask,
        c->tau_p, c->d_status, c->d_lam1);
    return cudaGetLastError();
  }
  return cnp_launch(c, k_trivar<L, MAXT, UNI, BUILD, APS>, dim3(c->H + 1), dim3(P), smem, what, zhat, c->d_lo, c->d_di,
                    c->d_up, c->d_sk, c->d_il2, c->d_vtab, c->nx, c->ld, t.padsh, t.smask, c->tau_p, c->d_status,
                    c->d_lam1);
}

#ifndef CNPINT_TRIVAR_APS
#define CNPINT_TRIVAR_APS 1
#endif
template <int L, int MAXT, bool BUILD>
static cudaError_t run_trivar_m(cnpint_ctx* c, const TriCfg& t, const double2* what, double2* zhat) {
  constexpr bool APS = CNPINT_TRIVAR_APS && !BUILD;
  return t.Lmin >= L - 1 ? run_trivar_t<L, MAXT, true, BUILD, APS>(c, t, what, zhat)
                         : run_trivar_t<L, MAXT, false, BUILD, APS>(c, t, what, zhat);
}

template <int L, bool BUILD>
static cudaError_t run_trivar(cnpint_ctx* c, const TriCfg& t, const double2* what, double2* zhat) {
  switch (t.G) {
    case 1: return run_trivar_m<L, 32, BUILD>(c, t, what, zhat);
    case 2: return run_trivar_m<L, 64, BUILD>(c, t, what, zhat);
    case 4: return run_trivar_m<L, 128, BUILD>(c, t, what, zhat);
    case 8: return run_trivar_m<L, 256, BUILD>(c, t, what, zhat);
  }
  return cudaErrorInvalidValue;
}

// complex entries per frequency of the variable-row table (0: no table for this operator)
int trivar_table_stride(int m) {
  const TriCfg t = tri_cfg(m, 0);
  return t.small || t.L < 0 ? 0 : trv_ts(32 * t.G);
}

// (Re)builds the per-handle variable-row table (cnpint_create, cnpint_set_debug); synchronous
cudaError_t build_trivar_table(cnpint_ctx* c) {
  if (c->dim != 1 || c->toeplitz || !c->d_vtab) return cudaSuccess;
  const TriCfg t = tri_cfg(c->nx, 0);
  if (t.small) return cudaSuccess;
  cudaError_t e = t.L == 4 ? run_trivar<4, true>(c, t, nullptr, nullptr)
                : t.L == 8 ? run_trivar<8, true>(c, t, nullptr, nullptr) : cudaErrorInvalidValue;
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return e;
}

// fault injection (debug bit 2048): the shifted solve reports a singular pivot, as a genuinely singular
// system would — exercises the status-word path of cnpint_device_status / cnpint_gmres* deterministically
__global__ void k_inject_singular(int* status) { atomicOr(status, 1); }

cudaError_t launch_shifted_solve(cnpint_ctx* c, const double2* what, double2* zhat) {
  if (c->debug & 2048) {
    k_inject_singular<<<1, 1, 0, c->stream>>>(c->d_status);
    if (cudaError_t e = cudaGetLastError()) return e;
  }
  const int m = c->nx;
  const int K = c->H + 1;
  const int64_t W = c->ld;
  cnp_prof_begin(c, KID_TRIDIAG);
  const double bytes = 32.0 * cnp_spec_units(c);
  const TriCfg t = tri_cfg(m, c->toeplitz);
  cudaError_t e;
  if (t.small) {
    k_tridiag_small<<<(K + 127) / 128, 128, 0, c->stream>>>(what, zhat, c->d_lo, c->d_di, c->d_up, c->d_sk, c->d_il2,
                                                            m, W, c->tau_p, K, c->d_status, c->d_lam1);
    e = cudaGetLastError();
  } else if (!c->toeplitz && !(c->debug & 512)) {
    e = t.L == 4 ? run_trivar<4, false>(c, t, what, zhat) : t.L == 8 ? run_trivar<8, false>(c, t, what, zhat)
                                                                      : cudaErrorInvalidValue;
  } else if (!c->toeplitz) {  // debug 512: the first-generation variable-row kernel
    e = t.L == 4 ? run_tri<MODE_VAR, 4>(c, t, what, zhat) : t.L == 8 ? run_tri<MODE_VAR, 8>(c, t, what, zhat)
                                                                     : cudaErrorInvalidValue;
  } else if (t.fast && !(c->debug & 4)) {
    e = t.L == 4 ? run_tri<MODE_FAST, 4>(c, t, what, zhat)
      : t.L == 8 ? run_tri<MODE_FAST, 8>(c, t, what, zhat)
      : t.L == 16 ? run_tri<MODE_FAST, 16>(c, t, what, zhat)
                  : cudaErrorInvalidValue;
  } else {
    e = t.L == 4 ? run_tri<MODE_TOEP, 4>(c, t, what, zhat)
      : t.L == 8 ? run_tri<MODE_TOEP, 8>(c, t, what, zhat)
      : t.L == 16 ? run_tri<MODE_TOEP, 16>(c, t, what, zhat)
                  : cudaErrorInvalidValue;
  }
  cnp_prof_end(c, KID_TRIDIAG, bytes);
  return e;
}
