// The reduced system of the x-sharded shifted solve (shard.cu), shared by the device kernel and the
// host test entry point.  Per frequency k, with X_r = (xs_r, xe_r) the first / last unknown of rank r:
//   X_r = G_r + P_r X_{r−1} + Q_r X_{r+1},   G_r = ((g_r)_1, (g_r)_m),
//   P_r = [[0, α_r (v_r)_1], [0, α_r (v_r)_m]],   Q_r = [[β_r (w_r)_1, 0], [β_r (w_r)_m, 0]],
// solved by block Thomas with 2×2 complex blocks: D_0 = I, Y_0 = G_0; M_r = P_r D_{r−1}⁻¹,
// D_r = I − M_r Q_{r−1}, Y_r = G_r + M_r Y_{r−1}; X_{R−1} = D_{R−1}⁻¹ Y_{R−1},
// X_r = D_r⁻¹ (Y_r + Q_r X_{r+1}).  Layouts: red[(k R + r) 4 + (v1, vm, w1, wm)], ab[2r + (α, β)],
// ends_all[(r K + k) 2 + (g1, gm)] (the all-gather of every rank's [K][2]).
#pragma once
#include <cuda_runtime.h>

#define SHD __host__ __device__ inline

SHD double2 hd_c(double x, double y) { double2 r; r.x = x; r.y = y; return r; }
SHD double2 hd_cadd(double2 a, double2 b) { return hd_c(a.x + b.x, a.y + b.y); }
SHD double2 hd_csub(double2 a, double2 b) { return hd_c(a.x - b.x, a.y - b.y); }
SHD double2 hd_cmul(double2 a, double2 b) { return hd_c(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
SHD double2 hd_cscale(double2 a, double s) { return hd_c(a.x * s, a.y * s); }
SHD double hd_cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
SHD double2 hd_cdiv(double2 a, double2 b) {
  const double d = hd_cabs2(b);
  return hd_c((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

struct Blk2 {  // 2×2 complex matrix [[a, b], [c, d]]
  double2 a, b, c, d;
};
SHD Blk2 blk_mul(const Blk2& X, const Blk2& Y) {
  return Blk2{hd_cadd(hd_cmul(X.a, Y.a), hd_cmul(X.b, Y.c)), hd_cadd(hd_cmul(X.a, Y.b), hd_cmul(X.b, Y.d)),
              hd_cadd(hd_cmul(X.c, Y.a), hd_cmul(X.d, Y.c)), hd_cadd(hd_cmul(X.c, Y.b), hd_cmul(X.d, Y.d))};
}
SHD void blk_apply(const Blk2& X, double2 s, double2 e, double2* os, double2* oe) {
  *os = hd_cadd(hd_cmul(X.a, s), hd_cmul(X.b, e));
  *oe = hd_cadd(hd_cmul(X.c, s), hd_cmul(X.d, e));
}
// inverse; ok = false when det cancels below 1e-13 of its terms (singular to working precision)
SHD Blk2 blk_inv(const Blk2& X, bool* ok) {
  const double2 p = hd_cmul(X.a, X.d), q = hd_cmul(X.b, X.c);
  const double2 det = hd_csub(p, q);
  const double dd = hd_cabs2(det);
  if (!(dd > 1e-26 * (hd_cabs2(p) + hd_cabs2(q))) || !(dd < 1e300)) *ok = false;
  const double2 m = hd_c(-1.0, 0.0);
  return Blk2{hd_cdiv(X.d, det), hd_cdiv(hd_cmul(m, X.b), det), hd_cdiv(hd_cmul(m, X.c), det), hd_cdiv(X.a, det)};
}

#define SHARD_RMAX 64

// Returns xe_{rank−1} (left, 0 for rank 0) and xs_{rank+1} (right, 0 for the last rank).
SHD bool shard_reduced_neighbours(int k, int K, int R, int rank, const double2* red, const double* ab,
                                  const double2* ends_all, double2* left, double2* right) {
  Blk2 Dinv[SHARD_RMAX];
  double2 Ys[SHARD_RMAX], Ye[SHARD_RMAX];
  bool ok = true;
  const double2 z = hd_c(0.0, 0.0), one = hd_c(1.0, 0.0);
  auto P = [&](int r) {
    const double2* c = red + ((size_t)k * R + r) * 4;
    return Blk2{z, hd_cscale(c[0], ab[2 * r]), z, hd_cscale(c[1], ab[2 * r])};
  };
  auto Q = [&](int r) {
    const double2* c = red + ((size_t)k * R + r) * 4;
    return Blk2{hd_cscale(c[2], ab[2 * r + 1]), z, hd_cscale(c[3], ab[2 * r + 1]), z};
  };
  for (int r = 0; r < R; ++r) {
    const double2 gs = ends_all[((size_t)r * K + k) * 2], ge = ends_all[((size_t)r * K + k) * 2 + 1];
    if (r == 0) {
      Dinv[0] = Blk2{one, z, z, one};
      Ys[0] = gs;
      Ye[0] = ge;
      continue;
    }
    const Blk2 Mr = blk_mul(P(r), Dinv[r - 1]);
    const Blk2 MQ = blk_mul(Mr, Q(r - 1));
    const Blk2 D = Blk2{hd_csub(one, MQ.a), hd_csub(z, MQ.b), hd_csub(z, MQ.c), hd_csub(one, MQ.d)};
    Dinv[r] = blk_inv(D, &ok);
    double2 ms, me;
    blk_apply(Mr, Ys[r - 1], Ye[r - 1], &ms, &me);
    Ys[r] = hd_cadd(gs, ms);
    Ye[r] = hd_cadd(ge, me);
  }
  // back substitution from the last rank down to rank − 1
  double2 xs_next = z, xe_next = z;  // X_{r+1}
  *left = z;
  *right = z;
  const int lo = rank > 0 ? rank - 1 : 0;
  for (int r = R - 1; r >= lo; --r) {
    double2 ts = Ys[r], te = Ye[r];
    if (r < R - 1) {
      double2 qs, qe;
      blk_apply(Q(r), xs_next, xe_next, &qs, &qe);
      ts = hd_cadd(ts, qs);
      te = hd_cadd(te, qe);
    }
    double2 xs, xe;
    blk_apply(Dinv[r], ts, te, &xs, &xe);
    if (r == rank + 1) *right = xs;
    if (r == rank - 1) *left = xe;
    xs_next = xs;
    xe_next = xe;
  }
  return ok;
}
