// GMRES kernels (K7 Arnoldi CGS2, K8 Hessenberg/Givens on device, K9 cycle end helpers).
//
// Right-preconditioned restarted GMRES (textbook algorithm, Saad Alg. 9.5).  The
// Krylov basis is stored UNNORMALISED: v_i = s_i Ṽ_i with s_i on device, so no separate
// normalisation pass is needed (the consumer of Ṽ_{j+1} — K2's Γ-scaling, or the dot/update
// kernels — folds s_i in).  Classical Gram–Schmidt with one reorthogonalisation (CGS2):
//   pass 1  c1 = Ṽᵀw                          (k_dots)
//   pass 2  w ← w − Σ c1_i s_i² Ṽ_i ; c2 = Ṽᵀw  (k_update, fused dots)
//   pass 3  w ← w − Σ c2_i s_i² Ṽ_i ; ‖w‖²      (k_update, fused norm) → stored as Ṽ_{j+1}
// Every reduction is two-stage and deterministic: a fixed grid writes per-block partial sums,
// one block per output sums them in a fixed order (bitwise reproducible runs, no atomics).
#include "common.cuh"
#include "internal.h"
#include "post_op.cuh"

struct VPtrs {
  const double* p[CNP_MAX_DOT];
};

// per-block reduction of NV accumulators; writes part[blockIdx.x * stride + i]
template <int NV>
CNP_DEV void block_reduce_write(double (&acc)[NV], double* part, int stride) {
  __shared__ double red[CNP_RED_THREADS / 32][NV > 0 ? NV : 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double v = warp_sum(acc[i]);
    if (lane == 0) red[w][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int k = 0; k < CNP_RED_THREADS / 32; ++k) s += red[k][threadIdx.x];
    part[(size_t)blockIdx.x * stride + threadIdx.x] = s;
  }
}

// partial dots: part[b][i] = Σ Ṽ_i·w over block b's elements (grid-stride over double2)
template <int NV>
__global__ void __launch_bounds__(CNP_RED_THREADS) k_dots(VPtrs V, const double* __restrict__ w, size_t n2,
                                                           double* __restrict__ part, int stride,
                                                           double* __restrict__ out, unsigned* counter) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n2; e += (size_t)gridDim.x * blockDim.x) {
    const double2 x = w2[e];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 v = ldg_cs2(reinterpret_cast<const double2*>(V.p[i]) + e);
      acc[i] = fma(v.x, x.x, fma(v.y, x.y, acc[i]));
    }
  }
  block_reduce_write<NV>(acc, part, stride);
  if (out) grid_fold(part, gridDim.x, stride, NV, out, counter);
}

// Σ w² (one read of w), folded into out
__global__ void __launch_bounds__(CNP_RED_THREADS) k_norm2(const double* __restrict__ w, size_t n2,
                                                            double* __restrict__ part, int stride,
                                                            double* __restrict__ out, unsigned* counter,
                                                            PostOp post) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  double acc[1] = {0.0};
  const double2* w2 = reinterpret_cast<const double2*>(w);
  // four independent loads in flight per thread (a one-load grid-stride loop leaves the HBM idle
  // between a load and its use); fixed per-thread summation order, so still deterministic
  const size_t stride_e = (size_t)gridDim.x * blockDim.x;
  size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  double a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (; e + 3 * stride_e < n2; e += 4 * stride_e) {
    const double2 x0 = ldg_cs2(w2 + e), x1 = ldg_cs2(w2 + e + stride_e);
    const double2 x2 = ldg_cs2(w2 + e + 2 * stride_e), x3 = ldg_cs2(w2 + e + 3 * stride_e);
    acc[0] = fma(x0.x, x0.x, fma(x0.y, x0.y, acc[0]));
    a1 = fma(x1.x, x1.x, fma(x1.y, x1.y, a1));
    a2 = fma(x2.x, x2.x, fma(x2.y, x2.y, a2));
    a3 = fma(x3.x, x3.x, fma(x3.y, x3.y, a3));
  }
  for (; e < n2; e += stride_e) {
    const double2 x = ldg_cs2(w2 + e);
    acc[0] = fma(x.x, x.x, fma(x.y, x.y, acc[0]));
  }
  acc[0] += (a1 + a2) + a3;
  block_reduce_write<1>(acc, part, stride);
  if (grid_fold(part, gridDim.x, stride, 1, out, counter)) run_post(post);
}

// w_out = w − Σ_i coef_i Ṽ_i with coef_i = (cd[i] + cd2[i])·s_i² (MODE 0; cd2 may be null) or
// coef_i = cd[i] (MODE 1, combine, w may be null), optionally fused partial dots with Ṽ (DOTS) or
// Σ w_out² (NORM).  NOWRITE: w_out is only formed in registers (its dots are the product), nothing
// is stored — CGS2's second projection c2 = Ṽᵀ(w − Ṽ s²c1) without writing the intermediate.
#ifndef UPD_REVERSE
#define UPD_REVERSE 1
#endif
// GDOTS (with NORM): also Ṽᵢᵀ w_out — the Gram row of the new basis vector for Gram CGS2; the fold
// writes out[0] = Σ w_out², out[1 + i] = Ṽᵢᵀ w_out.
template <int NV, int MODE, bool DOTS, bool NORM, bool NOWRITE = false, bool GDOTS = false>
__global__ void __launch_bounds__(CNP_RED_THREADS) k_update(VPtrs V, const double* __restrict__ cd,
                                                             const double* __restrict__ scl, const double* w,
                                                             double* wout, size_t n2, double* __restrict__ part,
                                                             int stride, double* __restrict__ out, unsigned* counter,
                                                             const double* __restrict__ cd2 = nullptr,
                                                             PostOp post = PostOp{}) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  double coef[NV];
  if constexpr (GDOTS) {
    // Gram CGS2: the second projection from the stored Gram matrix, c2 = c1 − G̃ S² c1 (every block
    // forms the same NV² products; post_op.cuh gram_c2_dev), coefficient (c1 + c2) s²
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double c2 = cd[i];
#pragma unroll
      for (int k = 0; k < NV; ++k) c2 -= post.G[(size_t)i * post.ldh + k] * (scl[k] * scl[k] * cd[k]);
      coef[i] = (cd[i] + c2) * scl[i] * scl[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i) coef[i] = MODE == 0 ? (cd[i] + (cd2 ? cd2[i] : 0.0)) * scl[i] * scl[i] : cd[i];
  }
  constexpr int NA = DOTS ? NV : GDOTS ? NV + 1 : 1;
  double acc[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) acc[i] = 0.0;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* o2 = reinterpret_cast<double2*>(wout);
  // GDOTS (Gram update, always right after the matvec that wrote w front to back): walk the vectors
  // back to front, so the tail of w the matvec left in the 126-MB L2 is read before this kernel's own
  // traffic evicts it (a front-to-back reader evicts each line just before it needs it)
  for (size_t e0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e0 < n2; e0 += (size_t)gridDim.x * blockDim.x) {
    const size_t e = (GDOTS && UPD_REVERSE) ? n2 - 1 - e0 : e0;
    double2 x = w2 ? w2[e] : make_double2(0.0, 0.0);
    double2 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      v[i] = DOTS ? reinterpret_cast<const double2*>(V.p[i])[e] : ldg_cs2(reinterpret_cast<const double2*>(V.p[i]) + e);
      if (MODE == 0) { x.x = fma(-coef[i], v[i].x, x.x); x.y = fma(-coef[i], v[i].y, x.y); }
      else { x.x = fma(coef[i], v[i].x, x.x); x.y = fma(coef[i], v[i].y, x.y); }
    }
    if (!NOWRITE) o2[e] = x;
    if constexpr (DOTS) {
#pragma unroll
      for (int i = 0; i < NV; ++i) acc[i] = fma(v[i].x, x.x, fma(v[i].y, x.y, acc[i]));
    }
    if constexpr (NORM) acc[0] = fma(x.x, x.x, fma(x.y, x.y, acc[0]));
    if constexpr (GDOTS) {
#pragma unroll
      for (int i = 0; i < NV; ++i) acc[1 + i] = fma(v[i].x, x.x, fma(v[i].y, x.y, acc[1 + i]));
    }
  }
  if constexpr (DOTS) {
    block_reduce_write<NV>(acc, part, stride);
    if (out) grid_fold(part, gridDim.x, stride, NV, out, counter);
  } else if constexpr (NORM) {
    block_reduce_write<NA>(acc, part, stride);
    if (out && grid_fold(part, gridDim.x, stride, NA, out, counter)) run_post(post);
  }
}

// out[i] (+)= Σ_b part[b*stride + i], one block per column, fixed order
__global__ void __launch_bounds__(256) k_reduce(const double* __restrict__ part, int nparts, int stride,
                                                double* __restrict__ out) {
  __shared__ double red[256];
  const int i = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nparts; b += 256) s += part[(size_t)b * stride + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = red[0];
}

// ---------------------------------------------------------------- tiny single-thread kernels
// scal[0] = ||b||, scal[1] = estimate, scal[2] = ||w||² (reduced), scal[3] = non-finite flag,
// scal[4] = true residual ||r||/||b||
__global__ void k_cycle_start(double* scl, double* g, double* scal, int first, int rmax) {
  if (threadIdx.x == 0) cycle_start_dev(scl, g, scal, first, rmax);
}

__global__ void k_arnoldi_finalize(int j, int ldh, const double* c1, const double* c2, double* scl, double* H,
                                   double* cs, double* sn, double* g, double* scal) {
  if (threadIdx.x == 0) arnoldi_finalize_dev(j, ldh, c1, c2, scl, H, cs, sn, g, scal);
}

// y = H[0:k,0:k]^{-1} g[0:k]; coef_i = y_i s_i  (combination Σ coef_i Ṽ_i = V y)
__global__ void k_backsolve(int k, int ldh, const double* H, const double* g, const double* scl, double* y,
                            double* coef) {
  if (threadIdx.x != 0) return;
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int l = i + 1; l < k; ++l) s -= H[i + (size_t)l * ldh] * y[l];
    y[i] = s / H[i + (size_t)i * ldh];
  }
  for (int i = 0; i < k; ++i) coef[i] = y[i] * scl[i];
}

// ---------------------------------------------------------------- launchers
static size_t n2_of(const cnpint_ctx* c) { return (size_t)c->vec / 2; }

template <int NV>
static void dots_nv(cnpint_ctx* c, const VPtrs& V, const double* w, double* part, double* out) {
  cnp_launch(c, k_dots<NV>, dim3(CNP_RED_BLOCKS), dim3(CNP_RED_THREADS), 0, V, w, n2_of(c), part, CNP_MAX_DOT + 1,
             out, c->d_counter);
}

cudaError_t launch_dots(cnpint_ctx* c, double* const* Vp, int nv, const double* w, double* part, double* out) {
  VPtrs V;
  for (int i = 0; i < CNP_MAX_DOT; ++i) V.p[i] = i < nv ? Vp[i] : nullptr;
  cnp_prof_begin(c, KID_DOTS);
  switch (nv) {
    case 1: dots_nv<1>(c, V, w, part, out); break;
    case 2: dots_nv<2>(c, V, w, part, out); break;
    case 3: dots_nv<3>(c, V, w, part, out); break;
    case 4: dots_nv<4>(c, V, w, part, out); break;
    case 5: dots_nv<5>(c, V, w, part, out); break;
    case 6: dots_nv<6>(c, V, w, part, out); break;
    case 7: dots_nv<7>(c, V, w, part, out); break;
    case 8: dots_nv<8>(c, V, w, part, out); break;
    default: return cudaErrorInvalidValue;
  }
  cnp_prof_end(c, KID_DOTS, 8.0 * cnp_units(c) * (nv + 1));
  return cudaGetLastError();
}

cudaError_t launch_norm2(cnpint_ctx* c, const double* w, double* part, double* out) {
  cnp_prof_begin(c, KID_DOTS);
  const PostOp post = c->post;
  c->post = PostOp{};
  cnp_launch(c, k_norm2, dim3(CNP_RED_BLOCKS), dim3(CNP_RED_THREADS), 0, w, n2_of(c), part, CNP_MAX_DOT + 1, out,
             c->d_counter, post);
  cnp_prof_end(c, KID_DOTS, 8.0 * cnp_units(c));
  return cudaGetLastError();
}

cudaError_t launch_reduce_n(cnpint_ctx* c, const double* part, int nparts, int stride, int ncols, double* out) {
  cnp_prof_begin(c, KID_REDUCE);
  k_reduce<<<ncols, 256, 0, c->stream>>>(part, nparts, stride, out);
  cnp_prof_end(c, KID_REDUCE, 0.0);
  return cudaGetLastError();
}

cudaError_t launch_reduce(cnpint_ctx* c, const double* part, int ncols, double* out, int /*unused*/) {
  return launch_reduce_n(c, part, CNP_RED_BLOCKS, CNP_MAX_DOT + 1, ncols, out);
}

template <int NV, int MODE, bool DOTS, bool NORM>
static void upd(cnpint_ctx* c, const VPtrs& V, const double* cd, const double* w, double* wout, double* part,
                double* out) {
  cnp_launch(c, k_update<NV, MODE, DOTS, NORM>, dim3(CNP_RED_BLOCKS), dim3(CNP_RED_THREADS), 0, V, cd,
             (const double*)c->d_scl, w, wout, n2_of(c), part, CNP_MAX_DOT + 1, out, c->d_counter,
             (const double*)nullptr, PostOp{});
}

// Cycle end with the Hessenberg back-substitution folded in: every block solves y = H[0:NV,0:NV]⁻¹g
// (NV ≤ CNP_MAX_DOT, a few hundred flops, H from L2) into shared memory, then u ← u + Σ coef_i X_i
// with coef_i = y_i (right preconditioning, X = Z) or y_i s_i (left, X = Ṽ).  Replaces k_backsolve
// + k_update<MODE 1>.  u_in may be null (fresh u).
template <int NV>
__global__ void __launch_bounds__(CNP_RED_THREADS) k_combine_bs(VPtrs X, const double* __restrict__ H, int ldh,
                                                                 const double* __restrict__ g,
                                                                 const double* __restrict__ scl, int scaled,
                                                                 const double* u_in, double* u_out, size_t n2) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  __shared__ double cs_[NV];
  if (threadIdx.x == 0) {
    double y[NV];
#pragma unroll
    for (int i = NV - 1; i >= 0; --i) {
      double s = g[i];
#pragma unroll
      for (int l = i + 1; l < NV; ++l) s -= H[i + (size_t)l * ldh] * y[l];
      y[i] = s / H[i + (size_t)i * ldh];
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) cs_[i] = scaled ? y[i] * scl[i] : y[i];
  }
  __syncthreads();
  double coef[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) coef[i] = cs_[i];
  const double2* w2 = reinterpret_cast<const double2*>(u_in);
  double2* o2 = reinterpret_cast<double2*>(u_out);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n2; e += (size_t)gridDim.x * blockDim.x) {
    double2 x = w2 ? w2[e] : make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 v = ldg_cs2(reinterpret_cast<const double2*>(X.p[i]) + e);
      x.x = fma(coef[i], v.x, x.x);
      x.y = fma(coef[i], v.y, x.y);
    }
    o2[e] = x;
  }
}

cudaError_t launch_combine_backsolve(cnpint_ctx* c, double* const* Xp, int nv, int scaled, const double* u_in,
                                     double* u_out) {
  VPtrs X;
  for (int i = 0; i < CNP_MAX_DOT; ++i) X.p[i] = i < nv ? Xp[i] : nullptr;
  const int ldh = c->restart_max + 1;
  cnp_prof_begin(c, KID_UPDATE);
#define CB_CASE(K) \
  case K: cnp_launch(c, k_combine_bs<K>, dim3(CNP_RED_BLOCKS), dim3(CNP_RED_THREADS), 0, X, (const double*)c->d_H, ldh, (const double*)c->d_g, (const double*)c->d_scl, scaled, u_in, u_out, n2_of(c)); break;
  switch (nv) {
    CB_CASE(1) CB_CASE(2) CB_CASE(3) CB_CASE(4) CB_CASE(5) CB_CASE(6) CB_CASE(7) CB_CASE(8)
    default: return cudaErrorInvalidValue;
  }
#undef CB_CASE
  cnp_prof_end(c, KID_UPDATE, 8.0 * cnp_units(c) * (nv + (u_in ? 2 : 1)));
  return cudaGetLastError();
}

template <int NV>
static void upd_cgs(cnpint_ctx* c, const VPtrs& V, const double* c1, const double* c2, double* w, double* part,
                    double* out, int phase) {
  if (phase == 0)  // c2 = Ṽᵀ(w − Ṽ s² c1), nothing written
    cnp_launch(c, k_update<NV, 0, true, false, true>, dim3(CNP_RED_BLOCKS), dim3(CNP_RED_THREADS), 0, V, c1,
               (const double*)c->d_scl, (const double*)w, w, n2_of(c), part, CNP_MAX_DOT + 1, out, c->d_counter,
               (const double*)nullptr, PostOp{});
  else if (phase == 1) {  // w ← w − Ṽ s² (c1 + c2), ‖w‖², then the pending post-fold step (Arnoldi finalize)
    const PostOp post = c->post;
    c->post = PostOp{};
    cnp_launch(c, k_update<NV, 0, false, true, false>, dim3(CNP_RED_BLOCKS), dim3(CNP_RED_THREADS), 0, V, c1,
               (const double*)c->d_scl, (const double*)w, w, n2_of(c), part, CNP_MAX_DOT + 1, out, c->d_counter,
               c2, post);
  } else {  // phase 2 (Gram CGS2): as phase 1, plus the Gram row Ṽᵢᵀ w of the new vector; out = [‖w‖², Ṽᵀw]
    const PostOp post = c->post;
    c->post = PostOp{};
    cnp_launch(c, k_update<NV, 0, false, true, false, true>, dim3(CNP_RED_BLOCKS), dim3(CNP_RED_THREADS), 0, V, c1,
               (const double*)c->d_scl, (const double*)w, w, n2_of(c), part, CNP_MAX_DOT + 1, out, c->d_counter,
               c2, post);
  }
}

// CGS2 with one write: phase 0 forms c2 = Ṽᵀ(w − Ṽ s²c1) (reads Ṽ and w, writes nothing), phase 1
// applies both projections at once, w ← w − Ṽ s²(c1 + c2), with ‖w‖² fused.
cudaError_t launch_cgs2_pass(cnpint_ctx* c, double* const* Vp, int nv, const double* c1, const double* c2,
                             double* w, double* part, double* out, int phase) {
  VPtrs V;
  for (int i = 0; i < CNP_MAX_DOT; ++i) V.p[i] = i < nv ? Vp[i] : nullptr;
  cnp_prof_begin(c, KID_UPDATE);
  switch (nv) {
    case 1: upd_cgs<1>(c, V, c1, c2, w, part, out, phase); break;
    case 2: upd_cgs<2>(c, V, c1, c2, w, part, out, phase); break;
    case 3: upd_cgs<3>(c, V, c1, c2, w, part, out, phase); break;
    case 4: upd_cgs<4>(c, V, c1, c2, w, part, out, phase); break;
    case 5: upd_cgs<5>(c, V, c1, c2, w, part, out, phase); break;
    case 6: upd_cgs<6>(c, V, c1, c2, w, part, out, phase); break;
    case 7: upd_cgs<7>(c, V, c1, c2, w, part, out, phase); break;
    case 8: upd_cgs<8>(c, V, c1, c2, w, part, out, phase); break;
    default: return cudaErrorInvalidValue;
  }
  cnp_prof_end(c, KID_UPDATE, 8.0 * cnp_units(c) * (nv + (phase == 0 ? 1 : 2)));  // phase 2: same bytes as 1
  return cudaGetLastError();
}

template <int NV>
static void upd_sel(cnpint_ctx* c, const VPtrs& V, const double* cd, int mode, const double* w, double* wout,
                    int dots, int norm, double* part, double* out) {
  if (mode == 1) upd<NV, 1, false, false>(c, V, cd, w, wout, part, nullptr);
  else if (dots) upd<NV, 0, true, false>(c, V, cd, w, wout, part, out);
  else if (norm) upd<NV, 0, false, true>(c, V, cd, w, wout, part, out);
  else upd<NV, 0, false, false>(c, V, cd, w, wout, part, nullptr);
}

// coefmode 0: w_out = w − Σ cd_i s_i² Ṽ_i.  coefmode 1: w_out = w + Σ cd_i Ṽ_i (w may be null).
cudaError_t launch_update(cnpint_ctx* c, double* const* Vp, int nv, const double* cd, int coefmode, double* w,
                          double* wout, int want_dots, int want_norm, double* part, double* out) {
  VPtrs V;
  for (int i = 0; i < CNP_MAX_DOT; ++i) V.p[i] = i < nv ? Vp[i] : nullptr;
  cnp_prof_begin(c, KID_UPDATE);
  switch (nv) {
    case 1: upd_sel<1>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    case 2: upd_sel<2>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    case 3: upd_sel<3>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    case 4: upd_sel<4>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    case 5: upd_sel<5>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    case 6: upd_sel<6>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    case 7: upd_sel<7>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    case 8: upd_sel<8>(c, V, cd, coefmode, w, wout, want_dots, want_norm, part, out); break;
    default: return cudaErrorInvalidValue;
  }
  cnp_prof_end(c, KID_UPDATE, 8.0 * cnp_units(c) * (nv + (w ? 2 : 1)));
  return cudaGetLastError();
}

// GMRES scalars d_scal[0..7] and the status word → the handle's mapped pinned host buffer, written by
// the SM over PCIe instead of a copy-engine transfer: with several handles solving at once (bench.py
// e2e), an 8-byte cudaMemcpyAsync waits behind the other handles' 134-MB vector copies on the shared
// copy engine (measured: 2.4 ms per wait at c2), this write does not.
__global__ void k_to_host(const double* __restrict__ scal, const int* __restrict__ status, volatile double* h) {
  pdl_enter();  // PDL: wait for the previous kernel on the stream before any global access
  const int i = threadIdx.x;
  if (i < 8) h[i] = scal[i];
  if (i == 8) h[8] = (double)*status;
}
cudaError_t launch_scal_to_host(cnpint_ctx* c) {
  cnp_launch(c, k_to_host, dim3(1), dim3(32), 0, (const double*)c->d_scal, (const int*)c->d_status, c->d_hmap);
  return cudaGetLastError();
}

// takes back the derived-norm probe's finalize of column j (post op 5): g[j] as it was before
__global__ void k_probe_undo(int j, double* g, double* scal) {
  if (threadIdx.x == 0) {
    g[j] = scal[13];
    g[j + 1] = 0.0;
    scal[6] = 0.0;
  }
}

// op 0: cycle_start(first = arg); op 1: arnoldi_finalize(j); op 2: backsolve(k = j); op 3: undo the probe of column j
cudaError_t launch_small(cnpint_ctx* c, int op, int j, int arg) {
  const int ldh = c->restart_max + 1;
  cnp_prof_begin(c, KID_SMALL);
  if (op == 0) k_cycle_start<<<1, 32, 0, c->stream>>>(c->d_scl, c->d_g, c->d_scal, arg, c->restart_max);
  else if (op == 1)
    k_arnoldi_finalize<<<1, 32, 0, c->stream>>>(j, ldh, c->d_c1, c->d_c2, c->d_scl, c->d_H, c->d_cs, c->d_sn, c->d_g,
                                                c->d_scal);
  else if (op == 3) k_probe_undo<<<1, 32, 0, c->stream>>>(j, c->d_g, c->d_scal);
  else k_backsolve<<<1, 32, 0, c->stream>>>(j, ldh, c->d_H, c->d_g, c->d_scl, c->d_y, c->d_coef);
  cnp_prof_end(c, KID_SMALL, 0.0);
  return cudaGetLastError();
}
