// NEXT #3: the 1D AaO system sharded along x over R ranks (one GPU each).
//
// The paper's parallelism is across the N/2+1 shifted solves of step (b) (Remark
// 3.1; `parfor` at PAPER.md:795).  Across GPUs the cheaper cut for a 1D operator is along x: the time
// transforms of steps (a) and (c) act per column (local), and each frequency's tridiagonal system
//   (λ1_k I − λ2_k Ã) ẑ_k = ŵ_k
// is solved by a two-level partition method.  Rank r owns rows [x0_r, x1_r).  With the scaled system
// B = s_k I − Ã (s_k = λ1_k/λ2_k, rows a_i = −τ lo_i, b_i = s_k − τ di_i, c_i = −τ up_i, as K3) and
// B_r its local diagonal block (Dirichlet-cut: the couplings a_{x0_r}, c_{x1_r−1} removed):
//   z_r = g_r + α_r xe_{r−1} v_r + β_r xs_{r+1} w_r,   g_r = B_r⁻¹ d_r,  v_r = B_r⁻¹ e_1,  w_r = B_r⁻¹ e_m,
//   α_r = τ lo_{x0_r}, β_r = τ up_{x1_r−1}  (0 at the domain ends),  xs_r / xe_r = first / last entry of z_r.
// Evaluated at the chunk ends this gives a block-tridiagonal 2R × 2R system in (xs_r, xe_r) whose only
// data-dependent entries are (g_r)_1, (g_r)_m: each rank all-gathers those 2 complex per frequency
// (the only exchange of a P_α⁻¹), solves the reduced system redundantly (one thread per frequency) and
// re-solves its block with the two corrected end rows, instead of storing the spikes v_r, w_r.  The
// spike ends (v_r)_1, (v_r)_m, (w_r)_1, (w_r)_m depend only on k and the operator: tabulated at create
// (host, long double) for every rank.
//   𝓜u (K1) needs the neighbours' boundary columns (N values per side): all-gathered, then the local
// Dirichlet-cut matvec is corrected in its first / last column.  GMRES all-reduces its dot products.
// Collectives go through a caller-supplied callback (the binding uses torch.distributed / NCCL).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "shard_reduced.cuh"

struct ShardInfo {
  int R, rank, K, m;
  double alpha_c, beta_c;   // this rank's α_r, β_r
  double2* d_red;           // [K][R][4] spike ends (v1, vm, w1, wm) of every rank's scaled block
  double* d_ab;             // [R][2] α_r, β_r
  double2* d_ends;          // [K][2] this rank's (g_1, g_m)  (all-gather send)
  double2* d_ends_all;      // [R][K][2]                     (all-gather receive)
  double2* d_spec2;         // [K][ld] K3 output (the K3 input ŵ stays in d_spec for the second solve)
  double* d_edges;          // [2][N] this rank's first / last column (halo send)
  double* d_halo_all;       // [R][2][N]                          (halo receive)
  cnpint_collective_fn coll;
  void* user;
};

void cnp_shard_free(cnpint_ctx* c) {
  if (c && c->shard) {
    delete c->shard;
    c->shard = nullptr;
  }
}

namespace {

const size_t SALIGN = 256;
size_t salign(size_t v) { return (v + SALIGN - 1) & ~(SALIGN - 1); }

struct ShardLayout {
  size_t red, ab, ends, ends_all, spec2, edges, halo_all, total;
};

ShardLayout shard_layout(int N, int R, int m) {
  const int K = N / 2 + 1;
  const int64_t ld = ((int64_t)m + 3) / 4 * 4;
  ShardLayout L;
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += salign(b ? b : 1); return o; };
  L.red = take((size_t)K * R * 4 * 16);
  L.ab = take((size_t)R * 2 * 8);
  L.ends = take((size_t)K * 2 * 16);
  L.ends_all = take((size_t)R * K * 2 * 16);
  L.spec2 = take((size_t)K * ld * 16);
  L.edges = take((size_t)2 * N * 8);
  L.halo_all = take((size_t)R * 2 * N * 8);
  L.total = off;
  return L;
}

const char* check_shard(int N, const cnpint_operator* op, int R, const int* x0, int rank, double alpha) {
  if (!op || op->dim != 1) return "sharding is for 1D operators";
  if (R < 1 || R > 64 || !x0 || rank < 0 || rank >= R) return "bad rank / world size";
  if (x0[0] != 0 || x0[R] != op->nx) return "x0 must run from 0 to nx";
  for (int r = 0; r < R; ++r)
    if (x0[r + 1] - x0[r] < 2) return "every chunk needs >= 2 rows";
  if (!(alpha > 0.0 && alpha < 1.0)) return "sharded P_alpha needs 0 < alpha < 1";
  if (N < 2 || (N & (N - 1))) return "N must be a power of two";
  return nullptr;
}

// local operator of rank r: rows [x0_r, x1_r) (Toeplitz stays Toeplitz; the Dirichlet cut is implicit)
struct LocalOp {
  cnpint_operator op;
  std::vector<double> sub, diag, sup;
};
LocalOp local_op(const cnpint_operator* g, int a, int b) {
  LocalOp L;
  L.op = *g;
  L.op.nx = b - a;
  L.op.ny = 1;
  if (!g->toeplitz) {
    L.sub.assign(g->sub + a, g->sub + b);
    L.diag.assign(g->diag + a, g->diag + b);
    L.sup.assign(g->sup + a, g->sup + b);
    L.op.sub = L.sub.data();
    L.op.diag = L.diag.data();
    L.op.sup = L.sup.data();
  }
  return L;
}

double row(const cnpint_operator* op, const double* arr, double cst, int i) { return op->toeplitz ? cst : arr[i]; }

// spike ends of every rank's scaled block, long double Thomas (k = 0..N/2)
void spike_ends(int N, double T, double alpha, const cnpint_operator* op, int R, const int* x0,
                std::vector<double2>& red, std::vector<double>& ab) {
  typedef std::complex<long double> cld;
  const int K = N / 2 + 1;
  const long double PI = 3.141592653589793238462643383279502884L;
  const long double tau = (long double)T / N;
  const long double lna = logl((long double)alpha), a = expl(lna / N), one_m_a = -expm1l(lna / N);
  red.assign((size_t)K * R * 4, make_double2(0.0, 0.0));
  ab.assign((size_t)R * 2, 0.0);
  for (int r = 0; r < R; ++r) {
    ab[2 * r] = r > 0 ? (double)(tau * row(op, op->sub, op->xs, x0[r])) : 0.0;
    ab[2 * r + 1] = r < R - 1 ? (double)(tau * row(op, op->sup, op->xu, x0[r + 1] - 1)) : 0.0;
  }
  std::vector<cld> cp, dv, dw;
  for (int k = 0; k < K; ++k) {
    const long double th = 2.0L * PI * k / N;
    long double sh = sinl(0.5L * th), sn = sinl(th), cs = cosl(th);
    if (2 * k == N) { sh = 1.0L; sn = 0.0L; cs = -1.0L; }
    const cld l1(one_m_a + 2.0L * a * sh * sh, a * sn), l2(0.5L * (1.0L + a * cs), -0.5L * a * sn);
    const cld s = l1 / l2;
    for (int r = 0; r < R; ++r) {
      const int i0 = x0[r], m = x0[r + 1] - x0[r];
      cp.assign(m, cld(0)); dv.assign(m, cld(0)); dw.assign(m, cld(0));
      // forward sweep for the two right-hand sides e_1 and e_m at once
      for (int i = 0; i < m; ++i) {
        const long double ai = i ? -tau * row(op, op->sub, op->xs, i0 + i) : 0.0L;
        const long double ci = i < m - 1 ? -tau * row(op, op->sup, op->xu, i0 + i) : 0.0L;
        const cld bi = s - cld(tau * row(op, op->diag, op->xd, i0 + i), 0.0L);
        const cld piv = i ? bi - ai * cp[i - 1] : bi;
        cp[i] = ci / piv;
        const cld ev = i == 0 ? cld(1.0L) : cld(0.0L), ew = i == m - 1 ? cld(1.0L) : cld(0.0L);
        dv[i] = (ev - (i ? ai * dv[i - 1] : cld(0.0L))) / piv;
        dw[i] = (ew - (i ? ai * dw[i - 1] : cld(0.0L))) / piv;
      }
      for (int i = m - 2; i >= 0; --i) {
        dv[i] -= cp[i] * dv[i + 1];
        dw[i] -= cp[i] * dw[i + 1];
      }
      double2* o = red.data() + ((size_t)k * R + r) * 4;
      auto d2 = [](cld z) { return make_double2((double)z.real(), (double)z.imag()); };
      o[0] = d2(dv[0]); o[1] = d2(dv[m - 1]); o[2] = d2(dw[0]); o[3] = d2(dw[m - 1]);
    }
  }
}

// ---------------------------------------------------------------------------------- kernels
__global__ void k_shard_ends(const double2* __restrict__ spec, double2* __restrict__ ends, int K, int m, int64_t ld) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  ends[2 * k] = spec[(int64_t)k * ld];
  ends[2 * k + 1] = spec[(int64_t)k * ld + m - 1];
}

// per frequency: the reduced block-tridiagonal solve, then the end rows of this rank's ŵ corrected by
// λ2_k (α xe_{r−1} e_1 + β xs_{r+1} e_m) for the second local solve
__global__ void k_shard_reduced(int K, int R, int rank, const double2* __restrict__ red, const double* __restrict__ ab,
                                const double2* __restrict__ ends_all, const double2* __restrict__ lam2,
                                double2* __restrict__ spec, int m, int64_t ld, int* __restrict__ status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double2 left, right;
  const bool ok = shard_reduced_neighbours(k, K, R, rank, red, ab, ends_all, &left, &right);
  const double2 l2 = lam2[k];
  const double al = ab[2 * rank], be = ab[2 * rank + 1];
  double2* row = spec + (int64_t)k * ld;
  if (rank > 0) row[0] = hd_cadd(row[0], hd_cscale(hd_cmul(l2, left), al));
  if (rank < R - 1) row[m - 1] = hd_cadd(row[m - 1], hd_cscale(hd_cmul(l2, right), be));
  if (!ok) atomicOr(status, 1);
}

__global__ void k_shard_edges(const double* __restrict__ u, double* __restrict__ edges, int N, int m, int64_t ld) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  edges[t] = u[(int64_t)t * ld];
  edges[N + t] = u[(int64_t)t * ld + m - 1];
}

// y_t (local Dirichlet-cut 𝓜u) += the neighbour couplings: −½α(hl_t + hl_{t−1}) in column 0,
// −½β(hr_t + hr_{t−1}) in column m−1 (Q1 u_t − Q2 u_{t−1} with L_h's off-block entries); sign = −1 for
// the residual b − 𝓜u
__global__ void k_shard_fix(double* __restrict__ y, const double* __restrict__ halo_all, int N, int m, int64_t ld,
                            int R, int rank, double al, double be, double sign) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  if (rank > 0) {
    const double* hl = halo_all + (size_t)(rank - 1) * 2 * N + N;  // left neighbour's last column
    const double s = hl[t] + (t ? hl[t - 1] : 0.0);
    y[(int64_t)t * ld] -= sign * 0.5 * al * s;
  }
  if (rank < R - 1) {
    const double* hr = halo_all + (size_t)(rank + 1) * 2 * N;      // right neighbour's first column
    const double s = hr[t] + (t ? hr[t - 1] : 0.0);
    y[(int64_t)t * ld + m - 1] -= sign * 0.5 * be * s;
  }
}

cnpint_status sfail(cnpint_ctx* c, cudaError_t e, const char* where) {
  snprintf(c->err, sizeof(c->err), "CUDA error in %s: %s", where, cudaGetErrorString(e));
  return CNPINT_ECUDA;
}
#define SCK(expr)                                          \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return sfail(c, _e, #expr);     \
  } while (0)

cnpint_status coll(cnpint_ctx* c, int op, const double* send, double* recv, size_t count) {
  ShardInfo* S = c->shard;
  if (S->R == 1) {  // a world of one: the collective is the identity
    if (op == 0 && send != recv)
      SCK(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    return CNPINT_OK;
  }
  if (!S->coll) {
    snprintf(c->err, sizeof(c->err), "shard: no collective callback (cnpint_shard_set_collective)");
    return CNPINT_EINVAL;
  }
  if (S->coll(S->user, op, send, recv, count, (void*)c->stream) != 0) {
    snprintf(c->err, sizeof(c->err), "shard: collective callback failed (op %d)", op);
    return CNPINT_ECUDA;
  }
  return CNPINT_OK;
}

cnpint_status pinv_begin(cnpint_ctx* c, const double* v, const double* vscale) {
  ShardInfo* S = c->shard;
  SCK(launch_time_fft(c, v, vscale, c->d_spec));
  SCK(launch_shifted_solve(c, c->d_spec, S->d_spec2));
  k_shard_ends<<<(S->K + 127) / 128, 128, 0, c->stream>>>(S->d_spec2, S->d_ends, S->K, S->m, c->ld);
  SCK(cudaGetLastError());
  return CNPINT_OK;
}

cnpint_status pinv_end(cnpint_ctx* c, double* z) {
  ShardInfo* S = c->shard;
  k_shard_reduced<<<(S->K + 127) / 128, 128, 0, c->stream>>>(S->K, S->R, S->rank, S->d_red, S->d_ab, S->d_ends_all,
                                                              c->d_lam2, c->d_spec, S->m, c->ld, c->d_status);
  SCK(cudaGetLastError());
  SCK(launch_shifted_solve(c, c->d_spec, S->d_spec2));
  SCK(launch_time_ifft(c, S->d_spec2, z, 0));
  return CNPINT_OK;
}

cnpint_status pinv(cnpint_ctx* c, const double* v, const double* vscale, double* z) {
  ShardInfo* S = c->shard;
  if (cnpint_status st = pinv_begin(c, v, vscale)) return st;
  if (cnpint_status st = coll(c, 0, (const double*)S->d_ends, (double*)S->d_ends_all, (size_t)S->K * 4)) return st;
  return pinv_end(c, z);
}

cnpint_status halo_begin(cnpint_ctx* c, const double* u) {
  ShardInfo* S = c->shard;
  k_shard_edges<<<(c->N + 127) / 128, 128, 0, c->stream>>>(u, S->d_edges, c->N, S->m, c->ld);
  SCK(cudaGetLastError());
  return CNPINT_OK;
}

// mode 0: y = 𝓜u; mode 2: y = b − 𝓜u
cnpint_status matvec_end(cnpint_ctx* c, const double* u, double* y, int mode, const double* b) {
  ShardInfo* S = c->shard;
  SCK(launch_matvec(c, u, y, mode, b, nullptr));
  k_shard_fix<<<(c->N + 127) / 128, 128, 0, c->stream>>>(y, S->d_halo_all, c->N, S->m, c->ld, S->R, S->rank,
                                                          S->alpha_c, S->beta_c, mode == 2 ? -1.0 : 1.0);
  SCK(cudaGetLastError());
  return CNPINT_OK;
}

cnpint_status matvec(cnpint_ctx* c, const double* u, double* y, int mode, const double* b) {
  ShardInfo* S = c->shard;
  if (cnpint_status st = halo_begin(c, u)) return st;
  if (cnpint_status st = coll(c, 0, S->d_edges, S->d_halo_all, (size_t)2 * c->N)) return st;
  return matvec_end(c, u, y, mode, b);
}

cnpint_status shard_ok(cnpint_ctx* c) {
  if (!c) return CNPINT_EINVAL;
  if (!c->shard) {
    snprintf(c->err, sizeof(c->err), "not a sharded handle (cnpint_shard_create)");
    return CNPINT_EINVAL;
  }
  return CNPINT_OK;
}

}  // namespace

extern "C" {

size_t cnpint_shard_workspace_bytes(int N, const cnpint_operator* op, int R, const int* x0, int rank,
                                    int restart_max) {
  if (check_shard(N, op, R, x0, rank, 0.5)) return 0;
  LocalOp L = local_op(op, x0[rank], x0[rank + 1]);
  const size_t base = cnpint_workspace_bytes(N, &L.op, restart_max);
  if (!base) return 0;
  return salign(base) + shard_layout(N, R, x0[rank + 1] - x0[rank]).total;
}

cnpint_status cnpint_shard_create(cnpint_ctx** out, int N, double T, double alpha, const cnpint_operator* op, int R,
                                  const int* x0, int rank, int restart_max, void* d_workspace, size_t ws_bytes,
                                  void* cuda_stream) {
  if (!out) return CNPINT_EINVAL;
  *out = nullptr;
  if (check_shard(N, op, R, x0, rank, alpha)) return CNPINT_EINVAL;
  const int m = x0[rank + 1] - x0[rank];
  LocalOp L = local_op(op, x0[rank], x0[rank + 1]);
  const size_t base = cnpint_workspace_bytes(N, &L.op, restart_max);
  if (!base) return CNPINT_EUNSUPPORTED;
  const ShardLayout SL = shard_layout(N, R, m);
  if (ws_bytes < salign(base) + SL.total) return CNPINT_EINVAL;
  cnpint_ctx* c = nullptr;
  cnpint_status st = cnpint_create(&c, N, T, alpha, &L.op, restart_max, d_workspace, base, cuda_stream);
  if (st != CNPINT_OK) return st;
  ShardInfo* S = new (std::nothrow) ShardInfo();
  if (!S) { cnpint_destroy(c); return CNPINT_EINVAL; }
  char* w = (char*)d_workspace + salign(base);
  S->R = R; S->rank = rank; S->K = N / 2 + 1; S->m = m;
  S->d_red = (double2*)(w + SL.red); S->d_ab = (double*)(w + SL.ab); S->d_ends = (double2*)(w + SL.ends);
  S->d_ends_all = (double2*)(w + SL.ends_all); S->d_spec2 = (double2*)(w + SL.spec2);
  S->d_edges = (double*)(w + SL.edges); S->d_halo_all = (double*)(w + SL.halo_all);
  std::vector<double2> red;
  std::vector<double> ab;
  spike_ends(N, T, alpha, op, R, x0, red, ab);
  S->alpha_c = ab[2 * rank];
  S->beta_c = ab[2 * rank + 1];
  c->shard = S;
  cudaError_t e = cudaMemcpyAsync(S->d_red, red.data(), red.size() * 16, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(S->d_ab, ab.data(), ab.size() * 8, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(w + SL.ends, 0, SL.total - SL.ends, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    cnpint_destroy(c);
    return CNPINT_ECUDA;
  }
  *out = c;
  return CNPINT_OK;
}

cnpint_status cnpint_shard_set_collective(cnpint_ctx* c, cnpint_collective_fn fn, void* user) {
  if (cnpint_status st = shard_ok(c)) return st;
  c->shard->coll = fn;
  c->shard->user = user;
  return CNPINT_OK;
}

cnpint_status cnpint_shard_buffers(cnpint_ctx* c, double** ends_send, double** ends_recv, size_t* ends_count,
                                   double** halo_send, double** halo_recv, size_t* halo_count) {
  if (cnpint_status st = shard_ok(c)) return st;
  ShardInfo* S = c->shard;
  if (ends_send) *ends_send = (double*)S->d_ends;
  if (ends_recv) *ends_recv = (double*)S->d_ends_all;
  if (ends_count) *ends_count = (size_t)S->K * 4;
  if (halo_send) *halo_send = S->d_edges;
  if (halo_recv) *halo_recv = S->d_halo_all;
  if (halo_count) *halo_count = (size_t)2 * c->N;
  return CNPINT_OK;
}

cnpint_status cnpint_shard_pinv_begin(cnpint_ctx* c, const double* d_v) {
  if (cnpint_status st = shard_ok(c)) return st;
  if (!d_v) return CNPINT_EINVAL;
  return pinv_begin(c, d_v, nullptr);
}
cnpint_status cnpint_shard_pinv_end(cnpint_ctx* c, double* d_z) {
  if (cnpint_status st = shard_ok(c)) return st;
  if (!d_z) return CNPINT_EINVAL;
  return pinv_end(c, d_z);
}
cnpint_status cnpint_shard_halo_begin(cnpint_ctx* c, const double* d_u) {
  if (cnpint_status st = shard_ok(c)) return st;
  if (!d_u) return CNPINT_EINVAL;
  return halo_begin(c, d_u);
}
cnpint_status cnpint_shard_apply_A_end(cnpint_ctx* c, const double* d_u, double* d_y) {
  if (cnpint_status st = shard_ok(c)) return st;
  if (!d_u || !d_y || d_u == d_y) return CNPINT_EINVAL;
  return matvec_end(c, d_u, d_y, 0, nullptr);
}
cnpint_status cnpint_shard_apply_Pinv(cnpint_ctx* c, const double* d_v, double* d_z) {
  if (cnpint_status st = shard_ok(c)) return st;
  if (!d_v || !d_z || d_v == d_z) return CNPINT_EINVAL;
  return pinv(c, d_v, nullptr, d_z);
}
cnpint_status cnpint_shard_apply_A(cnpint_ctx* c, const double* d_u, double* d_y) {
  if (cnpint_status st = shard_ok(c)) return st;
  if (!d_u || !d_y || d_u == d_y) return CNPINT_EINVAL;
  return matvec(c, d_u, d_y, 0, nullptr);
}

// Right-preconditioned restarted GMRES on the sharded system: the algorithm of cnpint_gmres with
// classic CGS2 (two reading passes, grouped by CNP_MAX_DOT vectors) whose dot products and norms are
// all-reduced across the ranks before the (replicated) Hessenberg / Givens step; every rank returns
// the same report.
cnpint_status cnpint_shard_gmres(cnpint_ctx* c, const double* d_b, double* d_u, double tol, int restart, int maxit,
                                 cnpint_gmres_report* rep) {
  if (cnpint_status st = shard_ok(c)) return st;
  if (!d_b || !d_u || d_b == d_u || c->restart_max < 1 || !(tol > 0.0 && tol < 1.0) || restart < 1 ||
      restart > c->restart_max || maxit < 1)
    return CNPINT_EINVAL;
  auto t0 = std::chrono::steady_clock::now();
  c->post = PostOp{};
  const int64_t vec = c->vec;
  double* h = c->h_pinned;
  std::vector<double*> V(restart + 1), Z(restart);
  for (int i = 0; i <= restart; ++i) V[i] = c->d_V + (size_t)i * vec;
  for (int i = 0; i < restart; ++i) Z[i] = c->d_Z + (size_t)i * vec;
  int its = 0, cycles = 0, converged = 0;
  double est = 1.0, relres = 1.0;
  cnpint_status result = CNPINT_OK;
  auto sync_scal = [&]() -> cnpint_status {
    SCK(launch_scal_to_host(c));
    SCK(cudaStreamSynchronize(c->stream));
    return CNPINT_OK;
  };
  // pass over groups of ≤ CNP_MAX_DOT vectors: dots into cd (then all-reduced), or the update
  auto dots = [&](int nv, double* w, double* cd) -> cnpint_status {
    for (int g0 = 0; g0 < nv; g0 += CNP_MAX_DOT) {
      const int ng = nv - g0 < CNP_MAX_DOT ? nv - g0 : CNP_MAX_DOT;
      SCK(launch_dots(c, V.data() + g0, ng, w, c->d_part, cd + g0));
    }
    return coll(c, 1, cd, cd, (size_t)nv);
  };
  auto update = [&](int nv, double* w, const double* cd, bool norm) -> cnpint_status {
    for (int g0 = 0; g0 < nv; g0 += CNP_MAX_DOT) {
      const int ng = nv - g0 < CNP_MAX_DOT ? nv - g0 : CNP_MAX_DOT;
      const bool last = norm && g0 + ng == nv;
      double* saved = c->d_scl;
      c->d_scl = saved + g0;
      cudaError_t e = launch_update(c, V.data() + g0, ng, cd + g0, 0, w, w, 0, last ? 1 : 0, c->d_part,
                                    last ? c->d_scal + 2 : nullptr);
      c->d_scl = saved;
      SCK(e);
    }
    return norm ? coll(c, 1, c->d_scal + 2, c->d_scal + 2, 1) : CNPINT_OK;
  };
  SCK(cudaMemsetAsync(c->d_scal, 0, 16 * sizeof(double), c->stream));
  SCK(launch_norm2(c, d_b, c->d_part, c->d_scal + 2));
  if (cnpint_status st = coll(c, 1, c->d_scal + 2, c->d_scal + 2, 1)) return st;
  SCK(launch_small(c, 0, 0, 1));  // cycle start: ‖b‖, s_0, g
  if (cnpint_status st = sync_scal()) return st;
  if (h[0] == 0.0) {
    SCK(cudaMemsetAsync(d_u, 0, vec * sizeof(double), c->stream));
    SCK(cudaStreamSynchronize(c->stream));
    if (rep) { rep->iterations = 0; rep->restarts = 0; rep->converged = 1; rep->relres_est = 0; rep->relres_true = 0; }
    return CNPINT_OK;
  }
  if (!std::isfinite(h[0])) { snprintf(c->err, sizeof(c->err), "shard_gmres: ||b|| not finite"); return CNPINT_EBREAKDOWN; }
  V[0] = const_cast<double*>(d_b);
  while (true) {
    int jdone = 0;
    for (int j = 0; j < restart; ++j) {
      if (cnpint_status st = pinv(c, V[j], c->d_scl + j, Z[j])) return st;
      double* w = V[j + 1];
      if (cnpint_status st = matvec(c, Z[j], w, 0, nullptr)) return st;
      const int nv = j + 1;
      if (cnpint_status st = dots(nv, w, c->d_c1)) return st;           // c1 = Ṽᵀw
      if (cnpint_status st = update(nv, w, c->d_c1, false)) return st;  // w −= Ṽ s² c1
      if (cnpint_status st = dots(nv, w, c->d_c2)) return st;           // c2 = Ṽᵀw (reorthogonalisation)
      if (cnpint_status st = update(nv, w, c->d_c2, true)) return st;   // w −= Ṽ s² c2, ‖w‖²
      SCK(launch_small(c, 1, j, 0));                                     // H column, Givens, estimate
      if (cnpint_status st = sync_scal()) return st;
      ++its;
      jdone = j + 1;
      est = h[1];
      if (rep && rep->history && its - 1 < rep->history_cap) rep->history[its - 1] = est;
      if (h[8] != 0.0) return cnpint_device_status(c) != CNPINT_OK ? CNPINT_ESINGULAR : CNPINT_ESINGULAR;
      if (h[3] != 0.0) { snprintf(c->err, sizeof(c->err), "shard_gmres: non-finite Arnoldi scalar"); return CNPINT_EBREAKDOWN; }
      if (est <= tol || its >= maxit || h[5] != 0.0) break;
    }
    // cycle end: y = H⁻¹g, u += Σ y_j z_j
    SCK(launch_small(c, 2, jdone, 0));
    for (int g0 = 0; g0 < jdone; g0 += CNP_MAX_DOT) {
      const int ng = jdone - g0 < CNP_MAX_DOT ? jdone - g0 : CNP_MAX_DOT;
      const bool fresh = cycles == 0 && g0 == 0;
      SCK(launch_update(c, Z.data() + g0, ng, c->d_y + g0, 1, fresh ? nullptr : d_u, d_u, 0, 0, c->d_part, nullptr));
    }
    // r = b − 𝓜u into the workspace slot of Ṽ_0, ‖r‖ (all-reduced), next cycle start
    V[0] = c->d_V;
    if (cnpint_status st = matvec(c, d_u, V[0], 2, d_b)) return st;
    SCK(launch_norm2(c, V[0], c->d_part, c->d_scal + 2));
    if (cnpint_status st = coll(c, 1, c->d_scal + 2, c->d_scal + 2, 1)) return st;
    SCK(launch_small(c, 0, 0, 0));
    if (cnpint_status st = sync_scal()) return st;
    relres = h[4];
    ++cycles;
    if (relres <= tol) { converged = 1; break; }
    if (its >= maxit) { result = CNPINT_ENOCONV; break; }
    if (!std::isfinite(relres)) { result = CNPINT_EBREAKDOWN; break; }
  }
  cnpint_status dst = cnpint_device_status(c);
  if (rep) {
    rep->iterations = its; rep->restarts = cycles - 1; rep->converged = converged; rep->relres_est = est;
    rep->relres_true = relres;
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  if (dst != CNPINT_OK) return dst;
  return result;
}

// Host entry points of the partition arithmetic (no GPU needed): the spike-end table the handles build
// at create, and the reduced solve the device runs per frequency — for host-side tests of the
// partitioning (world-size-2 gloo tests, tests/test_shard_host.py).
cnpint_status cnpint_shard_spike_ends_host(int N, double T, double alpha, const cnpint_operator* op, int R,
                                           const int* x0, double* red_out, double* ab_out) {
  if (check_shard(N, op, R, x0, 0, alpha) || !red_out || !ab_out) return CNPINT_EINVAL;
  std::vector<double2> red;
  std::vector<double> ab;
  spike_ends(N, T, alpha, op, R, x0, red, ab);
  std::memcpy(red_out, red.data(), red.size() * 16);
  std::memcpy(ab_out, ab.data(), ab.size() * 8);
  return CNPINT_OK;
}

cnpint_status cnpint_shard_reduced_host(int K, int R, int rank, const double* red, const double* ab,
                                        const double* ends_all, double* neighbours) {
  if (K < 1 || R < 1 || rank < 0 || rank >= R || !red || !ab || !ends_all || !neighbours) return CNPINT_EINVAL;
  bool ok = true;
  for (int k = 0; k < K; ++k) {
    double2 l, r;
    ok &= shard_reduced_neighbours(k, K, R, rank, (const double2*)red, ab, (const double2*)ends_all, &l, &r);
    neighbours[4 * k] = l.x; neighbours[4 * k + 1] = l.y; neighbours[4 * k + 2] = r.x; neighbours[4 * k + 3] = r.y;
  }
  return ok ? CNPINT_OK : CNPINT_ESINGULAR;
}

}  // extern "C"
