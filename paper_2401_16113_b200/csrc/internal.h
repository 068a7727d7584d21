// Internal (non-ABI) declarations shared by the cnpint host code and kernel launchers.
#pragma once
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/cnpint.h"

#define CNP_NUM_SMS_DEFAULT 148
// Deterministic two-stage reductions use a fixed number of partial-sum blocks.
#define CNP_RED_BLOCKS 1184   // 8 x 148
#define CNP_RED_THREADS 256
#define CNP_MAX_DOT 8         // basis vectors handled per dot/update launch

// kernel classes for the per-class event profiler (cnpint_profile_*)
enum {
  KID_MATVEC = 0, KID_FFT_FWD, KID_TRIDIAG, KID_FFT_INV, KID_TIMEPASS2D, KID_DST_X, KID_DST_Y,
  KID_DOTS, KID_UPDATE, KID_REDUCE, KID_SMALL, KID_DST_XY, KID_UPD_DST, KID_COUNT
};

// K3 launch configuration (k_tridiag.cu): G warps per system, L = max rows per thread chunk,
// Lmin = shortest chunk, tabstride = complex entries per frequency of the Toeplitz chunk table.
struct TriCfg {
  int small, G, logG, L, Lmin, tabstride, NS, padsh, smask, fast, nlv;
  size_t smem;
};
TriCfg tri_cfg(int m, int toeplitz);
// rows allocated per system in shared memory: m rounded up to the swizzle block (and to even)
static inline __host__ __device__ int tri_rows_alloc(int m, int padsh) {
  const int B = (1 << padsh) > 2 ? (1 << padsh) : 2;
  return (m + B - 1) / B * B;
}

// Small GMRES step run by the last block of a reducing kernel right after its deterministic fold
// (saves a single-thread kernel launch): op 1 = Arnoldi finalize of column j (Hessenberg column,
// Givens, estimate; reads the fold's ||w||² from scal[2]), op 2 = cycle start (β = sqrt(scal[2]),
// first: ||b||, scale s_0 = 1/β, g = β e_1).  Set in cnpint_ctx::post by the host before the launch
// of the reducing kernel, which passes it on and clears it.
struct PostOp {
  int op, j, ldh, first, rmax;
  const double* c1;
  const double* c2;
  double* scl;
  double* H;
  double* cs;
  double* sn;
  double* g;
  double* scal;
  // Gram CGS2 (post_op.cuh): op 3 c2 = c1 − G̃S²c1 (into c2w); op 4 stores the Gram row j+1 from the
  // update's fold cg = [‖Ṽ_{j+1}‖², Ṽᵢᵀ Ṽ_{j+1}] and runs op 1; op 2 records G̃_00 when G is set
  const double* cg;
  double* G;
  double* c2w;
  // when set: after the step, scal[0..7] and the status word go to the handle's mapped host buffer
  // (what k_to_host does), so the host's per-step read needs no extra launch
  volatile double* hmap;
  const int* status;
};

struct cnpint_ctx {
  // problem
  int dim, nx, ny, N, H, toeplitz;
  int64_t ld, slice, vec, spec_rows, spec_elems;
  double T, tau, alpha, a, lnalpha;
  double tau_p;        // τ of the preconditioner's Ã: τ·d̄ for 𝓛(t) = d(t)𝓛, else τ
  double* d_dt;        // [N] d(t_{t+½}) of a time-dependent operator (Eq. 5.8), null when constant
  double xs, xd, xu, ys, yd, yu, shift;
  int restart_max;
  cudaStream_t stream;
  int debug;
  int num_sms;
  // workspace carve-up (device pointers)
  char* ws;
  size_t ws_bytes;
  double* d_lo;        // [ld] τ-free 1D rows (zero padded; lo[0] = up[nx-1] = 0)
  double* d_di;
  double* d_up;
  double2* d_tw;       // [N] ω_N^q = e^{-2πiq/N}
  double* d_gam;       // [N] γ_t = α^{t/N}
  double* d_igam;      // [N] 1/(N γ_t)
  double2* d_lam1;     // [H+1] λ1_k
  double2* d_lam2;     // [H+1] λ2_k
  double2* d_sk;       // [H+1] s_k = λ1_k/λ2_k
  double2* d_il2;      // [H+1] 1/λ2_k
  double2* d_tritab;   // [H+1][tabstride] Toeplitz chunk tables of K3 (1D Toeplitz only)
  double2* d_vtab;     // [H+1][trivar_table_stride] K3 variable-row upper-tree tables (built on the device)
  double2* d_spec;     // [(H+1)][ny][ld] half spectrum (1D) ; 2D: unused
  double* d_fsY;       // four-step FFT intermediate (1D N >= 2048, 2D N >= 256; k_fstep.cu), else null
  unsigned* d_fscnt;   // [nxb] per-block pass-A counters, then the work ticket (monotonic)
  unsigned fs_cnt;     // host mirror: Σ pass-A items per block over all launches so far
  unsigned fs_tick;    // host mirror: tickets consumed so far
  unsigned* d_xycnt;   // 2D: [N] per-slice counters + the ticket of the fused sine pass (k_dstxy.cu)
  double* d_tmp1;      // [vec] scratch vectors
  double* d_tmp2;
  double* d_tmp3;
  double* d_io1;       // [vec] host-API staging / 2D scratch
  double* d_io2;
  double* d_io3;
  // 2D fast diagonalisation tables
  double* d_dxi;       // [nx] D_x^{-1} entries   ρ_x^{-i}
  double* d_dx;        // [nx] D_x entries        ρ_x^{i} * 2/(nx+1) (DST normalisation folded)
  double* d_dyi;       // [ny]
  double* d_dy;        // [ny]
  double* d_ex;        // [nx] eigenvalues of L_x
  double* d_ey;        // [ny] eigenvalues of L_y
  double mu_max;       // 2D: max over the spatial modes of μ' = τ_p(e_x + e_y + shift); < 0 ⇒ the time
                       // recurrence of every mode is stable (k_tscan.cu)
  double2* d_twx;      // [nx+1] e^{-2πiq/(2(nx+1))}
  double2* d_twy;      // [ny+1]
  // GMRES
  double* d_V;         // [(restart_max+1)][vec]
  double* d_Z;         // [restart_max][vec] z_j = P_α⁻¹ v_j of the current restart cycle
  double* d_G;         // [(restart_max+1)²] Gram matrix Ṽᵢᵀ Ṽₖ of the cycle's basis (Gram CGS2)
  double* d_cg;        // [CNP_MAX_DOT+1] the Gram-CGS2 update's fold [‖w‖², Ṽᵀw]
  int pdl;              // launch the GMRES-loop kernels with programmatic dependent launch
  int l2pf;             // sine / time passes prefetch their next tile into L2 (CNPINT_L2PF=0: off, A/B)
  double* d_part;      // [CNP_RED_BLOCKS][CNP_MAX_DOT+1]
  double* d_c1;        // [restart_max+1] raw dots (pass 1)
  double* d_c2;        // [restart_max+1] raw dots (pass 2)
  double* d_scl;       // [restart_max+1] basis scales s_i (v_i = s_i Ṽ_i)
  double* d_H;         // [(restart_max+1) * restart_max] column-major Hessenberg (ld = restart_max+1)
  double* d_cs;        // [restart_max]
  double* d_sn;        // [restart_max]
  double* d_g;         // [restart_max+1]
  double* d_y;         // [restart_max]
  double* d_coef;      // [restart_max+1] combination coefficients
  double* d_scal;      // [8] misc scalars: 0 = ||b||, 1 = est, 2 = beta^2, 3 = nonfinite flag
  int* d_status;       // device status word (bit 0: singular pivot)
  unsigned* d_counter; // grid_fold ticket counter (zero between launches)
  double* h_pinned;    // mapped pinned host scalars [16]: d_scal[0..7], status at [8]
  double* d_hmap;      // its device alias
  PostOp post;         // pending post-fold operation for the next reducing launch (op 0 = none)
  struct ShardInfo* shard;  // 1D x-sharded handle (shard.cu, NEXT #3), null for a whole-domain handle
  cudaStream_t s_in, s_out;  // copy streams of cnpint_gmres_host_batch (created on first use)
  cudaEvent_t ev[8];         // its events: in[2], repacked[2], out_ready[2], out_done[2]
  const double* last_v0;  // Ṽ_0 of the last completed GMRES cycle (b itself in the first), test hook
  int last_nv;            // basis vectors Ṽ_0..Ṽ_{last_nv−1} of that cycle
  double* h_stage_in;  // (lazily) pinned host staging not used; host API copies pageable memory
  int64_t launches;
  // 2D right GMRES: the vector whose x sine pass the last Gram update already wrote into d_tmp1
  // (k_upd_dst4); the next pinv_dev of exactly that vector skips its first pass, any pinv_dev clears it
  const double* xdst_src;
  void* prof;          // CnpProf* (host event pools), null when profiling is off
  char err[512];
};

// ------------------------------------------------------------------ kernel launchers (return cudaError_t)
cudaError_t launch_stream_copy(const double* src, double* dst, size_t n, cudaStream_t s);

struct DotPtrs {
  const double* p[CNP_MAX_DOT];
};
// y = 𝓜u fused with the first CGS pass: out[i] = Ṽ_iᵀ y, i < nv <= CNP_MAX_DOT (deterministic fold)
bool fstep_ok(const cnpint_ctx* c);
size_t fstep_y_bytes(int dim, int N, int64_t W);
int fstep_nxb(int N, int64_t W);
cudaError_t launch_fstep_pass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale);
bool tpass_ok(const cnpint_ctx* c);
cudaError_t launch_tpass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale);
cudaError_t launch_fstep_fwd(cnpint_ctx* c, const double* v, const double* vscale, double2* what);
cudaError_t launch_fstep_inv(cnpint_ctx* c, const double2* zhat, double* z, int accumulate);
cudaError_t launch_matvec_dots(cnpint_ctx* c, const double* u, double* y, double* const* V, int nv, double* part,
                               double* out, int ww = 0);
// host-layout repack for the *_host entry points: dir 0 packed → padded, 1 padded → packed
cudaError_t launch_repack(cnpint_ctx* c, const double* src, double* dst, int dir);

// y = 𝓜u (mode 0), y = P_α u (mode 1), y = b − 𝓜u (mode 2, b given), mode 3 = mode 2 without storing y;
// optional Σ y² partials (folded into out when given)
cudaError_t launch_matvec(cnpint_ctx* c, const double* u, double* y, int mode, const double* b, double* part,
                          double* out = nullptr);

cudaError_t launch_time_fft(cnpint_ctx* c, const double* v, const double* vscale, double2* what);
cudaError_t launch_shifted_solve(cnpint_ctx* c, const double2* what, double2* zhat);
int trivar_table_stride(int m);
cudaError_t build_trivar_table(cnpint_ctx* c);
cudaError_t launch_time_ifft(cnpint_ctx* c, const double2* zhat, double* z, int accumulate);

// N <= 16384: x-pair packed thread-block-cluster variant (k_tfft.cu)
struct TfftCfg {
  int C, logN2, X, CS, T, ok;
  size_t smem;
};
TfftCfg tfft_cfg(int N, int mode = 0);  // mode: 0/1 1D forward/inverse, 2 the 2D time pass
cudaError_t launch_tfft_fwd(cnpint_ctx* c, const double* v, const double* vscale, double2* what);
cudaError_t launch_tfft_inv(cnpint_ctx* c, const double2* zhat, double* z, int accumulate);
cudaError_t launch_tfft_pass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale);

// 2D
cudaError_t launch_dst_x(cnpint_ctx* c, const double* in, double* out, const double* vscale, int inverse);
cudaError_t launch_dst_y(cnpint_ctx* c, const double* in, double* out, int inverse);
cudaError_t launch_time_pass_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale);
bool tscan_ok(const cnpint_ctx* c);  // the recurrence form of the 2D time pass applies (k_tscan.cu)
cudaError_t launch_tscan_2d(cnpint_ctx* c, const double* in, double* out, const double* vscale);

// GMRES helpers
cudaError_t launch_norm2(cnpint_ctx* c, const double* w, double* part, double* out);  // out = Σ w²
// partial sums into part; if out != nullptr the last block folds them (deterministically) into out
cudaError_t launch_dots(cnpint_ctx* c, double* const* V, int nv, const double* w, double* part, double* out);
cudaError_t launch_reduce(cnpint_ctx* c, const double* part, int ncols, double* out, int accumulate_sq);
cudaError_t launch_combine_backsolve(cnpint_ctx* c, double* const* X, int nv, int scaled, const double* u_in,
                                     double* u_out);
bool upd_dst_ok(const cnpint_ctx* c);
cudaError_t launch_cgs2_pass_dst(cnpint_ctx* c, double* const* Vp, int nv, const double* c1, double* w,
                                 double* part, double* out, double* dout);
cudaError_t launch_cgs2_pass(cnpint_ctx* c, double* const* V, int nv, const double* c1, const double* c2,
                             double* w, double* part, double* out, int phase);
cudaError_t launch_update(cnpint_ctx* c, double* const* V, int nv, const double* coefsrc, int coefmode,
                          double* w, double* wout, int want_dots, int want_norm, double* part, double* out);
cudaError_t launch_small(cnpint_ctx* c, int op, int j, int arg);
cudaError_t launch_scal_to_host(cnpint_ctx* c);

// profiler hooks (cnpint.cu); no-ops unless cnpint_profile_enable(ctx, 1)
// Kernel launch on the handle's stream with programmatic dependent launch when c->pdl (CNPINT_PDL=0
// turns it off): the kernel must start with pdl_enter() before touching data of earlier kernels.
template <typename... KArgs, typename... Args>
static inline cudaError_t cnp_launch(const cnpint_ctx* c, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
void cnp_prof_begin(cnpint_ctx* c, int kid);
void cnp_shard_free(cnpint_ctx* c);  // shard.cu
// Per-(key, CUDA device) cache of a launcher's one-time setup (cudaFuncSetAttribute is per-device
// state; occupancy-derived grid sizes depend on the device): compute(&v) runs until it succeeds once
// for the current device, under no lock (it must be idempotent); lookups and stores are mutex-guarded,
// so handles on several devices and host threads are safe.  key = the kernel's address.
bool cnp_dev_cache_get(const void* key, int* val);
void cnp_dev_cache_put(const void* key, int val);
template <class F>
static inline cudaError_t cnp_dev_cached(const void* key, int* out, F&& compute) {
  if (cnp_dev_cache_get(key, out)) return cudaSuccess;
  cudaError_t e = compute(out);
  if (e == cudaSuccess) cnp_dev_cache_put(key, *out);
  return e;
}
void cnp_prof_end(cnpint_ctx* c, int kid, double algo_bytes);
static inline double cnp_units(const cnpint_ctx* c) { return (double)c->N * c->nx * c->ny; }
static inline double cnp_spec_units(const cnpint_ctx* c) { return (double)(c->H + 1) * c->nx * c->ny; }
