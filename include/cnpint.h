/*
 * cnpint — B200-native (sm_100a, fp64) all-at-once Crank–Nicolson solver with the block
 * α-circulant parallel-in-time preconditioner of arxiv 2401.16113.
 *
 * C ABI.  Plain pointers and sizes only; no torch types.  The caller owns every buffer.
 *
 * Notation: N = number of time steps (the paper's M), m = number of spatial
 * unknowns (the paper's N), τ = T/N, Ã = τ L_h, Q1 = I − ½Ã, Q2 = I + ½Ã.
 *
 * ----------------------------------------------------------------------------------------
 * Device vector layout (every d_* vector argument)
 *   fp64, block t (0-based) holds u^{t+1} (Eq. 2.2 unknown ordering).
 *   1D:  [N][ld]          element (t, x)    at  t*ld + x,            0 <= x < nx
 *   2D:  [N][ny][ld]      element (t, y, x) at  (t*ny + y)*ld + x,   0 <= x < nx, 0 <= y < ny
 *   ld = cnpint_ld(ctx) >= nx (padded row pitch, multiple of 4 doubles = 32 B so that rows
 *   start 32-B aligned; x fastest).  Padding columns x >= nx must be zero on input and are
 *   written as zero on output.  Total length: cnpint_vec_elems(ctx) doubles.  The paper's
 *   lexicographic order fixes neither the fastest index nor padding: our choice.
 * Host vector layout (the *_host entry points): packed, no padding:
 *   1D [N][nx], 2D [N][ny][nx], fp64, C order.
 *
 * Streams and synchronisation
 *   Every call enqueues on the stream given to cnpint_create (a cudaStream_t passed as void*,
 *   e.g. torch.cuda.current_stream().cuda_stream) and returns without synchronising, EXCEPT
 *   cnpint_gmres*, cnpint_*_host and cnpint_device_status, which synchronise that stream.
 *   Outputs may not alias inputs.  One handle per host thread.
 *
 * Ownership
 *   The workspace (cnpint_workspace_bytes bytes of device memory, 256-B aligned) is owned by
 *   the caller and must outlive the handle.  The library never allocates device memory after
 *   cnpint_create, except a small pinned host staging area for residual estimates.  Host
 *   coefficient arrays are copied at create and may be freed afterwards.
 *
 * Errors
 *   Argument errors are detected synchronously (CNPINT_EINVAL / CNPINT_EUNSUPPORTED) and
 *   nothing is enqueued.  CUDA launch/runtime failures return CNPINT_ECUDA.  A zero or
 *   non-finite pivot in the shifted tridiagonal solve — "zero" read relatively: a pivot or 2×2
 *   elimination determinant that cancels below 1e-13 of its terms — sets a device status word
 *   (SPEC.md:298 SingularPreconditioner) reported as CNPINT_ESINGULAR by cnpint_device_status and
 *   by cnpint_gmres* (which stop at the step whose P_α⁻¹ met it; the status word is cleared).
 *   cnpint_last_error(ctx) returns a human-readable message for the last failure.
 */
#ifndef CNPINT_H
#define CNPINT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cnpint_ctx cnpint_ctx;

typedef enum {
  CNPINT_OK = 0,
  CNPINT_EINVAL = -1,        /* bad argument (sizes, alpha, tol, null pointers, workspace) */
  CNPINT_EUNSUPPORTED = -2,  /* valid but unsupported (N not a power of two, N > 65536, ...) */
  CNPINT_ECUDA = -3,         /* CUDA runtime/launch error */
  CNPINT_ESINGULAR = -4,     /* zero / non-finite pivot in a shifted solve (device status) */
  CNPINT_ENOCONV = -5,       /* GMRES reached maxit without meeting tol (report filled in) */
  CNPINT_EBREAKDOWN = -6     /* non-finite GMRES scalar (NaN/Inf in the Arnoldi process) */
} cnpint_status;

/* Spatial operator L_h (NOT multiplied by τ; the library forms Ã = τ L_h).
 * "A ∈ R^{N×N} the spatial discretization matrix of 𝓛"; Assumption 3.1
 * (PAPER.md:235-238): negative semi-definite and diagonalisable.
 *   1D (dim = 1, ny = 1):  (L_h u)_i = sub_i u_{i−1} + diag_i u_i + sup_i u_{i+1},
 *                          u_{−1} = u_{nx} = 0 (homogeneous Dirichlet).
 *       toeplitz = 1: constant rows (sub, diag, sup) = (xs, xd, xu); the arrays are ignored.
 *       toeplitz = 0: per-row host arrays sub/diag/sup of length nx (sub[0], sup[nx−1] unused).
 *   2D (dim = 2):          L_h = I_y ⊗ L_x + L_y ⊗ I_x + shift·I,  L_x = tridiag(xs, xd, xu)
 *                          (nx×nx Toeplitz), L_y = tridiag(ys, yd, yu) (ny×ny Toeplitz).
 *       Requires xs*xu > 0 and ys*yu > 0 (diagonal similarity to a symmetric Toeplitz matrix,
 *       diagonalised by DST-I) and nx + 1, ny + 1 powers of two in [4, 1024].
 *   1D sizes: 2 <= nx <= 4096 (Toeplitz) or 2048 (variable rows).  N: power of two, 2..65536
 *   (1D time-axis FFT: thread-block clusters for N < 2048, the four-step L2-resident kernel for
 *   N >= 2048); 2D: N <= 16384 (cluster / one-column time pass). */
typedef struct {
  int dim;
  int nx, ny;
  int toeplitz;
  const double* sub;
  const double* diag;
  const double* sup;
  double xs, xd, xu;
  double ys, yd, yu;
  double shift;
} cnpint_operator;

typedef struct {
  int iterations;      /* total inner Arnoldi steps ("Its") */
  int restarts;        /* completed restart cycles that did not converge */
  int converged;       /* 1 if the true residual ||b − 𝓜u||/||b|| <= tol */
  double relres_est;   /* last Givens estimate |g_{j+1}|/||b|| */
  double relres_true;  /* ||b − 𝓜u||/||b|| at the last cycle end */
  double seconds;      /* host wall time inside the call */
  double* history;     /* caller host array (may be NULL): estimate after every inner step */
  int history_cap;     /* capacity of history */
  double relres_prec;  /* cnpint_gmres_left: ||P_α⁻¹(b − 𝓜u)|| / ||P_α⁻¹b|| at the last cycle end
                        * (the residual of PAPER.md:578-579); cnpint_gmres: not written */
} cnpint_gmres_report;

/* Bytes of device workspace for a handle with these sizes (0 on invalid arguments).
 * restart_max >= 1 sizes the GMRES Krylov basis (restart_max + 1 vectors); pass 0 to size
 * a handle for apply_A / apply_P / apply_Pinv only (cnpint_gmres then returns EINVAL). */
size_t cnpint_workspace_bytes(int N, const cnpint_operator* op, int restart_max);

/* Create a handle.  N: time steps, power of two, 2 <= N <= 65536 (1D; 2D: N <= 16384).  T > 0: horizon (τ = T/N).
 * alpha in (0, 1]: the α of C1^(α), C2^(α).  α = 1 is the block circulant P_1 of
 * the paper's comparison (NEXT #2): its k = N/2 shifted system degenerates to λ1 z = w, and P_1 is
 * singular iff Ã is (Remark 3.2) — create checks that and returns CNPINT_ESINGULAR
 * (Toeplitz / 2D: the closed-form spectrum; variable rows: long-double elimination of L_h with a
 * relative 1e-13 pivot test); a zero / non-finite pivot met later on the device is reported by
 * cnpint_device_status / cnpint_gmres*.
 * d_workspace: device pointer, >= cnpint_workspace_bytes bytes, 256-B aligned.
 * cuda_stream: cudaStream_t (may be NULL = legacy default stream). */
cnpint_status cnpint_create(cnpint_ctx** out, int N, double T, double alpha, const cnpint_operator* op,
                            int restart_max, void* d_workspace, size_t ws_bytes, void* cuda_stream);

/* Waits for the handle's stream, then frees the handle (not the caller's workspace). */
void cnpint_destroy(cnpint_ctx* ctx);
const char* cnpint_last_error(const cnpint_ctx* ctx);
/* Moves the handle to another stream; if it differs from the current one, the current stream is
 * synchronised first (the handle's kernels are ordered on one stream at a time). */
cnpint_status cnpint_set_stream(cnpint_ctx* ctx, void* cuda_stream);

int64_t cnpint_ld(const cnpint_ctx* ctx);          /* row pitch in doubles */
int64_t cnpint_vec_elems(const cnpint_ctx* ctx);   /* doubles per device vector (incl. padding) */
int64_t cnpint_spec_elems(const cnpint_ctx* ctx);  /* complex entries of the half spectrum */

/* y = 𝓜u,  𝓜 = B1 ⊗ I − B2 ⊗ Ã (Eq. 2.2), i.e. by the block form of
 * y_0 = Q1 u_0, y_t = Q1 u_t − Q2 u_{t−1}.  Kernel K1, one HBM pass. */
cnpint_status cnpint_apply_A(cnpint_ctx* ctx, const double* d_u, double* d_y);

/* v = P_α z  (PAPER.md:344-350 block form; test hook): as 𝓜 plus (Pz)_0 −= α Q2 z_{N−1}. */
cnpint_status cnpint_apply_P(cnpint_ctx* ctx, const double* d_z, double* d_v);

/* z = P_α⁻¹ v via the diagonalisation P_α = (V⊗I)(D1⊗I − D2⊗Ã)(V⁻¹⊗I), V = Λ_α⁻¹𝔽*
 * (Eq. 3.2), solving only k = 0..N/2 (Remark 3.1).
 * v must be real (the conjugate halving relies on it).  1D: K2 (Γ_α-scaled real FFT along t)
 * → K3 (N/2+1 complex tridiagonal solves) → K4 (C2R inverse FFT, Γ_α⁻¹, 1/N).
 * 2D: DST fast diagonalisation in space around a fused time pass, which per
 * spatial mode μ inverts the N×N α-circulant C1^(α) − μC2^(α) — by Eq. 3.2's transform on chip
 * (Γ_α·FFT, ÷ (λ1_k − λ2_kμ), iFFT·Γ_α⁻¹) or, by default when every mode is stable (μ < 0), as the
 * equivalent first-order recurrence (1 − μ/2) z_t − (1 + μ/2) z_{t−1} = v_t, z_{−1} = α z_{N−1}, run as a
 * chunked scan over the time axis (k_tscan.cu; cnpint_set_debug bit 524288 selects the transform). */
cnpint_status cnpint_apply_Pinv(cnpint_ctx* ctx, const double* d_v, double* d_z);

/* Stage entry points of the 1D P_α⁻¹ (per-kernel parity tests and timing).
 * Half spectrum layout: complex128 interleaved (re, im), [N/2+1][ld] (row k = frequency k),
 * unnormalised forward DFT: d_what[k][x] = Σ_t e^{−2πikt/N} α^{t/N} v[t][x] (step (a) times √N).
 * cnpint_shifted_solve solves (λ1_k I − λ2_k Ã) ẑ_k = ŵ_k with λ1_k = 1 − a e^{−2πik/N},
 * λ2_k = ½(1 + a e^{−2πik/N}), a = α^{1/N} (FFT-consistent reading of Eq. eigCx, R3).
 * cnpint_time_ifft applies z[t][x] = α^{−t/N} (1/N) Σ_{k<N} e^{+2πikt/N} ẑ_k (ẑ_{N−k} = conj ẑ_k). */
cnpint_status cnpint_time_fft(cnpint_ctx* ctx, const double* d_v, double* d_what);
cnpint_status cnpint_shifted_solve(cnpint_ctx* ctx, const double* d_what, double* d_zhat);
cnpint_status cnpint_time_ifft(cnpint_ctx* ctx, const double* d_zhat, double* d_z);

/* Right-preconditioned restarted GMRES(restart) on 𝓜P_α⁻¹ y = b, u = P_α⁻¹ y, zero initial
 * guess.  Stops when the Givens estimate |g_{j+1}|/||b|| <= tol and then
 * confirms the true residual ||b − 𝓜u||/||b|| <= tol at the cycle end (else restarts).
 * Arnoldi: classical Gram–Schmidt with one reorthogonalisation (CGS2), fused device kernels;
 * Hessenberg least squares (Givens) on device; one 64-byte device→host read per inner step.
 * The preconditioned directions z_j = P_α⁻¹ v_j are kept for the cycle, so the update is
 * u += Σ_j y_j z_j (= P_α⁻¹ V y, same iterate) without a further P_α⁻¹ application.
 * 0 < tol < 1, 1 <= restart <= restart_max, maxit >= 1 (total inner steps).
 * Returns CNPINT_OK, CNPINT_ENOCONV (maxit reached; u holds the last iterate, so
 * maxit = j <= restart returns the j-th GMRES iterate) or an error.  rep may be NULL. */
cnpint_status cnpint_gmres(cnpint_ctx* ctx, const double* d_b, double* d_u, double tol, int restart,
                           int maxit, cnpint_gmres_report* rep);

/* Left-preconditioned restarted GMRES(restart) on P_α⁻¹𝓜u = P_α⁻¹b, zero initial guess: the
 * variant the paper's convergence analysis is stated for (§4; Theorem 4.5,
 * PAPER.md:771-784).  r_0 = P_α⁻¹b; each inner step forms
 * w = P_α⁻¹(𝓜 v_j) (K1 then the P_α⁻¹ kernels, the basis scale folded into the Γ-scaling) and
 * orthogonalises it with the same CGS2 kernels as cnpint_gmres; the cycle end is u += V y (no
 * P_α⁻¹), then r = P_α⁻¹(b − 𝓜u) starts the next cycle.
 * history[k−1] = Givens estimate of ||r_k|| / ||r_0||, r_k = P_α⁻¹(b − 𝓜u^(k)) (R28).
 * Converged iff ||P_α⁻¹(b − 𝓜u)|| / ||P_α⁻¹b|| <= tol at a cycle end (rep->relres_prec);
 * rep->relres_true is the unpreconditioned ||b − 𝓜u|| / ||b||.  Arguments, workspace, errors and
 * the maxit semantics as cnpint_gmres (the first preconditioned direction slot serves as the
 * 𝓜v_j temporary). */
cnpint_status cnpint_gmres_left(cnpint_ctx* ctx, const double* d_b, double* d_u, double tol, int restart,
                                int maxit, cnpint_gmres_report* rep);

/* Host-buffer variants (end-to-end: H2D copy of the input, the device computation, D2H copy of
 * the result, all on the handle's stream; synchronises).  Host layout: packed (see top). */
cnpint_status cnpint_apply_Pinv_host(cnpint_ctx* ctx, const double* h_v, double* h_z);
cnpint_status cnpint_apply_A_host(cnpint_ctx* ctx, const double* h_u, double* h_y);
cnpint_status cnpint_gmres_host(cnpint_ctx* ctx, const double* h_b, double* h_u, double tol, int restart,
                                int maxit, cnpint_gmres_report* rep);

/* End-to-end GMRES over `count` right-hand sides in host memory (packed layout; pinned memory for the
 * copies to overlap): solve i runs on the handle's stream while the H2D copy of b_{i+1} and the D2H
 * copy of u_{i−1} run on two internal copy streams, so PCIe traffic in both directions hides behind
 * the computation.  d_stage: caller-owned device scratch of 4·cnpint_vec_elems doubles, 16-B aligned.
 * reps: NULL or an array of `count` reports.  Synchronises; returns CNPINT_OK, CNPINT_ENOCONV (some
 * solve reached maxit; its report says which) or the first error. */
cnpint_status cnpint_gmres_host_batch(cnpint_ctx* ctx, int count, const double* const* h_b, double* const* h_u,
                                      double tol, int restart, int maxit, double* d_stage, cnpint_gmres_report* reps);

/* Time-dependent operator 𝓛(t) = d(t)𝓛 (Eq. 5.8).
 * d_half: host array of the N values d(t_{t+½}), t = 0..N−1 (finite, > 0), copied; NULL restores the
 * constant-coefficient method.  Afterwards 𝓜 = B1⊗I − (D̃B2)⊗Ã with D̃ = diag(d_half) in apply_A,
 * gmres and the true residual, and the preconditioner uses d̄·C2^(α), d̄ = mean(d_half)
 * (apply_P, apply_Pinv and the stage kernels).  The caller forms ξ₀ = (I + ½d(t_½)Ã)u⁰ in b.
 * Synchronises; rebuilds the tables that depend on the preconditioner's τ. */
cnpint_status cnpint_set_time_dependence(cnpint_ctx* ctx, const double* d_half);

/* Synchronise the stream and report deferred device errors (CNPINT_ESINGULAR), clearing them. */
cnpint_status cnpint_device_status(cnpint_ctx* ctx);

/* Number of kernels this handle has launched since create (instrumentation for bench.py). */
int64_t cnpint_launch_count(const cnpint_ctx* ctx);

/* Per-kernel-class profiler (bench.py's live roofline): CUDA events recorded on the handle's stream
 * around every launch while enabled.  enable(ctx, 1) (re)starts the counters (synchronises);
 * enable(ctx, 0) frees the events.  read() synchronises and returns, for kernel class kid
 * (0 <= kid < cnpint_kernel_name() == NULL), the summed event durations in ms, the launch count and
 * the ALGORITHMIC bytes those launches must move.  Classes:
 * 0 K1 matvec, 1 K2 time FFT, 2 K3 tridiagonal, 3 K4 inverse time FFT, 4 K6 2D time pass,
 * 5 K5 DST x, 6 K5 DST y, 7 K7 dots, 8 K7 update, 9 reductions, 10 GMRES scalar kernels,
 * 11 K5 fused x+y sine pass. */
cnpint_status cnpint_profile_enable(cnpint_ctx* ctx, int on);
cnpint_status cnpint_profile_read(cnpint_ctx* ctx, int kernel_class, double* ms_total, int64_t* launches,
                                  double* algo_bytes);
const char* cnpint_kernel_name(int kernel_class);

/* K0: fp64 stream copy dst[i] = src[i], i < n (128-bit loads/stores) — the same-run HBM
 * bandwidth reference.  Enqueued on cuda_stream. */
cnpint_status cnpint_stream_copy(const double* d_src, double* d_dst, size_t n, void* cuda_stream);

/* Test hook (orthogonality measurements of the Arnoldi basis, K7): vector i of the LAST
 * restart cycle of the most recent cnpint_gmres call, v_i = s_i·Ṽ_i with 0 <= i < *count (count may
 * be read with i = 0 even when the call fails).  *d_vec = Ṽ_i (device, the vector layout above; the
 * first cycle's Ṽ_0 is the caller's b; valid until the next call on the handle), *scale = s_i (host
 * copy; synchronises the stream).  *count = steps of the cycle + 1, or = steps when the cycle's last step
 * took its norm from the Gram matrix and wrote no vector (the derived-norm probe, debug 2097152 off).
 * Any out pointer may be NULL.  EINVAL for i out of range. */
cnpint_status cnpint_krylov_basis(cnpint_ctx* ctx, int i, const double** d_vec, double* scale, int* count);

/* Same-run compute ceilings: enqueues on cuda_stream a kernel of 8 CTAs x 256
 * threads per SM doing `iters` rounds of dependent fp64 FMAs (kind 0, 8 chains per thread) or of
 * mma.sync.m8n8k4 f64 DMMA (kind 1, 4 accumulators per warp).  d_out: device scratch of
 * >= 8·SMs·256 doubles (one result per thread, so no work is eliminated).  *flops = the floating-point
 * operations one launch performs (FMA = 2; one m8n8k4 = 512); the caller times the launch with
 * events on the same stream.  EINVAL for bad arguments, ECUDA on launch failure. */
cnpint_status cnpint_peak_kernel(int kind, double* d_out, int iters, void* cuda_stream, double* flops);

/* ---------------------------------------------------------------------------------------------
 * 1D x-sharded handles.  R ranks (one GPU each) split the
 * spatial index of a 1D operator into contiguous chunks [x0[r], x0[r+1]), x0[0] = 0, x0[R] = nx, every
 * chunk >= 2 rows; rank r's vectors are [N][ld_r] over its chunk (ld_r = cnpint_ld).  P_α⁻¹ (PAPER.md
 * Eq. 3.2): the time transforms are per column (local); each frequency's tridiagonal system
 * (λ1_k I − λ2_k Ã) ẑ_k = ŵ_k is solved by a partition method — a local solve, an
 * all-gather of 2 complex per frequency (the local solution's end values), a redundant block-
 * tridiagonal 2R × 2R reduced solve, a local re-solve with corrected end rows.  𝓜u
 * all-gathers every rank's two boundary columns (2N doubles).  GMRES all-reduces its dot products.
 * Constant-coefficient operators, 0 < α < 1.
 *
 * Collectives are the caller's (e.g. NCCL through torch.distributed): op 0 = all-gather
 * (d_recv[r·count + i] = rank r's d_send[i], r < R), op 1 = in-place all-reduce sum of d_send (==
 * d_recv); device buffers of the handle's workspace; enqueue on cuda_stream or synchronise it; return 0
 * on success.  With R = 1 no callback is needed. */
typedef int (*cnpint_collective_fn)(void* user, int op, const double* d_send, double* d_recv, size_t count,
                                    void* cuda_stream);

size_t cnpint_shard_workspace_bytes(int N, const cnpint_operator* op, int R, const int* x0, int rank,
                                    int restart_max);
/* Arguments as cnpint_create, with op the GLOBAL 1D operator, R ranks, chunk bounds x0[R+1] and this
 * rank.  Builds rank `rank`'s handle (local operator = rows x0[rank]..x0[rank+1]−1, the couplings to the
 * neighbours kept aside) and the spike-end table of every rank (host, long double). */
cnpint_status cnpint_shard_create(cnpint_ctx** out, int N, double T, double alpha, const cnpint_operator* op, int R,
                                  const int* x0, int rank, int restart_max, void* d_workspace, size_t ws_bytes,
                                  void* cuda_stream);
cnpint_status cnpint_shard_set_collective(cnpint_ctx* ctx, cnpint_collective_fn fn, void* user);
/* The exchange buffers inside the workspace (device): the end values (send ends_count doubles, receive
 * R·ends_count) and the boundary columns (send halo_count = 2N, receive R·2N).  Any pointer may be NULL. */
cnpint_status cnpint_shard_buffers(cnpint_ctx* ctx, double** ends_send, double** ends_recv, size_t* ends_count,
                                   double** halo_send, double** halo_recv, size_t* halo_count);
/* Whole operations through the collective callback (rank-local vectors in, rank-local out). */
cnpint_status cnpint_shard_apply_Pinv(cnpint_ctx* ctx, const double* d_v, double* d_z);
cnpint_status cnpint_shard_apply_A(cnpint_ctx* ctx, const double* d_u, double* d_y);
/* Right-preconditioned restarted GMRES on the sharded system (the algorithm of cnpint_gmres with classic
 * CGS2 and all-reduced dot products); every rank receives the same report.  Synchronises. */
cnpint_status cnpint_shard_gmres(cnpint_ctx* ctx, const double* d_b, double* d_u, double tol, int restart,
                                 int maxit, cnpint_gmres_report* rep);
/* Phase-split operations (the caller moves the exchange buffers between the phases): P_α⁻¹ =
 * pinv_begin → all-gather of the end values → pinv_end; 𝓜u = halo_begin → all-gather of the boundary
 * columns → apply_A_end. */
cnpint_status cnpint_shard_pinv_begin(cnpint_ctx* ctx, const double* d_v);
cnpint_status cnpint_shard_pinv_end(cnpint_ctx* ctx, double* d_z);
cnpint_status cnpint_shard_halo_begin(cnpint_ctx* ctx, const double* d_u);
cnpint_status cnpint_shard_apply_A_end(cnpint_ctx* ctx, const double* d_u, double* d_y);
/* Host-only partition arithmetic (no GPU; the same code the handles run): the spike-end table
 * red[(k R + r) 4 + (v1, vm, w1, wm)] (complex, K = N/2+1 frequencies) and ab[2r + (α_r, β_r)]; and the
 * reduced solve for rank `rank` given every rank's end values ends_all[(r K + k) 2 + (g_1, g_m)] (complex),
 * writing neighbours[k] = (xe_{rank−1}, xs_{rank+1}) (complex pairs).  ESINGULAR if a 2×2 block cancels. */
cnpint_status cnpint_shard_spike_ends_host(int N, double T, double alpha, const cnpint_operator* op, int R,
                                           const int* x0, double* red_out, double* ab_out);
cnpint_status cnpint_shard_reduced_host(int K, int R, int rank, const double* red, const double* ab,
                                        const double* ends_all, double* neighbours);

/* Test hook (negative controls): 0 = none, 1 = flip the sign of the FFT twiddles,
 * 2 = use the printed Eq. eigCx ordering λ1_k = 1 − a e^{+2πik/N} (R3).
 * The parity suite must fail with either set.  Kernel-variant bits (not negative controls; the
 * parity suite runs the alternatives on the same inputs): 4 = Toeplitz shifted solves through the
 * generic merge tree instead of the tabulated fast tree; 8 = the one-column time FFT kernel
 * (N <= 16384); 16 = the cluster time FFT instead of the four-step kernel for 1D N >= 2048;
 * 32 = the shared-memory Stockham DST kernel for every 2D sine pass; 64 = the cluster kernel instead
 * of the register time pass for 2D N = 256, 512; 128 = classic CGS2 in cnpint_gmres (a second
 * reading pass c2 = Ṽᵀ(w − Ṽs²c1)) instead of the Gram form c2 = c1 − G̃s²c1, whose Gram row
 * Ṽᵀ Ṽ_j is reduced inside the matvec (K7); 256 = the pipelined half-length DST kernel
 * (k_dst2.cu: TMA bulk-copy ring, n + 1 ∈ {64, …, 512}, square grids) for the 2D sine passes;
 * 512 = the first-generation variable-row K3 kernel (every merge of the tree computed in the solve)
 * instead of k_trivar (upper tree from the per-handle table built at create; c3);
 * 1024 = the register DST kernel for every 2D sine pass with 2(n+1) ∈ {256, 512, 1024} (A/B);
 * 2048 = fault injection: every 1D shifted solve reports a singular pivot (status-word tests);
 * 4096 = the first-generation Stockham x pass instead of the lean register x pass (k_dst4.cu);
 * 8192 = the first-generation y pass (register / Stockham) instead of the lean y pass (k_dst5.cu);
 * 16384 = the lean 2D time pass (k_tpass2.cu) also at N = 512 (default at N = 256, 1024; debug 64 turns
 * both register time passes off in favour of the cluster kernel); 32768 = the three-pass 2D P_α⁻¹: W⁻¹
 * and W each as one fused x+y sine pass (k_dstxy.cu, n + 1 ∈ {64, …, 512}; 48 instead of 80 B of HBM
 * traffic per unknown, but no faster on B200: the passes are bound on chip, K5);
 * 131072 = no fusion of the 2D Gram update with the next x sine pass (k_upd_dst4; cnpint_gmres fuses them
 * when the lean x pass applies and the next Arnoldi step is expected to run);
 * 262144 = the first-generation lean time pass (divide by λ1_k − λ2_kμ) instead of the second (k_tpass2
 * GEN 2: ½/λ2_k folded into the forward output, then ÷ (c_k − μ) with c_k = λ1_k/λ2_k from per-mode tables);
 * 524288 = the 2D time pass as Eq. 3.2's transform (Γ_α·FFT along time, ÷ (λ1_k − λ2_kμ), iFFT·Γ_α⁻¹ on chip)
 * instead of the default recurrence form of the same α-circulant solve (k_tscan.cu: per spatial mode
 * (1 − μ/2) z_t − (1 + μ/2) z_{t−1} = v_t with z_{−1} = α z_{N−1}, a chunked scan over the time axis; used when
 * every mode has μ < 0 and N is a power of two in [8, 2048]);
 * 1048576 = the register 2D matvec (k_matvec2d: own row and both y neighbours loaded into registers, four
 * time rows per batch) instead of the staged one (k_matvec2d_s: rows of u through a cp.async shared-memory
 * ring, eight time rows in flight per warp); the same arithmetic per element;
 * 2097152 = no derived-norm probe in cnpint_gmres: by default a step expected to be the last takes
 * h_{j+1,j} from the Gram matrix (β² = ww − 2aᵀc1 + aᵀG̃a, trusted when β² ≥ 1e-8·wᵀw) and, if the estimate
 * then meets the tolerance, skips the update pass that would write a basis vector nobody reads;
 * 4194304 = probe every step (exercises the take-back path; the results are those of the plain steps).  Bits 1, 2, 8, 16, 64, 16384 and 262144 — the
 * transform's negative controls and kernel selections — also keep the transform path. */
cnpint_status cnpint_set_debug(cnpint_ctx* ctx, int flags);

#ifdef __cplusplus
}
#endif
#endif /* CNPINT_H */
