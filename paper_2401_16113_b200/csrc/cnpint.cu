// cnpint host side: the C ABI of include/cnpint.h — handle, workspace carve-up, fp64 tables, the
// P_α⁻¹ pipelines and the restarted right-preconditioned GMRES control loop.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdlib>
#include <algorithm>
#include <complex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <utility>
#include <vector>

#include "internal.h"


int matvec_partial_blocks(const cnpint_ctx* c);

// ------------------------------------------------------------------------------ profiler
// Per-kernel-class CUDA-event timing on the handle's stream.  Events come from a pool that grows
// during warm-up and is reused; recording an event pair costs ~1 µs of GPU time per launch.
struct CnpProf {
  std::vector<cudaEvent_t> ev[KID_COUNT];  // pairs: [2i] start, [2i+1] stop
  size_t used[KID_COUNT];
  double bytes[KID_COUNT];
};

static const char* const KNAMES[KID_COUNT] = {"K1_matvec", "K2_time_fft", "K3_tridiag", "K4_time_ifft",
                                              "K6_time_pass_2d", "K5_dst_x", "K5_dst_y", "K7_dots",
                                              "K7_update", "reduce", "K8_small", "K5_dst_xy",
                                              "K7_update+K5_dst_x"};

void cnp_prof_begin(cnpint_ctx* c, int kid) {
  CnpProf* p = (CnpProf*)c->prof;
  if (!p) return;
  size_t i = p->used[kid];
  if (p->ev[kid].size() < 2 * (i + 1)) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    p->ev[kid].push_back(a);
    p->ev[kid].push_back(b);
  }
  cudaEventRecord(p->ev[kid][2 * i], c->stream);
}

void cnp_prof_end(cnpint_ctx* c, int kid, double algo_bytes) {
  c->launches++;
  CnpProf* p = (CnpProf*)c->prof;
  if (!p) return;
  size_t i = p->used[kid];
  cudaEventRecord(p->ev[kid][2 * i + 1], c->stream);
  p->used[kid] = i + 1;
  p->bytes[kid] += algo_bytes;
}

static void prof_free(cnpint_ctx* c) {
  CnpProf* p = (CnpProf*)c->prof;
  if (!p) return;
  for (int k = 0; k < KID_COUNT; ++k)
    for (cudaEvent_t e : p->ev[k]) cudaEventDestroy(e);
  delete p;
  c->prof = nullptr;
}
// ------------------------------------------------------------------------------ per-device cache
static std::mutex g_cache_mu;
static std::map<std::pair<const void*, int>, int> g_cache;

bool cnp_dev_cache_get(const void* key, int* val) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find({key, dev});
  if (it == g_cache.end()) return false;
  *val = it->second;
  return true;
}

void cnp_dev_cache_put(const void* key, int val) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache[{key, dev}] = val;
}

cudaError_t launch_reduce_n(cnpint_ctx* c, const double* part, int nparts, int stride, int ncols, double* out);
cudaError_t launch_dstxy(cnpint_ctx* c, const double* in, double* out, int inverse, int accumulate);
cudaError_t launch_dst_x_acc(cnpint_ctx* c, const double* in, double* out);

namespace {

const size_t ALIGN = 256;
size_t up_align(size_t v) { return (v + ALIGN - 1) & ~(ALIGN - 1); }

bool is_pow2(long v) { return v > 0 && (v & (v - 1)) == 0; }

struct Layout {
  size_t lo, di, up, tw, gam, igam, lam1, lam2, sk, il2, tri, vtab, tables_end, spec, fsy, fscnt, tmp1, tmp2, tmp3, io1, io2, io3;
  size_t dxi, dx, dyi, dy, ex, ey, twx, twy;
  size_t dt, V, Z, part, c1, c2, scl, H, cs, sn, g, y, coef, G, cg, scal, status, xycnt;
  size_t total;
};

int64_t ld_of(int nx) { return ((int64_t)nx + 3) / 4 * 4; }

// Validates sizes; returns a message or nullptr.
const char* check_op(int N, const cnpint_operator* op, int* unsupported) {
  *unsupported = 0;
  if (!op) return "operator is NULL";
  if (op->dim != 1 && op->dim != 2) return "op->dim must be 1 or 2";
  if (op->nx < 1 || (op->dim == 2 && op->ny < 1)) return "nx/ny must be >= 1";
  if (op->dim == 1 && op->ny != 1 && op->ny != 0) return "1D operator requires ny = 1";
  if (N < 2) return "N must be >= 2";
  if (!is_pow2(N) || N > 65536) { *unsupported = 1; return "N must be a power of two in [2, 65536]"; }
  if (op->dim == 1) {
    if (!op->toeplitz && (!op->sub || !op->diag || !op->sup)) return "non-Toeplitz 1D operator needs sub/diag/sup";
    // K3 keeps <= 16 (Toeplitz) / 8 (variable) rows per thread in registers, <= 256 threads per system
    if (op->nx > (op->toeplitz ? 4096 : 2048) || op->nx < 2) {
      *unsupported = 1;
      return "1D needs 2 <= nx <= 4096 (Toeplitz) / 2048 (variable rows)";
    }
  } else {
    if (!is_pow2((long)op->nx + 1) || !is_pow2((long)op->ny + 1)) {
      *unsupported = 1;
      return "2D requires nx+1 and ny+1 powers of two (DST-I via FFT)";
    }
    if (op->nx + 1 > 1024 || op->ny + 1 > 1024) { *unsupported = 1; return "2D n+1 > 1024 unsupported"; }
    if (op->nx < 3 || op->ny < 3) { *unsupported = 1; return "2D needs nx, ny >= 3"; }
    if (N > 16384) { *unsupported = 1; return "2D needs N <= 16384 (time pass on chip)"; }
    if (!(op->xs * op->xu > 0.0) || !(op->ys * op->yu > 0.0))
      return "2D requires xs*xu > 0 and ys*yu > 0 (diagonal symmetrisation)";
  }
  return nullptr;
}

Layout layout(int N, const cnpint_operator* op, int restart_max) {
  Layout L;
  std::memset(&L, 0, sizeof(L));
  const int nx = op->nx, ny = op->dim == 2 ? op->ny : 1;
  const int64_t ld = ld_of(nx);
  const int64_t vec = (int64_t)N * ny * ld;
  const int H = N / 2;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += up_align(bytes ? bytes : 1); return o; };
  L.lo = take(ld * 8); L.di = take(ld * 8); L.up = take(ld * 8);
  L.tw = take((size_t)N * 16);
  L.gam = take((size_t)N * 8); L.igam = take((size_t)N * 8);
  L.lam1 = take((size_t)(H + 1) * 16); L.lam2 = take((size_t)(H + 1) * 16);
  L.sk = take((size_t)(H + 1) * 16); L.il2 = take((size_t)(H + 1) * 16);
  if (op->dim == 1 && op->toeplitz) {
    const TriCfg t = tri_cfg(nx, 1);
    L.tri = take(t.small ? 16 : (size_t)(H + 1) * t.tabstride * 16);
  }
  if (op->dim == 2) {
    L.dxi = take(nx * 8); L.dx = take(nx * 8); L.dyi = take(ny * 8); L.dy = take(ny * 8);
    L.ex = take(ld * 8); L.ey = take(ny * 8);
    L.twx = take((size_t)2 * (nx + 1) * 16); L.twy = take((size_t)2 * (ny + 1) * 16);
  }
  L.tables_end = off;
  if (op->dim == 1 && !op->toeplitz) {  // built on the device after the upload (outside the host image)
    const int ts = trivar_table_stride(nx);
    L.vtab = ts ? take((size_t)(H + 1) * ts * 16) : 0;
  }
  L.spec = op->dim == 1 ? take((size_t)(H + 1) * ld * 16) : take(16);
  L.fsy = take(fstep_y_bytes(op->dim, N, (int64_t)ny * ld));
  L.fscnt = take(fstep_y_bytes(op->dim, N, (int64_t)ny * ld) ? (size_t)(fstep_nxb(N, (int64_t)ny * ld) + 1) * 4 : 4);
  L.tmp1 = take(vec * 8); L.tmp2 = take(vec * 8); L.tmp3 = take(vec * 8);
  L.io1 = take(vec * 8); L.io2 = take(vec * 8); L.io3 = take(vec * 8);
  if (restart_max >= 1) {
    L.V = take((size_t)(restart_max + 1) * vec * 8);
    L.Z = take((size_t)restart_max * vec * 8);  // z_j = P_α⁻¹ v_j of the current cycle
    L.c1 = take((restart_max + 2) * 8); L.c2 = take((restart_max + 2) * 8); L.scl = take((restart_max + 2) * 8);
    L.H = take((size_t)(restart_max + 1) * restart_max * 8);
    L.cs = take(restart_max * 8); L.sn = take(restart_max * 8); L.g = take((restart_max + 2) * 8);
    L.y = take(restart_max * 8); L.coef = take((restart_max + 2) * 8);
    L.G = take((size_t)(restart_max + 1) * (restart_max + 1) * 8); L.cg = take((CNP_MAX_DOT + 1) * 8);
  }
  // partial sums: dots/updates use CNP_RED_BLOCKS rows of (MAX_DOT+1), the matvec one row per block
  {
    cnpint_ctx tmp;
    std::memset(&tmp, 0, sizeof(tmp));
    tmp.dim = op->dim; tmp.N = N; tmp.ld = ld; tmp.ny = ny;
    size_t mv = (size_t)matvec_partial_blocks(&tmp);
    size_t blocks = mv > CNP_RED_BLOCKS ? mv : CNP_RED_BLOCKS;
    L.part = take(blocks * (CNP_MAX_DOT + 1) * 8);
  }
  L.scal = take(16 * 8);
  L.status = take(64);
  L.dt = take((size_t)N * 8);  // d(t_{t+½}) of a time-dependent operator (cnpint_set_time_dependence)
  L.xycnt = op->dim == 2 ? take((size_t)(N + 1) * 4) : 0;  // fused sine pass: per-slice counters + ticket
  L.total = off;
  return L;
}

void seterr(cnpint_ctx* c, const char* fmt, ...) {
  if (!c) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c->err, sizeof(c->err), fmt, ap);
  va_end(ap);
}

cnpint_status cuda_fail(cnpint_ctx* c, cudaError_t e, const char* where) {
  seterr(c, "CUDA error in %s: %s", where, cudaGetErrorString(e));
  return CNPINT_ECUDA;
}

#define CK(expr)                                          \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return cuda_fail(c, _e, #expr); \
  } while (0)

// ------------------------------------------------------------------------- tables (host, long double)
void make_tables(cnpint_ctx* c, const cnpint_operator* op, std::vector<char>& img, const Layout& L) {
  const int N = c->N, H = c->H;
  const long double PI = 3.141592653589793238462643383279502884L;
  auto put = [&](size_t off, const void* src, size_t bytes) { std::memcpy(img.data() + off, src, bytes); };
  // rows
  std::vector<double> lo(c->ld, 0.0), di(c->ld, 0.0), up(c->ld, 0.0);
  if (c->dim == 1) {
    for (int i = 0; i < c->nx; ++i) {
      lo[i] = op->toeplitz ? op->xs : op->sub[i];
      di[i] = op->toeplitz ? op->xd : op->diag[i];
      up[i] = op->toeplitz ? op->xu : op->sup[i];
    }
    lo[0] = 0.0;
    up[c->nx - 1] = 0.0;
  }
  put(L.lo, lo.data(), c->ld * 8); put(L.di, di.data(), c->ld * 8); put(L.up, up.data(), c->ld * 8);
  // twiddles ω_N^q = e^{-2πiq/N}
  std::vector<double2> tw(N);
  for (int q = 0; q < N; ++q) {
    long double th = 2.0L * PI * (long double)q / (long double)N;
    tw[q] = make_double2((double)cosl(th), (double)(-sinl(th)));
    if (c->debug & 1) tw[q].y = -tw[q].y;
  }
  put(L.tw, tw.data(), N * 16);
  // γ_t = α^{t/N}, 1/(N γ_t)
  std::vector<double> gam(N), igam(N);
  const long double lna = logl((long double)c->alpha);
  for (int t = 0; t < N; ++t) {
    long double g = expl(lna * (long double)t / (long double)N);
    gam[t] = (double)g;
    igam[t] = (double)(1.0L / ((long double)N * g));
  }
  put(L.gam, gam.data(), N * 8); put(L.igam, igam.data(), N * 8);
  // λ1_k = 1 − a e^{−iθ_k}, λ2_k = ½(1 + a e^{−iθ_k}), θ_k = 2πk/N (FFT-consistent, R3)
  std::vector<double2> l1(H + 1), l2(H + 1), sk(H + 1), il2(H + 1);
  const long double a = expl(lna / (long double)N);
  const long double a_ld = a;
  const long double one_m_a = -expm1l(lna / (long double)N);
  for (int k = 0; k <= H; ++k) {
    long double th = 2.0L * PI * (long double)k / (long double)N;
    long double sh = sinl(0.5L * th);
    long double sn = sinl(th), cs = cosl(th);
    if (2 * k == N) { sh = 1.0L; sn = 0.0L; cs = -1.0L; }  // exact at θ = π (λ2 = 0 when α = 1)
    if (c->debug & 2) sn = -sn;  // printed Eq. eigCx ordering (negative control)
    long double r1 = one_m_a + 2.0L * a * sh * sh, i1 = a * sn;        // 1 − a cos θ + i a sin θ
    long double r2 = 0.5L * (1.0L + a * cs), i2 = -0.5L * a * sn;      // ½(1 + a cos θ) − ½ i a sin θ
    long double den = r2 * r2 + i2 * i2;
    l1[k] = make_double2((double)r1, (double)i1);
    l2[k] = make_double2((double)r2, (double)i2);
    if (den == 0.0L) {
      // α = 1, k = N/2: λ2 = 0, the shifted system is λ1 z = w (no spatial coupling).  K3 recognises
      // il2 = 0 and divides by λ1.
      sk[k] = make_double2(0.0, 0.0);
      il2[k] = make_double2(0.0, 0.0);
      continue;
    }
    sk[k] = make_double2((double)((r1 * r2 + i1 * i2) / den), (double)((i1 * r2 - r1 * i2) / den));
    il2[k] = make_double2((double)(r2 / den), (double)(-i2 / den));
  }
  put(L.lam1, l1.data(), (H + 1) * 16); put(L.lam2, l2.data(), (H + 1) * 16);
  put(L.sk, sk.data(), (H + 1) * 16); put(L.il2, il2.data(), (H + 1) * 16);
  if (c->dim == 1 && c->toeplitz) {
    // K3 Toeplitz chunk tables (k_tridiag.cu): forward pivots and backward spike coefficients of a
    // chunk of Lc = Lmin or Lmin+1 rows of (s_k I − Ã)/1 with a = −τ lo, c = −τ up, b = s_k − τ di.
    const TriCfg t = tri_cfg(c->nx, 1);
    if (!t.small) {
      typedef std::complex<long double> cld;
      const int Lt = t.L, st = t.tabstride;
      std::vector<double2> tab((size_t)(H + 1) * st, make_double2(0.0, 0.0));
      const long double tau = (long double)c->tau_p;  // preconditioner τ (d̄τ for 𝓛(t) = d(t)𝓛)
      const long double a = -tau * (long double)op->xs, cc = -tau * (long double)op->xu;
      std::vector<cld> inv(Lt), al(Lt), ga(Lt), ap(Lt), gp(Lt);
      auto d2 = [](cld z) { return make_double2((double)z.real(), (double)z.imag()); };
      for (int k = 0; k <= H; ++k) {
        long double th = 2.0L * PI * (long double)k / (long double)N;
        long double sh = sinl(0.5L * th), sn = sinl(th), cs = cosl(th);
        if (2 * k == N) { sh = 1.0L; sn = 0.0L; cs = -1.0L; }
        if (c->debug & 2) sn = -sn;
        const cld l1(one_m_a + 2.0L * a_ld * sh * sh, a_ld * sn), l2(0.5L * (1.0L + a_ld * cs), -0.5L * a_ld * sn);
        if (std::norm(l2) == 0.0L) continue;  // diagonal-only system (α = 1, k = N/2): no table
        const cld b = l1 / l2 - cld(tau * (long double)op->xd, 0.0L);
        double2* tb = tab.data() + (size_t)k * st;
        for (int j = 1; j < Lt; ++j) {
          const cld piv = (j == 1) ? b : b - a * ga[j - 1];
          inv[j] = 1.0L / piv;
          ga[j] = cc * inv[j];
          al[j] = (j == 1) ? a * inv[j] : -a * al[j - 1] * inv[j];
          tb[j] = d2(inv[j]);
        }
        struct SegC { cld fa, fb, fc, ga, gb, gc; };
        SegC chunk[2];
        for (int v = 0; v < 2; ++v) {
          const int Lc = t.Lmin + v;
          if (Lc < 2 || Lc > Lt) continue;
          double2* tv = tb + Lt + v * (2 * Lt + 3);
          cld fb, fc;
          if (Lc >= 3) {
            ap[Lc - 2] = al[Lc - 2];
            gp[Lc - 2] = ga[Lc - 2];
            for (int j = Lc - 3; j >= 1; --j) {
              ap[j] = al[j] - ga[j] * ap[j + 1];
              gp[j] = -ga[j] * gp[j + 1];
            }
            for (int j = 1; j <= Lc - 2; ++j) { tv[3 + j] = d2(ap[j]); tv[3 + Lt + j] = d2(gp[j]); }
            fb = b - cc * ap[1];
            fc = -cc * gp[1];
          } else {
            fb = b;
            fc = cld(cc, 0.0L);
          }
          tv[0] = d2(al[Lc - 1]);
          tv[1] = d2(fb);
          tv[2] = d2(fc);
          chunk[v] = SegC{cld(a, 0.0L), fb, fc, al[Lc - 1], cld(1.0L, 0.0L), ga[Lc - 1]};
        }
        if (t.fast) {
          // fast tree (k_tridiag.cu MODE_FAST): standard segments S (chunks of Ls rows) and the
          // last segment Z (its last chunk has Lmin rows) merged level by level.
          const int P = 32 * t.G;
          const int nlong = c->nx - P * t.Lmin;
          SegC S = chunk[nlong ? 1 : 0], Z = chunk[0];
          double2* tt = tb + 5 * Lt + 6;
          auto merge = [&](const SegC& A, const SegC& B, double2* cf) {
            const cld det = A.gb * B.fb - A.gc * B.fa;
            const cld id = 1.0L / det;
            const cld P1 = -B.fb * A.ga * id, P2 = A.gc * B.fc * id;
            const cld R1 = B.fa * A.ga * id, R2 = -A.gb * B.fc * id;
            cf[0] = d2(B.fb * id); cf[1] = d2(-A.gc * id);   // P0 = pa gd_A + pb fd_B
            cf[2] = d2(A.gb * id); cf[3] = d2(-B.fa * id);   // R0 = ra fd_B + rb gd_A
            cf[4] = d2(P1); cf[5] = d2(P2); cf[6] = d2(R1); cf[7] = d2(R2);
            cf[8] = d2(A.fc); cf[9] = d2(B.ga);
            return SegC{A.fa, A.fb + A.fc * P1, A.fc * P2, B.ga * R1, B.gb + B.ga * R2, B.gc};
          };
          for (int q = 0; q < t.nlv; ++q) {
            const SegC S2 = merge(S, S, tt + (2 * q) * 10);
            const SegC Z2 = merge(S, Z, tt + (2 * q + 1) * 10);
            S = S2;
            Z = Z2;
          }
          const cld det = Z.fb * Z.gb - Z.fc * Z.ga;
          const cld id = 1.0L / det;
          double2* r = tt + t.nlv * 20;
          r[0] = d2(Z.gb * id); r[1] = d2(-Z.fc * id);
          r[2] = d2(-Z.ga * id); r[3] = d2(Z.fb * id);
        }
      }
      put(L.tri, tab.data(), tab.size() * 16);
    }
  }
  if (c->dim == 2) {
    long double emax[2] = {0.0L, 0.0L};
    int axis_i = 0;
    auto axis = [&](int n, double s, double d, double u, size_t offi, size_t offd, size_t offe, size_t offtw,
                    int64_t elen) {
      std::vector<double> Di(n), Dd(n), e(elen, 0.0);
      // D⁻¹ tridiag(s, d, u) D with D = diag(ρ^j), ρ = √(s/u) is the symmetric Toeplitz
      // tridiag(σ, d, σ), σ = sgn(s)·√(su) (s·u > 0): eigenvalues d + 2σ cos(jπ/(n+1)), DST-I modes
      long double rho = sqrtl((long double)s / (long double)u);
      long double sq = (s < 0.0 ? -1.0L : 1.0L) * sqrtl((long double)s * (long double)u);
      for (int j = 1; j <= n; ++j) {
        Di[j - 1] = (double)powl(rho, -(long double)j);
        Dd[j - 1] = (double)(powl(rho, (long double)j) * 2.0L / (long double)(n + 1));
        e[j - 1] = (double)((long double)d + 2.0L * sq * cosl(PI * (long double)j / (long double)(n + 1)));
        if (j == 1 || (long double)e[j - 1] > emax[axis_i]) emax[axis_i] = (long double)e[j - 1];
      }
      ++axis_i;
      std::vector<double2> t2(2 * (n + 1));
      for (int q = 0; q < 2 * (n + 1); ++q) {
        long double th = PI * (long double)q / (long double)(n + 1);
        t2[q] = make_double2((double)cosl(th), (double)(-sinl(th)));
      }
      put(offi, Di.data(), n * 8); put(offd, Dd.data(), n * 8); put(offe, e.data(), elen * 8);
      put(offtw, t2.data(), 2 * (n + 1) * 16);
    };
    axis(c->nx, op->xs, op->xd, op->xu, L.dxi, L.dx, L.ex, L.twx, c->ld);
    axis(c->ny, op->ys, op->yd, op->yu, L.dyi, L.dy, L.ey, L.twy, c->ny);
    c->mu_max = (double)((long double)c->tau_p * (emax[0] + emax[1] + (long double)c->shift));
  }
}

// P_α⁻¹ on device.  in/out may coincide only for 2D (in is consumed by the first pass).
cnpint_status pinv_dev(cnpint_ctx* c, const double* in, const double* vscale, double* out, int accumulate) {
  if (c->dim == 1) {
    CK(launch_time_fft(c, in, vscale, c->d_spec));
    CK(launch_shifted_solve(c, c->d_spec, c->d_spec));
    CK(launch_time_ifft(c, c->d_spec, out, accumulate));
  } else {
    // W⁻¹ (x then y), fused time pass, W (y then x)
    double* a = (in == c->d_tmp1 || out == c->d_tmp1) ? c->d_io2 : c->d_tmp1;
    double* b = (in == c->d_tmp2 || out == c->d_tmp2) ? c->d_io2 : c->d_tmp2;
    if (a == b) b = c->d_io1;
    if (c->debug & 32768) {
      // three HBM passes: W⁻¹ fused over both axes, the time pass, W fused (k_dstxy.cu; the scratch
      // intermediate tmp3 stays in L2).  Opt-in: it moves 48 instead of 80 B per unknown but measured
      // 3-6 % slower than the five passes below (profiles/r02_dstxy_ab.txt): both are bound on chip.
      cnp_prof_begin(c, KID_DST_XY);
      cudaError_t e = launch_dstxy(c, in, b, 0, 0);
      cnp_prof_end(c, KID_DST_XY, 16.0 * cnp_units(c));
      if (e == cudaSuccess) {
        CK(launch_time_pass_2d(c, b, a, vscale));  // GMRES scale folded into the Γ-scaling
        cnp_prof_begin(c, KID_DST_XY);
        e = launch_dstxy(c, a, out, 1, accumulate);
        cnp_prof_end(c, KID_DST_XY, (accumulate ? 24.0 : 16.0) * cnp_units(c));
        CK(e);
        return CNPINT_OK;
      }
      if (e != cudaErrorNotSupported) return cuda_fail(c, e, "launch_dstxy");
      (void)cudaGetLastError();
    }
    // the first pass may already be done: the Gram update that wrote `in` also wrote its x pass into tmp1
    const bool have_x = c->xdst_src == in && a == c->d_tmp1;
    c->xdst_src = nullptr;
    if (!have_x) CK(launch_dst_x(c, in, a, nullptr, 0));
    CK(launch_dst_y(c, a, b, 0));
    CK(launch_time_pass_2d(c, b, a, vscale));  // GMRES scale folded into the Γ-scaling
    CK(launch_dst_y(c, a, b, 1));
    if (accumulate) CK(launch_dst_x_acc(c, b, out));
    else CK(launch_dst_x(c, b, out, nullptr, 1));
  }
  return CNPINT_OK;
}

cnpint_status check_vec(cnpint_ctx* c, const void* p, const char* name) {
  if (!p) { seterr(c, "%s is NULL", name); return CNPINT_EINVAL; }
  if (((uintptr_t)p) & 15) { seterr(c, "%s must be 16-byte aligned", name); return CNPINT_EINVAL; }
  return CNPINT_OK;
}

}  // namespace

// ============================================================================== C ABI
extern "C" {

size_t cnpint_workspace_bytes(int N, const cnpint_operator* op, int restart_max) {
  int uns = 0;
  if (check_op(N, op, &uns) || restart_max < 0) return 0;
  return layout(N, op, restart_max).total;
}

cnpint_status cnpint_create(cnpint_ctx** out, int N, double T, double alpha, const cnpint_operator* op,
                            int restart_max, void* d_workspace, size_t ws_bytes, void* cuda_stream) {
  if (!out) return CNPINT_EINVAL;
  *out = nullptr;
  int uns = 0;
  const char* msg = check_op(N, op, &uns);
  if (msg) return uns ? CNPINT_EUNSUPPORTED : CNPINT_EINVAL;
  if (!(T > 0.0) || !std::isfinite(T)) return CNPINT_EINVAL;
  if (!(alpha > 0.0 && alpha <= 1.0)) return CNPINT_EINVAL;  // α = 1: P₁ (NEXT #2)
  if (restart_max < 0 || restart_max > 1000) return CNPINT_EINVAL;
  Layout L = layout(N, op, restart_max);
  if (!d_workspace || ws_bytes < L.total || ((uintptr_t)d_workspace & (ALIGN - 1))) return CNPINT_EINVAL;
  if (alpha == 1.0 && (op->dim == 2 || op->toeplitz)) {
    // P₁ is singular iff Ã is (Remark 3.2): λ1 = 0 at k = 0 leaves −λ2Ã.  Closed-form
    // spectrum of the Toeplitz (Kronecker-sum) operator: μ = d + 2 sgn(s)√(su) cos(jπ/(n+1)).
    auto eig = [](double s, double d, double u, int n, int j) {
      const double r = s * u > 0.0 ? std::sqrt(s * u) * (s > 0.0 ? 1.0 : -1.0) : 0.0;
      return d + 2.0 * r * std::cos(M_PI * j / (n + 1.0));
    };
    double mn = HUGE_VAL, mx = 0.0;
    if (op->dim == 1) {
      if (op->xs * op->xu > 0.0)
        for (int j = 1; j <= op->nx; ++j) {
          const double e = std::fabs(eig(op->xs, op->xd, op->xu, op->nx, j));
          mn = std::min(mn, e); mx = std::max(mx, e);
        }
    } else {
      for (int j = 1; j <= op->ny; ++j)
        for (int i = 1; i <= op->nx; ++i) {
          const double e = std::fabs(eig(op->xs, op->xd, op->xu, op->nx, i) + eig(op->ys, op->yd, op->yu, op->ny, j) +
                                     op->shift);
          mn = std::min(mn, e); mx = std::max(mx, e);
        }
    }
    if (mx > 0.0 && mn <= 1e-13 * mx) return CNPINT_ESINGULAR;
  }
  if (op->dim == 1 && !op->toeplitz) {
    for (int i = 0; i < op->nx; ++i)
      if (!std::isfinite(op->sub[i]) || !std::isfinite(op->diag[i]) || !std::isfinite(op->sup[i])) return CNPINT_EINVAL;
    if (alpha == 1.0) {
      // P₁ is singular iff Ã is (Remark 3.2): Gaussian elimination of the variable-row
      // L_h in long double; a pivot that cancels below 1e-13 of its terms means singular to working
      // precision (the partitioned device elimination need not produce an exact zero for it)
      long double cp = 0.0L;
      for (int i = 0; i < op->nx; ++i) {
        const long double a = i ? op->sub[i] : 0.0L, c = i < op->nx - 1 ? op->sup[i] : 0.0L;
        const long double t = i ? a * cp : 0.0L;
        const long double piv = (long double)op->diag[i] - t;
        if (fabsl(piv) <= 1e-13L * (fabsl((long double)op->diag[i]) + fabsl(t))) return CNPINT_ESINGULAR;
        cp = c / piv;
      }
    }
  } else {
    double v[7] = {op->xs, op->xd, op->xu, op->ys, op->yd, op->yu, op->shift};
    for (double x : v)
      if (!std::isfinite(x)) return CNPINT_EINVAL;
  }
  cnpint_ctx* c = new (std::nothrow) cnpint_ctx;
  if (!c) return CNPINT_EINVAL;
  std::memset(c, 0, sizeof(*c));
  { const char* e = getenv("CNPINT_PDL"); c->pdl = (e && atoi(e) == 0) ? 0 : 1; }
  { const char* e = getenv("CNPINT_L2PF"); c->l2pf = (e && atoi(e) == 0) ? 0 : 1; }
  c->dim = op->dim; c->nx = op->nx; c->ny = op->dim == 2 ? op->ny : 1; c->N = N; c->H = N / 2;
  c->toeplitz = op->dim == 2 ? 1 : op->toeplitz;
  c->ld = ld_of(op->nx); c->slice = (int64_t)c->ny * c->ld; c->vec = (int64_t)N * c->slice;
  c->spec_rows = c->H + 1; c->spec_elems = c->spec_rows * c->slice;
  c->T = T; c->tau = T / N; c->tau_p = T / N; c->d_dt = nullptr; c->alpha = alpha; c->lnalpha = std::log(alpha); c->a = std::exp(c->lnalpha / N);
  c->xs = op->xs; c->xd = op->xd; c->xu = op->xu; c->ys = op->ys; c->yd = op->yd; c->yu = op->yu;
  c->shift = op->dim == 2 ? op->shift : 0.0;
  c->restart_max = restart_max;
  c->stream = (cudaStream_t)cuda_stream;
  int dev = 0;
  cudaGetDevice(&dev);
  c->num_sms = CNP_NUM_SMS_DEFAULT;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  c->ws = (char*)d_workspace; c->ws_bytes = ws_bytes;
  char* w = c->ws;
  c->d_lo = (double*)(w + L.lo); c->d_di = (double*)(w + L.di); c->d_up = (double*)(w + L.up);
  c->d_tw = (double2*)(w + L.tw); c->d_gam = (double*)(w + L.gam); c->d_igam = (double*)(w + L.igam);
  c->d_lam1 = (double2*)(w + L.lam1); c->d_lam2 = (double2*)(w + L.lam2);
  c->d_sk = (double2*)(w + L.sk); c->d_il2 = (double2*)(w + L.il2);
  c->d_tritab = (double2*)(w + L.tri);
  c->d_vtab = L.vtab ? (double2*)(w + L.vtab) : nullptr;
  c->d_spec = (double2*)(w + L.spec);
  c->d_fsY = fstep_y_bytes(op->dim, N, c->slice) ? (double*)(w + L.fsy) : nullptr;
  c->d_fscnt = (unsigned*)(w + L.fscnt);
  c->fs_cnt = 0;
  c->fs_tick = 0;
  c->d_tmp1 = (double*)(w + L.tmp1); c->d_tmp2 = (double*)(w + L.tmp2); c->d_tmp3 = (double*)(w + L.tmp3);
  c->d_io1 = (double*)(w + L.io1); c->d_io2 = (double*)(w + L.io2); c->d_io3 = (double*)(w + L.io3);
  if (op->dim == 2) {
    c->d_dxi = (double*)(w + L.dxi); c->d_dx = (double*)(w + L.dx); c->d_dyi = (double*)(w + L.dyi);
    c->d_dy = (double*)(w + L.dy); c->d_ex = (double*)(w + L.ex); c->d_ey = (double*)(w + L.ey);
    c->d_twx = (double2*)(w + L.twx); c->d_twy = (double2*)(w + L.twy);
  }
  if (restart_max >= 1) {
    c->d_V = (double*)(w + L.V); c->d_Z = (double*)(w + L.Z); c->d_c1 = (double*)(w + L.c1); c->d_c2 = (double*)(w + L.c2);
    c->d_scl = (double*)(w + L.scl); c->d_H = (double*)(w + L.H); c->d_cs = (double*)(w + L.cs);
    c->d_sn = (double*)(w + L.sn); c->d_g = (double*)(w + L.g); c->d_y = (double*)(w + L.y);
    c->d_coef = (double*)(w + L.coef);
  }
  c->d_part = (double*)(w + L.part);
  if (restart_max >= 1) { c->d_G = (double*)(w + L.G); c->d_cg = (double*)(w + L.cg); }
  c->d_scal = (double*)(w + L.scal);
  c->d_xycnt = op->dim == 2 ? (unsigned*)(w + L.xycnt) : nullptr;
  c->d_status = (int*)(w + L.status);
  c->d_counter = (unsigned*)(w + L.status + 32);
  // tables: build a host image of the table region [0, tables_end), upload, zero the rest
  cnpint_status st = CNPINT_OK;
  {
    std::vector<char> img(L.tables_end, 0);
    make_tables(c, op, img, L);
    cudaError_t e = cudaMemcpyAsync(w, img.data(), L.tables_end, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(w + L.tables_end, 0, L.total - L.tables_end, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&c->h_pinned, 16 * sizeof(double), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&c->d_hmap, c->h_pinned, 0);
    if (e != cudaSuccess) st = cuda_fail(c, e, "cnpint_create");
  }
  if (st == CNPINT_OK) {  // K3 variable-row tables (coefficient-only part of the upper merge tree)
    cudaError_t e = build_trivar_table(c);
    if (e != cudaSuccess) st = cuda_fail(c, e, "build_trivar_table");
  }
  if (st != CNPINT_OK) {
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    delete c;
    return st;
  }
  *out = c;
  return CNPINT_OK;
}

void cnpint_destroy(cnpint_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);  // the caller may release the workspace right after this call
  prof_free(c);
  cnp_shard_free(c);
  if (c->s_in) {
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    cudaStreamDestroy(c->s_in);
    cudaStreamDestroy(c->s_out);
  }
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  delete c;
}

const char* cnpint_last_error(const cnpint_ctx* c) { return c ? c->err : "null handle"; }

cnpint_status cnpint_set_stream(cnpint_ctx* c, void* s) {
  if (!c) return CNPINT_EINVAL;
  if ((cudaStream_t)s != c->stream) {
    // the persistent four-step kernels carry per-handle counters from launch to launch, so the work
    // already enqueued on the old stream must finish before anything runs on the new one
    CK(cudaStreamSynchronize(c->stream));
    c->stream = (cudaStream_t)s;
  }
  return CNPINT_OK;
}

int64_t cnpint_ld(const cnpint_ctx* c) { return c ? c->ld : -1; }
int64_t cnpint_vec_elems(const cnpint_ctx* c) { return c ? c->vec : -1; }
int64_t cnpint_spec_elems(const cnpint_ctx* c) { return c ? c->spec_elems : -1; }
int64_t cnpint_launch_count(const cnpint_ctx* c) { return c ? c->launches : -1; }

cnpint_status cnpint_apply_A(cnpint_ctx* c, const double* u, double* y) {
  if (!c) return CNPINT_EINVAL;
  if (check_vec(c, u, "u") || check_vec(c, y, "y")) return CNPINT_EINVAL;
  if (u == y) { seterr(c, "apply_A: output aliases input"); return CNPINT_EINVAL; }
  CK(launch_matvec(c, u, y, 0, nullptr, nullptr));
  return CNPINT_OK;
}

cnpint_status cnpint_apply_P(cnpint_ctx* c, const double* z, double* v) {
  if (!c) return CNPINT_EINVAL;
  if (check_vec(c, z, "z") || check_vec(c, v, "v")) return CNPINT_EINVAL;
  if (z == v) { seterr(c, "apply_P: output aliases input"); return CNPINT_EINVAL; }
  CK(launch_matvec(c, z, v, 1, nullptr, nullptr));
  return CNPINT_OK;
}

cnpint_status cnpint_apply_Pinv(cnpint_ctx* c, const double* v, double* z) {
  if (!c) return CNPINT_EINVAL;
  if (check_vec(c, v, "v") || check_vec(c, z, "z")) return CNPINT_EINVAL;
  if (v == z) { seterr(c, "apply_Pinv: output aliases input"); return CNPINT_EINVAL; }
  return pinv_dev(c, v, nullptr, z, 0);
}

cnpint_status cnpint_time_fft(cnpint_ctx* c, const double* v, double* what) {
  if (!c) return CNPINT_EINVAL;
  if (check_vec(c, v, "v") || check_vec(c, what, "what")) return CNPINT_EINVAL;
  if (c->dim != 1) { seterr(c, "stage entry points are 1D only"); return CNPINT_EUNSUPPORTED; }
  CK(launch_time_fft(c, v, nullptr, (double2*)what));
  return CNPINT_OK;
}

cnpint_status cnpint_shifted_solve(cnpint_ctx* c, const double* what, double* zhat) {
  if (!c) return CNPINT_EINVAL;
  if (check_vec(c, what, "what") || check_vec(c, zhat, "zhat")) return CNPINT_EINVAL;
  if (c->dim != 1) { seterr(c, "stage entry points are 1D only"); return CNPINT_EUNSUPPORTED; }
  CK(launch_shifted_solve(c, (const double2*)what, (double2*)zhat));
  return CNPINT_OK;
}

cnpint_status cnpint_time_ifft(cnpint_ctx* c, const double* zhat, double* z) {
  if (!c) return CNPINT_EINVAL;
  if (check_vec(c, zhat, "zhat") || check_vec(c, z, "z")) return CNPINT_EINVAL;
  if (c->dim != 1) { seterr(c, "stage entry points are 1D only"); return CNPINT_EUNSUPPORTED; }
  CK(launch_time_ifft(c, (const double2*)zhat, z, 0));
  return CNPINT_OK;
}

cnpint_status cnpint_device_status(cnpint_ctx* c) {
  if (!c) return CNPINT_EINVAL;
  CK(launch_scal_to_host(c));  // status word via the mapped buffer (no copy-engine transfer)
  CK(cudaStreamSynchronize(c->stream));
  if (c->h_pinned[8] != 0.0) {
    CK(cudaMemsetAsync(c->d_status, 0, sizeof(int), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    seterr(c, "zero or non-finite pivot in a shifted solve (P_alpha singular to working precision)");
    return CNPINT_ESINGULAR;
  }
  return CNPINT_OK;
}

cnpint_status cnpint_profile_enable(cnpint_ctx* c, int on) {
  if (!c) return CNPINT_EINVAL;
  if (!on) {
    if (c->prof) CK(cudaStreamSynchronize(c->stream));
    prof_free(c);
    return CNPINT_OK;
  }
  if (!c->prof) c->prof = new (std::nothrow) CnpProf();
  CnpProf* p = (CnpProf*)c->prof;
  if (!p) return CNPINT_EINVAL;
  CK(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < KID_COUNT; ++k) { p->used[k] = 0; p->bytes[k] = 0.0; }
  return CNPINT_OK;
}

cnpint_status cnpint_profile_read(cnpint_ctx* c, int kid, double* ms_total, int64_t* launches, double* algo_bytes) {
  if (!c || kid < 0 || kid >= KID_COUNT) return CNPINT_EINVAL;
  CnpProf* p = (CnpProf*)c->prof;
  double ms = 0.0;
  int64_t n = 0;
  double by = 0.0;
  if (p) {
    CK(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < p->used[kid]; ++i) {
      float f = 0.f;
      CK(cudaEventElapsedTime(&f, p->ev[kid][2 * i], p->ev[kid][2 * i + 1]));
      ms += f;
    }
    n = (int64_t)p->used[kid];
    by = p->bytes[kid];
  }
  if (ms_total) *ms_total = ms;
  if (launches) *launches = n;
  if (algo_bytes) *algo_bytes = by;
  return CNPINT_OK;
}

const char* cnpint_kernel_name(int kid) { return (kid >= 0 && kid < KID_COUNT) ? KNAMES[kid] : nullptr; }

cnpint_status cnpint_stream_copy(const double* src, double* dst, size_t n, void* stream) {
  if (!src || !dst) return CNPINT_EINVAL;
  cudaError_t e = launch_stream_copy(src, dst, n, (cudaStream_t)stream);
  return e == cudaSuccess ? CNPINT_OK : CNPINT_ECUDA;
}

cnpint_status cnpint_set_time_dependence(cnpint_ctx* c, const double* d_half) {
  if (!c) return CNPINT_EINVAL;
  if (!d_half) {
    c->tau_p = c->tau;
    c->d_dt = nullptr;
  } else {
    long double sum = 0.0L;
    for (int t = 0; t < c->N; ++t) {
      if (!std::isfinite(d_half[t]) || !(d_half[t] > 0.0)) {
        seterr(c, "set_time_dependence: d(t) must be finite and positive");
        return CNPINT_EINVAL;
      }
      sum += (long double)d_half[t];
    }
    cnpint_operator op;
    std::memset(&op, 0, sizeof(op));
    op.dim = c->dim; op.nx = c->nx; op.ny = c->ny; op.toeplitz = c->toeplitz;
    Layout L = layout(c->N, &op, c->restart_max);
    double* dd = (double*)(c->ws + L.dt);
    CK(cudaMemcpyAsync(dd, d_half, (size_t)c->N * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->d_dt = dd;
    c->tau_p = (double)((long double)c->tau * (sum / (long double)c->N));  // τ·d̄
  }
  // the K3 chunk tables depend on the preconditioner's τ: rebuild them
  return cnpint_set_debug(c, c->debug);
}

cnpint_status cnpint_set_debug(cnpint_ctx* c, int flags) {
  if (!c) return CNPINT_EINVAL;
  c->debug = flags;
  // rebuild the table region with the new flags (synchronous)
  cnpint_operator op;
  std::memset(&op, 0, sizeof(op));
  op.dim = c->dim; op.nx = c->nx; op.ny = c->ny; op.toeplitz = c->toeplitz;
  op.xs = c->xs; op.xd = c->xd; op.xu = c->xu; op.ys = c->ys; op.yd = c->yd; op.yu = c->yu; op.shift = c->shift;
  // the coefficient rows precede L.tw and are not re-uploaded: placeholders for variable rows
  std::vector<double> dummy(c->dim == 1 && !c->toeplitz ? c->nx : 0, 0.0);
  if (!dummy.empty()) { op.sub = dummy.data(); op.diag = dummy.data(); op.sup = dummy.data(); }
  Layout L = layout(c->N, &op, c->restart_max);
  std::vector<char> img(L.tables_end, 0);
  make_tables(c, &op, img, L);
  // only the twiddle, λ and K3 chunk tables depend on the flags: [tw, tables_end)
  const size_t hi = L.tables_end;
  CK(cudaMemcpyAsync(c->ws + L.tw, img.data() + L.tw, hi - L.tw, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  CK(build_trivar_table(c));  // depends on s_k (debug 2) and τ
  return CNPINT_OK;
}

// ------------------------------------------------------------------------------ GMRES
static cnpint_status gmres_args(cnpint_ctx* c, const double* d_b, double* d_u, double tol, int restart, int maxit) {
  if (!c) return CNPINT_EINVAL;
  if (check_vec(c, d_b, "b") || check_vec(c, d_u, "u")) return CNPINT_EINVAL;
  if (d_b == d_u) { seterr(c, "gmres: u aliases b"); return CNPINT_EINVAL; }
  if (c->restart_max < 1) { seterr(c, "handle created with restart_max = 0"); return CNPINT_EINVAL; }
  if (!(tol > 0.0 && tol < 1.0) || restart < 1 || restart > c->restart_max || maxit < 1) {
    seterr(c, "gmres: need 0 < tol < 1, 1 <= restart <= restart_max, maxit >= 1");
    return CNPINT_EINVAL;
  }
  return CNPINT_OK;
}

// Post-fold GMRES steps (see PostOp): the reducing kernel that produces ||w||² runs them in its last
// block instead of a separate single-thread launch.
static PostOp post_cycle_start(const cnpint_ctx* c, int first) {
  PostOp p{};
  p.op = 2; p.first = first; p.rmax = c->restart_max; p.scl = c->d_scl; p.g = c->d_g; p.scal = c->d_scal;
  p.G = c->d_G;  // G̃_00 for Gram CGS2 (null without a GMRES workspace)
  p.hmap = c->d_hmap; p.status = c->d_status;
  return p;
}
static PostOp post_finalize(const cnpint_ctx* c, int j) {
  PostOp p{};
  p.op = 1; p.j = j; p.ldh = c->restart_max + 1; p.c1 = c->d_c1; p.c2 = c->d_c2; p.scl = c->d_scl; p.H = c->d_H;
  p.cs = c->d_cs; p.sn = c->d_sn; p.g = c->d_g; p.scal = c->d_scal;
  p.hmap = c->d_hmap; p.status = c->d_status;
  return p;
}
static PostOp post_gram_probe(const cnpint_ctx* c, int j) {  // op 5: see gram_probe_dev (post_op.cuh)
  PostOp p = post_finalize(c, j);
  p.op = 5; p.G = c->d_G; p.c2w = c->d_c2;
  return p;
}
static PostOp post_gram_finalize(const cnpint_ctx* c, int j) {
  PostOp p = post_finalize(c, j);
  p.op = 4; p.cg = c->d_cg; p.G = c->d_G; p.c2w = c->d_c2;
  return p;
}

// CGS2 of w (already in its basis slot) against Ṽ_0..Ṽ_{nv−1}: c1 = Ṽᵀw (unless the producer fused
// it: have_c1), c2 = Ṽᵀ(w − Ṽs²c1), w −= Ṽ s²(c1 + c2) with ||w||² fused into scal[2].
// More than CNP_MAX_DOT vectors: groups of CNP_MAX_DOT (dots, update, dots, update, norm).
static cnpint_status cgs2(cnpint_ctx* c, double* const* V, int nv, double* w, bool have_c1) {
  if (nv <= CNP_MAX_DOT) {
    if (!have_c1) CK(launch_dots(c, V, nv, w, c->d_part, c->d_c1));
    // c2 = Ṽᵀ(w − Ṽs²c1) without storing the intermediate, then w ← w − Ṽs²(c1 + c2) with ‖w‖²:
    // the same two projections (CGS2) with one write of w instead of two
    CK(launch_cgs2_pass(c, V, nv, c->d_c1, nullptr, w, c->d_part, c->d_c2, 0));
    CK(launch_cgs2_pass(c, V, nv, c->d_c1, c->d_c2, w, c->d_part, c->d_scal + 2, 1));
    return CNPINT_OK;
  }
  for (int pass = 0; pass < 2; ++pass) {
    double* cd = pass == 0 ? c->d_c1 : c->d_c2;
    for (int g0 = 0; g0 < nv; g0 += CNP_MAX_DOT) {
      int ng = nv - g0 < CNP_MAX_DOT ? nv - g0 : CNP_MAX_DOT;
      CK(launch_dots(c, V + g0, ng, w, c->d_part, cd + g0));
    }
    for (int g0 = 0; g0 < nv; g0 += CNP_MAX_DOT) {
      int ng = nv - g0 < CNP_MAX_DOT ? nv - g0 : CNP_MAX_DOT;
      // coefficients cd[g0..] with scales scl[g0..]: shift the scale pointer via a temporary swap
      double* saved = c->d_scl;
      c->d_scl = saved + g0;
      const bool last = pass == 1 && g0 + ng == nv;
      cudaError_t e = launch_update(c, V + g0, ng, cd + g0, 0, w, w, 0, last ? 1 : 0, c->d_part,
                                    last ? c->d_scal + 2 : nullptr);
      c->d_scl = saved;
      CK(e);
    }
  }
  return CNPINT_OK;
}

cnpint_status cnpint_gmres(cnpint_ctx* c, const double* d_b, double* d_u, double tol, int restart, int maxit,
                           cnpint_gmres_report* rep) {
  if (cnpint_status a = gmres_args(c, d_b, d_u, tol, restart, maxit)) return a;
  c->post = PostOp{};
  c->xdst_src = nullptr;
  auto t0 = std::chrono::steady_clock::now();
  const int64_t vec = c->vec;
  double* h = c->h_pinned;
  std::vector<double*> V(restart + 1);
  for (int i = 0; i <= restart; ++i) V[i] = c->d_V + (size_t)i * vec;
  int its = 0, cycles = 0, converged = 0;
  double est = 1.0, relres_true = 1.0;
  cnpint_status result = CNPINT_OK;
  // u needs no zero fill: the first cycle end writes u = Σ y_j z_j (b = 0 is handled below)
  CK(cudaMemsetAsync(c->d_scal, 0, 16 * sizeof(double), c->stream));
  // ||b||: first basis vector is b itself (x0 = 0 ⇒ r0 = b)
  double* b_nc = const_cast<double*>(d_b);
  V[0] = b_nc;
  c->post = post_cycle_start(c, 1);  // run by launch_norm2's folding block
  CK(launch_norm2(c, d_b, c->d_part, c->d_scal + 2));
  // no host read here: ‖b‖ (h[0]) arrives with the first Arnoldi step's scalars, where b = 0 (every
  // quantity of that step is then 0 or NaN and is discarded) and a non-finite b are handled
  std::vector<double*> Z(restart);
  for (int i = 0; i < restart; ++i) Z[i] = c->d_Z + (size_t)i * vec;
  // the latest residual estimate (relative) and the one before, for the update + x-pass fusion: it is
  // used when the next Arnoldi step is expected to run, est_next ≈ est·min(1, est/est_before) > tol
  double est_now = 1.0, est_before = -1.0;
  while (true) {
    int jdone = 0;
    bool stop_inner = false;
    bool last_skipped = false;  // the cycle's last step took its norm from the Gram matrix: no Ṽ_{jdone} written
    for (int j = 0; j < restart && !stop_inner; ++j) {
      // z_j = P_α⁻¹ v_j  (v_j = s_j Ṽ_j; the scale is folded into the Γ-scaling), kept for the update
      cnpint_status st = pinv_dev(c, V[j], c->d_scl + j, Z[j], 0);
      if (st != CNPINT_OK) return st;
      // w = 𝓜 z_j, written straight into the slot of Ṽ_{j+1}
      double* w = V[j + 1];
      const int nv = j + 1;
      if (nv <= CNP_MAX_DOT && !(c->debug & 128)) {
        // Gram CGS2: w = 𝓜 z_j with c1 = Ṽᵀw; one update w −= Ṽs²(c1 + c2) whose blocks form
        // c2 = Ṽᵀ(w − Ṽs²c1) = c1 − G̃s²c1 from the stored Gram matrix and which also reduces ‖w‖²
        // and the Gram row Ṽᵀw of the new vector (post op 4 stores it, then the Arnoldi finalize)
        // — the same two projections as classic CGS2, one reading pass fewer
        const double est_next = est_before > 0.0 ? est_now * std::min(1.0, est_now / est_before) : est_now;
        // A step expected to be the last: its new basis vector would never be used, only its norm
        // h_{j+1,j} — which the Gram matrix gives without a pass over the vectors (post op 5, run by the
        // matvec's folding block: β² = ww − 2aᵀc1 + aᵀG̃a, trusted when β² ≥ 1e-8·ww).  If the estimate
        // then meets the tolerance, the update pass is skipped; otherwise the probe is taken back and the
        // step runs as usual.  debug 2097152 turns the probe off, 4194304 probes every step (tests: the
        // take-back path).
        // The probe runs when the predicted estimate is within 10× of the tolerance (a failed probe costs one
        // stream synchronisation and a one-thread kernel; measured histories: c2 α = 0.01 predicts 2.0e-10
        // and reaches 9.6e-11).
        bool update = true;
        if (!(c->debug & 2097152) && est_before > 0.0 && (est_next <= 10.0 * tol || (c->debug & 4194304))) {
          c->post = post_gram_probe(c, j);
          CK(launch_matvec_dots(c, Z[j], w, V.data(), nv, c->d_part, c->d_c1, 1));
          CK(cudaStreamSynchronize(c->stream));
          if (h[6] != 0.0 && h[1] <= tol && h[3] == 0.0 && h[5] == 0.0 && h[8] == 0.0) {
            last_skipped = true;
            update = false;
          } else if (h[6] != 0.0) {
            CK(launch_small(c, 3, j, 0));
          }
        } else {
          CK(launch_matvec_dots(c, Z[j], w, V.data(), nv, c->d_part, c->d_c1));
        }
        if (update) {
          c->post = post_gram_finalize(c, j);
          if (upd_dst_ok(c) && j + 1 < restart && its + 1 < maxit && est_next > tol) {
            // 2D: the update also writes the x sine pass of Ṽ_{j+1} (the first pass of the next P⁻¹)
            CK(launch_cgs2_pass_dst(c, V.data(), nv, c->d_c1, w, c->d_part, c->d_cg, c->d_tmp1));
            c->xdst_src = w;
          } else {
            CK(launch_cgs2_pass(c, V.data(), nv, c->d_c1, c->d_c2, w, c->d_part, c->d_cg, 2));
          }
        }
      } else {
        if (nv <= CNP_MAX_DOT) {
          // w = 𝓜 z_j fused with CGS pass 1 (c1 = Ṽᵀw); classic second pass (debug bit 128)
          CK(launch_matvec_dots(c, Z[j], w, V.data(), nv, c->d_part, c->d_c1));
        } else {
          CK(launch_matvec(c, Z[j], w, 0, nullptr, nullptr));
        }
        if (nv <= CNP_MAX_DOT) c->post = post_finalize(c, j);  // run by CGS2's last (norm) pass
        if (cnpint_status cs = cgs2(c, V.data(), nv, w, nv <= CNP_MAX_DOT)) return cs;
        if (nv > CNP_MAX_DOT) CK(launch_small(c, 1, j, 0));
      }
      if (nv > CNP_MAX_DOT) CK(launch_scal_to_host(c));  // else the finalize post op wrote them
      CK(cudaStreamSynchronize(c->stream));
      if (its == 0 && cycles == 0) {  // ‖b‖ of the cycle start
        if (h[0] == 0.0) {  // b = 0 ⇒ u = 0
          CK(cudaMemsetAsync(d_u, 0, vec * sizeof(double), c->stream));
          CK(cudaStreamSynchronize(c->stream));
          if (rep) { rep->iterations = 0; rep->restarts = 0; rep->converged = 1; rep->relres_est = 0; rep->relres_true = 0; }
          return CNPINT_OK;
        }
        if (!std::isfinite(h[0])) {
          if (cnpint_status ds = cnpint_device_status(c)) return ds;
          seterr(c, "gmres: ||b|| not finite");
          return CNPINT_EBREAKDOWN;
        }
      }
      ++its;
      jdone = j + 1;
      est = h[1];
      est_before = est_now;
      est_now = est;
      if (rep && rep->history && its - 1 < rep->history_cap) rep->history[its - 1] = est;
      if (h[8] != 0.0) {  // the step's P⁻¹ met a singular shifted system: stop now (status word read back)
        cnpint_status ds = cnpint_device_status(c);
        return ds != CNPINT_OK ? ds : CNPINT_ESINGULAR;
      }
      if (h[3] != 0.0) {
        // a singular shifted solve (zero / non-finite pivot, e.g. P_1 with a singular variable-row Ã)
        // poisons P⁻¹ first: report it as such (and clear the status word) before calling it breakdown
        if (cnpint_status ds = cnpint_device_status(c)) return ds;
        seterr(c, "gmres: non-finite scalar in the Arnoldi process");
        return CNPINT_EBREAKDOWN;
      }
      if (est <= tol || its >= maxit || h[5] != 0.0) stop_inner = true;
    }
    // cycle end: y = H⁻¹g, u += Σ y_j z_j  (= P⁻¹ V y: the stored z_j make the extra P⁻¹ unnecessary)
    c->xdst_src = nullptr;  // a speculative x pass of the last Ṽ_{j+1} is not used
    if (jdone <= CNP_MAX_DOT) {  // back-substitution inside the combine kernel
      CK(launch_combine_backsolve(c, Z.data(), jdone, 0, cycles == 0 ? nullptr : d_u, d_u));
    } else {
      CK(launch_small(c, 2, jdone, 0));
      for (int g0 = 0; g0 < jdone; g0 += CNP_MAX_DOT) {
        int ng = jdone - g0 < CNP_MAX_DOT ? jdone - g0 : CNP_MAX_DOT;
        const bool fresh = cycles == 0 && g0 == 0;  // u = Σ y_j z_j (no read of an initial zero u)
        CK(launch_update(c, Z.data() + g0, ng, c->d_y + g0, 1, fresh ? nullptr : d_u, d_u, 0, 0, c->d_part, nullptr));
      }
    }
    c->last_v0 = V[0];     // cnpint_krylov_basis (test hook): this cycle's basis
    c->last_nv = last_skipped ? jdone : jdone + 1;
    // true residual ‖b − 𝓜u‖: when the estimate says converged only its norm is needed (mode 3, no
    // store); otherwise r is written into the workspace slot of Ṽ_0 for the next cycle (b is kept)
    V[0] = c->d_V;
    const bool likely_done = est <= tol;
    c->post = post_cycle_start(c, 0);  // run by the residual matvec's folding block
    CK(launch_matvec(c, d_u, V[0], likely_done ? 3 : 2, d_b, c->d_part, c->d_scal + 2));  // post op writes h
    CK(cudaStreamSynchronize(c->stream));
    relres_true = h[4];
    ++cycles;
    if (relres_true <= tol) { converged = 1; break; }
    if (likely_done) {  // estimate and true residual disagree: form r for the restart after all
      c->post = post_cycle_start(c, 0);
      CK(launch_matvec(c, d_u, V[0], 2, d_b, c->d_part, c->d_scal + 2));
    }
    if (its >= maxit) { result = CNPINT_ENOCONV; break; }
    if (!std::isfinite(relres_true)) { seterr(c, "gmres: residual not finite"); result = CNPINT_EBREAKDOWN; break; }
  }
  cnpint_status dst = cnpint_device_status(c);
  auto t1 = std::chrono::steady_clock::now();
  if (rep) {
    rep->iterations = its;
    rep->restarts = cycles - 1;
    rep->converged = converged;
    rep->relres_est = est;
    rep->relres_true = relres_true;
    rep->seconds = std::chrono::duration<double>(t1 - t0).count();
  }
  if (dst != CNPINT_OK) return dst;
  if (result == CNPINT_ENOCONV) seterr(c, "gmres: maxit reached (relres %.3e > tol %.3e)", relres_true, tol);
  return result;
}

// Left preconditioning (NEXT #4).  scal[0] = ||P⁻¹b|| (the r_0 norm the estimates
// are relative to), scal[6] = ||b − 𝓜u||² of the last cycle end, scal[7] = ||b||².
cnpint_status cnpint_gmres_left(cnpint_ctx* c, const double* d_b, double* d_u, double tol, int restart, int maxit,
                                cnpint_gmres_report* rep) {
  if (cnpint_status a = gmres_args(c, d_b, d_u, tol, restart, maxit)) return a;
  c->post = PostOp{};
  auto t0 = std::chrono::steady_clock::now();
  const int64_t vec = c->vec;
  double* h = c->h_pinned;
  std::vector<double*> V(restart + 1);
  for (int i = 0; i <= restart; ++i) V[i] = c->d_V + (size_t)i * vec;
  double* tmp = c->d_Z;  // 𝓜v_j and b − 𝓜u (the preconditioned-direction slots are unused here)
  int its = 0, cycles = 0, converged = 0;
  double est = 1.0, relres_true = 1.0, relres_prec = 1.0;
  cnpint_status result = CNPINT_OK;
  CK(cudaMemsetAsync(c->d_scal, 0, 16 * sizeof(double), c->stream));
  CK(launch_norm2(c, d_b, c->d_part, c->d_scal + 7));
  // r_0 = P⁻¹b (x0 = 0), β = ||r_0||
  if (cnpint_status st = pinv_dev(c, d_b, nullptr, V[0], 0)) return st;
  c->post = post_cycle_start(c, 1);
  CK(launch_norm2(c, V[0], c->d_part, c->d_scal + 2));
  CK(launch_scal_to_host(c));
  CK(cudaStreamSynchronize(c->stream));
  const double bnorm = std::sqrt(h[7]);
  if (h[7] == 0.0) {  // b = 0 ⇒ u = 0
    CK(cudaMemsetAsync(d_u, 0, vec * sizeof(double), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (rep) {
      rep->iterations = 0; rep->restarts = 0; rep->converged = 1;
      rep->relres_est = 0; rep->relres_true = 0; rep->relres_prec = 0;
    }
    return CNPINT_OK;
  }
  if (!std::isfinite(h[0]) || !std::isfinite(bnorm) || h[0] == 0.0) {
    if (cnpint_status dst = cnpint_device_status(c)) return dst;
    seterr(c, "gmres_left: ||P^-1 b|| = %g (b != 0)", h[0]);
    return CNPINT_EBREAKDOWN;
  }
  while (true) {
    int jdone = 0;
    bool stop_inner = false;
    for (int j = 0; j < restart && !stop_inner; ++j) {
      // w = P⁻¹(𝓜 v_j), v_j = s_j Ṽ_j: 𝓜Ṽ_j, then s_j folded into the Γ-scaling of P⁻¹
      CK(launch_matvec(c, V[j], tmp, 0, nullptr, nullptr));
      double* w = V[j + 1];
      if (cnpint_status st = pinv_dev(c, tmp, c->d_scl + j, w, 0)) return st;
      if (j + 1 <= CNP_MAX_DOT) c->post = post_finalize(c, j);
      if (cnpint_status cs = cgs2(c, V.data(), j + 1, w, false)) return cs;
      if (j + 1 > CNP_MAX_DOT) CK(launch_small(c, 1, j, 0));
      CK(launch_scal_to_host(c));
      CK(cudaStreamSynchronize(c->stream));
      ++its;
      jdone = j + 1;
      est = h[1];
      if (rep && rep->history && its - 1 < rep->history_cap) rep->history[its - 1] = est;
      if (h[8] != 0.0) {  // singular shifted system in this step's P⁻¹ (see cnpint_gmres)
        cnpint_status ds = cnpint_device_status(c);
        return ds != CNPINT_OK ? ds : CNPINT_ESINGULAR;
      }
      if (h[3] != 0.0) {
        if (cnpint_status ds = cnpint_device_status(c)) return ds;  // singular pivot first (see cnpint_gmres)
        seterr(c, "gmres_left: non-finite scalar in the Arnoldi process");
        return CNPINT_EBREAKDOWN;
      }
      if (est <= tol || its >= maxit || h[5] != 0.0) stop_inner = true;
    }
    // cycle end: y = H⁻¹g, u += V y = Σ (y_i s_i) Ṽ_i  (no P⁻¹ with left preconditioning)
    if (jdone <= CNP_MAX_DOT) {  // back-substitution inside the combine kernel (coef = y s)
      CK(launch_combine_backsolve(c, V.data(), jdone, 1, cycles == 0 ? nullptr : d_u, d_u));
    } else {
      CK(launch_small(c, 2, jdone, 0));
      for (int g0 = 0; g0 < jdone; g0 += CNP_MAX_DOT) {
        int ng = jdone - g0 < CNP_MAX_DOT ? jdone - g0 : CNP_MAX_DOT;
        const bool fresh = cycles == 0 && g0 == 0;
        CK(launch_update(c, V.data() + g0, ng, c->d_coef + g0, 1, fresh ? nullptr : d_u, d_u, 0, 0, c->d_part,
                         nullptr));
      }
    }
    // b − 𝓜u (its norm²: the unpreconditioned residual), r = P⁻¹(b − 𝓜u) → Ṽ_0 of the next cycle
    CK(launch_matvec(c, d_u, tmp, 2, d_b, c->d_part, c->d_scal + 6));
    if (cnpint_status st = pinv_dev(c, tmp, nullptr, V[0], 0)) return st;
    c->post = post_cycle_start(c, 0);
    CK(launch_norm2(c, V[0], c->d_part, c->d_scal + 2));
    CK(launch_scal_to_host(c));
    CK(cudaStreamSynchronize(c->stream));
    relres_prec = h[4];
    relres_true = std::sqrt(h[6]) / bnorm;
    ++cycles;
    if (relres_prec <= tol) { converged = 1; break; }
    if (its >= maxit) { result = CNPINT_ENOCONV; break; }
    if (!std::isfinite(relres_prec)) { seterr(c, "gmres_left: residual not finite"); result = CNPINT_EBREAKDOWN; break; }
  }
  cnpint_status dst = cnpint_device_status(c);
  auto t1 = std::chrono::steady_clock::now();
  if (rep) {
    rep->iterations = its;
    rep->restarts = cycles - 1;
    rep->converged = converged;
    rep->relres_est = est;
    rep->relres_true = relres_true;
    rep->relres_prec = relres_prec;
    rep->seconds = std::chrono::duration<double>(t1 - t0).count();
  }
  if (dst != CNPINT_OK) return dst;
  if (result == CNPINT_ENOCONV)
    seterr(c, "gmres_left: maxit reached (preconditioned relres %.3e > tol %.3e)", relres_prec, tol);
  return result;
}

cnpint_status cnpint_krylov_basis(cnpint_ctx* c, int i, const double** d_vec, double* scale, int* count) {
  if (!c) return CNPINT_EINVAL;
  if (count) *count = c->last_nv;
  if (i < 0 || i >= c->last_nv || !c->last_v0) { seterr(c, "krylov_basis: no such vector"); return CNPINT_EINVAL; }
  if (d_vec) *d_vec = i == 0 ? c->last_v0 : c->d_V + (size_t)i * c->vec;
  if (scale) {
    // s_0 was replaced by the cycle-end residual's cycle start, which saved it in scal[12]
    const double* src = i == 0 ? c->d_scal + 12 : c->d_scl + i;
    CK(cudaMemcpyAsync(scale, src, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return CNPINT_OK;
}

// ------------------------------------------------------------------------------ host variants
// Host ↔ device: one contiguous copy of the packed host array into / out of a device staging vector,
// and an on-device repack to / from the padded layout (a pitched 2D DMA copy of short rows is much
// slower over PCIe than one linear transfer).
static cnpint_status h2d_vec(cnpint_ctx* c, const double* h, double* d, double* stage) {
  const size_t rows = (size_t)c->N * c->ny;
  CK(cudaMemcpyAsync(stage, h, rows * c->nx * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(launch_repack(c, stage, d, 0));
  return CNPINT_OK;
}
static cnpint_status d2h_vec(cnpint_ctx* c, const double* d, double* h, double* stage) {
  const size_t rows = (size_t)c->N * c->ny;
  CK(launch_repack(c, d, stage, 1));
  CK(cudaMemcpyAsync(h, stage, rows * c->nx * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  return CNPINT_OK;
}

cnpint_status cnpint_apply_Pinv_host(cnpint_ctx* c, const double* h_v, double* h_z) {
  if (!c || !h_v || !h_z) return CNPINT_EINVAL;
  cnpint_status st;
  if ((st = h2d_vec(c, h_v, c->d_io1, c->d_io3))) return st;
  if ((st = pinv_dev(c, c->d_io1, nullptr, c->d_io2, 0))) return st;
  if ((st = d2h_vec(c, c->d_io2, h_z, c->d_io3))) return st;
  CK(cudaStreamSynchronize(c->stream));
  return CNPINT_OK;
}

cnpint_status cnpint_apply_A_host(cnpint_ctx* c, const double* h_u, double* h_y) {
  if (!c || !h_u || !h_y) return CNPINT_EINVAL;
  cnpint_status st;
  if ((st = h2d_vec(c, h_u, c->d_io1, c->d_io3))) return st;
  CK(launch_matvec(c, c->d_io1, c->d_io2, 0, nullptr, nullptr));
  if ((st = d2h_vec(c, c->d_io2, h_y, c->d_io3))) return st;
  CK(cudaStreamSynchronize(c->stream));
  return CNPINT_OK;
}

// Pipelined end-to-end solves: solve i on the handle's stream while the H2D copy of b_{i+1} (stream
// s_in) and the D2H copy of u_{i−1} (stream s_out) move over PCIe in both directions.  Staging: d_stage
// holds stage_in[2] and stage_out[2] (packed layout); b and u live in io2 / io3 as in cnpint_gmres_host.
cnpint_status cnpint_gmres_host_batch(cnpint_ctx* c, int count, const double* const* h_b, double* const* h_u,
                                      double tol, int restart, int maxit, double* d_stage, cnpint_gmres_report* reps) {
  if (!c || count < 1 || !h_b || !h_u || !d_stage || ((uintptr_t)d_stage & 15)) return CNPINT_EINVAL;
  for (int i = 0; i < count; ++i)
    if (!h_b[i] || !h_u[i]) return CNPINT_EINVAL;
  if (!c->s_in) {
    CK(cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
    for (cudaEvent_t& e : c->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t* ev_in = c->ev;
  cudaEvent_t* ev_rep = c->ev + 2;
  cudaEvent_t* ev_ready = c->ev + 4;
  cudaEvent_t* ev_done = c->ev + 6;
  const size_t bytes = (size_t)c->N * c->ny * c->nx * sizeof(double);
  double* stage_in[2] = {d_stage, d_stage + c->vec};
  double* stage_out[2] = {d_stage + 2 * c->vec, d_stage + 3 * c->vec};
  double* db = c->d_io2;
  double* du = c->d_io3;
  auto h2d = [&](int i) -> cnpint_status {
    const int s = i & 1;
    if (i >= 2) CK(cudaStreamWaitEvent(c->s_in, ev_rep[s], 0));  // stage_in[s] consumed by solve i − 2
    CK(cudaMemcpyAsync(stage_in[s], h_b[i], bytes, cudaMemcpyHostToDevice, c->s_in));
    CK(cudaEventRecord(ev_in[s], c->s_in));
    return CNPINT_OK;
  };
  cnpint_status first_err = CNPINT_OK;
  if (cnpint_status st = h2d(0)) return st;
  if (count > 1)
    if (cnpint_status st = h2d(1)) return st;
  for (int i = 0; i < count; ++i) {
    const int s = i & 1;
    CK(cudaStreamWaitEvent(c->stream, ev_in[s], 0));
    CK(launch_repack(c, stage_in[s], db, 0));
    CK(cudaEventRecord(ev_rep[s], c->stream));
    if (i + 2 < count)
      if (cnpint_status st = h2d(i + 2)) return st;
    cnpint_status st = cnpint_gmres(c, db, du, tol, restart, maxit, reps ? reps + i : nullptr);
    if (st != CNPINT_OK && st != CNPINT_ENOCONV) return st;
    if (st != CNPINT_OK && first_err == CNPINT_OK) first_err = st;
    if (i >= 2) CK(cudaStreamWaitEvent(c->stream, ev_done[s], 0));  // stage_out[s] copied out by solve i − 2
    CK(launch_repack(c, du, stage_out[s], 1));
    CK(cudaEventRecord(ev_ready[s], c->stream));
    CK(cudaStreamWaitEvent(c->s_out, ev_ready[s], 0));
    CK(cudaMemcpyAsync(h_u[i], stage_out[s], bytes, cudaMemcpyDeviceToHost, c->s_out));
    CK(cudaEventRecord(ev_done[s], c->s_out));
  }
  CK(cudaStreamSynchronize(c->s_out));
  CK(cudaStreamSynchronize(c->stream));
  return first_err;
}

cnpint_status cnpint_gmres_host(cnpint_ctx* c, const double* h_b, double* h_u, double tol, int restart, int maxit,
                                cnpint_gmres_report* rep) {
  if (!c || !h_b || !h_u) return CNPINT_EINVAL;
  // GMRES uses tmp1/tmp2 (1D) or tmp1-3 + io1 (2D) internally; b and u live in io2 / io3.
  double* db = c->d_io2;
  double* du = c->d_io3;
  cnpint_status st = h2d_vec(c, h_b, db, c->d_io1);
  if (st) return st;
  st = cnpint_gmres(c, db, du, tol, restart, maxit, rep);
  if (st != CNPINT_OK && st != CNPINT_ENOCONV) return st;
  cnpint_status st2 = d2h_vec(c, du, h_u, c->d_io1);
  if (st2) return st2;
  CK(cudaStreamSynchronize(c->stream));
  return st;
}

}  // extern "C"
