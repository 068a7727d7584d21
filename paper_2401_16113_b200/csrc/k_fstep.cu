// Four-step time FFTs of the 1D P_α⁻¹ for long horizons (N >= 2048): K2 (MODE 0) and K4 (MODE 1)
// of PAPER.md:296-323 (Eq. 3.2 steps (a) and (c), Remark 3.1), same definitions as k_tfft.cu:
//   K2  ŵ_k[x] = Σ_t e^{−2πikt/N} · γ_t · s · v_t[x],  k = 0..N/2
//   K4  z_t[x] = 1/(N γ_t) · Σ_{k<N} e^{+2πikt/N} ẑ_k[x],  ẑ_{N−k} = conj ẑ_k
//
// Why another decomposition.  The cluster kernel keeps all N rows of a column tile on chip, so at
// N = 4096 a tile is only 8 real columns wide (64-B row segments) and its loads run at ~2 TB/s
// (profiles/r01_tilecopy_pattern.txt, r01_tfft_phases.txt).  Here N = N1·N2, t = t1 + N1 t2,
// k = k2 + N2 k1 and
//   pass A  Y[t1][k2] = ω_N^{t1 k2} · FFT_{N2}( γ_t s v_{t1 + N1 t2} )[k2]            (per t1)
//   pass B  X[k2 + N2 k1] = FFT_{N1}( Y[·][k2] )[k1]                                 (per k2)
// (inverse: the same two passes backwards with conjugate twiddles).  Each pass moves tiles of
// 2·NC = 64 real columns (512-B row segments).  The intermediate Y of a column block (2 MB at
// c2) goes through L2 only: both passes run in ONE persistent kernel whose work items are handed
// out in ticket order — the A items of block b, then (L blocks later) the B items of block b — and
// a B item waits on a per-block counter until all A items of its block have landed.  A B item is
// the sole reader of its Y rows and drops them from L2 afterwards (discard.global.L2), so Y is
// never written back to HBM: HBM traffic is one read of the input and one write of the output.
// Deadlock freedom: a B item only waits for items with smaller tickets, which were taken by CTAs
// that are already running and whose A items never wait.
// Two real columns (a, b) are packed as one complex column z_t = v_t[a] + i v_t[b]; the Hermitian
// separation X_a[k] = (Z_k + conj Z_{N−k})/2, X_b[k] = (Z_k − conj Z_{N−k})/(2i) pairs k2 with
// N2 − k2, so pass B items are frequency families {k2, N2 − k2}, k2 = 0..N2/2.
#include "common.cuh"
#include "internal.h"

#include <cstdlib>

#include "fft_tile.cuh"

#ifndef FS_NT
#define FS_NT 128
#endif
#ifndef FS_MINB
#define FS_MINB 4
#endif

namespace {

CNP_DEV void fs_separate(double2 zk, double2 zm, double2& xa, double2& xb) {
  xa = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
  xb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
}
CNP_DEV double2 fs_pack(double2 xa, double2 xb) { return make_double2(xa.x - xb.y, xa.y + xb.x); }

CNP_DEV unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CNP_DEV void discard_l2(const void* p) { asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory"); }

// compile-time geometry.  t1 items hold NC pair columns × N2 rows; family items hold NF = NC/2 pair
// columns × 2 members × N1 rows (the same shared-memory footprint when N1 = N2).
template <int LOG1, int LOG2>
struct FsGeo {
  static constexpr int N1 = 1 << LOG1, N2 = 1 << LOG2, N = N1 * N2, H = N / 2;
  static constexpr int MX = LOG1 > LOG2 ? LOG1 : LOG2;
  static constexpr int NC = MX <= 6 ? 32 : MX == 7 ? 16 : 8;
  static constexpr int NF = NC / 2;
  static constexpr int CS1 = tf_cs(LOG1), CS2 = tf_cs(LOG2);
  static constexpr int dataA = NC * CS2, dataB = 2 * NF * CS1;
  static constexpr int data = dataA > dataB ? dataA : dataB;
  static constexpr int off_stw1 = data;
  static constexpr int off_stw2 = off_stw1 + tf_stage_tw(LOG1);
  static constexpr int off_tw = off_stw2 + tf_stage_tw(LOG2);           // per-item twiddles [2·max(N1,N2)]
  static constexpr int NTW = 2 * (N1 > N2 ? N1 : N2);
  static constexpr int HI = N / 64;
  static constexpr int off_g = off_tw + NTW;                            // doubles ghi[HI], glo[64]
  static constexpr size_t bytes = (size_t)(off_g + (HI + 64) / 2 + 1) * 16;
};

}  // namespace

// Work-item order: step s = 0 .. nxb−1+L: A items of block s (s < nxb), then B items of block s−L.
struct FsSched {
  int nxb, nA, nB, L;
  unsigned total;
};

CNP_DEV void fs_item(const FsSched& S, unsigned T, int& isB, int& xb, int& idx) {
  const unsigned r1 = (unsigned)S.L * S.nA;
  const unsigned per = (unsigned)(S.nA + S.nB);
  const unsigned r2 = (unsigned)(S.nxb - S.L) * per;
  if (T < r1) {
    isB = 0; xb = T / S.nA; idx = T - xb * S.nA;
  } else if (T < r1 + r2) {
    const unsigned u = T - r1;
    const int s = S.L + u / per;
    const int r = u - (s - S.L) * per;
    if (r < S.nA) { isB = 0; xb = s; idx = r; }
    else { isB = 1; xb = s - S.L; idx = r - S.nA; }
  } else {
    const unsigned u = T - r1 - r2;
    isB = 1; xb = S.nxb - S.L + u / S.nB; idx = u - (xb - (S.nxb - S.L)) * S.nB;
  }
}

// Item kinds.  MODE 0: A items (isB = 0) are t1 items, B items are family items.  MODE 1: A items are
// family items, B items are t1 items.  Family item index = 2·k2 + h (h: which half of the block's
// pair columns).
template <int MODE, int LOG1, int LOG2>
__global__ void __launch_bounds__(FS_NT, FS_MINB)
    k_fstep(const double* __restrict__ vin, const double2* __restrict__ spin, double* __restrict__ vout,
            double2* __restrict__ spout, double2* __restrict__ Y, const double* __restrict__ vscale, int W, int nx,
            const double* __restrict__ gtab, int accumulate, int debug_sign, FsSched S, unsigned* cnt,
            unsigned* ticket, unsigned tick_base, unsigned cnt_target, int no_discard) {
  using G = FsGeo<LOG1, LOG2>;
  constexpr int NT = FS_NT;
  constexpr int N1 = G::N1, N2 = G::N2, N = G::N, H = G::H, NC = G::NC, NF = G::NF;
  constexpr int CS1 = G::CS1, CS2 = G::CS2;
  constexpr int X = 2 * NC;  // real columns per block
  static_assert(NT % NC == 0, "pair column per thread must be fixed");
  const int tid = threadIdx.x;
  double2* const buf = tf_smem;
  double2* const stw1 = tf_smem + G::off_stw1;
  double2* const stw2 = tf_smem + G::off_stw2;
  double2* const tws = tf_smem + G::off_tw;
  double* const ghi = reinterpret_cast<double*>(tf_smem + G::off_g);
  double* const glo = ghi + G::HI;
  __shared__ unsigned s_ticket;

  // ---- per-CTA tables once: stage twiddles of both lengths, Γ_α (MODE 0) or 1/(NΓ_α) (MODE 1) as
  //      two-level tables g_t = ghi[t >> 6]·glo[t & 63] (glo of MODE 1 carries the factor N back)
  const double sg = debug_sign ? -1.0 : 1.0;
  fill_stage_twiddles(stw1, LOG1, sg, tid, NT);
  fill_stage_twiddles(stw2, LOG2, sg, tid, NT);
  for (int q = tid; q < G::HI; q += NT) ghi[q] = __ldg(gtab + q * 64);
  for (int q = tid; q < 64; q += NT) glo[q] = MODE == 0 ? __ldg(gtab + q) : (double)N * __ldg(gtab + q);
  const double s = (MODE == 0 && vscale) ? *vscale : 1.0;
  if (tid == 0) s_ticket = atomicAdd(ticket, 1u) - tick_base;

  for (;;) {
    __syncthreads();  // previous item done with buf / tws; s_ticket published
    const unsigned T = s_ticket;
    if (T >= S.total) break;
    // the next ticket is requested now and published at the end of this item (its latency hides
    // behind this item's work)
    unsigned nxt = 0;
    if (tid == 0) nxt = atomicAdd(ticket, 1u);
    int isB, xb, idx;
    fs_item(S, T, isB, xb, idx);
    const int col0 = xb * X;
    double2* const Yb = Y + (size_t)xb * N * NC;  // block's Y: [t1][k2][c], c < NC

    if ((MODE == 0 && !isB) || (MODE == 1 && isB)) {
      // ================= t1 items: MODE 0 pass A (rows t1 + N1 t2 → Y), MODE 1 pass B' (Y → rows)
      const int t1 = idx;
      const int cpair = tid % NC;  // fixed across the loops below
      const int mycol = col0 + 2 * cpair;
      const bool padA = mycol >= nx, padB = mycol + 1 >= nx, colok = mycol < W;
      if (MODE == 0) {
        for (int q = tid; q < N2 * NC; q += NT) {
          const int t2 = q / NC, c = q - t2 * NC;
          const int col = col0 + 2 * c;
          double2* dst = buf + c * CS2 + pd(t2);
          if (col < W) cp_async16(dst, vin + (int64_t)(t1 + N1 * t2) * W + col);
          else *dst = make_double2(0.0, 0.0);
        }
        for (int q = tid; q < N2; q += NT) {  // ω_N^{t1 k2}
          double2 w = expi_neg((t1 * q) & (N - 1), N);
          w.y *= sg;
          tws[q] = w;
        }
      } else {
        if (tid == 0) {
          while ((int)(ld_acquire(cnt + xb) - cnt_target) < 0) __nanosleep(32);
        }
        __syncthreads();
        const double2* src = Yb + (size_t)t1 * N2 * NC;
        for (int q = tid; q < N2 * NC; q += NT) {
          const int k2 = q / NC, c = q - k2 * NC;
          cp_async16(buf + c * CS2 + pd(k2), src + q);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      if (MODE == 0) {
        local_fft<false, TF_SCALE, LOG2, NC, NT>(buf, stw2, TfScale{ghi, glo, N1, t1, s});
        double2* dst = Yb + (size_t)t1 * N2 * NC;
        for (int q = tid; q < N2 * NC; q += NT) {
          const int k2 = q / NC, c = q - k2 * NC;
          dst[q] = cmul(buf[c * CS2 + pd(k2)], tws[k2]);
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();  // cumulative: orders the CTA's Y stores (bar.sync) before the count
          atomicAdd(cnt + xb, 1u);
        }
      } else {
        if (!no_discard) {
          const char* src = reinterpret_cast<const char*>(Yb + (size_t)t1 * N2 * NC);
          for (int q = tid; q < N2 * NC * 16 / 128; q += NT) discard_l2(src + q * 128);
        }
        local_fft<true, TF_PLAIN, LOG2, NC, NT>(buf, stw2, TfScale{nullptr, nullptr, 1, 0, 1.0});
        if (colok) {
          for (int q = tid; q < N2 * NC; q += NT) {
            const int t2 = q / NC;  // q % NC == cpair
            const int t = t1 + N1 * t2;
            const double g = ghi[t >> 6] * glo[t & 63];
            const double2 z = buf[cpair * CS2 + pd(t2)];
            double2 val = make_double2(padA ? 0.0 : z.x * g, padB ? 0.0 : z.y * g);
            double2* dst = reinterpret_cast<double2*>(vout + (int64_t)t * W + mycol);
            if (accumulate) {
              const double2 o = *dst;
              val.x += o.x;
              val.y += o.y;
            }
            stg_cs2(dst, val);
          }
        }
      }
    } else {
      // ================= family items {k2, N2 − k2} × half block h: MODE 0 pass B (Y → spectrum
      //                   rows), MODE 1 pass A' (spectrum rows → Y).  Columns: pairs h·NF + c, c < NF.
      const int k2 = idx >> 1, h = idx & 1;
      const int k2m = (N2 - k2) & (N2 - 1);
      const bool two = k2m != k2;
      const int cpair = tid % NF;
      const int gpair = h * NF + cpair;  // pair index within the block
      const int mycol = col0 + 2 * gpair;
      const bool padA = mycol >= nx, padB = mycol + 1 >= nx, colok = mycol < W;
      // spectrum rows of the family: member 0 k = k2 + N2 k1 <= H (n0 rows), member 1 k = k2m + N2 k1 <= H
      const int n0 = (H - k2) / N2 + 1;
      const int n1 = two ? (H - k2m) / N2 + 1 : 0;
      if (MODE == 0) {
        if (tid == 0) {
          while ((int)(ld_acquire(cnt + xb) - cnt_target) < 0) __nanosleep(32);
        }
        __syncthreads();
        for (int q = tid; q < N1 * NF; q += NT) {
          const int t1 = q / NF, c = q - t1 * NF;
          cp_async16(buf + c * CS1 + pd(t1), Yb + ((size_t)t1 * N2 + k2) * NC + h * NF + c);
          if (two) cp_async16(buf + (NF + c) * CS1 + pd(t1), Yb + ((size_t)t1 * N2 + k2m) * NC + h * NF + c);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        if (!no_discard) {  // NF·16 B per (t1, member) row
          constexpr int LPR = NF * 16 / 128;
          for (int q = tid; q < N1 * LPR * 2; q += NT) {
            const int m = q / (N1 * LPR), r = q - m * N1 * LPR;
            const int t1 = r / LPR, l = r - t1 * LPR;
            if (m == 1 && !two) continue;
            const char* p = reinterpret_cast<const char*>(Yb + ((size_t)t1 * N2 + (m ? k2m : k2)) * NC + h * NF);
            discard_l2(p + l * 128);
          }
        }
        local_fft<false, TF_PLAIN, LOG1, 2 * NF, NT>(buf, stw1, TfScale{nullptr, nullptr, 1, 0, 1.0});
        if (colok) {
          for (int q = tid; q < (n0 + n1) * NF; q += NT) {
            const int r = q / NF;  // q % NF == cpair
            double2 zk, zm;
            int k;
            if (r < n0) {
              const int k1 = r;
              k = k2 + N2 * k1;
              zk = buf[cpair * CS1 + pd(k1)];
              zm = k2 == 0 ? buf[cpair * CS1 + pd((N1 - k1) & (N1 - 1))]
                           : buf[((two ? NF : 0) + cpair) * CS1 + pd(N1 - 1 - k1)];
            } else {
              const int k1 = r - n0;
              k = k2m + N2 * k1;
              zk = buf[(NF + cpair) * CS1 + pd(k1)];
              zm = buf[cpair * CS1 + pd(N1 - 1 - k1)];
            }
            double2 xa, xbv;
            fs_separate(zk, zm, xa, xbv);
            if (padA) xa = make_double2(0.0, 0.0);
            if (padB) xbv = make_double2(0.0, 0.0);
            double2* o = spout + (int64_t)k * W + mycol;
            stg_cs2(o, xa);
            stg_cs2(o + 1, xbv);
          }
        }
      } else {
        // gather Z_k for both members from the stored rows min(k, N − k)
        for (int q = tid; q < (n0 + n1) * NF; q += NT) {
          const int r = q / NF;
          const bool m1 = r >= n0;
          const int k1 = m1 ? r - n0 : r;
          const int k = (m1 ? k2m : k2) + N2 * k1;
          double2 xa = make_double2(0.0, 0.0), xbv = xa;
          if (colok) {
            const double2* src = spin + (int64_t)k * W + mycol;
            xa = ldg_cs2(src);
            xbv = ldg_cs2(src + 1);
          }
          double2 zk, zp;
          if (k == 0 || k == H) {
            zk = zp = make_double2(xa.x, xbv.x);
          } else {
            zk = fs_pack(xa, xbv);
            zp = fs_pack(cconj(xa), cconj(xbv));
          }
          // Z_k at its own member position; Z_{N−k} = conj-packed at the partner's position
          buf[((m1 ? NF : 0) + cpair) * CS1 + pd(k1)] = zk;
          int pm, pk1;
          if (m1) { pm = 0; pk1 = N1 - 1 - k1; }
          else if (k2 == 0) { pm = 0; pk1 = (N1 - k1) & (N1 - 1); }
          else if (!two) { pm = 0; pk1 = N1 - 1 - k1; }
          else { pm = 1; pk1 = N1 - 1 - k1; }
          buf[(pm * NF + cpair) * CS1 + pd(pk1)] = zp;
        }
        for (int q = tid; q < N1; q += NT) {  // conj ω_N^{k2 t1}, conj ω_N^{k2m t1}
          double2 w0 = expi_neg((k2 * q) & (N - 1), N), w1 = expi_neg((k2m * q) & (N - 1), N);
          w0.y *= -sg;
          w1.y *= -sg;
          tws[q] = w0;
          tws[N1 + q] = w1;
        }
        __syncthreads();
        local_fft<true, TF_PLAIN, LOG1, 2 * NF, NT>(buf, stw1, TfScale{nullptr, nullptr, 1, 0, 1.0});
        for (int q = tid; q < N1 * NF * 2; q += NT) {
          const int m = q / (N1 * NF), r = q - m * N1 * NF;
          if (m == 1 && !two) continue;
          const int t1 = r / NF, c = r - t1 * NF;
          Yb[((size_t)t1 * N2 + (m ? k2m : k2)) * NC + h * NF + c] =
              cmul(buf[(m * NF + c) * CS1 + pd(t1)], tws[m * N1 + t1]);
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          atomicAdd(cnt + xb, 1u);
        }
      }
    }
    __syncthreads();  // everyone has read s_ticket and finished with buf
    if (tid == 0) s_ticket = nxt - tick_base;
  }
}

// ------------------------------------------------------------------------------------ host side
static void fs_logs(int N, int& l1, int& l2) {
  int logN = 0;
  while ((1 << logN) < N) ++logN;
  l1 = (logN + 1) / 2;
  l2 = logN - l1;
}

bool fstep_ok(const cnpint_ctx* c) { return c->dim == 1 && c->N >= 2048 && c->N <= 65536 && c->d_fsY; }

static int fs_nc(int N) {
  int l1, l2;
  fs_logs(N, l1, l2);
  const int mx = l1 > l2 ? l1 : l2;
  return mx <= 6 ? 32 : mx == 7 ? 16 : 8;
}
int fstep_nxb(int N, int64_t ld) { return (int)((ld + 2 * fs_nc(N) - 1) / (2 * fs_nc(N))); }
// Y: nxb blocks of N × NC complex (the last block padded to whole pairs of NC columns)
size_t fstep_y_bytes(int dim, int N, int64_t ld) {
  return (dim == 1 && N >= 2048 && N <= 65536) ? (size_t)fstep_nxb(N, ld) * N * fs_nc(N) * 16 : 0;
}

template <int MODE, int LOG1, int LOG2>
static cudaError_t fs_launch(cnpint_ctx* c, const double* vin, const double2* spin, double* vout, double2* spout,
                             const double* vscale, int accumulate) {
  using G = FsGeo<LOG1, LOG2>;
  auto kern = k_fstep<MODE, LOG1, LOG2>;
  static int per_sm = 0;
  if (!per_sm) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::bytes);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, FS_NT, G::bytes);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  const int W = (int)c->ld;
  FsSched S;
  S.nxb = (W + 2 * G::NC - 1) / (2 * G::NC);
  S.nA = MODE == 0 ? G::N1 : 2 * (G::N2 / 2 + 1);
  S.nB = MODE == 0 ? 2 * (G::N2 / 2 + 1) : G::N1;
  S.total = (unsigned)S.nxb * (S.nA + S.nB);
  const int grid_max = per_sm * c->num_sms;
  const int grid = (int)(S.total < (unsigned)grid_max ? S.total : (unsigned)grid_max);
  // lag: enough steps between a block's A and B items that the CTAs in flight (≈ grid) finish the
  // A items first
  int L = 2 * ((grid + S.nA + S.nB - 1) / (S.nA + S.nB)) + 1;
  if (const char* e = getenv("CNPINT_FS_LAG")) L = atoi(e) > 0 ? atoi(e) : L;
  S.L = L < S.nxb ? L : S.nxb;
  const unsigned target = c->fs_cnt + (unsigned)S.nA;
  static int no_discard = -1;
  if (no_discard < 0) no_discard = getenv("CNPINT_FS_NODISCARD") ? 1 : 0;
  kern<<<grid, FS_NT, G::bytes, c->stream>>>(vin, spin, vout, spout, (double2*)c->d_fsY, vscale, W, c->nx,
                                            MODE == 0 ? c->d_gam : c->d_igam, accumulate, c->debug & 1, S,
                                            c->d_fscnt, c->d_fscnt + S.nxb, c->fs_tick, target, no_discard);
  c->fs_cnt = target;
  c->fs_tick += S.total + (unsigned)grid;  // every CTA also takes one ticket past the end
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t fs_dispatch(cnpint_ctx* c, const double* vin, const double2* spin, double* vout, double2* spout,
                               const double* vscale, int accumulate) {
  int l1, l2;
  fs_logs(c->N, l1, l2);
#define FS_CASE(A, B) \
  if (l1 == A && l2 == B) return fs_launch<MODE, A, B>(c, vin, spin, vout, spout, vscale, accumulate);
  FS_CASE(6, 5) FS_CASE(6, 6) FS_CASE(7, 6) FS_CASE(7, 7) FS_CASE(8, 7) FS_CASE(8, 8)
#undef FS_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_fstep_fwd(cnpint_ctx* c, const double* v, const double* vscale, double2* what) {
  cnp_prof_begin(c, KID_FFT_FWD);
  cudaError_t e = fs_dispatch<0>(c, v, nullptr, nullptr, what, vscale, 0);
  cnp_prof_end(c, KID_FFT_FWD, 8.0 * cnp_units(c) + 16.0 * cnp_spec_units(c));
  return e;
}
cudaError_t launch_fstep_inv(cnpint_ctx* c, const double2* zhat, double* z, int accumulate) {
  cnp_prof_begin(c, KID_FFT_INV);
  cudaError_t e = fs_dispatch<1>(c, nullptr, zhat, z, nullptr, nullptr, accumulate);
  cnp_prof_end(c, KID_FFT_INV, 8.0 * cnp_units(c) * (accumulate ? 2.0 : 1.0) + 16.0 * cnp_spec_units(c));
  return e;
}
