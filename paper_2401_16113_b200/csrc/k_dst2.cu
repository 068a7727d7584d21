// K5 (second generation): one axis of the 2D fast diagonalisation W⁻¹ / W (step (b)
// of Eq. 3.2 with the DST; see k_dst.cu for the diagonal-similarity reading) as a pipelined,
// half-length sine transform.
//
// Transform (per line f_1..f_n, n = M − 1, M = 2^LOGM):
//   F_k = Σ_j f'_j sin(πjk/M),  f'_j = pre_j f_j  (forward: pre = ρ^{−j}),   out_k = post_k F_k  (inverse:
//   post = ρ^{k}·2/M),  k = 1..n.
// Half-length algorithm (the pre-combination of Cooley, Lewis & Welch): with
//   y_0 = 0,  y_j = sin(jπ/M)(f'_j + f'_{M−j}) + ½(f'_j − f'_{M−j}),  Y = FFT_M(y)  (real input),
// the even outputs are F_{2k} = −Im Y_k and the odd ones a prefix sum of the real parts,
// F_{2k+1} = ½Re Y_0 + Σ_{i=1}^{k} Re Y_i  (the symmetric part of y meets cos, the antisymmetric part
// sin).  Two lines a, b ride in one complex FFT of length M, z = y^a + i y^b, separated by Hermitian
// symmetry: Y^a_k = (Z_k + conj Z_{M−k})/2, Y^b_k = (Z_k − conj Z_{M−k})/(2i).  Per line that is half
// the butterflies and half the shared-memory traffic of the odd extension of length 2M (k_dst.cu).
//
// B200 design:
//   * persistent CTAs (two per SM), a ring of S shared-memory stages filled by TMA bulk copies
//     (cp.async.bulk + mbarrier transaction counts) issued by one thread: while the CTA transforms
//     tile i, tile i+1 is in flight — the loads no longer wait behind the butterflies;
//   * x pass: a tile is 2P consecutive rows (contiguous in HBM: ONE bulk copy per tile);
//     y pass: a tile is 2P adjacent columns of one time slice, n row segments of 16P bytes, landed
//     at an odd 16-B pitch (conflict-free column reads);
//   * the FFT is M = R1·R2·R3 in registers (radix 8/4 passes), TP = M/8 threads per line pair; the
//     exchanges ping-pong between a per-CTA area A and the (consumed) stage region;
//   * the prefix sum is a warp-shuffle scan: the TP/2 ≤ 32 threads of a line own 8 consecutive k;
//   * outputs are staged (XOR-swizzled, conflict-free) and leave as coalesced 16-B stores.
#include "common.cuh"
#include "internal.h"

#include "fft_device.cuh"

namespace {

CNP_DEV uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
CNP_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(bar)), "r"(count) : "memory");
}
CNP_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
CNP_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
CNP_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
CNP_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// swizzled position of output x inside a staged line (16 consecutive x per scan lane → distinct banks)
CNP_DEV int opos(int x) { return x ^ ((x >> 4) & 15); }
// swizzled position of Z_k (8 consecutive k per post lane, and 8 consecutive k1 per step-3 lane)
CNP_DEV int zpos(int k) { return k ^ ((k >> 3) & 7); }

}  // namespace

template <bool YPASS, int LOGM>
struct D2Plan {
  static constexpr int M = 1 << LOGM, H = M / 2, n = M - 1;
  static constexpr int R1 = 8;
  static constexpr int R2 = LOGM == 7 ? 4 : 8;
  static constexpr int R3 = M / (R1 * R2);                // 8, 4, 4, 1 for LOGM = 9, 8, 7, 6
  static constexpr int TP = M / 8;                        // threads per line pair
  // x pass: 256 threads, two CTAs per SM; y pass: 512 threads (P ≤ M/2 pairs per slice), one CTA
  static constexpr int NT = !YPASS ? 256 : (TP * (M / 2) < 512 ? TP * (M / 2) : 512);
  static constexpr int MINB = YPASS ? 1 : 2;
  static constexpr int P = NT / TP;                       // line pairs per tile
  static constexpr int S = 2;                             // pipeline stages
  static constexpr int I1 = (M / R1) / TP;                // step items per thread
  static constexpr int I2 = (M / R2) / TP;
  static constexpr int I3 = (M / R3) / TP;
  static constexpr int YPITCH = 2 * P + 2;                // y pass stage: [n rows][2P + 2] (odd 16-B pitch)
  static constexpr int OREG = M + 2;                      // staged output: [pair][line][OREG]
  static constexpr int IN = YPASS ? n * YPITCH : 2 * P * M;  // x pass stage: [2P rows][M]
  static constexpr int STAGE1 = IN > 2 * P * OREG ? IN : 2 * P * OREG;
  static constexpr int STAGE = (STAGE1 + 1) / 2 * 2;      // doubles, 16-B multiple
  static constexpr int AREA = P * M;                      // complex, area A
  static constexpr size_t off_area = (size_t)S * STAGE * 8;
  static constexpr size_t off_tw = off_area + (size_t)AREA * 16;
  static constexpr size_t off_bar = off_tw + (size_t)M * 16;
  static constexpr size_t bytes = off_bar + 64;
  static_assert(!YPASS || P <= M / 2, "y pass: at most M/2 pairs per slice");
};

template <bool YPASS, int LOGM>
__global__ void __launch_bounds__(D2Plan<YPASS, LOGM>::NT, D2Plan<YPASS, LOGM>::MINB)
    k_dst2(const double* __restrict__ in, double* __restrict__ out, int N, int ny, int64_t ld,
           const double* __restrict__ pre, const double* __restrict__ post, const double2* __restrict__ tw2M,
           int accumulate, int debug_sign, int nx) {
  using PL = D2Plan<YPASS, LOGM>;
  constexpr int M = PL::M, H = PL::H, n = PL::n, TP = PL::TP, P = PL::P, S = PL::S;
  constexpr int R1 = PL::R1, R2 = PL::R2, R3 = PL::R3;
  char* const smem = reinterpret_cast<char*>(fft_smem);
  double* const stage0 = reinterpret_cast<double*>(smem);
  double2* const area = reinterpret_cast<double2*>(smem + PL::off_area);
  double2* const twM = reinterpret_cast<double2*>(smem + PL::off_tw);  // ω_M^q, q < M
  uint64_t* const full = reinterpret_cast<uint64_t*>(smem + PL::off_bar);
  const int tid = threadIdx.x;
  const int pr = tid / TP;      // line pair of this thread within the tile
  const int r = tid % TP;       // role within the pair
  const double sg = debug_sign ? -1.0 : 1.0;
  // ---- tables (create-time constants): ω_M^q = ω_{2M}^{2q}
  for (int q = tid; q < M; q += PL::NT) {
    double2 w = tw2M[2 * q];
    w.y *= sg;
    twM[q] = w;
  }
  const int ldi = (int)ld;
  const int nlines = N * ny;
  const int tiles_per_t = (M / 2) / P;  // y pass: pairs per slice = ld/2 = M/2
  const int ntiles = YPASS ? N * tiles_per_t : (nlines / 2 + P - 1) / P;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_enter();  // PDL: the lines below come from the previous kernel
  // ---- producer (one thread / one warp): bulk copies of tile `tile` into stage s
  auto issue = [&](int tile, int s) {
    double* st = stage0 + (size_t)s * PL::STAGE;
    if (!YPASS) {
      if (tid == 0) {
        const int row0 = tile * 2 * P;
        const int rows = min(2 * P, nlines - row0);
        const unsigned bytes = (unsigned)rows * M * 8;
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(st, in + (int64_t)row0 * ld, bytes, &full[s]);
      }
    } else if (tid < 32) {
      const int t = tile / tiles_per_t, col0 = (tile - t * tiles_per_t) * 2 * P;
      if (tid == 0) mbar_expect_tx(&full[s], (unsigned)n * 2 * P * 8);
      __syncwarp();
      for (int y = tid; y < n; y += 32)
        bulk_g2s(st + y * PL::YPITCH, in + ((int64_t)t * ny + y) * ld + col0, 2 * P * 8, &full[s]);
    }
  };
  int it = 0;
  for (int s = 0; s < S; ++s)
    if ((int)blockIdx.x + s * (int)gridDim.x < ntiles) issue(blockIdx.x + s * gridDim.x, s);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % S;
    double* const st = stage0 + (size_t)s * PL::STAGE;
    double2* const stc = reinterpret_cast<double2*>(st);  // the stage as complex scratch (C, then staging)
    mbar_wait(&full[s], (unsigned)((it / S) & 1));
    // ---- this pair's lines
    int t = 0, col0 = 0, row0 = 0;
    if (YPASS) {
      t = tile / tiles_per_t;
      col0 = (tile - t * tiles_per_t) * 2 * P;
    } else {
      row0 = tile * 2 * P;
    }
    // sample j (1 ≤ j ≤ n) of the pair as (f^a_j, f^b_j), pre-scaled
    auto fget = [&](int j) -> double2 {
      double2 v;
      if (YPASS) v = *reinterpret_cast<const double2*>(st + (j - 1) * PL::YPITCH + 2 * pr);
      else v = make_double2(st[(2 * pr) * M + j - 1], st[(2 * pr + 1) * M + j - 1]);
      const double g = pre ? __ldg(pre + j - 1) : 1.0;
      return cscale(v, g);
    };
    double2* const A = area + pr * M;
    double2* const C = stc + pr * M;
    // ---- step 1: z_j = y^a_j + i y^b_j at j = m + (M/R1) n1; DFT_R1; twiddle ω_M^{m k1}; B[k1][m] → A
#pragma unroll
    for (int i1 = 0; i1 < PL::I1; ++i1) {
      const int m = r + i1 * TP;
      double2 v[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int j = m + (M / R1) * n1;
        double2 z = make_double2(0.0, 0.0);
        if (j > 0) {
          const double2 fj = fget(j), fm = fget(M - j);  // f_{M−j}: j = M − j only at j = M/2
          const double sj = -__ldg(&tw2M[j].y);  // sin(jπ/M) = −Im ω_{2M}^j
          z = make_double2(fma(sj, fj.x + fm.x, 0.5 * (fj.x - fm.x)), fma(sj, fj.y + fm.y, 0.5 * (fj.y - fm.y)));
        }
        v[n1] = z;
      }
      dftR<R1, false>(v);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) A[k1 * (M / R1) + m] = k1 ? cmul(v[k1], twM[m * k1]) : v[0];
    }
    __syncthreads();  // B complete; every stage sample consumed (the stage becomes scratch)
    // ---- step 2: item (k1, m3): B[k1][m3 + R3 m2] → DFT_R2 → ω_M^{R1 m3 k2} → C[(k2 R1 + k1) R3 + m3']
#pragma unroll
    for (int i2 = 0; i2 < PL::I2; ++i2) {
      const int q = r + i2 * TP;
      const int m3 = q % R3, k1 = q / R3;
      double2 u[R2];
#pragma unroll
      for (int m2 = 0; m2 < R2; ++m2) u[m2] = A[k1 * (M / R1) + m3 + R3 * m2];
      dftR<R2, false>(u);
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) {
        const double2 w = (k2 && m3) ? cmul(u[k2], twM[R1 * m3 * k2]) : u[k2];
        C[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))] = w;
      }
    }
    __syncthreads();
    // ---- step 3: item (k1, k2): C → DFT_R3 → Z_k, k = k1 + R1 k2 + R1 R2 k3 → A (swizzled)
#pragma unroll
    for (int i3 = 0; i3 < PL::I3; ++i3) {
      const int q = r + i3 * TP;
      const int k1 = q % R1, k2 = q / R1;
      double2 w[R3];
#pragma unroll
      for (int m3 = 0; m3 < R3; ++m3) w[m3] = C[(k2 * R1 + k1) * R3 + (m3 ^ (k1 & (R3 - 1)))];
      if constexpr (R3 > 1) dftR<R3, false>(w);
#pragma unroll
      for (int k3 = 0; k3 < R3; ++k3) A[zpos(k1 + R1 * k2 + R1 * R2 * k3)] = w[k3];
    }
    __syncthreads();
    // ---- post: line ℓ of the pair (threads [0, TP/2) → a, [TP/2, TP) → b); lane q owns k ∈ [8q, 8q+8]
    const int ln = r / (TP / 2), q = r % (TP / 2);
    double Fo[16];  // outputs x = 16q + i: even i → F_{2k+1}, odd i → F_{2k+2}
    {
      double Rk[8];
      double loc = 0.0;
#pragma unroll
      for (int i = 0; i <= 8; ++i) {
        const int k = 8 * q + i;
        const double2 Zk = A[zpos(k & (M - 1))];
        const double2 Zm = A[zpos((M - k) & (M - 1))];
        // Y^a = (Z_k + conj Z_{M−k})/2, Y^b = (Z_k − conj Z_{M−k})/(2i)
        const double re = ln == 0 ? 0.5 * (Zk.x + Zm.x) : 0.5 * (Zk.y + Zm.y);
        const double im = ln == 0 ? 0.5 * (Zk.y - Zm.y) : -0.5 * (Zk.x - Zm.x);
        if (i < 8) {
          Rk[i] = (k == 0) ? 0.5 * re : re;
          loc += Rk[i];
        }
        if (i > 0) Fo[2 * i - 1] = (k < H) ? -im : 0.0;  // F_{2k} at x = 2k − 1; F_M (x = n, pad) = 0
      }
      // exclusive scan of the lane totals over the TP/2 lanes of this line (one warp or a part of it)
      constexpr int W = TP / 2 < 32 ? TP / 2 : 32;
      double incl = loc;
#pragma unroll
      for (int o = 1; o < W; o <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, incl, o, W);
        if (q % W >= o) incl += u;
      }
      double run = incl - loc;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        run += Rk[i];
        Fo[2 * i] = run;  // F_{2k+1}, k = 8q + i, at x = 16q + 2i
      }
    }
    __syncthreads();  // Z consumed (A free); the stage region takes the staged outputs
    {
      double* const ob = st + (2 * pr + ln) * PL::OREG;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int x = 16 * q + i;
        const double g = (post && x < n) ? __ldg(post + x) : 1.0;
        ob[opos(x)] = x < n ? Fo[i] * g : 0.0;
      }
    }
    __syncthreads();
    // ---- coalesced stores
    if (!YPASS) {
      // rows row0 + 2c + ℓ: thread → (line, x pair), consecutive threads consecutive x
      const int rows = min(2 * P, nlines - row0);
      for (int e = tid; e < rows * (M / 2); e += PL::NT) {
        const int lr = e / (M / 2), x = 2 * (e - lr * (M / 2));
        const double* ob = st + lr * PL::OREG;
        const int p0 = opos(x);
        const double2 v2 = *reinterpret_cast<const double2*>(ob + (p0 & ~1));
        double2 v = (p0 & 1) ? make_double2(v2.y, v2.x) : v2;
        double2* o = reinterpret_cast<double2*>(out + (int64_t)(row0 + lr) * ld + x);
        if (accumulate) {
          const double2 w = *o;
          v.x += w.x;
          v.y += w.y;
        }
        stg_cs2(o, v);
      }
    } else {
      // (row y, pair c): (F^a_y, F^b_y) → 16 B at column col0 + 2c; P pairs = 16P-byte row segments
      for (int e = tid; e < n * P; e += PL::NT) {
        const int y = e / P, c = e - y * P;
        const int py = opos(y);
        double2 v = make_double2(st[(2 * c) * PL::OREG + py], st[(2 * c + 1) * PL::OREG + py]);
        const int col = col0 + 2 * c;
        if (col >= nx) v.x = 0.0;  // padding columns stay exactly zero
        if (col + 1 >= nx) v.y = 0.0;
        double2* o = reinterpret_cast<double2*>(out + ((int64_t)t * ny + y) * ld + col);
        if (accumulate) {
          const double2 w = *o;
          v.x += w.x;
          v.y += w.y;
        }
        stg_cs2(o, v);
      }
    }
    fence_proxy_async();  // this thread's generic accesses of the stage before the async-proxy refill
    __syncthreads();      // stage s fully consumed
    const int next = tile + S * (int)gridDim.x;
    if (next < ntiles) issue(next, s);
  }
  (void)ldi;
}

template <bool YPASS, int LOGM>
static cudaError_t run_dst2(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                            int accumulate) {
  using PL = D2Plan<YPASS, LOGM>;
  auto kern = k_dst2<YPASS, LOGM>;
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
  const int nlines = c->N * c->ny;
  const int ntiles = YPASS ? c->N * ((PL::M / 2) / PL::P) : (nlines / 2 + PL::P - 1) / PL::P;
  const int grid = ntiles < grid_max ? ntiles : grid_max;
  const double2* tw = YPASS ? c->d_twy : c->d_twx;
  return cnp_launch(c, kern, dim3(grid), dim3(PL::NT), PL::bytes, in, out, c->N, c->ny, c->ld, pre, post, tw,
                    accumulate, c->debug & 1, c->nx);
}

// 2D sine pass through the pipelined half-length kernel when n + 1 ∈ {64, …, 512} and the operator is
// square in the sense of the DST tables (x pass: n = nx; y pass: n = ny, with ld = nx + 1 = M); returns
// cudaErrorNotSupported when not applicable (the caller keeps k_dst / k_dst_r).
cudaError_t launch_dst2(cnpint_ctx* c, bool ypass, const double* in, double* out, const double* pre,
                        const double* post, int accumulate) {
  const int n = ypass ? c->ny : c->nx;
  if (c->ld != c->nx + 1 || (ypass && c->ny != c->nx)) return cudaErrorNotSupported;
  switch (n + 1) {
    case 64: return ypass ? run_dst2<true, 6>(c, in, out, pre, post, accumulate) : run_dst2<false, 6>(c, in, out, pre, post, accumulate);
    case 128: return ypass ? run_dst2<true, 7>(c, in, out, pre, post, accumulate) : run_dst2<false, 7>(c, in, out, pre, post, accumulate);
    case 256: return ypass ? run_dst2<true, 8>(c, in, out, pre, post, accumulate) : run_dst2<false, 8>(c, in, out, pre, post, accumulate);
    case 512: return ypass ? run_dst2<true, 9>(c, in, out, pre, post, accumulate) : run_dst2<false, 9>(c, in, out, pre, post, accumulate);
    default: return cudaErrorNotSupported;
  }
}
