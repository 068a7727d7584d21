// K5, lean y pass (round 2): the y axis of W⁻¹ / W with the half-length sine
// transform and the low instruction count of k_dst4.cu, for lines that are COLUMNS of a time slice.
//
// A tile is P = 8 adjacent column pairs (16 columns = one 128-B row segment) of one slice.  Threads are
// interleaved pair-fastest (tid = c + P·r), so every warp load/store of the samples touches whole
// 128-B segments (4 rows × 8 pairs), and the exchange regions of the P pairs sit at an odd stride
// (M + 1 complex) so the 8 pairs of a shared-memory phase hit distinct banks.  The FFT (M = R1·R2·R3,
// radix-8 register passes) and the exchanges are k_dst4's with CTA-wide barriers; the prefix-sum phase
// re-maps threads pair-contiguously (lines own consecutive lanes for the warp scan), stages its
// results line by line (XOR-swizzled, conflict free) and the tile leaves as 128-B row segments.
#include "common.cuh"
#include "internal.h"

#include "fft_device.cuh"

namespace {

CNP_DEV int zpos5(int k) { return k ^ ((k >> 3) & 7); }
CNP_DEV int opos5(int x) { return x ^ ((x >> 4) & 15); }

}  // namespace

template <int LOGM>
struct D5Plan {
  static constexpr int M = 1 << LOGM, H = M / 2, n = M - 1;
  static constexpr int R1 = 8;
  static constexpr int R2 = LOGM == 7 ? 4 : 8;
  static constexpr int R3 = M / (R1 * R2);
  static constexpr int TP = M / 8;
  static constexpr int P = 8;                 // column pairs per tile
  static constexpr int NT = P * TP;           // 512, 256, 128, 64 threads for LOGM = 9..6
  static constexpr int MINB = 1024 / NT;
  static constexpr int RS = M + 1;            // region stride (complex), odd
  static constexpr int LS = M + 1;            // staged line stride (doubles), odd
  static constexpr int I1 = (M / R1) / TP, I2 = (M / R2) / TP, I3 = (M / R3) / TP;
  static constexpr size_t off_t1 = (size_t)P * RS * 16;
  static constexpr size_t off_t2 = off_t1 + (size_t)M * 16;
  static constexpr size_t off_ab = off_t2 + (size_t)(M / R1) * 16;
  static constexpr size_t off_post = off_ab + (size_t)M * 16;
  static constexpr size_t bytes = off_post + (size_t)M * 8;
  static_assert(2 * P * LS <= 2 * P * RS, "staging fits the exchange regions");
};

template <int LOGM>
__global__ void __launch_bounds__(D5Plan<LOGM>::NT, D5Plan<LOGM>::MINB)
    k_dst5(const double* __restrict__ in, double* __restrict__ out, int N, int ny, int64_t ld,
           const double* __restrict__ pre, const double* __restrict__ post, const double2* __restrict__ tw2M,
           int accumulate, int debug_sign, int nx) {
  using PL = D5Plan<LOGM>;
  constexpr int M = PL::M, H = PL::H, n = PL::n, TP = PL::TP, P = PL::P, NT = PL::NT, RS = PL::RS, LS = PL::LS;
  constexpr int R1 = PL::R1, R2 = PL::R2, R3 = PL::R3;
  char* const smem = reinterpret_cast<char*>(fft_smem);
  double2* const reg0 = reinterpret_cast<double2*>(smem);
  double* const stage = reinterpret_cast<double*>(smem);
  double2* const T1 = reinterpret_cast<double2*>(smem + PL::off_t1);
  double2* const T2 = reinterpret_cast<double2*>(smem + PL::off_t2);
  double2* const ab = reinterpret_cast<double2*>(smem + PL::off_ab);
  double2* const post2 = reinterpret_cast<double2*>(smem + PL::off_post);
  const int tid = threadIdx.x;
  const int c = tid % P, r = tid / P;  // load / FFT mapping: pair-fastest
  double2* const A = reg0 + c * RS;
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
      post2[q] = make_double2(x < n ? (post ? post[x] : 1.0) : 0.0, x + 1 < n ? (post ? post[x + 1] : 1.0) : 0.0);
    }
    double a = 0.0, b = 0.0;
    if (q > 0) {
      const double s = -tw2M[q].y;  // sin(qπ/M)
      const double gj = pre ? pre[q - 1] : 1.0, gm = pre ? pre[M - q - 1] : 1.0;
      a = (s + 0.5) * gj;
      b = (s - 0.5) * gm;
    }
    ab[q] = make_double2(a, b);
  }
  __syncthreads();
  pdl_enter();  // PDL: the slices below come from the previous kernel
  constexpr int TPS = (M / 2) / P;  // tiles per slice (ld = M columns = M/2 pairs)
  const int ntiles = N * TPS;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int t = tile / TPS, col0 = (tile - t * TPS) * 2 * P;
    const double* slice = in + (int64_t)t * ny * ld + col0 + 2 * c;
    // ---- step 1: z_j from rows j and M − j of this pair's two columns (16-B loads)
#pragma unroll
    for (int i1 = 0; i1 < PL::I1; ++i1) {
      const int m = r + i1 * TP;
      double2 v[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int j = m + (M / R1) * n1;
        double2 z = make_double2(0.0, 0.0);
        if (j > 0) {
          const double2 cf = ab[j];
          const double2 f = __ldg(reinterpret_cast<const double2*>(slice + (int64_t)(j - 1) * ld));
          const double2 fm = __ldg(reinterpret_cast<const double2*>(slice + (int64_t)(M - j - 1) * ld));
          z = make_double2(fma(cf.x, f.x, cf.y * fm.x), fma(cf.x, f.y, cf.y * fm.y));
        }
        v[n1] = z;
      }
      dftR<R1, false>(v);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) A[k1 * (M / R1) + m] = k1 ? cmul(v[k1], T1[k1 * (M / R1) + m]) : v[0];
    }
    __syncthreads();
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
      for (int k3 = 0; k3 < R3; ++k3) A[zpos5(k1 + R1 * k2 + R1 * R2 * k3)] = w3[i3][k3];
    }
    __syncthreads();
    // ---- post, pair-contiguous: pair cp, line ln, lane q owns k ∈ [8q, 8q+8]
    const int cp = tid / TP, rr = tid % TP, ln = rr / (TP / 2), q = rr % (TP / 2);
    const double2* Z = reg0 + cp * RS;
    double Rk[8], Ik[8];
    double loc = 0.0;
#pragma unroll
    for (int i = 0; i <= 8; ++i) {
      const int k = 8 * q + i;
      const double2 Zk = Z[zpos5(k & (M - 1))];
      const double2 Zm = Z[zpos5((M - k) & (M - 1))];
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
    __syncthreads();  // every Z read: the regions take the staged lines
    {
      double* sl = stage + (2 * cp + ln) * LS;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        run += Rk[i];
        const double2 ps = post2[i * (TP / 2) + q];
        const int x = 16 * q + 2 * i;
        sl[opos5(x)] = run * ps.x;
        sl[opos5(x + 1)] = Ik[i] * ps.y;
      }
    }
    __syncthreads();
    // ---- rows x < n of the 16 columns: (line 2c, line 2c+1) → 16 B at column col0 + 2c
    for (int e = tid; e < n * P; e += NT) {
      const int x = e / P, cc = e - x * P;
      const int px = opos5(x);
      double2 v2 = make_double2(stage[(2 * cc) * LS + px], stage[(2 * cc + 1) * LS + px]);
      const int col = col0 + 2 * cc;
      if (col >= nx) v2.x = 0.0;  // padding columns stay exactly zero
      if (col + 1 >= nx) v2.y = 0.0;
      double2* o = reinterpret_cast<double2*>(out + ((int64_t)t * ny + x) * ld + col);
      if (accumulate) {
        const double2 pv = *o;
        v2.x += pv.x;
        v2.y += pv.y;
      }
      stg_cs2(o, v2);
    }
    __syncthreads();  // staging read: the regions are free for the next tile
  }
}

template <int LOGM>
static cudaError_t run_dst5(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                            int accumulate) {
  using PL = D5Plan<LOGM>;
  auto kern = k_dst5<LOGM>;
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
  const int ntiles = c->N * ((PL::M / 2) / PL::P);
  const int grid = ntiles < grid_max ? ntiles : grid_max;
  return cnp_launch(c, kern, dim3(grid), dim3(PL::NT), PL::bytes, in, out, c->N, c->ny, c->ld, pre, post,
                    (const double2*)c->d_twy, accumulate, c->debug & 1, c->nx);
}

// y pass through the lean kernel on square grids with ny + 1 = ld ∈ {64, …, 512}; else NotSupported
cudaError_t launch_dst5_y(cnpint_ctx* c, const double* in, double* out, const double* pre, const double* post,
                          int accumulate) {
  if (c->ld != c->nx + 1 || c->ny != c->nx) return cudaErrorNotSupported;
  switch (c->ny + 1) {
    case 64: return run_dst5<6>(c, in, out, pre, post, accumulate);
    case 128: return run_dst5<7>(c, in, out, pre, post, accumulate);
    case 256: return run_dst5<8>(c, in, out, pre, post, accumulate);
    case 512: return run_dst5<9>(c, in, out, pre, post, accumulate);
    default: return cudaErrorNotSupported;
  }
}
