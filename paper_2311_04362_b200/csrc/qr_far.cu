// Far trailing update of the blocked Householder QR (qr2.cu, two-level
// blocking).  The panels of an outer block of OB <= 128 columns [b0, b0+ob)
// are factored (and update each other) first; their reflectors are then
// applied to the far columns [c0, c0+Nf) in one compact-WY step with
// tensor-core tiles:
//
//   Y = V' W_far          k_far_y   (split over row ranges, fixed-order sum)
//   Z = T' Y              k_far_z   (z_i = tau_i (y_i - sum_{k<i} G_ki z_k),
//                                    G = V'V: (T')^{-1} = diag(1/tau) +
//                                    strict_lower(G'), no explicit T)
//   W_far -= V Z          k_far_apply
//
// V (rows [b0, d), ob columns) is the unit lower trapezoid stored below the
// block's diagonal in W (dlarfb's V; linalg.py:42 dgeqrf).  With ob = 128
// the two GEMMs carry 2*128 flops per 8 bytes of W_far: DMMA-bound, where a
// 16-column panel's update is HBM-bound (qr2.cu k_qr_y / k_qr_apply, ~3
// flop/B).  Every sum runs in a fixed order: R is bitwise reproducible.
#include <algorithm>

#include "itsk_common.cuh"
#include "itsk_kernels.cuh"

namespace itsk {
namespace {

constexpr int FT = 256;          // threads per CTA
constexpr int FOB = 128;         // max block width (rows of Y / Z)
constexpr int FY_KC = 16;        // rows per stage in k_far_y
constexpr int FY_ST = 4;         // stages
constexpr int FY_VS = FOB + 8;   // [k][i] tiles: stride = 8 (mod 16) doubles -> conflict-free fragments
constexpr int FY_BS = 64 + 8;
constexpr int FA_KC = 32;        // k per stage in k_far_apply
constexpr int FA_VS = FA_KC + 4; // [row][k] tile: stride = 4 (mod 16)
constexpr int FA_ZS = 64 + 8;    // [k][col] tile

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// V(r, i) of the block whose first row / column is b0: zero above the
// diagonal, one on it, the stored reflector below
__device__ __forceinline__ double vv(double stored, int64_t r, int64_t b0, int i) {
  const int64_t jr = b0 + i;
  return r < jr ? 0.0 : (r == jr ? 1.0 : stored);
}
__device__ __forceinline__ int64_t split_lo(int s, int S, int64_t len) { return (static_cast<int64_t>(s) * len) / S; }

struct FarArgs {
  double* W;
  int64_t d, ldw;
  int64_t b0;          // first row and first column of the block
  int ob;              // block width (<= FOB)
  int64_t c0, Nf;      // far columns [c0, c0 + Nf)
  double* Yp;          // S x Nf x FOB partials (k_far_y, column-major: a column's FOB values
                       // contiguous), summed by k_far_z
  int S;
  const double* G;     // FOB x FOB: V'V of the block (k_far_z)
  const double* taus;  // global tau array, indexed b0 + i
  double* Z;           // Nf x FOB (column-major, like Yp)
};

// Y_s = V_s' B_s over the rows of split s; B = the far columns of W, or V
// itself (BV: the block's Gram matrix G = V'V).  CTA tile FOB x 64, 8 warps
// of 32 x 32 (4 x 4 DMMA 8x8 tiles), cp.async ring of FY_ST stages.
template <bool BV>
__global__ void __launch_bounds__(FT) k_far_y(FarArgs a) {
  extern __shared__ __align__(16) double fsm[];
  double* Vs = fsm;                              // FY_ST x FY_KC x FY_VS
  double* Bs = Vs + FY_ST * FY_KC * FY_VS;       // FY_ST x FY_KC x FY_BS
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int mw = warp >> 1, nw = warp & 1;       // warp's 32 x 32 sub-tile
  const int64_t cb = static_cast<int64_t>(blockIdx.x) * 64;
  const int cw = static_cast<int>(min(static_cast<int64_t>(64), a.Nf - cb));
  const int64_t len = a.d - a.b0;
  const int64_t rlo = a.b0 + split_lo(blockIdx.y, a.S, len), rhi = a.b0 + split_lo(blockIdx.y + 1, a.S, len);
  const int nch = static_cast<int>((rhi - rlo + FY_KC - 1) / FY_KC);
  const int ob = a.ob;
  auto load = [&](int ch) {
    const int st = ch % FY_ST;
    const int64_t r0 = rlo + static_cast<int64_t>(ch) * FY_KC;
    double* vs = Vs + st * FY_KC * FY_VS;
    double* bs = Bs + st * FY_KC * FY_BS;
    for (int idx = tid; idx < FY_KC * FOB; idx += FT) {
      const int rr = idx / FOB, i = idx - rr * FOB;
      const int64_t r = r0 + rr;
      const bool ok = r < rhi && i < ob;
      cp_async8(vs + rr * FY_VS + i, a.W + (ok ? r * a.ldw + a.b0 + i : 0), ok);
    }
    for (int idx = tid; idx < FY_KC * 64; idx += FT) {
      const int rr = idx >> 6, c = idx & 63;
      const int64_t r = r0 + rr;
      const bool ok = r < rhi && c < cw;
      cp_async8(bs + rr * FY_BS + c, a.W + (ok ? r * a.ldw + a.c0 + cb + c : 0), ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int ch = 0; ch < FY_ST - 1; ++ch) {
    if (ch < nch) load(ch);
    cp_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    cp_wait<FY_ST - 2>();
    __syncthreads();
    if (ch + FY_ST - 1 < nch) load(ch + FY_ST - 1);
    cp_commit();
    const int st = ch % FY_ST;
    const double* vs = Vs + st * FY_KC * FY_VS;
    const double* bs = Bs + st * FY_KC * FY_BS;
    const int64_t r0 = rlo + static_cast<int64_t>(ch) * FY_KC;
    const bool tri = r0 < a.b0 + ob;  // chunk meets the unit-diagonal triangle of V
#pragma unroll
    for (int k = 0; k < FY_KC; k += 4) {
      const int64_t r = r0 + k + t4;
      double af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = mw * 32 + mt * 8 + g4;
        const double v = vs[(k + t4) * FY_VS + i];
        af[mt] = tri ? vv(v, r, a.b0, i) : v;
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = nw * 32 + nt * 8 + g4;
        const double v = bs[(k + t4) * FY_BS + c];
        bf[nt] = (BV && tri) ? vv(v, r, a.b0, static_cast<int>(cb) + c) : v;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
  }
  cp_wait<0>();
  double* Y = a.Yp + static_cast<int64_t>(blockIdx.y) * FOB * a.Nf;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int i = mw * 32 + mt * 8 + g4, c = nw * 32 + nt * 8 + 2 * t4;
      if (i < ob) {
        if (c < cw) Y[(cb + c) * FOB + i] = acc[mt][nt][0];
        if (c + 1 < cw) Y[(cb + c + 1) * FOB + i] = acc[mt][nt][1];
      }
    }
}

// G[j][i] = sum_s Gp_s[j][i] (fixed order; Gp column-major as Yp, G with row
// stride FOB: G[k * FOB + i] = (V'V)_ki)
__global__ void k_far_gsum(const double* __restrict__ Gp, int S, int ob, double* G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= FOB * FOB) return;
  const int k = e / FOB, i = e - k * FOB;
  double v[8];
  double s = 0.0;
  if (k < ob && i < ob) {
    for (int s0 = 0; s0 < S; s0 += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = s0 + u < S ? __ldcg(Gp + static_cast<int64_t>(s0 + u) * FOB * ob + k * FOB + i) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < S) s += v[u];
    }
  }
  G[e] = s;
}

// Z = T' Y for one column per warp: lane j carries t_j (j = lane + 32 q);
// step i: z_i = tau_i t_i (lane i % 32), broadcast, lanes j > i subtract
// G_ij z_i.  G (128 KB) is read through L1 (no shared memory: the kernel
// fits beside the panel and GEMM kernels it overlaps); a column's partials
// and its Z are contiguous (column-major).
constexpr int FZ_WARPS = 8;
__global__ void __launch_bounds__(32 * FZ_WARPS) k_far_z(FarArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ob = a.ob;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * FZ_WARPS + warp;
  if (c >= a.Nf) return;
  double t[4];
  {
    const double* yp = a.Yp + c * FOB + lane;
    const int64_t stride = static_cast<int64_t>(FOB) * a.Nf;
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = 0.0;
    for (int sp = 0; sp < a.S; ++sp) {
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = lane + 32 * q < ob ? __ldcg(yp + sp * stride + 32 * q) : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] += v[q];
    }
  }
  double tau[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) tau[q] = lane + 32 * q < ob ? __ldg(a.taus + a.b0 + lane + 32 * q) : 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (32 * q >= ob) break;
#pragma unroll 4
    for (int il = 0; il < 32; ++il) {
      const int i = 32 * q + il;
      if (i >= ob) break;
      const double zi = __shfl_sync(FULL, tau[q] * t[q], il);
      const double* gr = a.G + i * FOB + lane;
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        if (q2 < q) continue;
        const int jj = lane + 32 * q2;
        const double g = __ldg(gr + 32 * q2);
        if (jj == i) t[q2] = zi;
        else if (jj > i) t[q2] = fma(-g, zi, t[q2]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int jj = lane + 32 * q;
    if (jj < ob) a.Z[c * FOB + jj] = t[q];
  }
}

// W_far -= V Z on a 128-row x 64-column tile: 8 warps of 32 x 32, the
// accumulators start from W and take the products with -V, k in chunks of
// FA_KC through a double-buffered cp.async ring.
__global__ void __launch_bounds__(FT) k_far_apply(FarArgs a) {
  extern __shared__ __align__(16) double fsm[];
  double* Vs = fsm;                      // 2 x 128 x FA_VS
  double* Zs = Vs + 2 * 128 * FA_VS;     // 2 x FA_KC x FA_ZS
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int mw = warp >> 1, nw = warp & 1;
  const int64_t r0 = a.b0 + static_cast<int64_t>(blockIdx.x) * 128;
  const int rh = static_cast<int>(min(static_cast<int64_t>(128), a.d - r0));
  const int64_t cb = static_cast<int64_t>(blockIdx.y) * 64;
  const int cw = static_cast<int>(min(static_cast<int64_t>(64), a.Nf - cb));
  const int ob = a.ob;
  const int nch = (ob + FA_KC - 1) / FA_KC;
  const bool tri = blockIdx.x == 0;  // rows [b0, b0 + 128) hold V's unit-diagonal triangle
  auto load = [&](int ch) {
    const int st = ch & 1;
    const int k0 = ch * FA_KC;
    double* vs = Vs + st * 128 * FA_VS;
    double* zs = Zs + st * FA_KC * FA_ZS;
    for (int idx = tid; idx < 128 * FA_KC; idx += FT) {
      const int rr = idx / FA_KC, k = idx - rr * FA_KC;
      const bool ok = rr < rh && k0 + k < ob;
      cp_async8(vs + rr * FA_VS + k, a.W + (ok ? (r0 + rr) * a.ldw + a.b0 + k0 + k : 0), ok);
    }
    for (int idx = tid; idx < FA_KC * 64; idx += FT) {
      const int k = idx >> 6, c = idx & 63;
      const bool ok = k0 + k < ob && c < cw;
      cp_async8(zs + k * FA_ZS + c, a.Z + (ok ? (cb + c) * FOB + k0 + k : 0), ok);
    }
  };
  load(0);
  cp_commit();
  double acc[4][4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int rr = mw * 32 + mt * 8 + g4, c = nw * 32 + nt * 8 + 2 * t4;
      const double* wp = a.W + (r0 + rr) * a.ldw + a.c0 + cb + c;
      acc[mt][nt][0] = (rr < rh && c < cw) ? wp[0] : 0.0;
      acc[mt][nt][1] = (rr < rh && c + 1 < cw) ? wp[1] : 0.0;
    }
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) load(ch + 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const int st = ch & 1;
    const double* vs = Vs + st * 128 * FA_VS;
    const double* zs = Zs + st * FA_KC * FA_ZS;
    const int k0 = ch * FA_KC;
#pragma unroll
    for (int k = 0; k < FA_KC; k += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int rr = mw * 32 + mt * 8 + g4;
        const double v = vs[rr * FA_VS + k + t4];
        af[mt] = -(tri ? vv(v, r0 + rr, a.b0, k0 + k + t4) : v);
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = zs[(k + t4) * FA_ZS + nw * 32 + nt * 8 + g4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
    __syncthreads();  // stage st is refilled by the next iteration's load
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int rr = mw * 32 + mt * 8 + g4, c = nw * 32 + nt * 8 + 2 * t4;
      if (rr < rh) {
        double* wp = a.W + (r0 + rr) * a.ldw + a.c0 + cb + c;
        if (c < cw) wp[0] = acc[mt][nt][0];
        if (c + 1 < cw) wp[1] = acc[mt][nt][1];
      }
    }
}

constexpr size_t FY_SMEM = static_cast<size_t>(FY_ST) * FY_KC * (FY_VS + FY_BS) * 8;
constexpr size_t FA_SMEM = static_cast<size_t>(2) * (128 * FA_VS + FA_KC * FA_ZS) * 8;

int far_attrs() {
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_y<false>)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_y<true>)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_apply)));
  return ITSK_OK;
}

}  // namespace

int64_t qr_far_yp_doubles() { return static_cast<int64_t>(FAR_YP_TILES) * FOB * 64; }

int launch_qr_far_gram(double* W, int64_t d, int64_t ldw, int64_t b0, int ob, double* Yp, double* G,
                       cudaStream_t s) {
  int rc = far_attrs();
  if (rc) return rc;
  FarArgs a{};
  a.W = W;
  a.d = d;
  a.ldw = ldw;
  a.b0 = b0;
  a.ob = ob;
  a.c0 = b0;
  a.Nf = ob;
  a.Yp = Yp;
  const int64_t len = d - b0;
  const int ncb = static_cast<int>((ob + 63) / 64);
  int S = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(FAR_YP_TILES / ncb, len / 64)));
  S = std::min(S, 2 * num_sms() / ncb);
  a.S = std::max(1, S);
  k_far_y<true><<<dim3(ncb, a.S), FT, FY_SMEM, s>>>(a);
  k_far_gsum<<<(FOB * FOB + 255) / 256, 256, 0, s>>>(Yp, a.S, ob, G);
  count_launch(2);
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

int launch_qr_far_update(double* W, int64_t d, int64_t ldw, int64_t b0, int ob, int64_t c0, int64_t Nf,
                         const double* G, const double* taus, double* Yp, double* Z, cudaStream_t s) {
  if (Nf <= 0) return ITSK_OK;
  int rc = far_attrs();
  if (rc) return rc;
  FarArgs a{};
  a.W = W;
  a.d = d;
  a.ldw = ldw;
  a.b0 = b0;
  a.ob = ob;
  a.c0 = c0;
  a.Nf = Nf;
  a.Yp = Yp;
  a.G = G;
  a.taus = taus;
  a.Z = Z;
  const int64_t len = d - b0;
  const int ncb = static_cast<int>((Nf + 63) / 64);
  // splits: ~2 CTAs per SM, Yp capacity, >= 64 rows each
  int64_t S = std::max<int64_t>(1, (2 * num_sms() + ncb - 1) / ncb);
  S = std::min<int64_t>(S, std::max<int64_t>(1, FAR_YP_TILES / ncb));
  S = std::min<int64_t>(S, std::max<int64_t>(1, len / 64));
  a.S = static_cast<int>(S);
  k_far_y<false><<<dim3(ncb, a.S), FT, FY_SMEM, s>>>(a);
  k_far_z<<<static_cast<unsigned>((Nf + FZ_WARPS - 1) / FZ_WARPS), 32 * FZ_WARPS, 0, s>>>(a);
  k_far_apply<<<dim3(static_cast<unsigned>((len + 127) / 128), ncb), FT, FA_SMEM, s>>>(a);
  count_launch(3);
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace itsk
