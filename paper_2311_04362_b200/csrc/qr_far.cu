// Far trailing update of the blocked Householder QR (qr2.cu, two-level
// blocking).  The panels of an outer block of OB <= 128 columns [b0, b0+ob)
// are factored (and update each other) first; their reflectors are then
// applied to the far columns [c0, c0+Nf) in one compact-WY step with
// tensor-core tiles:
//
//   Y = V' W_far          k_far_y   (split over row ranges, fixed-order sum)
//   G = V'V, T            k_far_y<true>, k_far_gsum, k_far_t (dlarft's
//                                    recurrence T[0:i,i] = -tau_i T G[0:i,i])
//   Z = T' Y              k_far_z   (a triangular mat-vec per column)
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
#ifdef ITSK_FARPROBE
__device__ unsigned long long g_far_prof[8];
#define FP(i)                                                     \
  do {                                                            \
    __syncthreads();                                              \
    if (threadIdx.x == 0) {                                       \
      const long long _t = clock64();                             \
      atomicAdd(&g_far_prof[i], static_cast<unsigned long long>(_t - _fp0)); \
      _fp0 = _t;                                                  \
    }                                                             \
  } while (0)
#else
#define FP(i) \
  do {        \
  } while (0)
#endif
namespace {

constexpr int FT = 256;          // threads per CTA
constexpr int FOB = 128;         // max block width (rows of Y / Z)
constexpr int FY_KC = 16;        // rows per stage in k_far_y
constexpr int FY_ST = 4;         // stages
constexpr int FY_VS = FOB + 8;   // [k][i] tiles: stride = 8 (mod 16) doubles -> conflict-free fragments
constexpr int FY_BS = 64 + 8;
constexpr int FA_KC = 32;        // k per stage in k_far_apply

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
// 16 bytes, the first `src_bytes` (0, 8 or 16) from global, the rest zero
__device__ __forceinline__ void cp_async16z(double* dst, const double* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
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
  const double* G;     // FOB x FOB: the block's T (k_far_t), read by k_far_z
  const double* taus;  // global tau array, indexed b0 + i
  double* Z;           // Nf x FOB (column-major, like Yp), stored NEGATED (-T'Y) for k_far_apply
  int vec16;           // W 16-byte aligned, even ldw, b0 and c0 even: 16-byte copies
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
    if (a.vec16) {
      for (int idx = tid; idx < FY_KC * (FOB / 2); idx += FT) {
        const int rr = idx / (FOB / 2), i = 2 * (idx - rr * (FOB / 2));
        const int64_t r = r0 + rr;
        const int sv = r < rhi ? 8 * max(0, min(2, ob - i)) : 0;
        cp_async16z(vs + rr * FY_VS + i, a.W + (sv ? r * a.ldw + a.b0 + i : 0), sv);
      }
      for (int idx = tid; idx < FY_KC * 32; idx += FT) {
        const int rr = idx >> 5, c = 2 * (idx & 31);
        const int64_t r = r0 + rr;
        const int sb = r < rhi ? 8 * max(0, min(2, cw - c)) : 0;
        cp_async16z(bs + rr * FY_BS + c, a.W + (sb ? r * a.ldw + a.c0 + cb + c : 0), sb);
      }
      return;
    }
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
    // chunks meeting V's unit-diagonal triangle select per element; the
    // others (all but the first few of split 0) use the stored values as is
    auto step = [&](auto tri_c) {
      constexpr bool TRI = decltype(tri_c)::value;
#pragma unroll
      for (int k = 0; k < FY_KC; k += 4) {
        const int64_t r = r0 + k + t4;
        double af[4], bf[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int i = mw * 32 + mt * 8 + g4;
          const double v = vs[(k + t4) * FY_VS + i];
          af[mt] = TRI ? vv(v, r, a.b0, i) : v;
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int c = nw * 32 + nt * 8 + g4;
          const double v = bs[(k + t4) * FY_BS + c];
          bf[nt] = (BV && TRI) ? vv(v, r, a.b0, static_cast<int>(cb) + c) : v;
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
      }
    };
    if (r0 < a.b0 + ob) step(std::true_type{});
    else step(std::false_type{});
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

// T of the block (upper triangular, FOB x FOB, row stride FOB), dlarft's T
// for V = [V_1 .. V_8] (16-column blocks), one CTA, by blocks: with T1 the
// finished leading j0 x j0 part and T_JJ the diagonal block of the next 16
// columns J,
//   T_JJ            dlarft's column recurrence on the 16 x 16 block alone
//                   (T[i][i] = tau_i, T[a][b] = -tau_b sum_{a<=k<b} T[a][k] G[k][b]);
//                   each lane owns a row and needs only its own row's
//                   earlier entries: one warp per block, all 8 at once
//   T[0:j0, J]    = -(T1 G[0:j0, J]) T_JJ     two parallel products, J = 1..7
// (T = [T1, -T1 V1'V2 T2; 0, T2], the recursive form of dlarft).  A zero
// tau gives a zero column (T_JJ's column b and so T[0:j0, b]), as dlarft.
// Z = T'Y then needs no sequential substitution (k_far_z).
constexpr int FT_THREADS = 512;
constexpr int FT_BLK = 16;
constexpr int FT_NB = FOB / FT_BLK;                        // diagonal blocks
constexpr int FT_GC = FT_BLK * FT_BLK * FT_NB * (FT_NB - 1) / 2;  // G[0:j0, J] for all J, [k][c]
constexpr size_t ft_smem() {
  return static_cast<size_t>(FOB * (FOB + 1) + FT_GC + FT_NB * FT_BLK * FT_BLK + FOB * FT_BLK) * 8;
}
__global__ void __launch_bounds__(FT_THREADS) k_far_t(const double* G, const double* __restrict__ taus,
                                                      int64_t b0, int ob, double* T) {
  extern __shared__ __align__(16) double tsm[];  // T: FOB x (FOB + 1) | Gc | Gd | P
  constexpr int TS = FOB + 1;
  double* Gc = tsm + FOB * TS;                   // block J's G[0:j0, J] at Gc + 256 J (J - 1) / 2, [k][c]
  double* Gd = Gc + FT_GC;                       // G's diagonal blocks, Gd[J][k][c]
  double* P = Gd + FT_NB * FT_BLK * FT_BLK;      // P[r * FT_BLK + c] = (T1 G[0:j0, J])[r][c]
  __shared__ double ts[FOB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef ITSK_FARPROBE
  long long _fp0 = clock64();
#endif
  const int nbk = (ob + FT_BLK - 1) / FT_BLK;
  for (int e = tid; e < FOB * TS; e += FT_THREADS) tsm[e] = 0.0;
  // every G element the recurrence reads, loaded up front (all in flight):
  // the diagonal blocks and, per block J, the rows above it
  for (int e = tid; e < FT_NB * FT_BLK * FT_BLK; e += FT_THREADS) {
    const int J = e >> 8, k = (e >> 4) & 15, c = e & 15;
    const int gk = J * FT_BLK + k, gc = J * FT_BLK + c;
    Gd[e] = (gk < ob && gc < ob) ? __ldcg(G + gk * FOB + gc) : 0.0;
  }
  for (int e = tid; e < FT_GC; e += FT_THREADS) {
    // e = 256 J (J - 1) / 2 + k * 16 + c with k < 16 J
    int J = 1;
    while (J + 1 < FT_NB && FT_BLK * FT_BLK * (J + 1) * J / 2 <= e) ++J;
    const int off = e - FT_BLK * FT_BLK * J * (J - 1) / 2;
    const int k = off >> 4, c = off & 15, gc = J * FT_BLK + c;
    Gc[e] = gc < ob ? __ldcg(G + k * FOB + gc) : 0.0;
  }
  if (tid < FOB) ts[tid] = tid < ob ? taus[b0 + tid] : 0.0;
  __syncthreads();
  FP(0);
  // (a) every diagonal block T_JJ (they depend on G_JJ and tau only): warp
  // J, lane a owns row a of the block and needs only its own row's earlier
  // entries (dlarft's recurrence T[a][b] = -tau_b sum_{a<=k<b} T[a][k] G[k][b])
  if (warp < nbk && lane < FT_BLK) {
    const int j0 = warp * FT_BLK, bw = min(FT_BLK, ob - j0);
    const double* gd = Gd + warp * FT_BLK * FT_BLK;
    double row[FT_BLK];
#pragma unroll
    for (int b = 0; b < FT_BLK; ++b) row[b] = 0.0;
#pragma unroll
    for (int b = 0; b < FT_BLK; ++b) {
      const double tb = b < bw ? ts[j0 + b] : 0.0;
      if (b == lane) {
        row[b] = tb;
      } else if (b > lane) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k < FT_BLK; k += 2) {
          if (k >= lane && k < b) s0 = fma(row[k], gd[k * FT_BLK + b], s0);
          if (k + 1 >= lane && k + 1 < b) s1 = fma(row[k + 1], gd[(k + 1) * FT_BLK + b], s1);
        }
        row[b] = -tb * (s0 + s1);
      }
    }
    if (lane < bw)
#pragma unroll
      for (int b = 0; b < FT_BLK; ++b)
        if (b < bw) tsm[(j0 + lane) * TS + j0 + b] = row[b];
  }
  __syncthreads();
  FP(2);
  // (b) T[0:j0, J] = -(T1 G[0:j0, J]) T_JJ, block after block
  for (int J = 1; J < nbk; ++J) {
    const int j0 = J * FT_BLK, bw = min(FT_BLK, ob - j0);
    const double* gc = Gc + FT_BLK * FT_BLK * J * (J - 1) / 2;
    // P: thread (r, c), 4 independent chains over k; 16 lanes share row r
    for (int e = tid; e < j0 * FT_BLK; e += FT_THREADS) {
      const int r = e / FT_BLK, c = e - r * FT_BLK;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const double* tr = tsm + r * TS;
      int k = r;
      for (; k + 3 < j0; k += 4) {
        a0 = fma(tr[k], gc[k * FT_BLK + c], a0);
        a1 = fma(tr[k + 1], gc[(k + 1) * FT_BLK + c], a1);
        a2 = fma(tr[k + 2], gc[(k + 2) * FT_BLK + c], a2);
        a3 = fma(tr[k + 3], gc[(k + 3) * FT_BLK + c], a3);
      }
      for (; k < j0; ++k) a0 = fma(tr[k], gc[k * FT_BLK + c], a0);
      P[e] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();
    FP(1);
    for (int e = tid; e < j0 * FT_BLK; e += FT_THREADS) {
      const int r = e / FT_BLK, c = e - r * FT_BLK;
      if (c >= bw) continue;
      double sum = 0.0;
      for (int k = 0; k <= c; ++k) sum = fma(P[r * FT_BLK + k], tsm[(j0 + k) * TS + j0 + c], sum);
      tsm[r * TS + j0 + c] = -sum;
    }
    __syncthreads();
    FP(3);
  }
  for (int e = tid; e < FOB * FOB; e += FT_THREADS) {
    const int rr = e / FOB, c = e - rr * FOB;
    T[e] = (rr < ob && c < ob) ? tsm[rr * TS + c] : 0.0;
  }
  FP(4);
}

// Z = T'Y, one column per warp: lane j holds z_j for j = lane + 32 q; y_k is
// the fixed-order sum of the split partials, broadcast by shuffle; z_j =
// sum_{k <= j} T_kj y_k in ascending k.  Y partials and Z are column-major
// (a column's FOB values contiguous); T is read through L1.
constexpr int FZ_WARPS = 8;
constexpr int FZ_CPW = 2;  // columns per warp, both at once (independent chains)
constexpr size_t FZ_SMEM = static_cast<size_t>(FOB) * FOB * 8;
__global__ void __launch_bounds__(32 * FZ_WARPS) k_far_z(FarArgs a) {
  extern __shared__ __align__(16) double Ts[];  // the block's T (k_far_t), FOB x FOB
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ob = a.ob;
  // T into shared memory first: the substitution-free mat-vec then reads it
  // at shared-memory latency (from L2 each of its ob steps waited ~1 us)
  if ((reinterpret_cast<uintptr_t>(a.G) & 15) == 0) {
    for (int e = 2 * tid; e < FOB * FOB; e += 2 * 32 * FZ_WARPS) cp_async16z(Ts + e, a.G + e, 16);
  } else {
    for (int e = tid; e < FOB * FOB; e += 32 * FZ_WARPS) cp_async8(Ts + e, a.G + e, true);
  }
  cp_commit();
  const int64_t stride = static_cast<int64_t>(FOB) * a.Nf;
  // y of columns c0, c1 (c1 < 0: none): the split partials in ascending
  // split order, 8 splits of both columns in flight per round
  auto ysum2 = [&](int64_t c0, int64_t c1, double (&y0)[4], double (&y1)[4]) {
    const double* yp0 = a.Yp + c0 * FOB + lane;
    const double* yp1 = a.Yp + (c1 >= 0 ? c1 : c0) * FOB + lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) y0[q] = y1[q] = 0.0;
    for (int s0 = 0; s0 < a.S; s0 += 8) {
      double v0[8][4], v1[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool ok = s0 + u < a.S && lane + 32 * q < ob;
          v0[u][q] = ok ? __ldcg(yp0 + (s0 + u) * stride + 32 * q) : 0.0;
          v1[u][q] = ok && c1 >= 0 ? __ldcg(yp1 + (s0 + u) * stride + 32 * q) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < a.S)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            y0[q] += v0[u][q];
            y1[q] += v1[u][q];
          }
    }
  };
  cp_wait<0>();
  __syncthreads();
  for (int cc = 0; cc < FZ_CPW; cc += 2) {
    const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * FZ_WARPS + warp) * FZ_CPW + cc;
    if (c0 >= a.Nf) break;
    const bool two = c0 + 1 < a.Nf;
    double y0[4], y1[4];
    ysum2(c0, two ? c0 + 1 : -1, y0, y1);
    double z0[4] = {0.0, 0.0, 0.0, 0.0}, z1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (32 * q >= ob) break;
#pragma unroll 8
      for (int kl = 0; kl < 32; ++kl) {
        const int k = 32 * q + kl;
        if (k >= ob) break;
        const double yk0 = __shfl_sync(FULL, y0[q], kl), yk1 = __shfl_sync(FULL, y1[q], kl);
        const double* tr = Ts + k * FOB + lane;
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          if (q2 < q) continue;
          const int j = lane + 32 * q2;
          if (k <= j) {
            const double t = tr[32 * q2];
            z0[q2] = fma(t, yk0, z0[q2]);
            z1[q2] = fma(t, yk1, z1[q2]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = lane + 32 * q;
      if (j < ob) {
        a.Z[c0 * FOB + j] = -z0[q];  // negated: k_far_apply accumulates W + V (-Z)
        if (two) a.Z[(c0 + 1) * FOB + j] = -z1[q];
      }
    }
  }
}

// W_far -= V Z on a 128-row x 64-column tile: 8 warps of 32 x 32, the
// accumulators start from W and take the products V (-Z) (k_far_z stores Z
// negated), k in chunks of FA_KC through a double-buffered cp.async ring.
// Shared tiles [row][k] for V and [col][k] for Z, 32 doubles per row with the
// 16-byte column index XOR-swizzled by the row's parity: each thread reads
// the k pair (2 t4, 2 t4 + 1) of its fragment row with ONE 16-byte load and
// feeds two DMMAs (the k = 8-step splits into the even and the odd k of the
// pairs), and the 8 lanes of every quarter-warp hit 8 distinct 16-byte bank
// groups.
__device__ __forceinline__ int fa_sw(int row, int k) { return row * FA_KC + (((k >> 1) ^ ((row & 1) << 2)) << 1); }

template <bool TRI>
__device__ __forceinline__ void far_apply_body(const FarArgs& a, double* Vs, double* Zs) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int mw = warp >> 1, nw = warp & 1;
  const int64_t r0 = a.b0 + static_cast<int64_t>(blockIdx.x) * 128;
  const int rh = static_cast<int>(min(static_cast<int64_t>(128), a.d - r0));
  const int64_t cb = static_cast<int64_t>(blockIdx.y) * 64;
  const int cw = static_cast<int>(min(static_cast<int64_t>(64), a.Nf - cb));
  const int ob = a.ob;
  const int nch = (ob + FA_KC - 1) / FA_KC;
  auto load = [&](int ch) {
    const int st = ch & 1;
    const int k0 = ch * FA_KC;
    double* vs = Vs + st * 128 * FA_KC;
    double* zs = Zs + st * 64 * FA_KC;
    if (a.vec16) {
      for (int idx = tid; idx < 128 * (FA_KC / 2); idx += FT) {
        const int rr = idx / (FA_KC / 2), k = 2 * (idx - rr * (FA_KC / 2));
        const int sv = rr < rh ? 8 * max(0, min(2, ob - k0 - k)) : 0;
        cp_async16z(vs + fa_sw(rr, k), a.W + (sv ? (r0 + rr) * a.ldw + a.b0 + k0 + k : 0), sv);
      }
      for (int idx = tid; idx < 64 * (FA_KC / 2); idx += FT) {
        const int c = idx / (FA_KC / 2), k = 2 * (idx - c * (FA_KC / 2));
        const int sz = c < cw ? 8 * max(0, min(2, ob - k0 - k)) : 0;
        cp_async16z(zs + fa_sw(c, k), a.Z + (sz ? (cb + c) * FOB + k0 + k : 0), sz);
      }
      return;
    }
    for (int idx = tid; idx < 128 * FA_KC; idx += FT) {
      const int rr = idx / FA_KC, k = idx - rr * FA_KC;
      const bool ok = rr < rh && k0 + k < ob;
      cp_async8(vs + fa_sw(rr, k) + (k & 1), a.W + (ok ? (r0 + rr) * a.ldw + a.b0 + k0 + k : 0), ok);
    }
    for (int idx = tid; idx < 64 * FA_KC; idx += FT) {
      const int c = idx / FA_KC, k = idx - c * FA_KC;
      const bool ok = k0 + k < ob && c < cw;
      cp_async8(zs + fa_sw(c, k) + (k & 1), a.Z + (ok ? (cb + c) * FOB + k0 + k : 0), ok);
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
    const double* vs = Vs + st * 128 * FA_KC;
    const double* zs = Zs + st * 64 * FA_KC;
    const int k0 = ch * FA_KC;
#pragma unroll
    for (int k = 0; k < FA_KC; k += 8) {
      double2 af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int rr = mw * 32 + mt * 8 + g4;
        af[mt] = *reinterpret_cast<const double2*>(vs + fa_sw(rr, k + 2 * t4));
        if (TRI) {
          af[mt].x = vv(af[mt].x, r0 + rr, a.b0, k0 + k + 2 * t4);
          af[mt].y = vv(af[mt].y, r0 + rr, a.b0, k0 + k + 2 * t4 + 1);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        bf[nt] = *reinterpret_cast<const double2*>(zs + fa_sw(nw * 32 + nt * 8 + g4, k + 2 * t4));
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt].x, bf[nt].x);
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt].y, bf[nt].y);
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

__global__ void __launch_bounds__(FT, 2) k_far_apply(FarArgs a) {
  extern __shared__ __align__(16) double fsm[];
  double* Vs = fsm;                   // 2 x 128 x FA_KC
  double* Zs = Vs + 2 * 128 * FA_KC;  // 2 x 64 x FA_KC
  // rows [b0, b0 + 128) hold V's unit-diagonal triangle
  if (blockIdx.x == 0) far_apply_body<true>(a, Vs, Zs);
  else far_apply_body<false>(a, Vs, Zs);
}

constexpr size_t FY_SMEM = static_cast<size_t>(FY_ST) * FY_KC * (FY_VS + FY_BS) * 8;
constexpr size_t FA_SMEM = static_cast<size_t>(2) * (128 + 64) * FA_KC * 8;

int far_attrs() {
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_y<false>)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_y<true>)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_apply)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_t)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_far_z)));
  return ITSK_OK;
}

}  // namespace

int64_t qr_far_yp_doubles() { return static_cast<int64_t>(FAR_YP_TILES) * FOB * 64; }

int launch_qr_far_gram(double* W, int64_t d, int64_t ldw, int64_t b0, int ob, const double* taus, double* Yp,
                       double* G, cudaStream_t s, cudaStream_t t_stream, cudaEvent_t ev_handoff) {
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
  a.vec16 = ((ldw | b0) & 1) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  const int64_t len = d - b0;
  const int ncb = static_cast<int>((ob + 63) / 64);
  int S = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(FAR_YP_TILES / ncb, len / 64)));
  S = std::min(S, 2 * num_sms() / ncb);
  a.S = std::max(1, S);
  k_far_y<true><<<dim3(ncb, a.S), FT, FY_SMEM, s>>>(a);
  k_far_gsum<<<(FOB * FOB + 255) / 256, 256, 0, s>>>(Yp, a.S, ob, G);
  count_launch(2);
  if (t_stream == nullptr) t_stream = s;
  else if (t_stream != s) {
    ITSK_CUDA(cudaEventRecord(ev_handoff, s));
    ITSK_CUDA(cudaStreamWaitEvent(t_stream, ev_handoff, 0));
  }
  // T from G and tau, written over G (read completely before the first write)
  k_far_t<<<1, FT_THREADS, ft_smem(), t_stream>>>(G, taus, b0, ob, G);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

int launch_qr_far_update(double* W, int64_t d, int64_t ldw, int64_t b0, int ob, int64_t c0, int64_t Nf,
                         const double* G, const double* taus, double* Yp, double* Z, cudaStream_t s, int parts) {
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
  a.vec16 = ((ldw | b0 | c0) & 1) == 0 && ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(Z)) & 15) == 0;
  const int64_t len = d - b0;
  const int ncb = static_cast<int>((Nf + 63) / 64);
  // splits: ~2 CTAs per SM, Yp capacity, >= 64 rows each
  int64_t S = std::max<int64_t>(1, (2 * num_sms() + ncb - 1) / ncb);
  S = std::min<int64_t>(S, std::max<int64_t>(1, FAR_YP_TILES / ncb));
  S = std::min<int64_t>(S, std::max<int64_t>(1, len / 64));
  a.S = static_cast<int>(S);
  if (parts & 1) {
    k_far_y<false><<<dim3(ncb, a.S), FT, FY_SMEM, s>>>(a);
    count_launch();
  }
  if (parts & 2) {
    k_far_z<<<static_cast<unsigned>((Nf + FZ_WARPS * FZ_CPW - 1) / (FZ_WARPS * FZ_CPW)), 32 * FZ_WARPS, FZ_SMEM,
              s>>>(a);
    k_far_apply<<<dim3(static_cast<unsigned>((len + 127) / 128), ncb), FT, FA_SMEM, s>>>(a);
    count_launch(2);
  }
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace itsk

#ifdef ITSK_FARPROBE
extern "C" void itsk_farprobe_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, itsk::g_far_prof, sizeof(unsigned long long) * 8);
}
#endif
