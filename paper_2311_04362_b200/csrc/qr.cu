// Householder QR of the augmented sketch [SA | Sb] (K2).
//
// Replaces householder_qr_econ (/root/reference/pkg/src/itsketch/linalg.py:30-47,
// LAPACK dgeqrf + dorgqr, then diag(R) >= 0) and the x0 right-hand side
// Q'·Sb (solvers.py:209).  Blocked right-looking Householder with LAPACK's
// dlarfg convention (beta = -sign(alpha) ||x||) and dlarft/dlarfb compact-WY
// trailing updates, run as ONE kernel whose CTAs each own a contiguous block
// of rows for the whole factorisation.  Q is never formed: the reflectors are
// applied to the Sb column like any other trailing column, which yields
// z = (Q'Sb)[:n] directly.
//
// Per column there is exactly ONE cross-CTA exchange: every CTA publishes
// [sum_{r>j} x_r^2, sum_{r>j} x_r a_rc (c in the panel)] for its rows (and
// the owner of row j appends row j), after which every CTA forms beta, tau
// and v'a_c = a_jc + scal * sum_{r>j} x_r a_rc locally — the quantities
// dgeqr2 computes with two passes (dnrm2, then dlarf's dgemv).  The CTA's
// rows of the current 32-wide panel live in shared memory.
//
// Two launch shapes share the code:
//   cluster mode  one thread-block cluster of <= 16 CTAs (small d, e.g. C2
//                 d = 4000): records are exchanged through distributed shared
//                 memory and synchronisation is barrier.cluster;
//   grid mode     a cooperative grid of up to 148 CTAs (large d): records in
//                 global memory, software grid barrier.
// All cross-CTA sums run in fixed CTA order, so R is bitwise reproducible and
// identical on every CTA.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "itsk_common.cuh"
#include "itsk_kernels.cuh"

namespace cg = cooperative_groups;

namespace itsk {
namespace {

constexpr int NB = 32;
constexpr int PSL = NB + 1;  // padded row stride of the panel cache: column walks are conflict-free
constexpr int QR_THREADS = 512;
constexpr int QR_WARPS = QR_THREADS / 32;
constexpr int REC = 2 * NB;  // [S_c (NB) | row j of the panel (NB, owner only)]

struct QrArgs {
  double* W;
  int64_t d, n, ldw, N;  // N = n + 1 (Sb column) or n
  double* R;
  double* z;
  int* singular;
  // grid-mode exchange buffers (global)
  double* grec;  // 2 x P x REC
  double* ggy;   // P x NB x (NB + N)
  double* gz;    // NB x N
  unsigned* bar;
  int64_t hmax;
};

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ int64_t split_lo(int q, int P, int64_t len) {
  return (static_cast<int64_t>(q) * len) / P;
}

// CTA q of P owning index j of a range of length len split by split_lo.
__device__ __forceinline__ int split_owner(int64_t j, int P, int64_t len) {
  int q = static_cast<int>((j * P) / len);
  while (q > 0 && split_lo(q, P, len) > j) --q;
  while (q + 1 < P && split_lo(q + 1, P, len) <= j) ++q;
  return q;
}

// Exchange through global memory + software grid barrier.
struct XGrid {
  double* rec;
  double* gy;
  double* z;
  unsigned* bar;
  int P, p;
  int64_t ldgy, N;
  // publish this CTA's record (n entries of `local`) before the exchange sync
  __device__ void publish(int buf, const double* local, int cnt) const {
    double* dst = rec + (static_cast<int64_t>(buf) * P + p) * REC;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = local[i];
  }
  __device__ double rec_r(int buf, int q, int i) const {
    return ldcg(rec + (static_cast<int64_t>(buf) * P + q) * REC + i);
  }
  __device__ double* gy_w() const { return gy + static_cast<int64_t>(p) * NB * ldgy; }
  __device__ double gy_r(int q, int jj, int64_t c) const {
    return ldcg(gy + (static_cast<int64_t>(q) * NB + jj) * ldgy + c);
  }
  // Z (NB x trailing columns) in global, ld N; CTA p writes its column slice.
  __device__ double* z_slice(int64_t c_lo) const { return z + c_lo; }
  __device__ int64_t z_ld() const { return N; }
  __device__ double z_at(int jj, int64_t c, int64_t) const { return ldcg(z + jj * N + c); }
  __device__ void sync() const { grid_barrier(bar); }
};

// Exchange through distributed shared memory inside one cluster.
struct XCluster {
  double* rec;  // local smem inbox, 2 x P x REC: every CTA pushes its record here
  double* gy;   // local smem, NB x ldgy
  double* z;    // local smem, NB x zld: this CTA's column slice of Z
  int P, p;
  int64_t ldgy, N, zld;
  // push model: remote stores into every CTA's inbox before the barrier, so
  // the reads after it are local (remote loads would sit on the critical path)
  __device__ void publish(int buf, const double* local, int cnt) const {
    cg::cluster_group cl = cg::this_cluster();
    for (int e = threadIdx.x; e < P * cnt; e += blockDim.x) {
      const int q = e / cnt, i = e - q * cnt;
      cl.map_shared_rank(rec, q)[(buf * P + p) * REC + i] = local[i];
    }
  }
  __device__ double rec_r(int buf, int q, int i) const { return rec[(buf * P + q) * REC + i]; }
  __device__ double* gy_w() const { return gy; }
  __device__ double gy_r(int q, int jj, int64_t c) const {
    const double* g = cg::this_cluster().map_shared_rank(gy, q);
    return g[jj * ldgy + c];
  }
  __device__ double* z_slice(int64_t) const { return z; }
  __device__ int64_t z_ld() const { return zld; }
  // Z[jj][c] (c trailing-relative) from the CTA whose slice holds column c
  __device__ double z_at(int jj, int64_t c, int64_t Nt) const {
    const int q = split_owner(c, P, Nt);
    const int64_t qlo = split_lo(q, P, Nt);
    const double* zq = cg::this_cluster().map_shared_rank(z, q);
    return zq[jj * zld + (c - qlo)];
  }
  __device__ void sync() const { cg::this_cluster().sync(); }
};

// fp64 tensor-core tile: D(8x8) += A(8x4) * B(4x8)  (DMMA.8x8x4 on sm_100a).
// Fragments (PTX m8n8k4 .f64): a = A[g][t], b = B[t][g], d = D[g][2t + {0,1}],
// with g = lane / 4 and t = lane % 4.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int RT = 32;        // row tile of the trailing update
constexpr int CB = 64;        // column chunk of the trailing update
constexpr int CBP = CB + 4;   // padded stride of the staged tiles

#ifdef ITSK_QR_PROFILE
__device__ unsigned long long g_qr_prof[16];
#define QPROF(i) do { __syncthreads(); if (threadIdx.x == 0 && x.p == 0) { long long _t = clock64(); _qacc[i] += _t - _qt; _qt = _t; } } while (0)
#else
#define QPROF(i) do { } while (0)
#endif

template <class X>
__device__ void qr_body(const QrArgs& a, const X& x, double* sm) {
#ifdef ITSK_QR_PROFILE
  long long _qt = clock64();
  long long _qacc[12] = {0};
#endif
  const int P = x.P, p = x.p, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int64_t d = a.d, n = a.n, ldw = a.ldw, N = a.N;
  double* W = a.W;
  const int64_t lo = split_lo(p, P, d), hi = split_lo(p + 1, P, d);
  const int64_t h = hi - lo;
  double* Ps = sm;                 // hmax x PSL: own rows of the current panel
  double* Ts = Ps + a.hmax * PSL;  // NB x NB
  double* Gs = Ts + NB * NB;       // NB x NB (also row j of the panel)
  double* wv = Gs + NB * NB;       // NB
  double* betas = wv + NB;         // n, identical on every CTA
  double* taus = betas + n;        // NB, current panel
  double* tile = taus + NB;        // RT x CBP: staged W tile / Y staging
  double* Zs = tile + RT * CBP;    // NB x CBP: staged Z chunk
  int owner = 0;  // owner CTA of row j, advanced monotonically

  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int kb = static_cast<int>(min(static_cast<int64_t>(NB), n - k0));
    for (int idx = tid; idx < static_cast<int>(h) * NB; idx += QR_THREADS) {
      const int rr = idx / NB, c = idx % NB;
      const int64_t r = lo + rr;
      Ps[rr * PSL + c] = (c < kb && r >= k0) ? W[r * ldw + k0 + c] : 0.0;
    }
    __syncthreads();
    // ---------------- panel: dgeqr2 with one exchange per column ----------------
    for (int jj = 0; jj < kb; ++jj) {
      const int64_t j = k0 + jj;
      const int buf = static_cast<int>(j & 1);  // records double-buffered by parity
      while (owner + 1 < P && split_lo(owner + 1, P, d) <= j) ++owner;
      double* rec = Gs + 128;  // local staging of this CTA's record
      const int ncol = kb - jj;
      const int64_t rs = max(lo, j + 1);
      const int c0 = warp, c1 = warp + QR_WARPS;  // each warp: two panel columns
      QPROF(0);
      if (c0 < ncol) {
        double s0 = 0.0, s1 = 0.0;
        for (int64_t r = rs + lane; r < hi; r += 32) {
          const double* row = Ps + (r - lo) * PSL + jj;
          const double xr = row[0];
          s0 = fma(xr, row[c0], s0);
          if (c1 < ncol) s1 = fma(xr, row[c1], s1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s0 += __shfl_xor_sync(FULL, s0, o);
          s1 += __shfl_xor_sync(FULL, s1, o);
        }
        if (lane == 0) {
          rec[c0] = s0;
          if (c1 < ncol) rec[c1] = s1;
        }
      }
      if (p == owner)
        for (int cc = tid; cc < ncol; cc += QR_THREADS) rec[NB + cc] = Ps[(j - lo) * PSL + jj + cc];
      __syncthreads();
      x.publish(buf, rec, p == owner ? REC : ncol);
      QPROF(1);
      x.sync();
      QPROF(2);
      if (tid >= QR_THREADS - 32 && tid - (QR_THREADS - 32) < ncol)
        Gs[tid - (QR_THREADS - 32)] = x.rec_r(buf, owner, NB + tid - (QR_THREADS - 32));
      if (c0 < ncol) {
        double s0 = 0.0, s1 = 0.0;
        for (int q = lane; q < P; q += 32) {
          s0 += x.rec_r(buf, q, c0);
          if (c1 < ncol) s1 += x.rec_r(buf, q, c1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s0 += __shfl_xor_sync(FULL, s0, o);
          s1 += __shfl_xor_sync(FULL, s1, o);
        }
        if (lane == 0) {
          wv[c0] = s0;
          if (c1 < ncol) wv[c1] = s1;
        }
      }
      __syncthreads();
      QPROF(3);
      // every thread forms the same dlarfg coefficients (no broadcast needed)
      const double xn2 = wv[0];
      const double alpha = Gs[0];
      double beta, tau, scal;
      if (xn2 == 0.0) {  // dlarfg: H = I
        tau = 0.0;
        beta = alpha;
        scal = 1.0;
      } else {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (tid == 0) {
        betas[j] = beta;
        taus[jj] = tau;
      }
      QPROF(4);
      if (tau != 0.0) {
        // warp per row, lane per panel column: a_rc += v_r * temp_c with
        // temp_c = -tau * (a_jc + scal * sum_{r>j} x_r a_rc), v_r = scal * x_r, v_j = 1
        const int cc = lane;
        const double temp = (cc > 0 && cc < ncol) ? -tau * (Gs[cc] + scal * wv[cc]) : 0.0;
        for (int64_t r = max(lo, j) + warp; r < hi; r += QR_WARPS) {
          double* row = Ps + (r - lo) * PSL + jj;
          const double xr = row[0];
          const double vr = (r == j) ? 1.0 : xr * scal;
          if (cc > 0 && cc < ncol) row[cc] += vr * temp;
          __syncwarp();
          if (lane == 0 && r != j) row[0] = vr;
        }
      }
      __syncthreads();
      QPROF(5);
    }
    for (int idx = tid; idx < static_cast<int>(h) * NB; idx += QR_THREADS) {
      const int rr = idx / NB, c = idx % NB;
      const int64_t r = lo + rr;
      if (c < kb && r >= k0) W[r * ldw + k0 + c] = Ps[rr * PSL + c];
    }
    // ---------------- trailing update: W -= V T' (V'W)  (dlarft + dlarfb) -----------
    const int64_t ct0 = k0 + kb;
    const int64_t Nt = N - ct0;
    if (Nt <= 0) {
      __syncthreads();
      continue;
    }
    for (int idx = tid; idx < static_cast<int>(h) * NB; idx += QR_THREADS) {
      const int rr = idx / NB, c = idx % NB;
      const int64_t r = lo + rr;
      if (c >= kb || r < k0 + c) Ps[rr * PSL + c] = 0.0;
      else if (r == k0 + c) Ps[rr * PSL + c] = 1.0;
    }
    __syncthreads();
    const int64_t r0 = max(lo, k0);
    const int hv = hi > r0 ? static_cast<int>(hi - r0) : 0;
    const double* V = Ps + (r0 - lo) * PSL;
    QPROF(6);
    // (1) partial [G | Y] = V_own' [V_own | W_own(:, ct0:)] on DMMA tiles:
    //     M = 32 (reflectors), N = CB columns per chunk, K = own rows.
    double* gyw = x.gy_w();
    const int ncols3 = kb + static_cast<int>(Nt);
    for (int cb = 0; cb < ncols3; cb += CB) {
      const int cw = min(CB, ncols3 - cb);
      double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};
      for (int rt = 0; rt < hv; rt += RT) {
        const int rh = min(RT, hv - rt);
        __syncthreads();
        for (int idx = tid; idx < RT * CB; idx += QR_THREADS) {
          const int rr = idx / CB, c = idx % CB, cg_ = cb + c;
          double v = 0.0;
          if (rr < rh && c < cw)
            v = (cg_ < kb) ? V[(rt + rr) * PSL + cg_] : W[(r0 + rt + rr) * ldw + ct0 + cg_ - kb];
          tile[rr * CBP + c] = v;
        }
        __syncthreads();
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          const int T = warp * 2 + tt;  // 32 output tiles: 4 (M) x 8 (N)
          const int mt = T >> 3, nt = T & 7;
#pragma unroll
          for (int k = 0; k < RT; k += 4) {
            const int rr = k + t4;
            const double av = (rr < rh) ? V[(rt + rr) * PSL + mt * 8 + g4] : 0.0;
            const double bv = tile[rr * CBP + nt * 8 + g4];
            dmma_8x8x4(d0[tt], d1[tt], av, bv);
          }
        }
      }
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const int T = warp * 2 + tt;
        const int mt = T >> 3, nt = T & 7;
        const int jj = mt * 8 + g4, c = nt * 8 + t4 * 2;
        if (jj < kb) {
          if (c < cw) gyw[jj * x.ldgy + cb + c] = d0[tt];
          if (c + 1 < cw) gyw[jj * x.ldgy + cb + c + 1] = d1[tt];
        }
      }
    }
    QPROF(7);
    x.sync();
    QPROF(8);
    // (2) G = V'V (fixed CTA order) and T (dlarft, forward / columnwise), on every CTA
    for (int idx = tid; idx < kb * kb; idx += QR_THREADS) {
      const int jj = idx / kb, kk = idx % kb;
      double s = 0.0;
      for (int q = 0; q < P; ++q) s += x.gy_r(q, jj, kk);
      Gs[jj * NB + kk] = s;
    }
    __syncthreads();
    if (warp == 0) {  // lane k owns row k of T
      for (int i = 0; i < kb; ++i) {
        const double ti = taus[i];
        const double g = (lane < i) ? -ti * Gs[lane * NB + i] : 0.0;
        double acc = 0.0;
        for (int l = 0; l < i; ++l) {
          const double gl = __shfl_sync(FULL, g, l);
          if (lane <= l) acc += Ts[lane * NB + l] * gl;
        }
        if (lane < i) Ts[lane * NB + i] = (ti == 0.0) ? 0.0 : acc;
        if (lane == i) Ts[i * NB + i] = ti;
        if (lane > i) Ts[lane * NB + i] = 0.0;
        __syncwarp();
      }
    }
    __syncthreads();
    // (3) this CTA's column slice of Y (fixed-order sum) -> Z = T'Y
    const int64_t c_lo = split_lo(p, P, Nt), c_hi = split_lo(p + 1, P, Nt);
    double* zw = x.z_slice(c_lo);
    const int64_t zld = x.z_ld();
    for (int64_t cb = c_lo; cb < c_hi; cb += CB) {
      const int w = static_cast<int>(min(static_cast<int64_t>(CB), c_hi - cb));
      for (int idx = tid; idx < kb * w; idx += QR_THREADS) {
        const int jj = idx / w, cc = idx % w;
        double s = 0.0;
        for (int q = 0; q < P; ++q) s += x.gy_r(q, jj, kb + cb + cc);
        tile[jj * CBP + cc] = s;
      }
      __syncthreads();
      for (int idx = tid; idx < kb * w; idx += QR_THREADS) {
        const int jj = idx / w, cc = idx % w;
        double s = 0.0;
        for (int kk = 0; kk <= jj; ++kk) s += Ts[kk * NB + jj] * tile[kk * CBP + cc];
        zw[jj * zld + (cb - c_lo) + cc] = s;
      }
      __syncthreads();
    }
    QPROF(9);
    x.sync();
    QPROF(10);
    // (4) W_own(:, ct0:) -= V_own Z on DMMA tiles: M = RT rows, N = CB, K = 32.
    for (int cb = 0; cb < Nt; cb += CB) {
      const int cw = static_cast<int>(min(static_cast<int64_t>(CB), Nt - cb));
      __syncthreads();
      for (int idx = tid; idx < NB * CB; idx += QR_THREADS) {
        const int c = idx / NB, jj = idx % NB;  // one column per 32 threads: one owner lookup
        Zs[jj * CBP + c] = (jj < kb && c < cw) ? x.z_at(jj, cb + c, Nt) : 0.0;
      }
      for (int rt = 0; rt < hv; rt += RT) {
        const int rh = min(RT, hv - rt);
        __syncthreads();
        for (int idx = tid; idx < RT * CB; idx += QR_THREADS) {
          const int rr = idx / CB, c = idx % CB;
          tile[rr * CBP + c] = (rr < rh && c < cw) ? W[(r0 + rt + rr) * ldw + ct0 + cb + c] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          const int T = warp * 2 + tt;  // 32 output tiles: 4 (M) x 8 (N)
          const int mt = T >> 3, nt = T & 7;
          const int rr = mt * 8 + g4, c = nt * 8 + t4 * 2;
          double d0 = tile[rr * CBP + c], d1 = tile[rr * CBP + c + 1];
#pragma unroll
          for (int k = 0; k < NB; k += 4) {
            const double av = (mt * 8 + g4 < rh) ? -V[(rt + mt * 8 + g4) * PSL + k + t4] : 0.0;
            const double bv = Zs[(k + t4) * CBP + nt * 8 + g4];
            dmma_8x8x4(d0, d1, av, bv);
          }
          if (rr < rh) {
            double* wp = W + (r0 + rt + rr) * ldw + ct0 + cb + c;
            if (c < cw) wp[0] = d0;
            if (c + 1 < cw) wp[1] = d1;
          }
        }
      }
    }
    __syncthreads();
    QPROF(11);
  }
  // R (sign-fixed upper triangle) and z = sign-fixed Q'Sb for own rows < n
  // (linalg.py:43-46); every value read here was written by this CTA.
  const int64_t ihi = min(hi, n);
  for (int64_t idx = tid; idx < (ihi > lo ? ihi - lo : 0) * n; idx += QR_THREADS) {
    const int64_t i = lo + idx / n, c = idx % n;
    const double bi = betas[i];
    const double sg = bi < 0.0 ? -1.0 : 1.0;
    const double rv = (c < i) ? 0.0 : (c == i ? sg * bi : sg * W[i * ldw + c]);
    a.R[i * n + c] = rv;
    if (!isfinite(rv)) atomicOr(a.singular, 2);  // bit 1: non-finite R or z (see k_qr_finish)
  }
  for (int64_t i = lo + tid; i < ihi; i += QR_THREADS) {
    const double bi = betas[i];
    const double sg = bi < 0.0 ? -1.0 : 1.0;
    if (a.z && N > n) {
      const double zv = sg * W[i * ldw + n];
      a.z[i] = zv;
      if (!isfinite(zv)) atomicOr(a.singular, 2);
    }
  }
  if (p == 0)
    for (int64_t i = tid; i < n; i += QR_THREADS)
      if (betas[i] == 0.0) atomicOr(a.singular, 1);
#ifdef ITSK_QR_PROFILE
  if (threadIdx.x == 0 && x.p == 0)
    for (int i = 0; i < 12; ++i) g_qr_prof[i] += _qacc[i];
#endif
}

__global__ void __launch_bounds__(QR_THREADS, 1) k_qr_grid(QrArgs a) {
  extern __shared__ double sm[];
  XGrid x;
  x.rec = a.grec;
  x.gy = a.ggy;
  x.z = a.gz;
  x.bar = a.bar;
  x.P = gridDim.x;
  x.p = blockIdx.x;
  x.ldgy = NB + a.N;
  x.N = a.N;
  qr_body(a, x, sm);
}

__host__ __device__ size_t common_doubles(int64_t hmax, int64_t n) {
  return static_cast<size_t>(hmax * PSL + 2 * NB * NB + NB + n + NB + RT * CBP + NB * CBP);
}

__global__ void __launch_bounds__(QR_THREADS, 1) k_qr_cluster(QrArgs a) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  XCluster x;
  x.P = static_cast<int>(cl.num_blocks());
  x.p = static_cast<int>(cl.block_rank());
  x.ldgy = NB + a.N;
  x.N = a.N;
  x.zld = (a.N + x.P - 1) / x.P + 1;
  x.rec = sm + common_doubles(a.hmax, a.n);
  x.gy = x.rec + 2 * x.P * REC;
  x.z = x.gy + NB * x.ldgy;
  cl.sync();
  qr_body(a, x, sm);
  cl.sync();  // keep shared memory alive until every CTA finished reading it
}

struct QrPlan {
  bool cluster;
  int P;
  int64_t hmax;
  size_t smem;
  int64_t ws_bytes;
  unsigned* bar;
  int* singular;
  double *grec, *ggy, *gz;
};

constexpr size_t QR_SMEM_MAX = 220 * 1024;

QrPlan qr_plan(void* ws, int64_t d, int64_t n, int has_rhs) {
  QrPlan L;
  const int64_t N = n + (has_rhs ? 1 : 0);
  // cluster mode: <= 16 CTAs (non-portable cluster limit); panel rows and the
  // exchange buffers in shared memory
  const int C = static_cast<int>(std::min<int64_t>(16, std::max<int64_t>(1, (d + 63) / 64)));
  const int64_t hmax_c = (d + C - 1) / C + 1;
  const int64_t zld = (N + C - 1) / C + 1;
  const size_t smem_cl = (common_doubles(hmax_c, n) + 2 * C * REC + NB * (NB + N) + NB * zld) * 8;
  L.cluster = smem_cl <= QR_SMEM_MAX;
  const int grid_cap = num_sms();
  if (L.cluster) {
    L.P = C;
    L.hmax = hmax_c;
    L.smem = smem_cl;
  } else {
    const int64_t P = std::min<int64_t>(grid_cap, std::max<int64_t>(1, (d + 31) / 32));
    L.P = static_cast<int>(P);
    L.hmax = (d + P - 1) / P + 1;
    L.smem = common_doubles(L.hmax, n) * 8;
  }
  Carver cv(ws, 1ll << 62);
  L.bar = cv.take<unsigned>(64);
  L.singular = cv.take<int>(64);
  if (L.cluster) {
    L.grec = L.ggy = L.gz = nullptr;
  } else {
    L.grec = cv.take<double>(2ll * L.P * REC);
    L.ggy = cv.take<double>(static_cast<int64_t>(L.P) * NB * (NB + N));
    L.gz = cv.take<double>(NB * N);
  }
  L.ws_bytes = cv.off + 256;
  return L;
}

}  // namespace
}  // namespace itsk

using namespace itsk;

constexpr int64_t V2_WS_OFFSET = 1024;  // bytes: [0,512) barrier, [512,1024) singular flag

namespace {
// A factorisation in one piece: the panel / update split (qr2.cu), or the
// single-kernel QR while its rows fit a CTA's shared memory (~50000 rows).
bool qr_direct_ok(int64_t d, int64_t n) {
  if (qr_v2_plan(d, n).NB > 0) return true;
  return qr_plan(nullptr, d, n, 1).smem <= QR_SMEM_MAX;
}
int64_t qr_direct_ws(int64_t d, int64_t n) {
  int64_t b = std::max(qr_plan(nullptr, d, n, 1).ws_bytes, qr_plan(nullptr, d, n, 0).ws_bytes);
  return std::max<int64_t>(b, V2_WS_OFFSET + 8 * qr_v2_plan(d, n).ws_doubles);
}
// Taller matrices: TSQR over row blocks (as stable as one Householder QR) —
// each block of <= QR_BLOCK_ROWS rows is factored with its share of the rhs
// column, the k stacked [R_i | z_i] (k n x (n+1)) are factored again; the
// final R and z are those of the whole [A | b].
constexpr int64_t QR_BLOCK_ROWS = 24000;
struct QrBlocks {
  int64_t k, hb;  // k blocks of hb rows (the last one shorter)
};
QrBlocks qr_blocks(int64_t d, int64_t n) {
  if (qr_direct_ok(d, n)) return {1, d};
  const int64_t k = (d + QR_BLOCK_ROWS - 1) / QR_BLOCK_ROWS;
  return {k, (d + k - 1) / k};
}
struct QrBlockWs {
  int64_t sub, total;           // bytes: the sub-factorisations' workspace, everything
  int64_t s_off, r_off, z_off;  // byte offsets of the stack, the block's R and z
};
int64_t qr_total_ws(int64_t d, int64_t n);
QrBlockWs qr_block_ws(int64_t d, int64_t n) {
  const QrBlocks B = qr_blocks(d, n);
  QrBlockWs w{};
  w.sub = align_up(std::max(qr_direct_ws(B.hb, n), qr_total_ws(B.k * n, n)), 256);
  w.s_off = w.sub;
  w.r_off = align_up(w.s_off + B.k * n * (n + 1) * 8, 256);
  w.z_off = align_up(w.r_off + n * n * 8, 256);
  w.total = align_up(w.z_off + n * 8, 256) + 256;
  return w;
}
int64_t qr_total_ws(int64_t d, int64_t n) {
  return qr_blocks(d, n).k == 1 ? qr_direct_ws(d, n) : qr_block_ws(d, n).total;
}
}  // namespace

extern "C" int itsk_qr_workspace(int64_t d, int64_t n, int64_t* bytes) {
  ITSK_REQUIRE(bytes && d >= n && n >= 1, "need d >= n >= 1");
  *bytes = qr_total_ws(d, n);
  return ITSK_OK;
}

extern "C" int itsk_qr_row_blocks(int64_t d, int64_t n, int64_t* blocks) {
  ITSK_REQUIRE(blocks && d >= n && n >= 1, "need d >= n >= 1");
  *blocks = qr_blocks(d, n).k;
  return ITSK_OK;
}

namespace {
// Launches the factorisation; *flag receives the device address of the
// "exact zero on diag(R)" flag (read by the caller, synchronously or not).
int qr_aug_core(double* W, int64_t d, int64_t n, int64_t ldw, double* R, double* z, void* ws, int64_t ws_bytes,
                itsk_stream_t stream, int** flag) {
  ITSK_REQUIRE(W && R && ws, "null pointer");
  ITSK_REQUIRE(n >= 1 && d >= n, "need m >= n, got %lld x %lld", (long long)d, (long long)n);
  const int has_rhs = z != nullptr;
  ITSK_REQUIRE(ldw >= n + has_rhs, "bad leading dimension");
  const QrBlocks B = qr_blocks(d, n);
  if (B.k > 1) {
    ITSK_REQUIRE(2 * n <= B.hb, "qr: n=%lld is too wide for the row-blocked factorisation of %lld rows",
                 (long long)n, (long long)d);
    const QrBlockWs bw = qr_block_ws(d, n);
    ITSK_REQUIRE(bw.total <= ws_bytes, "qr workspace too small (%lld < %lld)", (long long)ws_bytes,
                 (long long)bw.total);
    cudaStream_t bs = reinterpret_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(ws);
    double* S = reinterpret_cast<double*>(base + bw.s_off);
    double* Rt = reinterpret_cast<double*>(base + bw.r_off);
    double* zt = reinterpret_cast<double*>(base + bw.z_off);
    const int64_t N = n + has_rhs;
    for (int64_t i = 0; i < B.k; ++i) {
      const int64_t r0 = i * B.hb, rows = std::min(B.hb, d - r0);
      int* f = nullptr;
      int rc = qr_aug_core(W + r0 * ldw, rows, n, ldw, Rt, has_rhs ? zt : nullptr, ws, bw.sub, stream, &f);
      if (rc) return rc;
      ITSK_CUDA(cudaMemcpy2DAsync(S + i * n * N, N * 8, Rt, n * 8, n * 8, n, cudaMemcpyDeviceToDevice, bs));
      if (has_rhs)
        ITSK_CUDA(cudaMemcpy2DAsync(S + i * n * N + n, N * 8, zt, 8, 8, n, cudaMemcpyDeviceToDevice, bs));
    }
    // (a block's own zero pivot is not the matrix's: only the last factorisation's flags count)
    return qr_aug_core(S, B.k * n, n, N, R, z, ws, bw.sub, stream, flag);
  }
  QrPlan L = qr_plan(ws, d, n, has_rhs);
  ITSK_REQUIRE(L.ws_bytes <= ws_bytes, "qr workspace too small (%lld < %lld)", (long long)ws_bytes,
               (long long)L.ws_bytes);
  ITSK_REQUIRE(L.smem <= QR_SMEM_MAX, "qr: too many rows per CTA (d=%lld, n=%lld)", (long long)d,
               (long long)n);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // the panel / update split (qr2.cu) wherever its panel fits in a cluster's
  // shared memory; beyond (more than ~25600 rows at 16-wide panels) the
  // single-kernel QR below: one cluster, or the whole grid with barriers
  const QrV2Plan V2 = qr_v2_plan(d, n);
  if (V2.NB > 0) {
    ITSK_REQUIRE(V2_WS_OFFSET + 8 * V2.ws_doubles <= ws_bytes, "qr workspace too small");
    int* sing = reinterpret_cast<int*>(static_cast<char*>(ws) + 512);
    double* wsd = reinterpret_cast<double*>(static_cast<char*>(ws) + V2_WS_OFFSET);
    int rc = launch_qr_v2(W, d, n, ldw, n + has_rhs, R, z, sing, wsd, V2, s);
    if (rc) return rc;
    *flag = sing;
    return ITSK_OK;
  }
  ITSK_CUDA(cudaMemsetAsync(L.bar, 0, 512, s));
  QrArgs a;
  a.W = W;
  a.d = d;
  a.n = n;
  a.ldw = ldw;
  a.N = n + has_rhs;
  a.R = R;
  a.z = z;
  a.singular = L.singular;
  a.grec = L.grec;
  a.ggy = L.ggy;
  a.gz = L.gz;
  a.bar = L.bar;
  a.hmax = L.hmax;
  if (L.cluster) {
    ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_qr_cluster)));
    ITSK_CUDA(func_attr_once(reinterpret_cast<const void*>(k_qr_cluster),
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L.P);
    cfg.blockDim = dim3(QR_THREADS);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = L.P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ITSK_CUDA(cudaLaunchKernelEx(&cfg, k_qr_cluster, a));
  } else {
    ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_qr_grid)));
    void* args[] = {&a};
    ITSK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_qr_grid), dim3(L.P),
                                          dim3(QR_THREADS), args, L.smem, s));
  }
  count_launch();
  *flag = L.singular;
  return ITSK_OK;
}
}  // namespace


extern "C" int itsk_qr_aug(double* W, int64_t d, int64_t n, int64_t ldw, double* R, double* z,
                           void* ws, int64_t ws_bytes, itsk_stream_t stream) {
  int* flag = nullptr;
  int rc = qr_aug_core(W, d, n, ldw, R, z, ws, ws_bytes, stream, &flag);
  if (rc) return rc;
  int singular = 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ITSK_CUDA(cudaMemcpyAsync(&singular, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  ITSK_CUDA(cudaStreamSynchronize(s));
  if (singular & 1) {  // bit 1 (non-finite R or z) is the async entry's business: LAPACK's QR returns NaNs too
    set_error("zero diagonal entry in triangular factor");
    return ITSK_ESINGULAR;
  }
  return ITSK_OK;
}

extern "C" int itsk_qr_aug_async(double* W, int64_t d, int64_t n, int64_t ldw, double* R, double* z, void* ws,
                                 int64_t ws_bytes, int* singular, itsk_stream_t stream) {
  ITSK_REQUIRE(singular, "null singular flag");
  int* flag = nullptr;
  int rc = qr_aug_core(W, d, n, ldw, R, z, ws, ws_bytes, stream, &flag);
  if (rc) return rc;
  ITSK_CUDA(cudaMemcpyAsync(singular, flag, sizeof(int), cudaMemcpyDeviceToDevice,
                            reinterpret_cast<cudaStream_t>(stream)));
  return ITSK_OK;
}

#ifdef ITSK_QR_PROFILE
extern "C" void itsk_qr_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, itsk::g_qr_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(itsk::g_qr_prof, z, sizeof(z));
}
#endif
