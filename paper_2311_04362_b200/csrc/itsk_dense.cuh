// Single-CTA dense kernels on the n x n R factor, shared (inline) by the
// stand-alone entry points (trsv.cu) and the loop body (loop.cu).
//
// R: row-major, ld n, upper triangular.  Vectors live in shared memory.
// When the packed upper triangle fits (n <= ~220 for 190 KB), it is staged
// once per kernel into shared memory (RPacked); otherwise R is read from L2
// (RGlobal).  The substitution chains keep the 32x32 diagonal block of the
// current step in registers, so each of the n sequential steps costs a
// divide, a shuffle and an FMA — no memory round trip.
#pragma once
#include "itsk_common.cuh"

namespace itsk {

#ifdef ITSK_DENSE_PROBE
__device__ long long g_probe[8];
#endif

// 512 threads: the register-resident 32x32 diagonal block needs > 64 regs/thread.
constexpr int DENSE_THREADS = 512;

// Index math is 32-bit throughout (n <= 16384 is enforced by the entry points).
struct RGlobal {
  const double* __restrict__ R;
  int nn;
  __device__ __forceinline__ RGlobal(const double* r, int64_t n) : R(r), nn(static_cast<int>(n)) {}
  __device__ __forceinline__ double operator()(int i, int j) const { return R[i * nn + j]; }
};

// upper triangle packed by rows: row i holds R[i][i..n) starting at
// off(i) = i*n - i(i-1)/2; the accessor subtracts i from a per-row base.
struct RPacked {
  uint32_t base;  // shared-window address of the packed triangle
  int nn;
  __device__ __forceinline__ RPacked(const double* P, int64_t n)
      : base(static_cast<uint32_t>(__cvta_generic_to_shared(P))), nn(static_cast<int>(n)) {}
  __device__ __forceinline__ double operator()(int i, int j) const {
    const uint32_t off = static_cast<uint32_t>(i * nn - ((i * (i - 1)) >> 1) + (j - i));
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + off * 8u));  // read-only data: no volatile
    return v;
  }
};

__host__ __device__ __forceinline__ int64_t packed_doubles(int64_t n) { return n * (n + 1) / 2; }

__device__ __forceinline__ void stage_packed(const double* __restrict__ R, int64_t n, double* P) {
  // one flat sweep over R so every thread keeps several independent loads in
  // flight; consecutive threads read consecutive elements
  const int nn = static_cast<int>(n * n), ni = static_cast<int>(n);
#pragma unroll 4
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int i = e / ni, j = e - i * ni;
    const double v = R[e];
    if (j >= i) P[i * ni - ((i * (i - 1)) >> 1) + (j - i)] = v;
  }
  __syncthreads();
}

// Packed upper triangle in global memory (itsk_pack_upper) -> shared memory
// with ONE bulk copy (the row-by-row gather from the dense R is latency bound).
__host__ __device__ __forceinline__ int64_t packed_bytes(int64_t n) {
  return (packed_doubles(n) * 8 + 15) / 16 * 16;
}

__device__ __forceinline__ void stage_packed_bulk(const double* Rp, int64_t n, double* P) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned bytes = static_cast<unsigned>(packed_bytes(n));
    mbar_expect_tx(&bar, bytes);
    bulk_g2s_plain(P, Rp, bytes, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
}

// The kernels below need a scratch area `red` of at least
// 64 * (blockDim.x / 32) doubles in shared memory.

// Software-pipelined blocked substitution (32-wide blocks).  While warp 0
// runs the sequential chain of block I, the other warps already accumulate
// into block I+1 (I-1 for the back solve) the contributions of every block
// that is final; warp 0 then adds only the neighbouring block's 32x32 product
// before starting the next chain.  Per step the chain costs one multiply by
// the precomputed 1/R_kk, one shuffle and one FMA (dtrsv divides; y*(1/d)
// differs from y/d by at most one rounding — the solve stays backward
// stable).  All sums run in a fixed order: results are reproducible.

// y := R^{-T} y   (forward substitution)
template <class RA>
__device__ __forceinline__ void trsv_t_inplace(const RA& R, int n64, double* y, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  const int nw = blockDim.x >> 5, nh = nw - 1;  // helper warps 1..nw-1
  const int nblk = static_cast<int>((n + 31) / 32);
  for (int I = 0; I < nblk; ++I) {
    const int b0 = 32 * I;
    if (warp == 0) {
#ifdef ITSK_DENSE_PROBE
      long long _c0 = clock64();
#endif
      const int bs = static_cast<int>(min(32, n - b0));
      const int jl = min(b0 + lane, n - 1);
      // contributions of blocks < I-1 (helpers, previous step) and of block I-1
      double s = 0.0;
      if (I >= 2) {
        const double* pb = red + (I & 1) * 32 * nw;
        for (int w = 1; w < nw; ++w) s += pb[w * 32 + lane];
      }
      if (I >= 1) {
        const int pb0 = b0 - 32;
        double p2 = 0.0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) p2 = fma(R(pb0 + k, jl), y[pb0 + k], p2);
        s += p2;
      }
      double col[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double v = R(min(b0 + k, n - 1), jl);
        col[k] = (k < lane && lane < bs) ? v : 0.0;
      }
      const double dg = R(jl, jl);
      const double rinv = (lane < bs) ? 1.0 / dg : 0.0;
      const double yv = y[jl];
      double yi = (lane < bs) ? yv - s : 0.0;
#ifdef ITSK_DENSE_PROBE
      __syncwarp();
      long long _c1 = clock64();
#endif
      // straight-line chain: for k >= bs the step is a no-op (lane k holds 0,
      // col[k] == 0), so no per-step branch / reconvergence is needed
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (lane == k) yi *= rinv;
        const double yk = __shfl_sync(FULL, yi, k);
        yi = fma(-col[k], yk, yi);  // col[k] == 0 for lanes <= k
      }
#ifdef ITSK_DENSE_PROBE
      __syncwarp();
      long long _c2 = clock64();
      if (lane == 0) { g_probe[0] += _c1 - _c0; g_probe[1] += _c2 - _c1; }
#endif
      if (lane < bs) y[b0 + lane] = yi;
    } else if (I + 1 < nblk && nh > 0) {
      // helpers: rows [0, b0) (blocks < I, final) into block I+1
      const int t0 = b0 + 32;
      const int jl = min(t0 + lane, n - 1);
      const int k_lo = (b0 * (warp - 1)) / nh, k_hi = (b0 * warp) / nh;
      double acc = 0.0;
      for (int k = k_lo; k < k_hi; ++k) acc = fma(R(k, jl), y[k], acc);
      red[((I + 1) & 1) * 32 * nw + warp * 32 + lane] = acc;
    }
    __syncthreads();
  }
}

// x := R^{-1} x   (back substitution, blocks from the bottom)
template <class RA>
__device__ __forceinline__ void trsv_n_inplace(const RA& R, int n64, double* x, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  const int nw = blockDim.x >> 5, nh = nw - 1;
  const int nblk = static_cast<int>((n + 31) / 32);
  for (int I = nblk - 1; I >= 0; --I) {
    const int b0 = 32 * I;
    const int be = min(b0 + 32, n);
    const int bs = static_cast<int>(be - b0);
    if (warp == 0) {
      const int il = min(b0 + lane, n - 1);
      double s = 0.0;
      if (I + 1 < nblk) s = red[(I & 1) * 32 * nw + lane];  // columns beyond block I+1 (helpers)
      if (I + 1 < nblk) {  // block I+1's contribution: row il, columns [be, be+32)
        const int cb = be;
        const int cw = static_cast<int>(min(32, n - cb));
        double p2 = 0.0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const double rv = R(il, min(cb + k, n - 1));
          p2 = fma(k < cw ? rv : 0.0, x[min(cb + k, n - 1)], p2);
        }
        s += p2;
      }
      double row[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double v = R(il, min(b0 + k, n - 1));
        row[k] = (k > lane && k < bs) ? v : 0.0;
      }
      const double dg = R(il, il);
      const double rinv = (lane < bs) ? 1.0 / dg : 0.0;
      const double xv = x[il];
      double t = (lane < bs) ? xv - s : 0.0;
#pragma unroll
      for (int k = 31; k >= 0; --k) {  // no-op steps for k >= bs (see trsv_t_inplace)
        if (lane == k) t *= rinv;
        const double xk = __shfl_sync(FULL, t, k);
        t = fma(-row[k], xk, t);  // row[k] == 0 for lanes >= k
      }
      if (lane < bs) x[b0 + lane] = t;
    } else if (I >= 1 && nh > 0) {
      // helpers: columns [be + 32, n) (blocks > I+1, final) into the rows of block I-1
      const int tb0 = b0 - 32;
      const int c0 = be;  // blocks > I are final
      for (int rr = warp - 1; rr < 32; rr += nh) {
        const int i = tb0 + rr;
        double acc = 0.0;
        for (int j = c0 + lane; j < n; j += 32) acc = fma(R(i, j), x[j], acc);
        acc = warp_sum(acc);
        if (lane == 0) red[((I - 1) & 1) * 32 * nw + rr] = acc;
      }
    }
    __syncthreads();
  }
}

// out := R v  (upper): 4 rows per warp at a time, reductions interleaved
template <class RA>
__device__ __forceinline__ void trmv_n(const RA& R, int n64, const double* v, double* out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  const int nw = blockDim.x >> 5;
  for (int i0 = 4 * warp; i0 < n; i0 += 4 * nw) {
    double s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s[u] = 0.0;
      const int i = i0 + u;
      if (i < n)
        for (int j = i + lane; j < n; j += 32) s[u] = fma(R(i, j), v[j], s[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += __shfl_xor_sync(FULL, s[u], o);
    if (lane < 4 && i0 + lane < n) {
      double r = s[0];
#pragma unroll
      for (int u = 1; u < 4; ++u)
        if (lane == u) r = s[u];
      out[i0 + lane] = r;
    }
  }
  __syncthreads();
}

// out := R' v : per 32-column block, warps split the i-range, lanes the
// columns (contiguous row segments); fixed-order sum of the warp partials
template <class RA>
__device__ __forceinline__ void trmv_t(const RA& R, int n64, const double* v, double* out,
                                       double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  const int nw = blockDim.x >> 5;
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int bs = static_cast<int>(min(32, n - b0));
    const int top = b0 + bs;  // rows i < top contribute to this block
    const int k_lo = (top * warp) / nw, k_hi = (top * (warp + 1)) / nw;
    double acc = 0.0;
    const int j = min(b0 + lane, n - 1);
    for (int i = k_lo; i < k_hi; ++i) {
      const double rv = R(i, j);
      acc = fma(i <= j ? rv : 0.0, v[i], acc);
    }
    red[warp * 32 + lane] = (lane < bs) ? acc : 0.0;
    __syncthreads();
    if (warp == 0 && lane < bs) {
      double sum = 0.0;
      for (int w = 0; w < nw; ++w) sum += red[w * 32 + lane];
      out[b0 + lane] = sum;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double dot_sm(const double* a, const double* b, int64_t n, double* red) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += a[i] * b[i];
  return block_sum(s, red);
}

// Shared-memory budget of the single-CTA R kernels.
constexpr int64_t DENSE_SMEM_BUDGET = 200 * 1024;

__host__ __device__ __forceinline__ bool use_packed(int64_t n, int64_t other_doubles) {
  return (packed_doubles(n) + other_doubles) * 8 <= DENSE_SMEM_BUDGET;
}

}  // namespace itsk
