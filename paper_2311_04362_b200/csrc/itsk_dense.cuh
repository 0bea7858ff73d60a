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

// 512 threads: the register-resident 32x32 diagonal block needs > 64 regs/thread.
constexpr int DENSE_THREADS = 512;

struct RGlobal {
  const double* __restrict__ R;
  int64_t n;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const { return R[i * n + j]; }
};

// upper triangle packed by rows: row i holds R[i][i..n) starting at
// off(i) = i*n - i(i-1)/2; the accessor subtracts i from a per-row base.
struct RPacked {
  uint32_t base;  // shared-window address of the packed triangle
  int nn;
  __device__ __forceinline__ RPacked(const double* P, int64_t n)
      : base(static_cast<uint32_t>(__cvta_generic_to_shared(P))), nn(static_cast<int>(n)) {}
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    const int ii = static_cast<int>(i);
    const uint32_t off = static_cast<uint32_t>(ii * nn - ((ii * (ii - 1)) >> 1) + (static_cast<int>(j) - ii));
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + off * 8u));
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
// 32 * (blockDim.x / 32) + 32 doubles in shared memory.

// y := R^{-T} y   (forward substitution, LEFT-looking by 32-blocks).
// For block I the contribution of the solved entries, sum_{k<b0} R[k][i] y[k]
// (i in I), is split over the warps by k-range with lanes on the 32 columns
// of I (contiguous row segments of R); the per-warp partials are added in a
// fixed order.  The sequential chain per step is one multiply by the
// precomputed 1/R_kk, one shuffle and one FMA (dtrsv divides; y*(1/d) differs
// from y/d by at most one rounding — the solve stays backward stable).
template <class RA>
__device__ __forceinline__ void trsv_t_inplace(const RA& R, int64_t n, double* y, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += 32) {
    const int bs = static_cast<int>(min(static_cast<int64_t>(32), n - b0));
    // loads below are unconditional on clamped indices and masked afterwards:
    // predicated loads would compile into divergent branches around each load
    const int64_t jl = min(b0 + lane, n - 1);
    if (b0 > 0) {
      const int64_t k_lo = (b0 * warp) / nw, k_hi = (b0 * (warp + 1)) / nw;
      double acc = 0.0;
      for (int64_t k = k_lo; k < k_hi; ++k) acc = fma(R(k, jl), y[k], acc);
      red[warp * 32 + lane] = (lane < bs) ? acc : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      // lane i holds column i of the diagonal block: R[b0+k][b0+i], k < i
      double col[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double v = R(min(b0 + k, n - 1), jl);
        col[k] = (k < lane && lane < bs) ? v : 0.0;
      }
      const double dg = R(jl, jl);
      const double rinv = (lane < bs) ? 1.0 / dg : 0.0;
      double s = 0.0;
      if (b0 > 0) {
#pragma unroll 8
        for (int w = 0; w < nw; ++w) s += red[w * 32 + lane];
      }
      const double yv = y[jl];
      double yi = (lane < bs) ? yv - s : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < bs) {
          if (lane == k) yi *= rinv;
          const double yk = __shfl_sync(FULL, yi, k);
          yi = fma(-col[k], yk, yi);  // col[k] == 0 for lanes <= k
        }
      }
      if (lane < bs) y[b0 + lane] = yi;
    }
    __syncthreads();
  }
}

// x := R^{-1} x   (back substitution, left-looking by 32-blocks from the bottom;
// warps take rows of the block, lanes the contiguous solved tail of the row)
template <class RA>
__device__ __forceinline__ void trsv_n_inplace(const RA& R, int64_t n, double* x, double* tmp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t be = n; be > 0; be -= 32) {
    const int64_t b0 = max(static_cast<int64_t>(0), be - 32);
    const int bs = static_cast<int>(be - b0);
    for (int rr = warp; rr < bs; rr += nw) {
      const int64_t i = b0 + rr;
      double s = 0.0;
      for (int64_t j = be + lane; j < n; j += 32) s = fma(R(i, j), x[j], s);
      s = warp_sum(s);
      if (lane == 0) tmp[rr] = x[i] - s;
    }
    __syncthreads();
    if (warp == 0) {
      // lane i holds row i of the diagonal block: R[b0+i][b0+k], k > i
      const int64_t il = min(b0 + lane, n - 1);
      double row[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double v = R(il, min(b0 + k, n - 1));
        row[k] = (k > lane && k < bs) ? v : 0.0;
      }
      const double dg = R(il, il);
      const double rinv = (lane < bs) ? 1.0 / dg : 0.0;
      const double tv = tmp[lane];
      double t = (lane < bs) ? tv : 0.0;
#pragma unroll
      for (int k = 31; k >= 0; --k) {
        if (k < bs) {
          if (lane == k) t *= rinv;
          const double xk = __shfl_sync(FULL, t, k);
          t = fma(-row[k], xk, t);  // row[k] == 0 for lanes >= k
        }
      }
      if (lane < bs) x[b0 + lane] = t;
    }
    __syncthreads();
  }
}

// out := R v  (upper): 4 rows per warp at a time, reductions interleaved
template <class RA>
__device__ __forceinline__ void trmv_n(const RA& R, int64_t n, const double* v, double* out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t i0 = 4 * warp; i0 < n; i0 += 4 * nw) {
    double s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s[u] = 0.0;
      const int64_t i = i0 + u;
      if (i < n)
        for (int64_t j = i + lane; j < n; j += 32) s[u] = fma(R(i, j), v[j], s[u]);
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
__device__ __forceinline__ void trmv_t(const RA& R, int64_t n, const double* v, double* out,
                                       double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += 32) {
    const int bs = static_cast<int>(min(static_cast<int64_t>(32), n - b0));
    const int64_t top = b0 + bs;  // rows i < top contribute to this block
    const int64_t k_lo = (top * warp) / nw, k_hi = (top * (warp + 1)) / nw;
    double acc = 0.0;
    const int64_t j = min(b0 + lane, n - 1);
    for (int64_t i = k_lo; i < k_hi; ++i) {
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
