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
  const double* P;
  int64_t n;
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    const int ii = static_cast<int>(i), nn = static_cast<int>(n);
    return P[ii * nn - ((ii * (ii - 1)) >> 1) + (static_cast<int>(j) - ii)];
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

// y := R^{-T} y   (forward substitution, right-looking by 32-blocks).
// The sequential chain per step is one multiply by the precomputed 1/R_kk,
// one shuffle and one FMA (dtrsv divides; y*(1/d) differs from y/d by at most
// one rounding — the solve stays backward stable).
template <class RA>
__device__ __forceinline__ void trsv_t_inplace(const RA& R, int64_t n, double* y) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += 32) {
    const int bs = static_cast<int>(min(static_cast<int64_t>(32), n - b0));
    if (warp == 0) {
      // lane i holds column i of the diagonal block: R[b0+k][b0+i], k < i
      double col[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) col[k] = (k < lane && lane < bs) ? R(b0 + k, b0 + lane) : 0.0;
      const double rinv = (lane < bs) ? 1.0 / R(b0 + lane, b0 + lane) : 0.0;
      double yi = (lane < bs) ? y[b0 + lane] : 0.0;
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
    for (int64_t j = b0 + bs + tid; j < n; j += blockDim.x) {
      double acc = y[j];
      for (int k = 0; k < bs; ++k) acc -= R(b0 + k, j) * y[b0 + k];
      y[j] = acc;
    }
    __syncthreads();
  }
}

// x := R^{-1} x   (back substitution, left-looking by 32-blocks from the bottom)
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
      for (int64_t j = be + lane; j < n; j += 32) s += R(i, j) * x[j];
      s = warp_sum(s);
      if (lane == 0) tmp[rr] = x[i] - s;
    }
    __syncthreads();
    if (warp == 0) {
      // lane i holds row i of the diagonal block: R[b0+i][b0+k], k > i
      double row[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) row[k] = (k > lane && k < bs) ? R(b0 + lane, b0 + k) : 0.0;
      const double rinv = (lane < bs) ? 1.0 / R(b0 + lane, b0 + lane) : 0.0;
      double t = (lane < bs) ? tmp[lane] : 0.0;
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

// out := R v  (upper)
template <class RA>
__device__ __forceinline__ void trmv_n(const RA& R, int64_t n, const double* v, double* out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    double s = 0.0;
    for (int64_t j = i + lane; j < n; j += 32) s += R(i, j) * v[j];
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
  __syncthreads();
}

// out := R' v
template <class RA>
__device__ __forceinline__ void trmv_t(const RA& R, int64_t n, const double* v, double* out) {
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int64_t i = 0; i <= j; ++i) s += R(i, j) * v[i];
    out[j] = s;
  }
  __syncthreads();
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
