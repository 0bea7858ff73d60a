// Single-CTA dense kernels on the n x n R factor, shared (inline) by the
// stand-alone entry points (trsv.cu) and the loop body (loop.cu).
// R: row-major, ld n, upper triangular.  Vectors live in shared memory.
#pragma once
#include "itsk_common.cuh"

namespace itsk {

// y := R^{-T} y   (y in shared memory, length n)
__device__ __forceinline__ void trsv_t_inplace(const double* __restrict__ R, int64_t n, double* y) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += 32) {
    const int bs = static_cast<int>(min(static_cast<int64_t>(32), n - b0));
    if (warp == 0) {
      double yi = (lane < bs) ? y[b0 + lane] : 0.0;
      for (int k = 0; k < bs; ++k) {
        if (lane == k) yi = yi / R[(b0 + k) * n + b0 + k];
        const double yk = __shfl_sync(FULL, yi, k);
        if (lane > k && lane < bs) yi -= R[(b0 + k) * n + b0 + lane] * yk;
      }
      if (lane < bs) y[b0 + lane] = yi;
    }
    __syncthreads();
    for (int64_t j = b0 + bs + tid; j < n; j += blockDim.x) {
      double acc = y[j];
      for (int k = 0; k < bs; ++k) acc -= R[(b0 + k) * n + j] * y[b0 + k];
      y[j] = acc;
    }
    __syncthreads();
  }
}

// x := R^{-1} x   (x in shared memory, length n); tmp: 32 doubles of smem
__device__ __forceinline__ void trsv_n_inplace(const double* __restrict__ R, int64_t n, double* x, double* tmp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t be = n; be > 0; be -= 32) {
    const int64_t b0 = max(static_cast<int64_t>(0), be - 32);
    const int bs = static_cast<int>(be - b0);
    for (int rr = warp; rr < bs; rr += nw) {
      const int64_t i = b0 + rr;
      const double* row = R + i * n;
      double s = 0.0;
      for (int64_t j = be + lane; j < n; j += 32) s += row[j] * x[j];
      s = warp_sum(s);
      if (lane == 0) tmp[rr] = x[i] - s;
    }
    __syncthreads();
    if (warp == 0) {
      double t = (lane < bs) ? tmp[lane] : 0.0;
      for (int k = bs - 1; k >= 0; --k) {
        if (lane == k) t = t / R[(b0 + k) * n + b0 + k];
        const double xk = __shfl_sync(FULL, t, k);
        if (lane < k) t -= R[(b0 + lane) * n + b0 + k] * xk;
      }
      if (lane < bs) x[b0 + lane] = t;
    }
    __syncthreads();
  }
}

// out := R v  (upper), out/v in shared memory
__device__ __forceinline__ void trmv_n(const double* __restrict__ R, int64_t n, const double* v, double* out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const double* row = R + i * n;
    double s = 0.0;
    for (int64_t j = i + lane; j < n; j += 32) s += row[j] * v[j];
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
  __syncthreads();
}

// out := R' v
__device__ __forceinline__ void trmv_t(const double* __restrict__ R, int64_t n, const double* v, double* out) {
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int64_t i = 0; i <= j; ++i) s += R[i * n + j] * v[i];
    out[j] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ double dot_sm(const double* a, const double* b, int64_t n, double* red) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += a[i] * b[i];
  return block_sum(s, red);
}

}  // namespace itsk
