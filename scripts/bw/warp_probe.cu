#include <cstdio>
#include <vector>
#include "itsk_dense.cuh"
using namespace itsk;
namespace itsk { void set_error(const char*, ...) {} void count_launch(int64_t) {} int num_sms() { return 148; } cudaError_t allow_max_smem(const void*) { return cudaSuccess; } }

// single-warp forward solve R^T y = c
template <class RA>
__device__ void trsv_t_warp(const RA& R, int n, double* y) {
  const int lane = threadIdx.x & 31;
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int bs = min(32, n - b0);
    double acc = 0.0;
    if (lane < bs) {
      const int j = b0 + lane;
#pragma unroll 8
      for (int k = 0; k < b0; ++k) acc = fma(R(k, j), y[k], acc);
    }
    double col[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) col[k] = (k < lane && lane < bs) ? R(b0 + k, b0 + lane) : 0.0;
    const double rinv = (lane < bs) ? 1.0 / R(b0 + lane, b0 + lane) : 0.0;
    double yi = (lane < bs) ? y[b0 + lane] - acc : 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k < bs) {
        if (lane == k) yi *= rinv;
        const double yk = __shfl_sync(FULL, yi, k);
        yi = fma(-col[k], yk, yi);
      }
    }
    if (lane < bs) y[b0 + lane] = yi;
    __syncwarp();
  }
}
// single-warp back solve R x = y: partial dots 4 rows at a time
template <class RA>
__device__ void trsv_n_warp(const RA& R, int n, double* x) {
  const int lane = threadIdx.x & 31;
  for (int be = n; be > 0; be -= 32) {
    const int b0 = max(0, be - 32), bs = be - b0;
    double mine = 0.0;  // lane i: partial for row b0+i
    for (int r0 = 0; r0 < bs; r0 += 4) {
      double s[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r0 + u < bs)
          for (int j = be + lane; j < n; j += 32) s[u] = fma(R(b0 + r0 + u, j), x[j], s[u]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] += __shfl_xor_sync(FULL, s[u], o);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (lane == r0 + u) mine = s[u];
    }
    double row[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) row[k] = (k > lane && k < bs) ? R(b0 + lane, b0 + k) : 0.0;
    const double rinv = (lane < bs) ? 1.0 / R(b0 + lane, b0 + lane) : 0.0;
    double t = (lane < bs) ? x[b0 + lane] - mine : 0.0;
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (k < bs) {
        if (lane == k) t *= rinv;
        const double xk = __shfl_sync(FULL, t, k);
        t = fma(-row[k], xk, t);
      }
    }
    if (lane < bs) x[b0 + lane] = t;
    __syncwarp();
  }
}

__global__ void __launch_bounds__(512) probe(const double* Rp, int n, double* y, long long* cyc) {
  extern __shared__ double sm[];
  stage_packed_bulk(Rp, n, sm);
  double* v = sm + packed_doubles(n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = 1.0 + i;
  __syncthreads();
  RPacked R{sm, n};
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    trsv_t_warp(R, n, v);
    long long t1 = clock64();
    trsv_n_warp(R, n, v);
    long long t2 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = v[i];
}
int main() {
  for (int n : {64, 200}) {
    std::vector<double> P((n * (n + 1) / 2) + 2, 0.001);
    for (int i = 0; i < n; ++i) P[(long)i * n - (long)i * (i - 1) / 2] = 2.0;
    double *dP, *dy; long long* dc; cudaMalloc(&dP, P.size() * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dc, 64);
    cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = (packed_doubles(n) + 2 * n + 32) * 8;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long c[2];
    for (int it = 0; it < 3; ++it) probe<<<1, 512, smem>>>(dP, n, dy, dc);
    cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    printf("n=%d single-warp: trsv_t %lld  trsv_n %lld cycles (%s)\n", n, c[0], c[1], cudaGetErrorString(cudaGetLastError()));
  }
}
