#include <cstdio>
#include <vector>
#include "itsk_dense.cuh"
using namespace itsk;
namespace itsk { void set_error(const char*, ...) {} void count_launch(int64_t) {} int num_sms() { return 148; } cudaError_t allow_max_smem(const void*) { return cudaSuccess; } }
__device__ long long g_t[8];
template <bool FAST, class RA>
__device__ void trsv_t_prof(const RA& R, int64_t n, double* y, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  long long tp = 0, ts = 0, td = 0, ts2 = 0;
  for (int64_t b0 = 0; b0 < n; b0 += 32) {
    long long t0 = clock64();
    const int bs = static_cast<int>(min(static_cast<int64_t>(32), n - b0));
    if (b0 > 0) {
      const int64_t k_lo = (b0 * warp) / nw, k_hi = (b0 * (warp + 1)) / nw;
      double acc = 0.0;
      if (lane < bs)
        for (int64_t k = k_lo; k < k_hi; ++k) acc = fma(R(k, b0 + lane), y[k], acc);
      red[warp * 32 + lane] = acc;
    }
    long long t1 = clock64();
    __syncthreads();
    long long t2 = clock64();
    if (warp == 0 && bs == 32 && FAST) {
      long long a0 = clock64();
      double col[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) col[k] = (k < lane) ? R(b0 + k, b0 + lane) : 0.0;
      double acc0 = 0; for (int k = 0; k < 32; ++k) acc0 += col[k];
      __syncwarp();
      long long a1 = clock64();
      const double rinv = 1.0 / R(b0 + lane, b0 + lane);
      double s = rinv * 0.0 + acc0 * 0.0;
      __syncwarp();
      long long a2 = clock64();
      if (b0 > 0)
        for (int w = 0; w < nw; ++w) s += red[w * 32 + lane];
      double yi = y[b0 + lane] - s;
      __syncwarp();
      long long a3 = clock64();
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (lane == k) yi *= rinv;
        const double yk = __shfl_sync(FULL, yi, k);
        yi = fma(-col[k], yk, yi);
      }
      __syncwarp();
      long long a4 = clock64();
      y[b0 + lane] = yi;
      if (lane == 0) { atomicAdd((unsigned long long*)&g_t[4], (unsigned long long)(a1 - a0)); atomicAdd((unsigned long long*)&g_t[5], (unsigned long long)(a2 - a1)); atomicAdd((unsigned long long*)&g_t[6], (unsigned long long)(a3 - a2)); atomicAdd((unsigned long long*)&g_t[7], (unsigned long long)(a4 - a3)); }
    } else if (warp == 0) {
      double col[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) col[k] = (k < lane && lane < bs) ? R(b0 + k, b0 + lane) : 0.0;
      const double rinv = (lane < bs) ? 1.0 / R(b0 + lane, b0 + lane) : 0.0;
      double s = 0.0;
      if (b0 > 0)
        for (int w = 0; w < nw; ++w) s += red[w * 32 + lane];
      double yi = (lane < bs) ? y[b0 + lane] - s : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < bs) {
          if (lane == k) yi *= rinv;
          const double yk = __shfl_sync(FULL, yi, k);
          yi = fma(-col[k], yk, yi);
        }
      }
      if (lane < bs) y[b0 + lane] = yi;
    }
    long long t3 = clock64();
    __syncthreads();
    long long t4 = clock64();
    tp += t1 - t0; ts += t2 - t1; td += t3 - t2; ts2 += t4 - t3;
  }
  if (threadIdx.x == 0) { g_t[0] = tp; g_t[1] = ts; g_t[2] = td; g_t[3] = ts2; }
}
template <bool FAST>
__global__ void __launch_bounds__(512) probe(const double* Rp, int n, double* y) {
  extern __shared__ double sm[];
  __shared__ double red[32 * 16 + 32];
  stage_packed_bulk(Rp, n, sm);
  double* v = sm + packed_doubles(n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = 1.0 + i;
  __syncthreads();
  RPacked R{sm, n};
  trsv_t_prof<FAST>(R, n, v, red);
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = v[i];
}
int main() {
  int n = 200;
  std::vector<double> P((n * (n + 1) / 2) + 2, 0.001);
  for (int i = 0; i < n; ++i) P[(long)i * n - (long)i * (i - 1) / 2] = 2.0;
  double *dP, *dy; cudaMalloc(&dP, P.size() * 8); cudaMalloc(&dy, n * 8);
  cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
  size_t smem = (packed_doubles(n) + 2 * n + 32) * 8;
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long t[4];
  for (int it = 0; it < 3; ++it) probe<false><<<1, 512, smem>>>(dP, n, dy);
  cudaMemcpyFromSymbol(t, g_t, 32);
  printf("generic: partials %lld  sync1 %lld  diag %lld  sync2 %lld\n", t[0], t[1], t[2], t[3]);
  for (int it = 0; it < 3; ++it) probe<true><<<1, 512, smem>>>(dP, n, dy);
  cudaMemcpyFromSymbol(t, g_t, 32);
  printf("fast32 : partials %lld  sync1 %lld  diag %lld  sync2 %lld\n", t[0], t[1], t[2], t[3]);
  long long u[8]; cudaMemcpyFromSymbol(u, g_t, 64);
  printf("fast32 sub (3 runs, 6 full blocks each): col %lld rinv %lld redsum %lld chain %lld\n", u[4], u[5], u[6], u[7]);
}
