#include <cstdio>
#include <vector>
#include "itsk_dense.cuh"
using namespace itsk;
namespace itsk { void set_error(const char*, ...) {} void count_launch(int64_t) {} int num_sms() { return 148; } cudaError_t allow_max_smem(const void*) { return cudaSuccess; } }
__global__ void __launch_bounds__(512) probe(const double* Rp, int n, double* y, long long* cyc) {
  extern __shared__ double sm[];
  stage_packed_bulk(Rp, n, sm);
  RPacked R{sm, n};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    const int b0 = 64, bs = 32;
    long long t0 = clock64();
    double col[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) col[k] = (k < lane && lane < bs) ? R(b0 + k, b0 + lane) : 0.0;
    __syncwarp();
    long long t1 = clock64();
    const double dd = R(b0 + lane, b0 + lane);
    const double rinv = (lane < bs) ? 1.0 / dd : 0.0;
    __syncwarp();
    long long t2 = clock64();
    double yi = y[lane] + rinv * 0.0 + col[lane & 31] * 0.0;
    __syncwarp();
    long long t3 = clock64();
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k < bs) {
        if (lane == k) yi *= rinv;
        const double yk = __shfl_sync(FULL, yi, k);
        yi = fma(-col[k], yk, yi);
      }
    }
    __syncwarp();
    long long t4 = clock64();
    y[lane] = yi;
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t4 - t3; }
  }
}
int main() {
  int n = 200;
  std::vector<double> P((n * (n + 1) / 2) + 2, 0.5);
  double *dP, *dy; long long* dc; cudaMalloc(&dP, P.size() * 8); cudaMalloc(&dy, 256 * 8); cudaMalloc(&dc, 64);
  cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice); cudaMemset(dy, 0, 2048);
  size_t smem = (packed_doubles(n) + 2) * 8;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long c[4];
  for (int it = 0; it < 3; ++it) probe<<<1, 512, smem>>>(dP, n, dy, dc);
  cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
  printf("col loads %lld  rinv %lld  chain %lld cycles (%s)\n", c[0], c[1], c[2], cudaGetErrorString(cudaGetLastError()));
}
