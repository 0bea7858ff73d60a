// Cycle-level probe of the single-CTA dense primitives (n = 200, packed R in smem).
#include <cstdio>
#include <vector>
#include <cmath>
#define ITSK_DENSE_PROBE
#include "itsk_dense.cuh"
using namespace itsk;
namespace itsk { void set_error(const char*, ...) {} void count_launch(int64_t) {} int num_sms() { return 148; } cudaError_t allow_max_smem(const void*) { return cudaSuccess; } }

__global__ void __launch_bounds__(512) probe(const double* Rp, int n, double* y, long long* cyc) {
  extern __shared__ double sm[];
  __shared__ double red[64 * 16];
  long long t0 = clock64();
  stage_packed_bulk(Rp, n, sm);
  long long t1 = clock64();
  double* v = sm + packed_doubles(n);
  double* tmp = v + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = 1.0 + i;
  __syncthreads();
  RPacked R(sm, n);
  long long t2 = clock64();
  trsv_t_inplace(R, n, v, red);
  long long t3 = clock64();
  trsv_n_inplace(R, n, v, red);
  long long t4 = clock64();
  trmv_n(R, n, v, tmp);
  long long t5 = clock64();
  trmv_t(R, n, tmp, v, red);
  long long t6 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; cyc[2] = t4 - t3; cyc[3] = t5 - t4; cyc[4] = t6 - t5; }
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = v[i];
}
__global__ void empty_k(long long* c) { if (threadIdx.x == 0) c[7] = 1; }

int main() {
  for (int n : {32, 64, 200}) {
    std::vector<double> R(n * n, 0.0), P((n * (n + 1) / 2) + 2, 0.0);
    for (int i = 0; i < n; ++i) for (int j = i; j < n; ++j) R[i * n + j] = (i == j) ? n + 2.0 : 0.01 * ((i * 7 + j * 3) % 11 - 5);
    for (int i = 0; i < n; ++i) for (int j = i; j < n; ++j) P[(long)i * n - (long)i * (i - 1) / 2 + (j - i)] = R[i * n + j];
    double *dP, *dy; long long* dc; cudaMalloc(&dP, P.size() * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dc, 64);
    cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = (packed_doubles(n) + 2 * n + 32) * 8;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long c[8];
    for (int it = 0; it < 3; ++it) probe<<<1, 512, smem>>>(dP, n, dy, dc);
    cudaMemcpy(c, dc, 40, cudaMemcpyDeviceToHost);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); for (int it = 0; it < 20; ++it) probe<<<1, 512, smem>>>(dP, n, dy, dc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long gp[8]; cudaMemcpyFromSymbol(gp, g_probe, 64); long long z8[8] = {0}; cudaMemcpyToSymbol(g_probe, z8, 64);
    printf("   per-call (23 calls) prep %lld chain %lld\n", gp[0] / 23, gp[1] / 23);
    printf("n=%d stage %lld  trsv_t %lld  trsv_n %lld  trmv_n %lld  trmv_t %lld cycles ; kernel %.1f us  (%s)\n", n, c[0], c[1], c[2], c[3], c[4], ms * 1e3 / 20, cudaGetErrorString(cudaGetLastError()));
  }
  long long* dc; cudaMalloc(&dc, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  empty_k<<<1, 512>>>(dc);
  cudaEventRecord(e0); for (int it = 0; it < 100; ++it) empty_k<<<1, 512>>>(dc); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("empty kernel %.2f us\n", ms * 1e3 / 100);
  return 0;
}
