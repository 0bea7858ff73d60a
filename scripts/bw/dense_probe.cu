// Cycle-level probe of the single-CTA dense primitives (packed R in smem),
// with and without the diagonal-block inverses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_04362_b200/csrc \
//        -o scripts/bw/dense_probe scripts/bw/dense_probe.cu
#include <cstdio>
#include <vector>
#include <cmath>
#define ITSK_DENSE_PROBE
#include "itsk_dense.cuh"
using namespace itsk;
namespace itsk { void set_error(const char*, ...) {} void count_launch(int64_t) {} int num_sms() { return 148; } cudaError_t allow_max_smem(const void*) { return cudaSuccess; } }

__global__ void __launch_bounds__(512) probe(const double* Rp, int n, double* y, long long* cyc, int with_inv) {
  extern __shared__ double sm[];
  __shared__ double red[64 * 16];
  long long t0 = clock64();
  stage_packed_bulk(Rp, n, sm, with_inv != 0);
  long long t1 = clock64();
  double* v = sm + (with_inv ? rp_doubles(n) : packed_doubles(n));
  double* tmp = v + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = 1.0 + i;
  __syncthreads();
  RPacked R(sm, n);
  const DiagInv inv = diag_inv_at(sm, n, with_inv != 0);
  long long t2 = clock64();
  trsv_t_inplace(R, n, v, red, inv);
  long long t3 = clock64();
  trsv_n_inplace(R, n, v, red, inv);
  long long t4 = clock64();
  trmv_n(R, n, v, tmp);
  long long t5 = clock64();
  trmv_t(R, n, tmp, v, red);
  long long t6 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; cyc[2] = t4 - t3; cyc[3] = t5 - t4; cyc[4] = t6 - t5; }
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = v[i];
}

int main() {
  for (int n : {32, 64, 200}) {
    for (int with_inv = 0; with_inv < 2; ++with_inv) {
      std::vector<double> R(n * n, 0.0), P(rp_doubles(n), 0.0);
      for (int i = 0; i < n; ++i) for (int j = i; j < n; ++j) R[i * n + j] = (i == j) ? n + 2.0 : 0.01 * ((i * 7 + j * 3) % 11 - 5);
      for (int i = 0; i < n; ++i) for (int j = i; j < n; ++j) P[(long)i * n - (long)i * (i - 1) / 2 + (j - i)] = R[i * n + j];
      const long X0 = packed_bytes(n) / 8, K0 = X0 + invd_doubles(n);
      for (int B = 0; B * 32 < n; ++B) {
        const int b0 = 32 * B, bs = std::min(32, n - b0);
        for (int j = 0; j < bs; ++j) {
          double x[32] = {0};
          x[j] = 1.0 / R[(b0 + j) * n + b0 + j];
          for (int k = j - 1; k >= 0; --k) { double s = 0; for (int l = k + 1; l <= j; ++l) s += R[(b0 + k) * n + b0 + l] * x[l]; x[k] = -s / R[(b0 + k) * n + b0 + k]; }
          for (int k = 0; k <= j; ++k) P[X0 + B * 528 + k * bs - k * (k - 1) / 2 + (j - k)] = x[k];
        }
        P[K0 + B] = 1.0;
      }
      double *dP, *dy; long long* dc; cudaMalloc(&dP, P.size() * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dc, 64);
      cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
      size_t smem = (rp_doubles(n) + 2 * n + 32) * 8;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
      long long c[8];
      for (int it = 0; it < 3; ++it) probe<<<1, 512, smem>>>(dP, n, dy, dc, with_inv);
      cudaMemcpy(c, dc, 40, cudaMemcpyDeviceToHost);
      long long z8[8] = {0}; cudaMemcpyToSymbol(g_probe, z8, 64);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0); for (int it = 0; it < 20; ++it) probe<<<1, 512, smem>>>(dP, n, dy, dc, with_inv); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long gp[8]; cudaMemcpyFromSymbol(gp, g_probe, 64);
      std::vector<double> y(n); cudaMemcpy(y.data(), dy, n * 8, cudaMemcpyDeviceToHost);
      double cs = 0; for (double v : y) cs += v;
      printf("n=%d inv=%d stage %lld trsv_t %lld trsv_n %lld trmv_n %lld trmv_t %lld cycles; kernel %.1f us; t-blocks prep %lld (red %lld p2 %lld) chain %lld; checksum %.15e (%s)\n",
             n, with_inv, c[0], c[1], c[2], c[3], c[4], ms * 1e3 / 20, gp[0] / 20, gp[2] / 20, gp[3] / 20, gp[1] / 20, cs, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
