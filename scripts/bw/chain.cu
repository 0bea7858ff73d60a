#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_shfl(double* out, const double* col_in, int reps, long long* cyc) {
  int lane = threadIdx.x & 31;
  double col[32];
  for (int k = 0; k < 32; ++k) col[k] = col_in[k * 32 + lane];
  double rinv = 1.0 / (2.0 + lane);
  double yi = lane;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (lane == k) yi *= rinv;
      const double yk = __shfl_sync(0xffffffff, yi, k);
      yi = fma(-col[k], yk, yi);
    }
  }
  long long t1 = clock64();
  out[lane] = yi;
  if (lane == 0) *cyc = (t1 - t0);
}
// variant: broadcast via shared memory instead of shuffle
__global__ void chain_smem(double* out, const double* col_in, int reps, long long* cyc) {
  __shared__ volatile double bc[32];
  int lane = threadIdx.x & 31;
  double col[32];
  for (int k = 0; k < 32; ++k) col[k] = col_in[k * 32 + lane];
  double rinv = 1.0 / (2.0 + lane);
  double yi = lane;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (lane == k) { yi *= rinv; bc[k] = yi; }
      __syncwarp();
      const double yk = bc[k];
      yi = fma(-col[k], yk, yi);
    }
  }
  long long t1 = clock64();
  out[lane] = yi;
  if (lane == 0) *cyc = (t1 - t0);
}
int main() {
  double *out, *col; long long* cyc; cudaMalloc(&out, 256); cudaMalloc(&col, 8192); cudaMalloc(&cyc, 8);
  cudaMemset(col, 0, 8192);
  long long h;
  for (int v = 0; v < 2; ++v) {
    for (int it = 0; it < 2; ++it) {
      if (v == 0) chain_shfl<<<1, 32>>>(out, col, 1000, cyc); else chain_smem<<<1, 32>>>(out, col, 1000, cyc);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%s: %.1f cycles per step\n", v == 0 ? "shfl" : "smem", h / 32000.0);
  }
  return 0;
}
