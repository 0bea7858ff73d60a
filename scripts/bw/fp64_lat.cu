// Dependent-chain latency of FP64 ops on this GPU (single warp, clock64).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a, y = b;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = fma(x, a, y); x = fma(x, a, y); x = fma(x, a, y); x = fma(x, a, y); }
  long long t2 = clock64();
  float f = (float)x, g = (float)y;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { f = fmaf(f, g, 1.0f); f = fmaf(f, g, 1.0f); f = fmaf(f, g, 1.0f); f = fmaf(f, g, 1.0f); }
  long long t3 = clock64();
  double z = x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { z = __shfl_sync(0xffffffff, z, (threadIdx.x + 1) & 31); }
  long long t4 = clock64();
  double w = z;
#pragma unroll 1
  for (int i = 0; i < 200; ++i) { w = 1.0 / (w + 3.0); }
  long long t5 = clock64();
#pragma unroll 1
  for (int i = 0; i < 200; ++i) { w = sqrt(w + 3.0); }
  long long t6 = clock64();
  out[threadIdx.x] = x + f + z + w;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 1.0000001, 1e-9); k<<<1, 32>>>(o, c, 1.0000001, 1e-9);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("DADD %.1f  DFMA %.1f  FFMA %.1f  SHFL(f64) %.1f  DDIV %.1f  DSQRT %.1f cycles/op\n", h[0] / 4000.0, h[1] / 4000.0, h[2] / 4000.0, h[3] / 1000.0, h[4] / 200.0, h[5] / 200.0);
  return 0;
}
