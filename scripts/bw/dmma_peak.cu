// fp64 peak probes for the QR roofline (MEASURED_PEAKS.json
// has no fp64 figure).
//   dmma : mma.sync.aligned.m8n8k4.row.col.f64 (the DMMA tensor pipe),
//          NACC independent accumulators per warp, W warps per CTA, every SM
//   dfma : fma.rn.f64 chains on the fp64 pipe (the non-tensor path)
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bw/dmma_peak scripts/bw/dmma_peak.cu
// Run:    scripts/bw/dmma_peak            (prints one line per configuration)
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
static float time_it(K kern, int grid, int block, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, iters);  // warm
  cudaEventRecord(e0);
  kern<<<grid, block>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 64);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int ctas_per_sm : {1, 2}) {
      int grid = sms * ctas_per_sm, block = 32 * warps;
      float ms = time_it(k_dmma<8>, grid, block, out, iters);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid * warps;
      printf("dmma m8n8k4 nacc=8 warps/cta=%d ctas/sm=%d: %.3f ms  %.2f TFLOP/s\n", warps, ctas_per_sm, ms,
             flops / ms / 1e9);
    }
  }
  for (int warps : {8, 16, 32}) {
    int grid = sms * 2, block = 32 * warps;
    float ms = time_it(k_dfma<8>, grid, block, out, iters);
    double flops = 2.0 * 8 * iters * (double)grid * block;
    printf("dfma nacc=8 warps/cta=%d ctas/sm=2: %.3f ms  %.2f TFLOP/s\n", warps, ms, flops / ms / 1e9);
  }
  printf("sms=%d clock_khz=%d err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
