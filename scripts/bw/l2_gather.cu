// Gather-bandwidth probe for the sketch's roofline: warps gather random
// 1 KB row segments (128 doubles, the sketch's column block) from a source
// buffer and sum them, like k_sketch_gather.  With the source L2-resident
// (<= ~60 MB) this is the L2 -> SM gather ceiling; with a large source
// (>> L2) it is the HBM random-1KB ceiling.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bw/l2_gather scripts/bw/l2_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_gather(const double* __restrict__ src, int64_t rows, int64_t ld, const uint32_t* __restrict__ idx,
                         int per_warp, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t* my = idx + w * per_warp;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int k = 0; k < per_warp; k += 4) {
    double4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double* p = src + static_cast<int64_t>(my[k + u]) * ld + 4 * lane;
      v[u] = *reinterpret_cast<const double4*>(p);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 += v[u].x;
      a1 += v[u].y;
      a2 += v[u].z;
      a3 += v[u].w;
    }
  }
  if (a0 + a1 + a2 + a3 == 12345.0) out[0] = a0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t ld = 2048;  // a 16 KB row, 1 KB gathered per source (like C4's column blocks)
  const int per_warp = 1024;
  const int warps = sms * 64;
  uint32_t* idx;
  cudaMalloc(&idx, sizeof(uint32_t) * static_cast<int64_t>(warps) * per_warp);
  double* out;
  cudaMalloc(&out, 64);
  for (int64_t rows : {2048LL, 3072LL, 4096LL, 8192LL, 262144LL, 2097152LL}) {
    double* src;
    if (cudaMalloc(&src, rows * ld * 8) != cudaSuccess) break;
    cudaMemset(src, 0, rows * ld * 8);
    // random source rows (a fixed LCG) in each warp's list
    uint32_t* h = new uint32_t[static_cast<int64_t>(warps) * per_warp];
    uint64_t s = 12345;
    for (int64_t i = 0; i < static_cast<int64_t>(warps) * per_warp; ++i) {
      s = s * 6364136223846793005ULL + 1442695040888963407ULL;
      h[i] = static_cast<uint32_t>((s >> 33) % rows);
    }
    cudaMemcpy(idx, h, sizeof(uint32_t) * static_cast<int64_t>(warps) * per_warp, cudaMemcpyHostToDevice);
    delete[] h;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_gather<<<warps / 8, 256>>>(src, rows, ld, idx, per_warp, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_gather<<<warps / 8, 256>>>(src, rows, ld, idx, per_warp, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 5.0 * warps * per_warp * 1024;
    printf("gather 1 KB segments from %8.1f MB (%lld rows of 16 KB): %.3f ms  %.0f GB/s  err=%s\n",
           rows * ld * 8 / 1e6, static_cast<long long>(rows), ms / 5, bytes / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(src);
  }
  return 0;
}
