// Streaming-read bandwidth probe: TMA bulk ring (1D cp.async.bulk) vs LDG.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_tx(uint64_t* b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned par) {
  asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=; }" :: "r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su32(dst)), "l"(src), "r"(n), "r"(su32(bar)) : "memory");
}

// one producer lane per stage group; NC consumer warps touch one double per lane
__global__ void tma_stream(const char* A, long long bytes_per_cta, int chunk, int S, int NC, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm; uint64_t* empty = full + 64;
  unsigned char* buf = sm + 1024;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  long long nchunks = bytes_per_cta / chunk;
  const char* base = A + (long long)blockIdx.x * bytes_per_cta;
  if (tid == 0) { for (int s = 0; s < S; ++s) { mb_init(full + s, 1); mb_init(empty + s, NC); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  double acc = 0;
  if (warp == NC) {
    if (lane == 0) {
      for (long long t = 0; t < nchunks; ++t) {
        int s = t % S;
        if (t >= S) mb_wait(empty + s, ((t / S) - 1) & 1);
        mb_tx(full + s, chunk);
        bulk(buf + (long long)s * chunk, base + t * chunk, chunk, full + s);
      }
    }
  } else {
    for (long long t = 0; t < nchunks; ++t) {
      int s = t % S;
      mb_wait(full + s, (t / S) & 1);
      acc += ((const double*)(buf + (long long)s * chunk))[warp * 32 + lane];
      __syncwarp();
      if (lane == 0) mb_arrive(empty + s);
    }
  }
  if (acc == 12345.0) out[0] = acc;
}

__global__ void ldg_stream(const double2* A, long long n2_per_cta, double* out) {
  const double2* base = A + (long long)blockIdx.x * n2_per_cta;
  double acc = 0;
  #pragma unroll 8
  for (long long i = threadIdx.x; i < n2_per_cta; i += blockDim.x) { double2 v = __ldcs(base + i); acc += v.x + v.y; }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const long long total = 1536ll << 20;  // 1.5 GB
  char* A; double* out; cudaMalloc(&A, total); cudaMalloc(&out, 8); cudaMemset(A, 0, total);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int ctas_per_sm, chunk, S, NC; };
  std::vector<Cfg> cfgs = {{1, 16384, 12, 8}, {1, 8192, 24, 8}, {1, 4096, 48, 8}, {1, 32768, 6, 8},
                           {2, 16384, 6, 4}, {2, 8192, 12, 4}, {4, 8192, 6, 2}, {4, 4096, 12, 2}, {1, 16384, 13, 16}};
  for (auto c : cfgs) {
    int grid = sms * c.ctas_per_sm;
    long long per = (total / grid) / c.chunk * c.chunk;
    size_t smem = 1024 + (size_t)c.S * c.chunk;
    if (smem > 220 * 1024 / c.ctas_per_sm + 1024) { smem = 0; }
    int th = 32 * (c.NC + 1);
    for (int w = 0; w < 2; ++w) tma_stream<<<grid, th, smem>>>(A, per, c.chunk, c.S, c.NC, out);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) tma_stream<<<grid, th, smem>>>(A, per, c.chunk, c.S, c.NC, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("TMA ctas/sm=%d chunk=%6d S=%2d NC=%2d : %7.0f GB/s  (%s)\n", c.ctas_per_sm, c.chunk, c.S, c.NC,
           5.0 * per * grid / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  for (int bs : {256, 512, 1024}) for (int cps : {1, 2, 4, 8}) {
    if (bs * cps > 2048) continue;
    int grid = sms * cps; long long per2 = (total / 16) / grid;
    for (int w = 0; w < 2; ++w) ldg_stream<<<grid, bs>>>((const double2*)A, per2, out);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) ldg_stream<<<grid, bs>>>((const double2*)A, per2, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG bs=%4d ctas/sm=%d : %7.0f GB/s\n", bs, cps, 5.0 * per2 * 16 * grid / (ms * 1e-3) / 1e9);
  }
  return 0;
}
