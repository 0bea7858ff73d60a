// Pure streaming-read time vs size (is the fused pass's fixed cost at C2
// inherent to a 320 MB read?): TMA bulk ring, 148 CTAs x 1, 16 KB chunks,
// per-CTA start / end times from %globaltimer.
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
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void tma_stream(const char* A, long long bytes_per_cta, int chunk, int S, int NC, double* out,
                           unsigned long long* ts) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm; uint64_t* empty = full + 64;
  unsigned char* buf = sm + 1024;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0 && ts) ts[3 * blockIdx.x] = gt();
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
      if (t == 0 && tid == 0 && ts) ts[3 * blockIdx.x + 1] = gt();
      acc += ((const double*)(buf + (long long)s * chunk))[warp * 32 + lane];
      __syncwarp();
      if (lane == 0) mb_arrive(empty + s);
    }
  }
  if (acc == 12345.0) out[0] = acc;
  __syncthreads();
  if (tid == 0 && ts) ts[3 * blockIdx.x + 2] = gt();
}

__global__ void empty_k(double* out) { if (threadIdx.x == 9999) out[0] = 1; }

int main() {
  const long long maxb = 1280ll << 20;
  char* A; double* out; unsigned long long* ts;
  cudaMalloc(&A, maxb); cudaMalloc(&out, 8); cudaMemset(A, 0, maxb);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&ts, 3 * 8 * sms * sizeof(unsigned long long));
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (size_t smem : {0ul, 200ul * 1024}) {
    for (int w = 0; w < 3; ++w) empty_k<<<sms, 544, smem>>>(out);
    cudaEventRecord(e0);
    for (int it = 0; it < 50; ++it) empty_k<<<sms, 544, smem>>>(out);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("empty kernel 148x544 smem=%zu: %.2f us per launch\n", smem, ms * 1e3 / 50);
  }
  const int chunk = 16384, S = 12, NC = 16;
  for (long long mb : {40, 80, 160, 320, 640, 1280}) {
    long long total = mb << 20;
    int grid = sms;
    long long per = (total / grid) / chunk * chunk;
    size_t smem = 1024 + (size_t)S * chunk;
    int th = 32 * (NC + 1);
    for (int w = 0; w < 3; ++w) tma_stream<<<grid, th, smem>>>(A, per, chunk, S, NC, out, nullptr);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) tma_stream<<<grid, th, smem>>>(A, per, chunk, S, NC, out, nullptr);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1e3 / 20;
    tma_stream<<<grid, th, smem>>>(A, per, chunk, S, NC, out, ts);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(3 * grid);
    cudaMemcpy(h.data(), ts, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, tmax = 0; std::vector<double> st, fa, en;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[3 * b]);
    for (int b = 0; b < grid; ++b) { st.push_back((h[3*b]-t0)*1e-3); fa.push_back((h[3*b+1]-t0)*1e-3); en.push_back((h[3*b+2]-t0)*1e-3); }
    std::sort(st.begin(), st.end()); std::sort(fa.begin(), fa.end()); std::sort(en.begin(), en.end());
    printf("%5lld MB: %8.1f us  %6.0f GB/s | start max %.2f us, first-tile med %.2f max %.2f, end min %.1f med %.1f max %.1f us\n",
           mb, us, per * grid / (us * 1e-6) / 1e9, st.back(), fa[grid/2], fa.back(), en.front(), en[grid/2], en.back());
  }
  return 0;
}
