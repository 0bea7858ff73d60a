// Does a runtime-API (<<<>>>) launch into a green-context stream stay on the
// green context's SMs?  Splits the device's SMs into a 32-SM group and the
// rest, launches a kernel recording %smid into each group's stream, and a
// 16-CTA cluster kernel into the small group.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/bw/green_ctx_probe scripts/bw/green_ctx_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <set>
#include <cstdlib>

__global__ void k_smid(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(s);
  // keep the CTA resident a little while
  long long t0 = clock64();
  while (clock64() - t0 < 200000) {
  }
}
__global__ void k_smid_cl(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(s);
}

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* m; cuGetErrorString(r, &m); printf("%s -> %s\n", #x, m); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

int main(int argc, char** argv) {
  const unsigned want = argc > 1 ? atoi(argv[1]) : 32;
  RK(cudaFree(0));
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  CUdevResource parts[2], rest;
  unsigned nparts = 1;
  CK(cuDevSmResourceSplitByCount(parts, &nparts, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, want));
  printf("split: %u group(s) of %u SMs, rest %u SMs\n", nparts, parts[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc da, db;
  CK(cuDevResourceGenerateDesc(&da, &parts[0], 1));
  CK(cuDevResourceGenerateDesc(&db, &rest, 1));
  CUgreenCtx ga, gb;
  CK(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sa, sb;
  CK(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
  int *da_out, *db_out, *dc_out;
  RK(cudaMalloc(&da_out, 4096 * 4));
  RK(cudaMalloc(&db_out, 4096 * 4));
  RK(cudaMalloc(&dc_out, 4096 * 4));
  k_smid<<<1024, 128, 0, (cudaStream_t)sa>>>(da_out);
  RK(cudaGetLastError());
  k_smid<<<1024, 128, 0, (cudaStream_t)sb>>>(db_out);
  RK(cudaGetLastError());
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(64);
    cfg.blockDim = dim3(128);
    cfg.stream = (cudaStream_t)sa;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cs == 16) cudaFuncSetAttribute(k_smid_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_smid_cl, dc_out);
    cudaError_t e2 = cudaStreamSynchronize((cudaStream_t)sa);
    printf("cluster %2d in the small green context: launch %s, sync %s\n", cs, cudaGetErrorString(e), cudaGetErrorString(e2));
    if (e2 != cudaSuccess) return 1;
  }
  RK(cudaDeviceSynchronize());
  int ha[1024], hb[1024], hc[64];
  RK(cudaMemcpy(ha, da_out, sizeof(ha), cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(hb, db_out, sizeof(hb), cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(hc, dc_out, sizeof(hc), cudaMemcpyDeviceToHost));
  std::set<int> A(ha, ha + 1024), B(hb, hb + 1024), C(hc, hc + 64);
  int both = 0;
  for (int x : A) both += B.count(x);
  printf("group A kernel used %zu distinct SMs, group B kernel %zu, overlap %d; cluster kernel in A used %zu SMs (all in A: %s)\n",
         A.size(), B.size(), both, C.size(), [&] { for (int x : C) if (!A.count(x)) return "no"; return "yes"; }());
  return 0;
}
