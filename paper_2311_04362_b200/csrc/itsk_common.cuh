// Shared device/host helpers for the B200 iterative-sketching path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "itsk_b200.h"

namespace itsk {

// Thread-local last error message, surfaced through itsk_last_error().
void set_error(const char* fmt, ...);

#define ITSK_CUDA(expr)                                                        \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::itsk::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                        cudaGetErrorString(_e));                               \
      return ITSK_ECUDA;                                                       \
    }                                                                          \
  } while (0)

#define ITSK_CHECK_LAUNCH() ITSK_CUDA(cudaGetLastError())

#define ITSK_REQUIRE(cond, ...)                                                \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::itsk::set_error(__VA_ARGS__);                                          \
      return ITSK_EINVAL;                                                      \
    }                                                                          \
  } while (0)

// Counts every kernel launch issued through the C-ABI (for gpu_launches).
void count_launch(int64_t k = 1);

int num_sms();

// Raise `func`'s dynamic shared-memory limit to the device maximum (once per
// kernel per process; cudaFuncSetAttribute is too slow to call per launch).
cudaError_t allow_max_smem(const void* func);
// cudaFuncSetAttribute once per (device, function, attribute)
cudaError_t func_attr_once(const void* func, cudaFuncAttribute attr, int value);
cudaError_t keep_async_pool();  // default mempool keeps its freed blocks (once per device)

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Fixed-order block sum: every thread receives the same value; the order of
// the additions depends only on blockDim, so results are run-to-run
// deterministic.  `red` must hold blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

// Software grid barrier for cooperatively launched kernels.  bar[0] counts
// arrivals, bar[1] is the generation.  Both must start at zero.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned gen = ld_acquire(bar + 1);
    unsigned arrived;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                 : "=r"(arrived) : "l"(bar) : "memory");
    if (arrived == nb - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      while (ld_acquire(bar + 1) == gen) {
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
}

// Streaming loads for A (read once per pass): no L1 allocation and an
// L2 evict-first policy so A does not push R / x / r out of L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ double ldg_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// ---- programmatic dependent launch ----
// griddepcontrol.wait: block until the preceding kernel in the stream has
// completed and its memory is visible; launch_dependents: let the next kernel
// start its prologue.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch `func` with programmatic stream serialisation allowed (kernels that
// call pdl_wait() before touching their predecessor's output).  ITSK_NO_PDL=1
// launches without the attribute.
bool pdl_enabled();
template <class... Args>
cudaError_t launch_pdl(const void* func, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  void* ptrs[] = {static_cast<void*>(&args)...};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, func, ptrs);
}

// ---- mbarrier + 1D bulk copy (TMA) helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, unsigned bytes,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Carver {
  char* base;
  int64_t cap;
  int64_t off = 0;
  Carver(void* b, int64_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(int64_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * static_cast<int64_t>(sizeof(T));
    return p;
  }
  bool ok() const { return off <= cap; }
};

#ifdef ITSK_TIMELINE
// Diagnostic build only (build.py probe="timeline"): %globaltimer in ns.
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int TL_SLOTS = 64;
#endif

}  // namespace itsk
