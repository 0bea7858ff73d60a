// S·[A | b] — the sparse sign sketch (K1).
//
// Replaces SparseSignEmbedding.apply_dense / apply_vec
// (/root/reference/pkg/src/itsketch/embed.py:62-74), i.e. scipy's
// csc_matvecs, which computes  for j ascending: for each stored (i, v) of
// column j:  y[i, :] += v * a[j, :]  with the product rounded before the add.
// Here the pattern is grouped by sketch row i (CSR of S, sources ascending),
// one warp owns sketch row i x a column block and accumulates its sources in
// the same ascending order in registers — so every output is bitwise equal to
// scipy's, and the kernel is deterministic.  The b column rides along as
// column n of the output (apply_vec is the same sum, solvers.py:208).
#include <algorithm>
#include <cstdlib>

#include "itsk_common.cuh"

namespace itsk {
namespace {

// Source-row window of one launch: only sources j in [j0, j1) are summed,
// continuing from W's current value when `accum` is set.  Sources are
// ascending in each sketch row's list, so consecutive windows in row order
// add the same terms in the same order as one launch over all rows — the
// upload pipeline sketches A chunk by chunk as it arrives, bitwise the same.
struct SkRange {
  uint32_t j0, j1;
  int accum;
};

__device__ __forceinline__ uint32_t lower_src(const uint32_t* __restrict__ src, uint32_t lo, uint32_t hi,
                                              uint32_t key) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((src[mid] & 0x7fffffffu) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int CPL, int UNR>
__global__ void __launch_bounds__(128) k_sketch_gather(
    const double* __restrict__ A, int64_t lda, int64_t n, const double* __restrict__ b,
    const uint32_t* __restrict__ ptr, const uint32_t* __restrict__ src, int64_t d,
    double scale, double* __restrict__ W, int64_t ldw, SkRange rg) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= d) return;
  const int64_t ncol = n + (b ? 1 : 0);
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * 32 * CPL;
  // per column slot: 0 = A column, 1 = the b column, 2 = none
  int kind[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int64_t col = c0 + lane + 32 * q;
    kind[q] = col < n ? 0 : (col == n && b ? 1 : 2);
  }
  const double* Ac = A + c0 + lane;
  double acc[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int64_t col = c0 + lane + 32 * q;
    acc[q] = (rg.accum && col < ncol) ? W[i * ldw + col] : 0.0;
  }
  uint32_t e0 = ptr[i], e1 = ptr[i + 1];
  if (rg.j0 > 0) e0 = lower_src(src, e0, e1, rg.j0);
  if (rg.j1 != 0xffffffffu) e1 = lower_src(src, e0, e1, rg.j1);
  for (uint32_t e = e0; e < e1; e += 32) {
    const uint32_t mine = (e + lane < e1) ? src[e + lane] : 0u;
    const int cnt = static_cast<int>(min(32u, e1 - e));
    int k = 0;
    for (; k + UNR <= cnt; k += UNR) {
      double v[UNR][CPL];
      double sv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint32_t s = __shfl_sync(FULL, mine, k + u);
        const int64_t j = s & 0x7fffffffu;
        sv[u] = (s >> 31) ? -scale : scale;
        const double* arow = Ac + j * lda;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          v[u][q] = kind[q] == 0 ? arow[32 * q] : (kind[q] == 1 ? b[j] : 0.0);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int q = 0; q < CPL; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(sv[u], v[u][q]));
    }
    for (; k < cnt; ++k) {
      const uint32_t s = __shfl_sync(FULL, mine, k);
      const int64_t j = s & 0x7fffffffu;
      const double svk = (s >> 31) ? -scale : scale;
      const double* arow = Ac + j * lda;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const double a = kind[q] == 0 ? arow[32 * q] : (kind[q] == 1 ? b[j] : 0.0);
        acc[q] = __dadd_rn(acc[q], __dmul_rn(svk, a));
      }
    }
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int64_t col = c0 + lane + 32 * q;
    if (col < ncol) W[i * ldw + col] = acc[q];
  }
}

// Ring variant: warp per (sketch row, 32-column block), one column per lane,
// each lane streaming its element of the next RG_DEPTH source rows into a
// per-warp shared-memory ring with cp.async (8 bytes per lane per source,
// commit groups of RG_G sources) while it adds the landed ones in source
// order.  The register gather keeps only UNR sources in flight per warp,
// which starves the memory system when d x column blocks is small (few
// warps, long sequential chains: C5's d = 4n points); here ~RG_DEPTH are.
// Same sums in the same order: bitwise equal to the register gather.
constexpr int RG_DEPTH = 64;
constexpr int RG_G = 8;
constexpr int RG_NG = RG_DEPTH / RG_G;
constexpr int RG_WARPS = 4;

__device__ __forceinline__ void cp_async8_ring(double* dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int nbytes = valid ? 8 : 0;  // 0: zero-fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_commit_ring() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_n() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_wait_ring(int pending) {
  // pending groups allowed to stay in flight (an immediate operand)
  switch (pending < RG_NG - 1 ? pending : RG_NG - 1) {
    case 0: cp_wait_n<0>(); break;
    case 1: cp_wait_n<1>(); break;
    case 2: cp_wait_n<2>(); break;
    case 3: cp_wait_n<3>(); break;
    case 4: cp_wait_n<4>(); break;
    case 5: cp_wait_n<5>(); break;
    case 6: cp_wait_n<6>(); break;
    default: cp_wait_n<7>(); break;
  }
}

// Source words reach the issuing lanes as a 32-word register block (one
// coalesced load, the next block prefetched) and the consumer through a small
// shared-memory ring written at issue time: no dependent global load sits
// between consuming a group and issuing its refill.
__global__ void __launch_bounds__(32 * RG_WARPS) k_sketch_ring(
    const double* __restrict__ A, int64_t lda, int64_t n, const double* __restrict__ b,
    const uint32_t* __restrict__ ptr, const uint32_t* __restrict__ src, int64_t d,
    double scale, double* __restrict__ W, int64_t ldw, SkRange rg) {
  static_assert(RG_NG <= 8 && 32 % RG_G == 0, "ring shape");
  extern __shared__ __align__(16) double ring_sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = ring_sm + static_cast<int64_t>(warp) * RG_DEPTH * 32;
  uint32_t* rsrc = reinterpret_cast<uint32_t*>(ring_sm + RG_WARPS * RG_DEPTH * 32) + warp * RG_DEPTH;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * RG_WARPS + warp;
  if (i >= d) return;  // no CTA-wide barriers below
  const int64_t ncol = n + (b ? 1 : 0);
  const int64_t col = static_cast<int64_t>(blockIdx.y) * 32 + lane;
  const int kind = col < n ? 0 : (col == n && b ? 1 : 2);
  const double* base = kind == 0 ? A + col : (kind == 1 ? b : A);
  const int64_t stride = kind == 0 ? lda : (kind == 1 ? 1 : 0);
  double acc = (rg.accum && col < ncol) ? W[i * ldw + col] : 0.0;
  uint32_t e0 = ptr[i], e1 = ptr[i + 1];
  if (rg.j0 > 0) e0 = lower_src(src, e0, e1, rg.j0);
  if (rg.j1 != 0xffffffffu) e1 = lower_src(src, e0, e1, rg.j1);
  const uint32_t total = e1 - e0;
  const uint32_t ngroups = (total + RG_G - 1) / RG_G;
  double* my = ring + lane;
  // issue side: src words of the 32-block holding the next group, and the block after
  uint32_t blk = 0;
  uint32_t wcur = lane < total ? __ldg(src + e0 + lane) : 0u;
  uint32_t wnxt = 32 + lane < total ? __ldg(src + e0 + 32 + lane) : 0u;
  auto issue_group = [&](uint32_t g) {
    const uint32_t q0 = g * RG_G;
    if ((q0 >> 5) != blk) {  // next 32-block (uniform): rotate and prefetch the one after
      blk = q0 >> 5;
      wcur = wnxt;
      const uint32_t qn = (blk + 1) * 32 + lane;
      wnxt = qn < total ? __ldg(src + e0 + qn) : 0u;
    }
#pragma unroll
    for (int u = 0; u < RG_G; ++u) {
      const uint32_t q = q0 + u;
      const uint32_t w = __shfl_sync(FULL, wcur, (q0 & 31) + u);
      if (q < total) cp_async8_ring(my + (q % RG_DEPTH) * 32, base + static_cast<int64_t>(w & 0x7fffffffu) * stride,
                                    kind != 2);
    }
    const uint32_t wv = __shfl_sync(FULL, wcur, (q0 & 31) + (lane & (RG_G - 1)));
    if (lane < RG_G) rsrc[(q0 + lane) % RG_DEPTH] = wv;
    cp_commit_ring();
  };
  const uint32_t npro = ngroups < static_cast<uint32_t>(RG_NG) ? ngroups : static_cast<uint32_t>(RG_NG);
  for (uint32_t g = 0; g < npro; ++g) issue_group(g);
  for (uint32_t g = 0; g < ngroups; ++g) {
    const uint32_t left = ngroups - g - 1;
    cp_wait_ring(static_cast<int>(left));
    __syncwarp();  // rsrc entries written by other lanes
    double v[RG_G];
    uint32_t sw[RG_G];
#pragma unroll
    for (int u = 0; u < RG_G; ++u) {
      const uint32_t q = g * RG_G + u;
      sw[u] = rsrc[q % RG_DEPTH];
      v[u] = my[(q % RG_DEPTH) * 32];
    }
#pragma unroll
    for (int u = 0; u < RG_G; ++u) {
      const uint32_t q = g * RG_G + u;
      if (q < total) acc = __dadd_rn(acc, __dmul_rn((sw[u] >> 31) ? -scale : scale, v[u]));
    }
    __syncwarp();  // every lane has read the group's rsrc slots before they are rewritten
    // the slots just read are free: refill them with group g + RG_NG
    if (g + RG_NG < ngroups) issue_group(g + RG_NG);
  }
  if (col < ncol) W[i * ldw + col] = acc;
}

int launch_ring(const double* A, int64_t lda, int64_t n, const double* b, const uint32_t* ptr,
                const uint32_t* src, int64_t d, double scale, double* W, int64_t ldw, SkRange rg,
                cudaStream_t s) {
  const int64_t ncol = n + (b ? 1 : 0);
  dim3 grid(static_cast<unsigned>((d + RG_WARPS - 1) / RG_WARPS), static_cast<unsigned>((ncol + 31) / 32));
  const size_t smem = RG_WARPS * RG_DEPTH * (32 * sizeof(double) + sizeof(uint32_t));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_sketch_ring)));
  k_sketch_ring<<<grid, 32 * RG_WARPS, smem, s>>>(A, lda, n, b, ptr, src, d, scale, W, ldw, rg);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

// Tuning knobs (read per call so tests can sweep the variants in-process).
struct SketchTune {
  int ring = -1;      // 1: cp.async ring variant, 0: register gather, -1: by shape
  int gcpl = 0;       // register gather: cap on columns-per-lane (more column blocks)
  int unr = 0;        // register gather: sources per unrolled group (0 = heuristic)
  SketchTune() {
    if (const char* e = getenv("ITSK_SKETCH_RING")) ring = atoi(e);
    if (const char* e = getenv("ITSK_SKETCH_GCPL")) gcpl = atoi(e);
    if (const char* e = getenv("ITSK_SKETCH_UNR")) unr = atoi(e);
  }
};

SketchTune sketch_tune() { return SketchTune(); }

template <int CPL, int UNR>
int launch_gather(const double* A, int64_t lda, int64_t n, const double* b,
                  const uint32_t* ptr, const uint32_t* src, int64_t d, double scale, double* W,
                  int64_t ldw, SkRange rg, cudaStream_t s) {
  const int64_t ncol = n + (b ? 1 : 0);
  dim3 grid(static_cast<unsigned>((d * 32 + 127) / 128),
            static_cast<unsigned>((ncol + 32 * CPL - 1) / (32 * CPL)));
  k_sketch_gather<CPL, UNR><<<grid, 128, 0, s>>>(A, lda, n, b, ptr, src, d, scale, W, ldw, rg);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace
}  // namespace itsk

using namespace itsk;

extern "C" int itsk_sketch(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                           const uint32_t* sk_ptr, const uint32_t* sk_src, int64_t d,
                           int64_t zeta, double* SAb, int64_t ldw, itsk_stream_t stream) {
  return itsk_sketch_rows(A, m, n, lda, b, sk_ptr, sk_src, d, zeta, SAb, ldw, 0, m, 0, stream);
}

extern "C" int itsk_sketch_rows(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                                const uint32_t* sk_ptr, const uint32_t* sk_src, int64_t d, int64_t zeta,
                                double* SAb, int64_t ldw, int64_t row0, int64_t row1, int accumulate,
                                itsk_stream_t stream) {
  ITSK_REQUIRE(m >= 1 && n >= 0 && d >= 1 && zeta >= 1, "bad sketch shape");
  ITSK_REQUIRE(0 <= row0 && row0 <= row1 && row1 <= m && m < (1ll << 31), "bad source-row window");
  SkRange rg;
  rg.j0 = static_cast<uint32_t>(row0);
  rg.j1 = row1 >= m ? 0xffffffffu : static_cast<uint32_t>(row1);
  rg.accum = accumulate ? 1 : 0;
  ITSK_REQUIRE(lda >= n && ldw >= n + (b ? 1 : 0), "bad leading dimension");
  ITSK_REQUIRE(sk_ptr && sk_src && SAb && (A || n == 0), "null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // scale = 1/sqrt(zeta) exactly as embed.py:92 (correctly rounded sqrt, div)
  const double scale = 1.0 / sqrt(static_cast<double>(zeta));
  const int64_t ncol = n + (b ? 1 : 0);
  const SketchTune tu = sketch_tune();
  // columns per lane: at most 4 (4 columns x 4 sources = 16 loads in flight
  // per lane at ~70 registers; 8 columns needs ~110 registers and halves the
  // resident warps — 25% slower at C2), fewer when d is small so that the grid
  // still has >= ~6000 warps (the chains are sequential per output, so
  // parallelism comes only from d x column blocks).  A TMA-staged variant
  // (per-warp ring of bulk-copied row segments) measured 1.8-5x slower: the
  // per-copy cost of 0.25-2 KB bulk copies dominates.
  // few (sketch row x 32-column) chains — about one wave or less — leave the
  // register gather with too few loads in flight: the cp.async ring keeps 64
  // sources per warp in flight (C5 d = 400, n = 100: 1.4x; from d x blocks ~
  // 5000 up the gather wins, profiles/r04_sketch_ring_vs_gather.txt)
  const bool ring = tu.ring >= 0 ? tu.ring == 1
                                 : (tu.gcpl == 0 && tu.unr == 0 && d * ((ncol + 31) / 32) <= 2048);
  if (ring) return launch_ring(A, lda, n, b, sk_ptr, sk_src, d, scale, SAb, ldw, rg, s);
  int64_t need = (ncol + 31) / 32;
  int64_t cap = 4;
  while (cap > 1 && d * ((ncol + 32 * cap - 1) / (32 * cap)) < 6000) cap >>= 1;
  if (tu.gcpl > 0) cap = tu.gcpl;
  if (need > cap) need = cap;
  const int unr = tu.unr > 0 ? tu.unr : (need <= 2 ? 8 : 4);
#define ITSK_G(CPLV, UNRV) \
  if (unr == UNRV) return launch_gather<CPLV, UNRV>(A, lda, n, b, sk_ptr, sk_src, d, scale, SAb, ldw, rg, s);
  if (need <= 1) { ITSK_G(1, 8) ITSK_G(1, 2) return launch_gather<1, 4>(A, lda, n, b, sk_ptr, sk_src, d, scale, SAb, ldw, rg, s); }
  if (need <= 2) { ITSK_G(2, 8) ITSK_G(2, 2) return launch_gather<2, 4>(A, lda, n, b, sk_ptr, sk_src, d, scale, SAb, ldw, rg, s); }
  if (need <= 4) { ITSK_G(4, 8) ITSK_G(4, 2) return launch_gather<4, 4>(A, lda, n, b, sk_ptr, sk_src, d, scale, SAb, ldw, rg, s); }
  ITSK_G(8, 8) ITSK_G(8, 2)
#undef ITSK_G
  return launch_gather<8, 4>(A, lda, n, b, sk_ptr, sk_src, d, scale, SAb, ldw, rg, s);
}
