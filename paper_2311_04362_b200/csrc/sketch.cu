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

// Tuning knobs (read per call so tests can sweep the variants in-process).
struct SketchTune {
  int gcpl = 0;       // register gather: cap on columns-per-lane (more column blocks)
  int unr = 0;        // register gather: sources per unrolled group (0 = heuristic)
  SketchTune() {
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
