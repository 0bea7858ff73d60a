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
#include <type_traits>

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
  // source row x leading dimension as one 32 x 32 -> 64 multiply-add (the
  // entry point requires lda < 2^31); a block of columns that lies inside A
  // (block-uniform) loads without the per-column kind tests
  const uint32_t lda32 = static_cast<uint32_t>(lda);
  const bool interior = c0 + 32 * CPL <= n;
  auto sweep = [&](auto inner) {
    constexpr bool IN = decltype(inner)::value;
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
          const uint32_t j = s & 0x7fffffffu;
          sv[u] = (s >> 31) ? -scale : scale;
          const double* arow = Ac + static_cast<uint64_t>(j) * lda32;
#pragma unroll
          for (int q = 0; q < CPL; ++q)
            v[u][q] = IN ? arow[32 * q] : (kind[q] == 0 ? arow[32 * q] : (kind[q] == 1 ? b[j] : 0.0));
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < CPL; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(sv[u], v[u][q]));
      }
      for (; k < cnt; ++k) {
        const uint32_t s = __shfl_sync(FULL, mine, k);
        const uint32_t j = s & 0x7fffffffu;
        const double svk = (s >> 31) ? -scale : scale;
        const double* arow = Ac + static_cast<uint64_t>(j) * lda32;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const double a = IN ? arow[32 * q] : (kind[q] == 0 ? arow[32 * q] : (kind[q] == 1 ? b[j] : 0.0));
          acc[q] = __dadd_rn(acc[q], __dmul_rn(svk, a));
        }
      }
    }
  };
  if (interior) sweep(std::true_type{});
  else sweep(std::false_type{});
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int64_t col = c0 + lane + 32 * q;
    if (col < ncol) W[i * ldw + col] = acc[q];
  }
}

// Window sweep for a large A (the gather above re-reads A zeta times from
// HBM: at C4 504 GB of DRAM reads for 64 GB of A, L2 hit rate 2%,
// profiles/rd2_sketch_window_deadend.txt).  One persistent launch, one CTA
// per SM: a warp owns up to RPW sketch rows, and the grid sweeps the source
// rows in windows of R rows, 128 columns (a panel) at a time: every warp
// adds the sources of its rows that fall in the current window, in ascending
// order, then counts itself done with the window.  A warp may start window g
// only when every warp has finished window g - drift (arrival counters; they
// order nothing, A is read-only — they only bound the L2 working set), so
// all zeta readers of a source row find its panel segment in L2 and A is
// read from HBM about once.  Each row's running sum lives in shared memory
// between its window segments.  Every output is the same sum in the same
// order as k_sketch_gather: bitwise scipy's.
// CL adjacent columns per lane (a panel of 32 CL), U sources per chunk,
// NWARP warps per CTA with RPW sketch rows each
template <int CL, int NWARP, int RPW>
constexpr size_t sw_smem_bytes() { return sizeof(double) * NWARP * RPW * 32 * CL; }

// The stream: walking the windows one by one costs, per (panel, window) step
// and warp, a boundary load, a scan, a dependent source-word load and a
// partly filled last chunk (~2.4 us of the ~17 us a 20000-row window step
// takes at C4; that version ran 53-59 ms, profiles/rd2_sketch_sweep.txt).
// Here the prologue writes each warp's (row, source) pairs ONCE in processing order
// (window-major, rows ascending inside a window, sources ascending inside a
// row) as 8-byte entries {source word, local row}; a panel is then one
// uninterrupted stream of U-entry chunks: the entries of the next chunk are
// loaded under the current chunk's 16-byte row loads, windows only gate the
// issue (a chunk whose last entry lies in window w waits for window
// w - drift to be complete everywhere) and are counted as the stream passes
// them.  A warp owns a contiguous block of sketch rows, so its entries occupy
// the index range of its rows in the pattern's CSR.  Same sums in the same
// order: bitwise scipy's.
__host__ __device__ __forceinline__ uint32_t sw_win(uint32_t j, double inv_r) {
  // monotone in j; used wherever a source row is mapped to its window
  return static_cast<uint32_t>(static_cast<double>(j) * inv_r);
}

template <int CL, int U, int SW_WARPS, int SW_RPW, bool DIRECT>
__global__ void __launch_bounds__(32 * SW_WARPS, 1) k_sketch_stream(
    const double* __restrict__ A, int64_t lda, int64_t n, const double* __restrict__ b,
    const uint32_t* __restrict__ ptr, const uint32_t* __restrict__ src, int64_t d, double scale,
    double* __restrict__ W, int64_t ldw, double inv_r, int nwin, int npanel, unsigned* wdone,
    uint32_t* __restrict__ bnd, uint2* ord, int flags) {
  const int vec = flags & 1;
  const int drift = flags >> 8;  // windows a warp may run ahead of the slowest
  static_assert(CL == 2 || CL == 4, "columns per lane");
  static_assert(U <= 32 && (U & (U - 1)) == 0 && SW_RPW <= 32, "chunk / row shape");
  constexpr int PANEL = 32 * CL, NV = CL / 2;  // NV double2 per lane per source
  extern __shared__ __align__(16) double sw_sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t NW = static_cast<int64_t>(gridDim.x) * SW_WARPS;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * SW_WARPS + warp;
  const int64_t ncol = n + (b ? 1 : 0);
  double2* acc_sm = reinterpret_cast<double2*>(sw_sm + static_cast<int64_t>(warp) * SW_RPW * PANEL);
  // rows [row0, row0 + nrows) (d = q NW + rem: the first rem warps own q + 1).
  // Direct mode (no more sketch rows than the grid has warps): a warp owns at
  // most ONE sketch row — its processing order is the row's own CSR order, so
  // the entries are read straight from the pattern (no prologue, no scratch)
  // — and the owners are dealt warp-major, so that every SM gets its share of
  // the rows.
  // (a template parameter: the materialised-order kernel's code is untouched —
  // as a run-time branch the direct path cost the C4 sketch 46.3 -> 53.2 ms)
  const int64_t qr = d / NW, rem = d % NW;
  const int64_t gwp = static_cast<int64_t>(warp) * gridDim.x + blockIdx.x;
  const int64_t row0 = DIRECT ? (gwp < d ? gwp : 0) : gw * qr + (gw < rem ? gw : rem);
  const int nrows = DIRECT ? (gwp < d ? 1 : 0) : static_cast<int>(qr + (gw < rem ? 1 : 0));
  const bool rowok = lane < nrows;
  const uint32_t r0 = rowok ? ptr[row0 + lane] : 0u, r1 = rowok ? ptr[row0 + lane + 1] : 0u;
  const uint32_t e0 = ptr[row0];
  const uint32_t etot = ptr[row0 + nrows] - e0;
  // prologue 1: the end of every window's segment of every own row (positions
  // p-1, p in windows wp < wc end windows [wp, wc) at p; the row end is a
  // sentinel in window nwin)
  uint32_t* wb = bnd + gw * SW_RPW * static_cast<int64_t>(nwin);
  for (int k = 0; k < (DIRECT ? 0 : nrows); ++k) {
    const uint32_t a0 = __shfl_sync(FULL, r0, k), a1 = __shfl_sync(FULL, r1, k);
    int carry = 0;
    for (uint32_t q = a0; q <= a1; q += 32) {
      const uint32_t p = q + lane;
      const int wc = p < a1 ? static_cast<int>(sw_win(src[p] & 0x7fffffffu, inv_r)) : nwin;
      int wp = __shfl_up_sync(FULL, wc, 1);
      if (lane == 0) wp = carry;
      if (p <= a1)
        for (int w = wp; w < wc; ++w) wb[k * nwin + w] = p;
      carry = __shfl_sync(FULL, wc, 31);
    }
  }
  __syncwarp();
  // prologue 2: the entries in processing order
  if constexpr (!DIRECT) {
    uint32_t sk = r0, o = e0;
    for (int w = 0; w < nwin; ++w) {
      const uint32_t tk = rowok ? wb[lane * nwin + w] : 0u;
      const uint32_t cnt = rowok ? tk - sk : 0u;
      uint32_t incl = cnt;  // inclusive scan: row k covers flattened positions [incl - cnt, incl)
#pragma unroll
      for (int q = 1; q < 32; q <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, q);
        if (lane >= q) incl += t;
      }
      const uint32_t total = __shfl_sync(FULL, incl, 31);
      const uint32_t base = sk - (incl - cnt);  // source index = base_k + position
      for (uint32_t P = 0; P < total; P += 32) {
        const uint32_t pos = min(P + lane, total - 1);
        int k = 0;
#pragma unroll
        for (int kk = 0; kk < SW_RPW - 1; ++kk) k += pos >= __shfl_sync(FULL, incl, kk) ? 1 : 0;
        const uint32_t bk = __shfl_sync(FULL, base, k);
        if (P + lane < total) ord[o + pos] = make_uint2(src[bk + pos], static_cast<uint32_t>(k));
      }
      o += total;
      sk = tk;
    }
  }
  __syncwarp();
  // Window arrivals are counted per CTA in shared memory; the CTA's last warp
  // adds one to the window's global counter, and the grid's last CTA writes
  // the window's epoch (g + 1) into every CTA's own flag line, the only line
  // the CTA's warps poll.
  __shared__ unsigned cta_cnt[8];
  if (threadIdx.x < 8) cta_cnt[threadIdx.x] = 0u;
  __syncthreads();
  unsigned* wflag = wdone + static_cast<int64_t>(nwin) * npanel;  // gridDim.x lines of 32 words
  const volatile unsigned* myflag = wflag + 32 * static_cast<int64_t>(blockIdx.x);
  int known = -1;  // highest global window step known complete
  auto wait_for = [&](int gq) {
    if (gq > known) {
      if (lane == 0)
        while (myflag[gq & 7] < static_cast<unsigned>(gq) + 1u) __nanosleep(32);
      __syncwarp();
      known = gq;
    }
  };
  auto arrive = [&](int g) {
    // the CTA's counter slot g & 7 last counted window g - 8: a warp with few
    // or no entries must not run more than a slot ring ahead of the grid
    wait_for(g - 7);
    int bcast = 0;
    if (lane == 0) {
      if (atomicAdd(&cta_cnt[g & 7], 1u) == SW_WARPS - 1) {
        // the slot is next used 8 windows on, which no warp reaches before
        // window g + 8 - drift > g is complete everywhere (drift < 8)
        cta_cnt[g & 7] = 0u;
        __threadfence();
        bcast = atomicAdd(wdone + g, 1u) == gridDim.x - 1 ? 1 : 0;
      }
    }
    if (__shfl_sync(FULL, bcast, 0))
      for (unsigned c = lane; c < gridDim.x; c += 32)
        *reinterpret_cast<volatile unsigned*>(wflag + 32 * static_cast<int64_t>(c) + (g & 7)) =
            static_cast<unsigned>(g) + 1u;
  };
  const uint2* my = ord + e0;
  const uint32_t* mysrc = src + e0;
  const uint32_t lda32 = static_cast<uint32_t>(lda);  // lda < 2^31 (entry point)
  auto entry = [&](uint32_t idx) {
    if constexpr (DIRECT) return make_uint2(__ldg(mysrc + idx), 0u);
    else return my[idx];
  };
  for (int p = 0; p < npanel; ++p) {
    // this lane's columns: cA + 64 h + {0, 1}, h < NV (each 16-byte load of a
    // warp is one contiguous 512-byte segment)
    const int64_t cA = static_cast<int64_t>(p) * PANEL + 2 * lane;
    const bool allv = __all_sync(FULL, vec && cA + 64 * (NV - 1) + 1 < n);
    int kind[CL];
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      const int64_t col = cA + 64 * (c >> 1) + (c & 1);
      kind[c] = col < n ? 0 : (col == n && b ? 1 : 2);
    }
    const double* Ap = A + static_cast<int64_t>(p) * PANEL;
    const double* Ac = Ap + 2 * lane;
#pragma unroll
    for (int k = 0; k < SW_RPW; ++k)
#pragma unroll
      for (int h = 0; h < NV; ++h) acc_sm[k * 16 * CL + 32 * h + lane] = make_double2(0.0, 0.0);
    __syncwarp();
    const int g0 = p * nwin;
    int arrived = 0;  // windows of this panel this warp has counted itself done with
    int kcur = -1;
    double2 acc[NV];
    // lane u (mod U): entry P + u, clamped into the list
    uint2 ent = make_uint2(0u, 0u);
    if (etot > 0) ent = entry(min(static_cast<uint32_t>(lane & (U - 1)), etot - 1));
    for (uint32_t P = 0; P < etot; P += U) {
      uint2 entn = make_uint2(0u, 0u);
      if (P + U < etot) entn = entry(min(P + U + static_cast<uint32_t>(lane & (U - 1)), etot - 1));
      const int nu = static_cast<int>(min(etot - P, static_cast<uint32_t>(U)));
      const uint32_t sv = ent.x;
      const int wf = static_cast<int>(sw_win(__shfl_sync(FULL, sv, 0) & 0x7fffffffu, inv_r));
      const int wl = static_cast<int>(sw_win(__shfl_sync(FULL, sv, nu - 1) & 0x7fffffffu, inv_r));
      // everything before this chunk is added: windows below its first are done
      while (arrived < wf) arrive(g0 + arrived++);
      // gate: window wl - drift complete everywhere (never one this warp has
      // not counted itself done with: a chunk may span more than `drift`)
      wait_for(g0 + min(wl - drift, wf - 1));
      const double* pu = Ap + static_cast<uint64_t>(sv & 0x7fffffffu) * lda32;  // lane-independent start
      double2 v[U][NV];
      if (allv) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double2* q = reinterpret_cast<const double2*>(
                                 __shfl_sync(FULL, reinterpret_cast<uintptr_t>(pu), u)) + lane;
#pragma unroll
          for (int h = 0; h < NV; ++h) v[u][h] = u < nu ? __ldg(q + 32 * h) : make_double2(0.0, 0.0);
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j = __shfl_sync(FULL, sv, u) & 0x7fffffffu;
          const double* arow = Ac + j * lda;
#pragma unroll
          for (int h = 0; h < NV; ++h) {
            const int c0 = 2 * h, c1 = 2 * h + 1;
            v[u][h].x = u >= nu ? 0.0 : (kind[c0] == 0 ? arow[64 * h] : (kind[c0] == 1 ? b[j] : 0.0));
            v[u][h].y = u >= nu ? 0.0 : (kind[c1] == 0 ? arow[64 * h + 1] : (kind[c1] == 1 ? b[j] : 0.0));
          }
        }
      }
      // the chunk's row switches and signs as ballots (warp-uniform masks:
      // the per-source tests below are uniform branches); slots past the end
      // of the list hold zeros and add +0.0, which changes no sum (a sum that
      // starts at +0.0 is never -0.0)
      const int kme = static_cast<int>(ent.y);
      int kprev = __shfl_up_sync(FULL, kme, 1);
      if (lane == 0) kprev = kcur;
      const unsigned swm = __ballot_sync(FULL, lane < nu && kme != kprev);
      const unsigned sgm = __ballot_sync(FULL, lane < nu && (sv >> 31) != 0u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if ((swm >> u) & 1u) {
          const int k = __shfl_sync(FULL, kme, u);
          if (kcur >= 0)
#pragma unroll
            for (int h = 0; h < NV; ++h) acc_sm[kcur * 16 * CL + 32 * h + lane] = acc[h];
#pragma unroll
          for (int h = 0; h < NV; ++h) acc[h] = acc_sm[k * 16 * CL + 32 * h + lane];
          kcur = k;
        }
        const double sg = ((sgm >> u) & 1u) ? -scale : scale;
#pragma unroll
        for (int h = 0; h < NV; ++h) {
          acc[h].x = __dadd_rn(acc[h].x, __dmul_rn(sg, v[u][h].x));
          acc[h].y = __dadd_rn(acc[h].y, __dmul_rn(sg, v[u][h].y));
        }
      }
      ent = entn;
    }
    if (kcur >= 0)
#pragma unroll
      for (int h = 0; h < NV; ++h) acc_sm[kcur * 16 * CL + 32 * h + lane] = acc[h];
    __syncwarp();
    while (arrived < nwin) arrive(g0 + arrived++);
#pragma unroll
    for (int k = 0; k < SW_RPW; ++k) {
      const int64_t i = row0 + k;
      if (k >= nrows) continue;
#pragma unroll
      for (int h = 0; h < NV; ++h) {
        const double2 a = acc_sm[k * 16 * CL + 32 * h + lane];
        if (cA + 64 * h < ncol) W[i * ldw + cA + 64 * h] = a.x;
        if (cA + 64 * h + 1 < ncol) W[i * ldw + cA + 64 * h + 1] = a.y;
      }
    }
    __syncwarp();
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
  // 32-bit stride (the entry point requires lda < 2^31): source row x stride
  // is one wide multiply-add instead of a 64 x 64 product
  const uint32_t stride = kind == 0 ? static_cast<uint32_t>(lda) : (kind == 1 ? 1u : 0u);
  double acc = (rg.accum && col < ncol) ? W[i * ldw + col] : 0.0;
  uint32_t e0 = ptr[i], e1 = ptr[i + 1];
  if (rg.j0 > 0) e0 = lower_src(src, e0, e1, rg.j0);
  if (rg.j1 != 0xffffffffu) e1 = lower_src(src, e0, e1, rg.j1);
  const uint32_t total = e1 - e0;
  const uint32_t ngroups = (total + RG_G - 1) / RG_G;
  double* my = ring + lane;
  const uint32_t my_s = smem_u32(my);
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
    // (a group never straddles a ring wrap or a 32-block: RG_G divides both)
    const uint32_t dst0 = my_s + (q0 % RG_DEPTH) * 256u;
    const int nbytes = kind != 2 ? 8 : 0;  // 0: zero-fill
    if (q0 + RG_G <= total) {  // full group (uniform): no per-source predicates
#pragma unroll
      for (int u = 0; u < RG_G; ++u) {
        const uint32_t w = __shfl_sync(FULL, wcur, (q0 & 31) + u);
        const double* sp = base + static_cast<uint64_t>(w & 0x7fffffffu) * stride;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst0 + 256u * u), "l"(sp), "r"(nbytes)
                     : "memory");
      }
    } else {
#pragma unroll
      for (int u = 0; u < RG_G; ++u) {
        const uint32_t w = __shfl_sync(FULL, wcur, (q0 & 31) + u);
        const double* sp = base + static_cast<uint64_t>(w & 0x7fffffffu) * stride;
        if (q0 + u < total)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst0 + 256u * u), "l"(sp), "r"(nbytes)
                       : "memory");
      }
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
    const uint32_t s0 = (g * RG_G) % RG_DEPTH;
#pragma unroll
    for (int u = 0; u < RG_G; ++u) {
      sw[u] = rsrc[s0 + u];
      v[u] = my[(s0 + u) * 32];
    }
    // fl(-scale * v) = fl(scale * -v): the sign goes into the operand's sign
    // bit (one logic op) instead of selecting +-scale
    if ((g + 1) * RG_G <= total) {
#pragma unroll
      for (int u = 0; u < RG_G; ++u) {
        const double vs = __hiloint2double(__double2hiint(v[u]) ^ static_cast<int>(sw[u] & 0x80000000u),
                                           __double2loint(v[u]));
        acc = __dadd_rn(acc, __dmul_rn(scale, vs));
      }
    } else {
#pragma unroll
      for (int u = 0; u < RG_G; ++u) {
        const double vs = __hiloint2double(__double2hiint(v[u]) ^ static_cast<int>(sw[u] & 0x80000000u),
                                           __double2loint(v[u]));
        if (g * RG_G + u < total) acc = __dadd_rn(acc, __dmul_rn(scale, vs));
      }
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
  int swcl = 0;      // window sweep columns per lane (2: 64-column panels, else 128; same bits)
  int drift = 2;      // window sweep: windows a warp may run ahead (L2 working set; same bits)
  int sweep = -1;     // window sweep: -1 auto (large A), 0 off, 1 on, > 1 on with that many window rows (same bits)
  int direct = -1;    // window sweep, one row per warp read straight from the pattern: -1 auto, 0 off, 1 on (same bits)
  SketchTune() {
    if (const char* e = getenv("ITSK_SKETCH_SWEEP")) sweep = atoi(e);
    if (const char* e = getenv("ITSK_SKETCH_SWCL")) swcl = atoi(e);
    if (const char* e = getenv("ITSK_SKETCH_DIRECT")) direct = atoi(e);
    if (const char* e = getenv("ITSK_SKETCH_DRIFT")) drift = std::min(7, std::max(1, atoi(e)));
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
  ITSK_REQUIRE(lda >= n && ldw >= n + (b ? 1 : 0) && lda < (1ll << 31), "bad leading dimension");
  ITSK_REQUIRE(sk_ptr && sk_src && SAb && (A || n == 0), "null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // scale = 1/sqrt(zeta) exactly as embed.py:92 (correctly rounded sqrt, div)
  const double scale = 1.0 / sqrt(static_cast<double>(zeta));
  const int64_t ncol = n + (b ? 1 : 0);
  const SketchTune tu = sketch_tune();
  // columns per lane: at most 4 (4 columns x 4 sources = 16 loads in flight
  // per lane at ~70 registers; 8 columns needs ~110 registers and halves the
  // resident warps — 25% slower at C2), fewer when d is small so that the grid
  // still has >= ~2400 warps (the chains are sequential per output, so
  // parallelism comes only from d x column blocks; but these shapes are bound
  // by warp instructions per (source, column block), and two columns per lane
  // halve them: 16.7M x 100, d = 2000: 22.8 ms with 8000 one-column warps, 15.8
  // with 4000 two-column warps, 18.5 with 2000 four-column warps;
  // profiles/rd2_sketch_gather_ab.txt).  A TMA-staged variant
  // (per-warp ring of bulk-copied row segments) measured 1.8-5x slower: the
  // per-copy cost of 0.25-2 KB bulk copies dominates.
  // few (sketch row x 32-column) chains — about one wave or less — leave the
  // register gather with too few loads in flight: the cp.async ring keeps 64
  // sources per warp in flight (C5 d = 400, n = 100: 1.4x; from d x blocks ~
  // 5000 up the gather wins, profiles/r04_sketch_ring_vs_gather.txt)
  const bool ring = tu.ring >= 0 ? tu.ring == 1
                                 : (tu.gcpl == 0 && tu.unr == 0 && d * ((ncol + 31) / 32) <= 2048);
  // the window sweep: a whole-source call (not an upload window, no
  // accumulation) on an A several times the L2, with every sketch row of the
  // grid's warps in registers
  {
    const int nsm = num_sms();
    // kernel shapes (all the same bits): columns per lane, sources per chunk,
    // warps per CTA, sketch rows per warp
    struct SwShape { const void* fn; int cl, warps, rpw; size_t smem; };
    // 128-column panels with up to 12 sketch rows per warp; 64-column panels
    // with up to 24 for a d beyond that (and, 12 rows, for the tests: same bits)
    static const SwShape shapes[] = {
        {reinterpret_cast<const void*>(k_sketch_stream<4, 8, 16, 12, false>), 4, 16, 12, sw_smem_bytes<4, 16, 12>()},
        {reinterpret_cast<const void*>(k_sketch_stream<2, 16, 16, 12, false>), 2, 16, 12, sw_smem_bytes<2, 16, 12>()},
        {reinterpret_cast<const void*>(k_sketch_stream<2, 16, 16, 24, false>), 2, 16, 24, sw_smem_bytes<2, 16, 24>()},
        // direct mode: one row per warp (one row's running sums in shared memory)
        {reinterpret_cast<const void*>(k_sketch_stream<4, 8, 16, 1, true>), 4, 16, 1, sw_smem_bytes<4, 16, 1>()},
        {reinterpret_cast<const void*>(k_sketch_stream<2, 16, 16, 1, true>), 2, 16, 1, sw_smem_bytes<2, 16, 1>()}};
    const int64_t nw = static_cast<int64_t>(nsm) * 16;
    const SwShape& sh0 = shapes[d > nw * 12 ? 2 : (tu.swcl == 2 ? 1 : 0)];
    // automatic from 2 GB of [A|b] (streamed sweep vs gather, ms: C4 64 GB 46.6 / 72;
    // 32 GB 24.1 / 35.5; 16 GB 12.4 / 17.3; 8 GB 6.1 / 8.3; C3 4 GB 3.7 / 4.1;
    // C2 0.3 GB 0.50 / 0.27, where the gather finds A in L2) when the grid's
    // warps have rows to own (C5 cells, profiles/rd2_final_sketch_sweep_c5.txt):
    // d >= 2 rows per warp, and below 16 GB only with zeta >= 8 (the re-reads
    // it saves) or d >= 4 rows per warp; from 16 GB also a d of one row for
    // most warps when the rows are at least two panels wide
    const int64_t bytes = m * ncol * 8;
    const bool big =
        bytes >= (2ll << 30) &&
        ((d >= 2 * nw && (zeta >= 8 || d >= 4 * nw || bytes >= (16ll << 30))) ||
         (4 * d >= 3 * nw && ncol >= 256 && bytes >= (16ll << 30) && zeta >= 8));
    // direct mode (no more sketch rows than warps: a warp owns one row and
    // reads its entries straight from the pattern, no prologue and no scratch):
    // wide rows of a large A (16.7M x 500, d = 2000, zeta = 8: 71.5 -> 65.5 ms);
    // on C5's narrow cells (n = 100) one 8 KB chunk in flight per warp is too
    // little and the ring / gather stay ahead; so did a gated cp.async ring with up to
    // 64 segments in flight per owner: with one warp per row the warp's own
    // instruction stream is the limit (profiles/rd2_sketch_direct_ab.txt)
    const bool can_direct = d <= nw && tu.direct != 0;
    const bool direct = can_direct && (tu.direct == 1 || (ncol >= 256 && bytes >= (16ll << 30)));
    const SwShape& sh = direct ? shapes[tu.swcl == 2 ? 4 : 3] : sh0;
    if ((tu.sweep > 0 || (tu.sweep < 0 && (big || direct))) && tu.ring != 1 && tu.gcpl == 0 && tu.unr == 0 && rg.j0 == 0 &&
        rg.j1 == 0xffffffffu && !rg.accum && d <= nw * sh.rpw && m < (1ll << 31)) {
      const int cl = sh.cl;
      // a window holds ~20 MB of A: 20000 rows of a 128-column panel, 40000 of a 64-column one
      const uint32_t R = tu.sweep > 1 ? static_cast<uint32_t>(tu.sweep)
                                      : (cl == 2 ? 40000u : 20000u);
      const double inv_r = 1.0 / static_cast<double>(R);
      const int nwin = static_cast<int>(sw_win(static_cast<uint32_t>(m - 1), inv_r)) + 1;
      const int npanel = static_cast<int>((ncol + 32 * cl - 1) / (32 * cl));
      unsigned* wdone = nullptr;
      uint32_t* bnd = nullptr;
      // per-window counters, then one 128-byte flag line per CTA
      const size_t cbytes = sizeof(unsigned) * (static_cast<size_t>(nwin) * npanel + 32 * static_cast<size_t>(nsm));
      const size_t bbytes = direct ? 0 : sizeof(uint32_t) * static_cast<size_t>(nw) * sh.rpw * nwin;
      ITSK_CUDA(keep_async_pool());
      // one scratch block: counters and flag lines | window boundaries | the
      // entries in processing order (8 m zeta bytes: 256 MB at C4).  Without
      // room for it the gather below does the job (same bits).
      const size_t obytes = direct ? 0 : sizeof(uint2) * static_cast<size_t>(m) * zeta;
      const size_t c_al = (cbytes + 255) / 256 * 256, b_al = (bbytes + 255) / 256 * 256;
      unsigned char* scratch = nullptr;
      if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), c_al + b_al + obytes, s) != cudaSuccess) {
        cudaGetLastError();
        scratch = nullptr;
      }
      if (scratch) {
        wdone = reinterpret_cast<unsigned*>(scratch);
        bnd = reinterpret_cast<uint32_t*>(scratch + c_al);
        uint2* ord = reinterpret_cast<uint2*>(scratch + c_al + b_al);
        ITSK_CUDA(cudaMemsetAsync(wdone, 0, cbytes, s));
        int flags = ((lda % 2 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) ? 1 : 0) | (tu.drift << 8);
        const void* fn = sh.fn;
        const size_t smem = sh.smem;
        ITSK_CUDA(func_attr_once(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        void* args[] = {&A, &lda, &n, &b, &sk_ptr, &sk_src, &d, const_cast<double*>(&scale), &SAb, &ldw,
                        const_cast<double*>(&inv_r), const_cast<int*>(&nwin), const_cast<int*>(&npanel),
                        &wdone, &bnd, &ord, &flags};
        ITSK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(nsm), dim3(32 * sh.warps), args, smem, s));
        count_launch();
        ITSK_CUDA(cudaFreeAsync(scratch, s));
        return ITSK_OK;
      }
    }
  }
  if (ring) return launch_ring(A, lda, n, b, sk_ptr, sk_src, d, scale, SAb, ldw, rg, s);
  int64_t need = (ncol + 31) / 32;
  int64_t cap = 4;
  while (cap > 1 && d * ((ncol + 32 * cap - 1) / (32 * cap)) < 2400) cap >>= 1;
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
