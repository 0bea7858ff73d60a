// Sparse CSR A (§3.5).
//
// The reference accepts a scipy sparse A on the same path:
//   S·A      embed.py:76-80  (S_csc @ A.tocsc()).todense() — per output entry
//            SA[k, i] = sum over the sources j of S's row k, ascending, with
//            A[j, i] != 0 of fl(s_kj * A[j, i]), added sequentially from 0
//            (scipy csr_matmat on the transposes)
//   r        solvers.py:290,299  b - a @ x   (csr_matvec: a sequential row sum)
//   c        solvers.py:343      a.T @ r     (csc_matvec over rows ascending)
// Here:
//   k_sketch_csr  one warp per sketch row: its sources (CSR of S, ascending)
//                 in batches of 32, their entries applied in rank waves to a
//                 shared-memory accumulator row — every column receives its
//                 products in source order, so S·A is bitwise the
//                 reference's (b: the dense gather kernel, column n).
//   k_csr_rows    r_j = b_j - sum_t fl(A_jt x_t) in stored order (bitwise
//                 csr_matvec), r written, the four norm partials per CTA.
//   k_csc_chunks  c = A'r over the CSC copy of A built once per plan (stable
//                 radix sort of the entries by column): every column is cut
//                 into fixed chunks of CHUNK entries, a warp sums a chunk in a
//                 fixed lane/tree order.
//   k_csr_finish  per column the chunk partials in chunk order, and the norm
//                 partials in CTA order, into cs = [c | 4 norms] — the layout
//                 of the dense fused pass, so the loop's tail kernel is shared.
// Deterministic run to run; r is bitwise the reference's, c differs from the
// reference's sequential sum by rounding only.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "itsk_common.cuh"
#include "itsk_kernels.cuh"

namespace itsk {
namespace {

constexpr int CSR_THREADS = 256;
constexpr int CHUNK = 1024;      // CSC entries per warp chunk

__global__ void k_entry_rows(const int64_t* __restrict__ row_ptr, int64_t m, uint32_t* __restrict__ erow) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  for (int64_t e = row_ptr[j]; e < row_ptr[j + 1]; ++e) erow[e] = static_cast<uint32_t>(j);
}

__global__ void k_iota(uint32_t* __restrict__ v, int64_t nnz) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < nnz) v[e] = static_cast<uint32_t>(e);
}

__global__ void k_csc_gather(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ erow,
                             const double* __restrict__ val, int64_t nnz, int32_t* __restrict__ crow,
                             double* __restrict__ cval) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const uint32_t e = perm[p];
  crow[p] = static_cast<int32_t>(erow[e]);
  cval[p] = val[e];
}

// col_ptr[k] = first position of key >= k in the sorted column keys
__global__ void k_col_ptr(const uint32_t* __restrict__ keys, int64_t nnz, int64_t n, int64_t* __restrict__ col_ptr) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k > n) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < static_cast<uint32_t>(k)) lo = mid + 1; else hi = mid;
  }
  col_ptr[k] = lo;
}

__global__ void k_check_csr(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t m,
                            int64_t n, int64_t nnz, int* __restrict__ bad) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j > m) return;
  const int64_t p = row_ptr[j];
  if (p < 0 || p > nnz || (j == 0 && p != 0) || (j == m && p != nnz) || (j > 0 && row_ptr[j - 1] > p)) {
    atomicOr(bad, 1);
    return;
  }
  if (j < m)
    for (int64_t e = p; e < row_ptr[j + 1] && e < nnz; ++e)
      if (col[e] < 0 || col[e] >= n) atomicOr(bad, 2);
}

// ---------------------------------------------------------------------------
// S·A for CSR A
//
// A warp owns sketch row k and walks its sources in ascending order, 32 at a
// time.  The batch's entries (source-major, stored order inside a row) are
// taken 32 per round; inside a round, an entry's rank = the number of earlier
// entries of the round with the same column (__match_any_sync), and the
// round is applied in waves of equal rank — entries of one wave touch
// distinct columns, and every column still receives its products in source
// order, so each output is the same sequential sum as scipy's.  Rounds of a
// batch are loaded together (RND x 2 loads in flight per lane).  S·b (the
// b column) is one more sequential chain per row: the dense gather kernel
// computes it (itsk_sketch with n = 0).
// ---------------------------------------------------------------------------
constexpr int SK_RND = 4;  // rounds of 32 entries loaded per batch step

__global__ void __launch_bounds__(256) k_sketch_csr(
    const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const double* __restrict__ val,
    int64_t n, const uint32_t* __restrict__ ptr, const uint32_t* __restrict__ src, int64_t d, double scale,
    double* __restrict__ W, int64_t ldw, int smem_acc) {
  extern __shared__ double sacc[];
  __shared__ int soff[8][33];
  __shared__ int64_t sp0[8][32];
  __shared__ double ssv[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (i >= d) return;
  // the accumulator row: shared memory when it fits, else the output row itself
  double* acc = smem_acc ? sacc + static_cast<int64_t>(warp) * n : W + i * ldw;
  for (int64_t c = lane; c < n; c += 32) acc[c] = 0.0;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t e0 = ptr[i], e1 = ptr[i + 1];
  for (uint32_t e = e0; e < e1; e += 32) {
    const int cnt = static_cast<int>(min(32u, e1 - e));
    int len = 0;
    int64_t p0 = 0;
    double sv = 0.0;
    if (lane < cnt) {
      const uint32_t sj = src[e + lane];
      const int64_t j = sj & 0x7fffffffu;
      sv = (sj >> 31) ? -scale : scale;
      p0 = row_ptr[j];
      len = static_cast<int>(row_ptr[j + 1] - p0);
    }
    int inc = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    const int T = __shfl_sync(FULL, inc, 31);
    __syncwarp();
    soff[warp][lane] = inc - len;
    if (lane == 31) soff[warp][32] = T;
    sp0[warp][lane] = p0;
    ssv[warp][lane] = sv;
    __syncwarp();
    for (int t0 = 0; t0 < T; t0 += 32 * SK_RND) {
      int cr[SK_RND];
      double pr[SK_RND];
#pragma unroll
      for (int u = 0; u < SK_RND; ++u) {
        const int t = t0 + 32 * u + lane;
        cr[u] = -1 - lane;
        pr[u] = 0.0;
        if (t < T) {
          // source of entry t: the last q with soff[q] <= t
          int lo = 0, hi = cnt - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (soff[warp][mid] <= t) lo = mid; else hi = mid - 1;
          }
          const int64_t ei = sp0[warp][lo] + (t - soff[warp][lo]);
          cr[u] = col[ei];
          pr[u] = __dmul_rn(val[ei], ssv[warp][lo]);
        }
      }
#pragma unroll
      for (int u = 0; u < SK_RND; ++u) {
        if (t0 + 32 * u >= T) break;
        const bool act = cr[u] >= 0;
        const unsigned peers = __match_any_sync(FULL, cr[u]);
        const int rank = __popc(peers & lt);
        const int waves = __reduce_max_sync(FULL, act ? rank : 0);
        for (int w = 0; w <= waves; ++w) {
          if (act && rank == w) acc[cr[u]] = __dadd_rn(acc[cr[u]], pr[u]);
          __syncwarp();
        }
      }
    }
    __syncwarp();
  }
  if (smem_acc)
    for (int64_t c = lane; c < n; c += 32) W[i * ldw + c] = acc[c];
}

// ---------------------------------------------------------------------------
// The pass: r = bscale*b - A x (rows), c = A'r (CSC chunks), finish
// ---------------------------------------------------------------------------
struct CsrPassArgs {
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
  const int64_t* col_ptr;
  const int32_t* crow;
  const double* cval;
  const int32_t* chunk_col;
  const int64_t* chunk_ptr;
  double* chunk_part;
  double* row_part;  // g1 x 4
  int64_t m, n, nchunks, rows_per_cta;
  int g1;
  const double* b;
  double bscale;
  const double* x;
  const double* r_prev;
  double* r_out;
  const double* r_true;
  double* cs;
  // loop mode (as PassArgs): x / r_prev / r_out from ctl->it
  const LoopCtl* ctl;
  const double* xs;
  double* rs;
  int mode;
};

__device__ __forceinline__ bool resolve(const CsrPassArgs& a, const double*& x, const double*& r_prev,
                                        double*& r_out) {
  if (a.mode == 0) {
    x = a.x;
    r_prev = a.r_prev;
    r_out = a.r_out;
    return true;
  }
  const LoopCtl* ctl = a.ctl;
  if (ctl->result.done) return false;
  const int64_t S = ctl->r_slots;
  if (a.mode == 1) {
    const int64_t it = ctl->it;
    x = a.xs + (it + 1) * a.n;
    r_prev = a.rs + (it % S) * a.m;
    r_out = a.rs + ((it + 1) % S) * a.m;
  } else {
    x = a.xs;
    r_prev = nullptr;
    r_out = a.rs;
  }
  return true;
}

// Rows: a warp takes RPL*32 consecutive rows at a time (lane l owns rows
// l, l+32, ...); all their row pointers / b / r_prev loads are issued
// together, then the batch's entries (one contiguous CSR range) are staged in
// shared memory with coalesced, independent loads, and each lane sums its
// rows in stored order (the bitwise csr_matvec order).  x is staged per CTA
// when it fits.  A batch with more entries than the stage uses direct loads.
constexpr int RPL = 1;            // rows per lane per batch
constexpr int ROW_STAGE = 256;    // staged entries per warp (8 per row on average at RPL 1)
constexpr int X_STAGE = 8192;     // x staged in shared memory up to this n

__global__ void __launch_bounds__(CSR_THREADS) k_csr_rows(CsrPassArgs a) {
  __shared__ double red[CSR_THREADS / 32];
  // dynamic: staged values | staged columns | x (when n <= X_STAGE)
  extern __shared__ double dsm[];
  double(*sval)[ROW_STAGE] = reinterpret_cast<double(*)[ROW_STAGE]>(dsm);
  int(*scol)[ROW_STAGE] = reinterpret_cast<int(*)[ROW_STAGE]>(dsm + (CSR_THREADS / 32) * ROW_STAGE);
  double* xsm = dsm + (CSR_THREADS / 32) * ROW_STAGE * 3 / 2;
  pdl_wait();
  const double *x, *r_prev;
  double* r_out;
  if (!resolve(a, x, r_prev, r_out)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool xs = a.n <= X_STAGE;
  if (xs)
    for (int64_t c = threadIdx.x; c < a.n; c += CSR_THREADS) xsm[c] = x[c];
  __syncthreads();
  const double* xv = xs ? xsm : x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * a.rows_per_cta;
  const int64_t r1 = min(a.m, r0 + a.rows_per_cta);
  constexpr int BATCH = 32 * RPL;
  double s_rr = 0.0, s_dd = 0.0, s_tt = 0.0, s_bb = 0.0;
  for (int64_t j0 = r0 + BATCH * warp; j0 < r1; j0 += BATCH * (CSR_THREADS / 32)) {
    int64_t plo[RPL], phi[RPL];
    double bj[RPL], rp[RPL], rt[RPL];
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int64_t j = j0 + lane + 32 * u;
      const bool ok = j < r1;
      plo[u] = ok ? a.row_ptr[j] : 0;
      phi[u] = ok ? a.row_ptr[j + 1] : 0;
      bj[u] = ok ? a.b[j] : 0.0;
      rp[u] = (ok && r_prev) ? r_prev[j] : 0.0;
      rt[u] = (ok && a.r_true) ? a.r_true[j] : 0.0;
    }
    const int nrow = static_cast<int>(r1 - j0 < BATCH ? r1 - j0 : BATCH);
    const int last = nrow - 1;
    const int64_t base = __shfl_sync(FULL, plo[0], 0);
    int64_t end = 0;
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int64_t e = __shfl_sync(FULL, phi[u], last & 31);
      if (u == (last >> 5)) end = e;
    }
    const int64_t total = end - base;
    const bool staged = total <= ROW_STAGE;
    if (staged) {
      for (int t = lane; t < total; t += 32) {
        scol[warp][t] = a.col[base + t];
        sval[warp][t] = a.val[base + t];
      }
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int64_t j = j0 + lane + 32 * u;
      if (j >= r1) continue;
      double dot = 0.0;
      if (staged) {
        for (int64_t e = plo[u] - base; e < phi[u] - base; ++e)
          dot = __dadd_rn(dot, __dmul_rn(sval[warp][e], xv[scol[warp][e]]));
      } else {
        for (int64_t e = plo[u]; e < phi[u]; ++e) dot = __dadd_rn(dot, __dmul_rn(a.val[e], xv[a.col[e]]));
      }
      const double r = __dsub_rn(a.bscale == 1.0 ? bj[u] : __dmul_rn(a.bscale, bj[u]), dot);
      r_out[j] = r;
      s_rr += r * r;
      s_bb += bj[u] * bj[u];
      const double dd = r - rp[u];
      s_dd += dd * dd;
      const double tt = rt[u] - r;
      s_tt += tt * tt;
    }
    __syncwarp();
  }
  s_rr = block_sum(s_rr, red);
  s_dd = block_sum(s_dd, red);
  s_tt = block_sum(s_tt, red);
  s_bb = block_sum(s_bb, red);
  if (threadIdx.x == 0) {
    double* o = a.row_part + 4 * static_cast<int64_t>(blockIdx.x);
    o[0] = s_rr;
    o[1] = r_prev ? s_dd : 0.0;
    o[2] = a.r_true ? s_tt : 0.0;
    o[3] = s_bb;
  }
}

// A'r: a warp per chunk of CHUNK CSC entries (one column); lane l sums
// entries l, l+32, ... into 4 interleaved accumulators (8 loads in flight),
// combined in a fixed order, then a fixed shuffle tree.
__global__ void __launch_bounds__(CSR_THREADS) k_csc_chunks(CsrPassArgs a) {
  pdl_wait();
  const double *x, *r_prev;
  double* r;
  if (!resolve(a, x, r_prev, r)) return;
  const int lane = threadIdx.x & 31;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * (CSR_THREADS / 32) + (threadIdx.x >> 5);
  if (q >= a.chunk_ptr[a.n]) return;  // a.nchunks bounds the grid
  const int k = a.chunk_col[q];
  const int64_t lo = a.col_ptr[k] + (q - a.chunk_ptr[k]) * CHUNK;
  const int64_t hi = min(lo + CHUNK, a.col_ptr[k + 1]);
  constexpr int U = 8;  // accumulators: 16 loads in flight per lane, then 8 gathers
  double acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.0;
  int64_t p = lo + lane;
  for (; p + 32 * (U - 1) < hi; p += 32 * U) {
    int ri[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ri[u] = a.crow[p + 32 * u];
      v[u] = a.cval[p + 32 * u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = fma(v[u], r[ri[u]], acc[u]);
  }
  for (; p < hi; p += 32) acc[0] = fma(a.cval[p], r[a.crow[p]], acc[0]);
  double t = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) t += acc[u];
  const double s = warp_sum(t);
  if (lane == 0) a.chunk_part[q] = s;
}

// Finish: warp w of the grid sums column w's chunk partials (lane-strided,
// fixed tree); the last 4 warps sum the row kernel's norm partials.
__global__ void __launch_bounds__(CSR_THREADS) k_csr_finish(CsrPassArgs a) {
  pdl_wait();
  if (a.mode != 0 && a.ctl->result.done) return;
  const int lane = threadIdx.x & 31;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * (CSR_THREADS / 32) + (threadIdx.x >> 5);
  if (w < a.n) {
    double s = 0.0;
    for (int64_t q = a.chunk_ptr[w] + lane; q < a.chunk_ptr[w + 1]; q += 32) s += a.chunk_part[q];
    s = warp_sum(s);
    if (lane == 0) a.cs[w] = s;
  } else if (w < a.n + 4) {
    const int k = static_cast<int>(w - a.n);
    double s = 0.0;
    for (int g = lane; g < a.g1; g += 32) s += a.row_part[4 * static_cast<int64_t>(g) + k];
    s = warp_sum(s);
    if (lane == 0) a.cs[w] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Plan: the CSC copy, chunk table and partial buffers (one device allocation)
// ---------------------------------------------------------------------------
struct CsrPlan {
  int64_t m, n, nnz;
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
  int64_t* col_ptr;
  int32_t* crow;
  double* cval;
  int32_t* chunk_col;
  int64_t* chunk_ptr;
  double* chunk_part;
  double* row_part;
  double* r_tmp;
  int64_t nchunks;
  int g1;
  int64_t rows_per_cta;
  void* pool;
};

int csr_rows_grid(int64_t m) {
  int64_t g = (m + 2 * RPL * CSR_THREADS - 1) / (2 * RPL * CSR_THREADS);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  return static_cast<int>(std::max<int64_t>(1, std::min(g, cap)));
}

int launch_csr_pass(const CsrPlan* P, const double* b, double bscale, const double* x, const double* r_prev,
                    double* r_out, const double* r_true, double* cs, const LoopCtl* ctl, const double* xs,
                    double* rs, int mode, cudaStream_t s) {
  CsrPassArgs a{};
  a.row_ptr = P->row_ptr;
  a.col = P->col;
  a.val = P->val;
  a.col_ptr = P->col_ptr;
  a.crow = P->crow;
  a.cval = P->cval;
  a.chunk_col = P->chunk_col;
  a.chunk_ptr = P->chunk_ptr;
  a.chunk_part = P->chunk_part;
  a.row_part = P->row_part;
  a.m = P->m;
  a.n = P->n;
  a.nchunks = P->nchunks;
  a.rows_per_cta = P->rows_per_cta;
  a.g1 = P->g1;
  a.b = b;
  a.bscale = bscale;
  a.x = x;
  a.r_prev = r_prev;
  a.r_out = (mode == 0 && !r_out) ? P->r_tmp : r_out;
  a.r_true = r_true;
  a.cs = cs;
  a.ctl = ctl;
  a.xs = xs;
  a.rs = rs;
  a.mode = mode;
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_csr_rows)));
  const size_t xsmem = (CSR_THREADS / 32) * ROW_STAGE * 12 + (P->n <= X_STAGE ? static_cast<size_t>(P->n) * 8 : 0);
  ITSK_CUDA(launch_pdl(reinterpret_cast<const void*>(k_csr_rows), dim3(P->g1), dim3(CSR_THREADS), xsmem, s, a));
  count_launch();
  if (P->nchunks > 0) {
    const unsigned g2 = static_cast<unsigned>((P->nchunks + CSR_THREADS / 32 - 1) / (CSR_THREADS / 32));
    ITSK_CUDA(launch_pdl(reinterpret_cast<const void*>(k_csc_chunks), dim3(g2), dim3(CSR_THREADS), 0, s, a));
    count_launch();
  }
  const unsigned g3 = static_cast<unsigned>((P->n + 4 + CSR_THREADS / 32 - 1) / (CSR_THREADS / 32));
  ITSK_CUDA(launch_pdl(reinterpret_cast<const void*>(k_csr_finish), dim3(g3), dim3(CSR_THREADS), 0, s, a));
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace itsk

using namespace itsk;

namespace itsk {
namespace {
// chunks per column, then (after the scan) the chunk -> column map
__global__ void k_chunk_count(const int64_t* __restrict__ col_ptr, int64_t n, int64_t* __restrict__ cnt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) cnt[k] = (col_ptr[k + 1] - col_ptr[k] + CHUNK - 1) / CHUNK;
}
__global__ void k_chunk_fill(const int64_t* __restrict__ chunk_ptr, int64_t n, int32_t* __restrict__ chunk_col) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  for (int64_t q = chunk_ptr[k]; q < chunk_ptr[k + 1]; ++q) chunk_col[q] = static_cast<int32_t>(k);
}

// keep freed stream-ordered allocations in the device pool (plans are made
// per solve; returning the memory to the driver each time costs milliseconds)
void retain_pool_memory() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static bool done[64] = {};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}
}  // namespace
}  // namespace itsk

extern "C" int itsk_csr_plan_create(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t m,
                                    int64_t n, int64_t nnz, itsk_stream_t stream, itsk_csr_plan** plan) {
  ITSK_REQUIRE(plan && row_ptr && (nnz == 0 || (col && val)), "null pointer");
  ITSK_REQUIRE(m >= 1 && n >= 1 && nnz >= 0, "bad CSR shape");
  ITSK_REQUIRE(nnz < (1ll << 31) && m < (1ll << 31) && n < (1ll << 31), "CSR too large (nnz, m, n < 2^31)");
  *plan = nullptr;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  retain_pool_memory();
  CsrPlan* P = new CsrPlan();
  P->m = m;
  P->n = n;
  P->nnz = nnz;
  P->row_ptr = row_ptr;
  P->col = col;
  P->val = val;
  P->g1 = csr_rows_grid(m);
  P->rows_per_cta = align_up((m + P->g1 - 1) / P->g1, 32 * RPL);
  P->nchunks = n + (nnz + CHUNK - 1) / CHUNK;  // upper bound; the count is chunk_ptr[n]
  const int bits = std::max(1, 64 - __builtin_clzll(static_cast<unsigned long long>(n)));
  const int nsort = static_cast<int>(std::max<int64_t>(nnz, 1));
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, nsort, 0, bits, s);
  cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr,
                                static_cast<int>(n), s);
  // one stream-ordered allocation: the plan's arrays, then creation scratch
  Carver cv(nullptr, 1ll << 62);
  auto layout = [&](Carver& c, bool assign) {
    int64_t* a0 = c.take<int64_t>(n + 1);
    int32_t* a1 = c.take<int32_t>(nnz);
    double* a2 = c.take<double>(nnz);
    int32_t* a3 = c.take<int32_t>(P->nchunks);
    int64_t* a4 = c.take<int64_t>(n + 1);
    double* a5 = c.take<double>(P->nchunks);
    double* a6 = c.take<double>(4 * static_cast<int64_t>(P->g1));
    double* a7 = c.take<double>(m);
    int* a8 = c.take<int>(1);
    if (assign) {
      P->col_ptr = a0; P->crow = a1; P->cval = a2; P->chunk_col = a3;
      P->chunk_ptr = a4; P->chunk_part = a5; P->row_part = a6; P->r_tmp = a7;
    }
    return a8;
  };
  layout(cv, false);
  const int64_t keep = cv.off;
  cv.take<uint32_t>(nnz);  // sorted keys
  cv.take<uint32_t>(nnz);  // iota
  cv.take<uint32_t>(nnz);  // permutation
  cv.take<uint32_t>(nnz);  // entry rows
  cv.take<int64_t>(n);     // chunk counts
  cv.take<char>(static_cast<int64_t>(std::max(sort_bytes, scan_bytes)));
  auto fail = [&](int code) {
    if (P->pool) cudaFreeAsync(P->pool, s);
    delete P;
    return code;
  };
  if (cudaMallocAsync(&P->pool, cv.off + 256, s) != cudaSuccess) {
    set_error("csr plan: device allocation of %lld bytes failed", (long long)cv.off);
    cudaGetLastError();
    delete P;
    return ITSK_ECUDA;
  }
  Carver c2(P->pool, 1ll << 62);
  int* bad = layout(c2, true);
  uint32_t* keys = c2.take<uint32_t>(nnz);
  uint32_t* iota = c2.take<uint32_t>(nnz);
  uint32_t* perm = c2.take<uint32_t>(nnz);
  uint32_t* erow = c2.take<uint32_t>(nnz);
  int64_t* ccnt = c2.take<int64_t>(n);
  void* tmp = c2.take<char>(static_cast<int64_t>(std::max(sort_bytes, scan_bytes)));
  (void)keep;
  // validate the structure (monotone row_ptr, columns in range): the one sync
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), s);
  k_check_csr<<<static_cast<unsigned>((m + 1 + 255) / 256), 256, 0, s>>>(row_ptr, col, m, n, nnz, bad);
  count_launch();
  int hbad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    set_error("csr plan: %s", cudaGetErrorString(e));
    return fail(ITSK_ECUDA);
  }
  if (hbad) {
    set_error("invalid CSR structure (%s)", (hbad & 1) ? "row_ptr" : "column index out of range");
    return fail(ITSK_EINVAL);
  }
  // CSC: stable radix sort of the entry ids by column (entries are in row order)
  if (nnz > 0) {
    k_entry_rows<<<static_cast<unsigned>((m + 255) / 256), 256, 0, s>>>(row_ptr, m, erow);
    k_iota<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(iota, nnz);
    cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, reinterpret_cast<const uint32_t*>(col), keys, iota, perm,
                                    static_cast<int>(nnz), 0, bits, s);
    k_col_ptr<<<static_cast<unsigned>((n + 1 + 255) / 256), 256, 0, s>>>(keys, nnz, n, P->col_ptr);
    k_csc_gather<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(perm, erow, val, nnz, P->crow, P->cval);
    count_launch(5);
  } else {
    cudaMemsetAsync(P->col_ptr, 0, sizeof(int64_t) * (n + 1), s);
  }
  // chunk table on the device: counts, inclusive scan into chunk_ptr[1..n], fill
  k_chunk_count<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(P->col_ptr, n, ccnt);
  cudaMemsetAsync(P->chunk_ptr, 0, sizeof(int64_t), s);
  cub::DeviceScan::InclusiveSum(tmp, scan_bytes, ccnt, P->chunk_ptr + 1, static_cast<int>(n), s);
  k_chunk_fill<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(P->chunk_ptr, n, P->chunk_col);
  count_launch(3);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("csr plan: %s", cudaGetErrorString(e));
    return fail(ITSK_ECUDA);
  }
  *plan = reinterpret_cast<itsk_csr_plan*>(P);
  return ITSK_OK;
}

extern "C" void itsk_csr_plan_destroy(itsk_csr_plan* plan) {
  if (!plan) return;
  CsrPlan* P = reinterpret_cast<CsrPlan*>(plan);
  cudaDeviceSynchronize();  // no stream still reads the plan
  if (P->pool) cudaFreeAsync(P->pool, 0);
  delete P;
}

extern "C" int itsk_csr_shape(const itsk_csr_plan* plan, int64_t* m, int64_t* n, int64_t* nnz) {
  ITSK_REQUIRE(plan, "null plan");
  const CsrPlan* P = reinterpret_cast<const CsrPlan*>(plan);
  if (m) *m = P->m;
  if (n) *n = P->n;
  if (nnz) *nnz = P->nnz;
  return ITSK_OK;
}

extern "C" int itsk_csr_sketch(const itsk_csr_plan* plan, const double* b, const uint32_t* sk_ptr,
                               const uint32_t* sk_src, int64_t d, int64_t zeta, double* SAb, int64_t ldw,
                               itsk_stream_t stream) {
  ITSK_REQUIRE(plan && sk_ptr && sk_src && SAb, "null pointer");
  const CsrPlan* P = reinterpret_cast<const CsrPlan*>(plan);
  ITSK_REQUIRE(d >= 1 && zeta >= 1 && ldw >= P->n + (b ? 1 : 0), "bad sketch shape");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const double scale = 1.0 / sqrt(static_cast<double>(zeta));  // embed.py:92
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_sketch_csr)));
  const int64_t n = P->n;
  const int64_t budget = 180 * 1024;
  int warps = static_cast<int>(std::min<int64_t>(8, budget / (n * 8)));
  const int smem_acc = warps >= 1 ? 1 : 0;
  if (!smem_acc) warps = 8;
  const size_t smem = smem_acc ? static_cast<size_t>(warps) * n * 8 : 0;
  const unsigned grid = static_cast<unsigned>((d + warps - 1) / warps);
  k_sketch_csr<<<grid, 32 * warps, smem, s>>>(P->row_ptr, P->col, P->val, n, sk_ptr, sk_src, d, scale, SAb, ldw,
                                              smem_acc);
  count_launch();
  ITSK_CHECK_LAUNCH();
  // S·b into column n: the dense gather with no A columns (apply_vec's sum)
  if (b) return itsk_sketch(nullptr, P->m, 0, 0, b, sk_ptr, sk_src, d, zeta, SAb + n, ldw, stream);
  return ITSK_OK;
}

extern "C" int itsk_csr_pass(const itsk_csr_plan* plan, const double* b, double bscale, const double* x,
                             const double* r_prev, double* r_out, const double* r_true, double* cs,
                             itsk_stream_t stream) {
  ITSK_REQUIRE(plan && b && x && cs, "null pointer");
  return launch_csr_pass(reinterpret_cast<const CsrPlan*>(plan), b, bscale, x, r_prev, r_out, r_true, cs, nullptr,
                         nullptr, nullptr, 0, reinterpret_cast<cudaStream_t>(stream));
}
