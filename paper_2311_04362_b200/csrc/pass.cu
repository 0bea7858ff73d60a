// The fused streaming pass of the refinement loop (K3).
//
// The reference makes two BLAS-2 passes over A per iteration
// (/root/reference/pkg/src/itsketch/solvers.py:299 `r_next = b - a @ x_next`
// and :343 `a.T @ r`), plus m-vector passes for the norms (:300-302) and for
// _record's residual error (:250).  Row-major A (numpy C order) lets one pass
// do all of it: a warp owns a row, forms dot(A_j, x) with a shuffle reduce,
// r_j = b_j - dot, and immediately folds r_j * A_j into its register copy of
// c = A'r while the row is still in registers.  A is read exactly once per
// iteration (8 m n bytes: the HBM roofline of the loop), with evict-first
// streaming loads; each CTA owns a contiguous row range.  Per-CTA partials
// are summed by k_finalize in a fixed order, so c and the norms are
// bitwise reproducible run to run.
#include <algorithm>
#include <cstdlib>

#include "itsk_common.cuh"
#include "itsk_kernels.cuh"

namespace itsk {
namespace {

constexpr int PASS_THREADS = 256;
constexpr int PASS_WARPS = PASS_THREADS / 32;

template <int CPL>
__global__ void __launch_bounds__(PASS_THREADS) k_pass(PassArgs a) {
  extern __shared__ double sm[];
  constexpr int NC = 32 * CPL;
  constexpr bool XREG = CPL <= 8;
  constexpr int UNR = CPL <= 8 ? 2 : 1;
  double* xsm = sm;            // NC
  double* csm = sm + NC;       // PASS_WARPS x NC
  __shared__ double ssm[PASS_WARPS][4];

  const double* x;
  const double* r_prev;
  double* r_out;
  if (a.mode == 0) {
    x = a.x;
    r_prev = a.r_prev;
    r_out = a.r_out;
  } else {
    const LoopCtl* ctl = a.ctl;
    if (ctl->result.done) return;
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
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n, lda = a.lda;
  for (int c = tid; c < NC; c += PASS_THREADS) xsm[c] = (c < n) ? x[c] : 0.0;
  __syncthreads();

  double xv[XREG ? CPL : 1];
  if (XREG) {
#pragma unroll
    for (int q = 0; q < CPL; ++q) xv[q] = xsm[lane + 32 * q];
  }
  double acc[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) acc[q] = 0.0;
  double s_rr = 0.0, s_dd = 0.0, s_tt = 0.0, s_bb = 0.0;

  const int64_t r_begin = static_cast<int64_t>(blockIdx.x) * a.rows_per_cta;
  const int64_t r_end = min(a.m, r_begin + a.rows_per_cta);
  const double* b = a.b;
  const double* r_true = a.r_true;
  const uint64_t pol = evict_first_policy();

  for (int64_t row0 = r_begin + warp; row0 < r_end; row0 += PASS_WARPS * UNR) {
    double av[UNR][CPL];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t row = row0 + u * PASS_WARPS;
      const double* arow = a.A + row * lda;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        av[u][q] = (row < r_end && c < n) ? ldg_stream(arow + c, pol) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t row = row0 + u * PASS_WARPS;
      if (row >= r_end) break;
      double dot = 0.0;
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        dot = fma(av[u][q], XREG ? xv[XREG ? q : 0] : xsm[lane + 32 * q], dot);
      dot = warp_sum(dot);
      const double bj = b[row];
      const double r = (a.bscale == 1.0 ? bj : a.bscale * bj) - dot;
#pragma unroll
      for (int q = 0; q < CPL; ++q) acc[q] = fma(r, av[u][q], acc[q]);
      if (lane == 0) {
        if (r_out) r_out[row] = r;
        s_rr += r * r;
        s_bb += bj * bj;
        if (r_prev) {
          const double dd = r - r_prev[row];
          s_dd += dd * dd;
        }
        if (r_true) {
          const double tt = r_true[row] - r;
          s_tt += tt * tt;
        }
      }
    }
  }
  // CTA reduction in fixed warp order
#pragma unroll
  for (int q = 0; q < CPL; ++q) csm[warp * NC + lane + 32 * q] = acc[q];
  if (lane == 0) {
    ssm[warp][0] = s_rr;
    ssm[warp][1] = s_dd;
    ssm[warp][2] = s_tt;
    ssm[warp][3] = s_bb;
  }
  __syncthreads();
  double* out = a.part + static_cast<int64_t>(blockIdx.x) * (n + 4);
  for (int c = tid; c < n; c += PASS_THREADS) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < PASS_WARPS; ++w) s += csm[w * NC + c];
    out[c] = s;
  }
  if (tid < 4) {
    double s = 0.0;
    for (int w = 0; w < PASS_WARPS; ++w) s += ssm[w][tid];
    out[n + tid] = s;
  }
}

// ---------------------------------------------------------------------------
// Wide rows (n beyond the staged kernels' 2048 columns, or beyond 1024 at an
// odd leading dimension): the whole CTA takes one row at a time.  A thread
// owns the columns tid, tid + 512, ... (coalesced 8-byte loads, the next row
// in flight under the current one), so the row's elements stay in registers
// between the dot product and the c update — A is read once — and every
// column of c has exactly one owner (no CTA-level reduction of c).  One
// barrier per row (double-buffered warp partials, summed in warp order by
// every thread).  The per-CTA partials go through k_finalize like k_pass's.
// ---------------------------------------------------------------------------
constexpr int WIDE_THREADS = 512;
constexpr int WIDE_WARPS = WIDE_THREADS / 32;

template <int CPT>
__global__ void __launch_bounds__(WIDE_THREADS, 1) k_pass_wide(PassArgs a) {
  __shared__ double red[2][WIDE_WARPS];
  const double* x;
  const double* r_prev;
  double* r_out;
  if (a.mode == 0) {
    x = a.x;
    r_prev = a.r_prev;
    r_out = a.r_out;
  } else {
    const LoopCtl* ctl = a.ctl;
    if (ctl->result.done) return;
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
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n, lda = a.lda;
  double xv[CPT], acc[CPT], av[CPT], an[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int64_t c = tid + WIDE_THREADS * q;
    xv[q] = c < n ? x[c] : 0.0;
    acc[q] = 0.0;
  }
  double s_rr = 0.0, s_dd = 0.0, s_tt = 0.0, s_bb = 0.0;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.x) * a.rows_per_cta;
  const int64_t r_end = min(a.m, r_begin + a.rows_per_cta);
  const double* b = a.b;
  const double* r_true = a.r_true;
  const uint64_t pol = evict_first_policy();
  auto load_row = [&](int64_t row, double (&v)[CPT]) {
    const double* arow = a.A + row * lda;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int64_t c = tid + WIDE_THREADS * q;
      v[q] = (row < r_end && c < n) ? ldg_stream(arow + c, pol) : 0.0;
    }
  };
  load_row(r_begin, av);
  int buf = 0;
  for (int64_t row = r_begin; row < r_end; ++row) {
    load_row(row + 1, an);
    double dot = 0.0;
#pragma unroll
    for (int q = 0; q < CPT; ++q) dot = fma(av[q], xv[q], dot);
    dot = warp_sum(dot);
    if (lane == 0) red[buf][warp] = dot;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < WIDE_WARPS; ++w) tot += red[buf][w];
    buf ^= 1;
    const double bj = b[row];
    const double r = (a.bscale == 1.0 ? bj : a.bscale * bj) - tot;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      acc[q] = fma(r, av[q], acc[q]);
      av[q] = an[q];
    }
    if (tid == 0) {
      if (r_out) r_out[row] = r;
      s_rr += r * r;
      s_bb += bj * bj;
      if (r_prev) {
        const double dd = r - r_prev[row];
        s_dd += dd * dd;
      }
      if (r_true) {
        const double tt = r_true[row] - r;
        s_tt += tt * tt;
      }
    }
  }
  double* out = a.part + static_cast<int64_t>(blockIdx.x) * (n + 4);
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int64_t c = tid + WIDE_THREADS * q;
    if (c < n) out[c] = acc[q];
  }
  if (tid == 0) {
    out[n] = s_rr;
    out[n + 1] = s_dd;
    out[n + 2] = s_tt;
    out[n + 3] = s_bb;
  }
}

// ---------------------------------------------------------------------------
// TMA-staged variant (sm_100a): one producer warp streams contiguous tiles of
// T rows (T*lda*8 bytes, one cp.async.bulk each, L2 evict-first) into an
// S-stage shared-memory ring guarded by mbarriers; 8 consumer warps take rows
// round-robin from the ring.  The row is read twice from shared memory (dot,
// then c update), so registers hold only c (and x when it fits) — this keeps
// ~S*16 KB of HBM traffic in flight per SM independent of n.
// ---------------------------------------------------------------------------

struct TmaShape {
  int T;            // rows per tile (multiple of UNR)
  int S;            // stages
  int stage_bytes;  // T*lda*8, 128-aligned
};

// Consumer warps take batches of UNR consecutive rows (a batch never spans
// two tiles): the UNR dot products and their shuffle reductions are
// interleaved, so the per-row latency chain (LDS -> FMA chain -> 5 shuffles)
// is paid once per batch.  Only A goes through the bulk-copy ring — one copy
// per tile; per-copy cost, not bytes, limits TMA at small sizes — while lanes
// 0..UNR-1 prefetch b / r_prev / r_true of the warp's batch two steps ahead
// with ordinary loads.  stage_tile[s] names the tile a stage holds, so a
// consumer never waits on an mbarrier phase that aliases an older tile.
// Two-level "last CTA" reduction of the per-CTA partials (see PassArgs):
// the partial of this CTA is in a.part[blockIdx.x]; the last arriver of each
// group sums its group in CTA order, the last group sums the groups in group
// order, so the result does not depend on which CTA finishes last.  The
// partials are L2 reads: each level issues a whole chunk of them before the
// first add (RCH loads in flight per column) — a dependent load per partial
// was ~12 serialised L2 round trips at 148 CTAs, most of the pass's fixed
// cost at C2.  The adds keep the sequential order of the index.
constexpr int RCH = 16;

__device__ __forceinline__ double sum_strided(const double* p, int64_t stride, int cnt, double s) {
  for (int k0 = 0; k0 < cnt; k0 += RCH) {
    double v[RCH];
#pragma unroll
    for (int k = 0; k < RCH; ++k) v[k] = (k0 + k < cnt) ? __ldcg(p + (k0 + k) * stride) : 0.0;
#pragma unroll
    for (int k = 0; k < RCH; ++k)
      if (k0 + k < cnt) s += v[k];
  }
  return s;
}

// Ticket increment with acquire-release semantics at GPU scope, by one
// thread after a CTA barrier: the barrier orders the CTA's partial writes
// before the release, and the acquire orders the last arriver's loads of
// the other CTAs' partials after it (one fence per CTA instead of one per
// thread).
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* p) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

__device__ void group_reduce(const PassArgs& a, int64_t n) {
  __shared__ int s_last;
  const int64_t w = n + 4;
  const int G = a.group, gi = static_cast<int>(blockIdx.x) / G;
  const int gsz = min(G, static_cast<int>(gridDim.x) - gi * G);
  const int ng = (static_cast<int>(gridDim.x) + G - 1) / G;
  __syncthreads();
  if (threadIdx.x == 0) s_last = ticket_acq_rel(&a.tickets[gi]) == static_cast<unsigned>(gsz - 1);
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) a.tickets[gi] = 0;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x)
    a.gpart[static_cast<int64_t>(gi) * w + c] = sum_strided(a.part + static_cast<int64_t>(gi) * G * w + c, w, gsz, 0.0);
  if (a.tail_sums) return;  // the loop's tail sums the groups (tail_group_sum, same order)
  __syncthreads();
  if (threadIdx.x == 0) s_last = ticket_acq_rel(&a.tickets[ng]) == static_cast<unsigned>(ng - 1);
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) a.tickets[ng] = 0;
  // even groups into s0, odd groups into s1, then s0 + s1
  const int ne = (ng + 1) / 2, no = ng / 2;
  const PeerArgs& pe = a.peer;
  const bool send = pe.size > 0 && a.ctl != nullptr;
  const int64_t epoch = send ? a.ctl->epoch_base + (a.mode == 2 ? 0 : a.ctl->it + 1) : 0;
  const int64_t pw = peer_width(n);
  const int64_t slot = ((epoch & 1) * pe.size + pe.rank) * pw;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
    const double s0 = sum_strided(a.gpart + c, 2 * w, ne, 0.0);
    const double s1 = sum_strided(a.gpart + w + c, 2 * w, no, 0.0);
    const double v = s0 + s1;
    a.cs[c] = v;
    // peer exchange: this rank's partial into every rank's receive buffer
    if (send)
      for (int r = 0; r < pe.size; ++r) pe.recv[r][slot + c] = v;
  }
  if (send && threadIdx.x == 0) {
    const double rb = peer_ready_bit(pe);
    for (int r = 0; r < pe.size; ++r) pe.recv[r][slot + w] = rb;
  }
  if (send) {
    __threadfence_system();
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < pe.size)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pe.flags[threadIdx.x] + pe.rank),
                   "l"(static_cast<unsigned long long>(epoch))
                   : "memory");
  }
}

#ifdef ITSK_TIMELINE
// [slot][0] first CTA start, [1] last CTA end of streaming, [2] last CTA end
__device__ unsigned long long g_pass_tl[TL_SLOTS][4];
#endif

template <int CPL, int UNR, int NCW>
__global__ void __launch_bounds__(32 * NCW, 1) k_pass_tma(PassArgs a, TmaShape sh) {
  constexpr int THREADS = 32 * NCW;
#ifdef ITSK_TIMELINE
  const unsigned long long tl_t0 = gtime();
  int tl_slot = -1;
#endif
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int NC = 32 * CPL;
  constexpr bool XREG = CPL <= 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  unsigned* consumed = reinterpret_cast<unsigned*>(full + 32);  // batches of a stage's tile read so far
  int* stage_tile = reinterpret_cast<int*>(consumed + 32);
  double* xsm = reinterpret_cast<double*>(smraw + 1024);
  unsigned char* stages = smraw + 1024 + (XREG ? 0 : NC * 8);
  __shared__ double ssm[NCW][4];
  __shared__ int s_done;

  const double* r_true = a.r_true;
  const double* b = a.b;
  const double bscale = a.bscale;  // 1.0 except in LSQR's bidiagonalisation
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n, lda = a.lda;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.x) * a.rows_per_cta;
  const int64_t r_end = min(a.m, r_begin + a.rows_per_cta);
  const int nrows = r_end > r_begin ? static_cast<int>(r_end - r_begin) : 0;
  const int T = sh.T, S = sh.S;
  const int ntiles = (nrows + T - 1) / T;
  const int npre = min(S, ntiles);  // tiles issued before the dependency wait

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      consumed[s] = 0u;
      stage_tile[s] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Programmatic dependent launch: A does not depend on the previous kernel,
  // so the producer fills the ring while that kernel (the loop tail) still
  // runs; everything the previous kernel writes (x, the loop state) is read
  // after griddepcontrol.wait.
  pdl_trigger();
  // no producer warp: the consumer that reads the last batch of a stage's
  // tile refills the stage with tile t + S (a per-stage counter; the bulk
  // copy is ordered after every warp's reads of the stage by the counter's
  // acquire-release and a proxy fence)
  const uint64_t pol = evict_first_policy();
  if (tid == 0) {
    for (int t = 0; t < npre; ++t) {
      const int64_t row0 = r_begin + static_cast<int64_t>(t) * T;
      const int rows = min(T, nrows - t * T);
      const unsigned bytes = static_cast<unsigned>(rows * lda * 8);
      reinterpret_cast<volatile int*>(stage_tile)[t] = t;
      mbar_expect_tx(full + t, bytes);
      bulk_g2s(stages + static_cast<int64_t>(t) * sh.stage_bytes, a.A + row0 * lda, bytes, full + t, pol);
    }
  }
  pdl_wait();

  const double* x;
  const double* r_prev;
  double* r_out;
  if (a.mode == 0) {
    x = a.x;
    r_prev = a.r_prev;
    r_out = a.r_out;
  } else {
    const LoopCtl* ctl = a.ctl;
    if (tid == 0) s_done = ctl->result.done;
    __syncthreads();
    if (s_done) {
      // loop finished: drain the prefetched copies before the CTA exits
      if (tid == 0)
        for (int t = 0; t < npre; ++t) mbar_wait(full + t, 0u);
      return;
    }
    const int64_t S = ctl->r_slots;
#ifdef ITSK_TIMELINE
    tl_slot = a.mode == 1 ? static_cast<int>(ctl->it) + 1 : 0;
#endif
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
  }
  if (!XREG)
    for (int c = tid; c < NC; c += THREADS) xsm[c] = (c < n) ? x[c] : 0.0;
  __syncthreads();

  double acc[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) acc[q] = 0.0;

  {
    // ---------------- consumers ----------------
    double xv[XREG ? CPL : 1];
    if (XREG) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        xv[q] = (c < n) ? x[c] : 0.0;
      }
    }
    // lane u < UNR carries row u of the batch: prefetched scalars and sums
    double s_rr = 0.0, s_dd = 0.0, s_tt = 0.0, s_bb = 0.0;
    constexpr int STEP = NCW * UNR;
    auto fetch = [&](int k, double& fb, double& fp, double& ft) {
      const int kk = k + lane;
      const bool ok = lane < UNR && kk < nrows;
      const int64_t g = r_begin + kk;
      fb = ok ? b[g] : 0.0;
      fp = (ok && r_prev) ? r_prev[g] : 0.0;
      ft = (ok && r_true) ? r_true[g] : 0.0;
    };
    double cb, cp, ct, nb, np, nt;
    const int k_first = warp * UNR;
    fetch(k_first, cb, cp, ct);
    fetch(k_first + STEP, nb, np, nt);
    for (int k0 = k_first; k0 < nrows; k0 += STEP) {
      double fb, fp, ft;
      fetch(k0 + 2 * STEP, fb, fp, ft);
      const int t = k0 / T;
      const int s = t % S;
      while (reinterpret_cast<volatile int*>(stage_tile)[s] != t) __nanosleep(20);
      mbar_wait(full + s, static_cast<unsigned>((t / S) & 1));
      const double* base =
          reinterpret_cast<const double*>(stages + static_cast<int64_t>(s) * sh.stage_bytes) +
          static_cast<int64_t>(k0 - t * T) * lda;
      const int nu = min(UNR, nrows - k0);
      double dot[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) dot[u] = 0.0;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        if (c < n) {
          const double xq = XREG ? xv[XREG ? q : 0] : xsm[c];
#pragma unroll
          for (int u = 0; u < UNR; ++u)
            if (u < nu) dot[u] = fma(base[u * lda + c], xq, dot[u]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < UNR; ++u) dot[u] += __shfl_xor_sync(FULL, dot[u], o);
      double r[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) r[u] = bscale * __shfl_sync(FULL, cb, u) - dot[u];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        if (c < n) {
#pragma unroll
          for (int u = 0; u < UNR; ++u)
            if (u < nu) acc[q] = fma(r[u], base[u * lda + c], acc[q]);
        }
      }
      __syncwarp();
      if (lane == 0) {
        // the last of the tile's T / UNR batches read: refill the stage
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "r"(smem_u32(consumed + s)) : "memory");
        if (old == static_cast<unsigned>(T / UNR - 1)) {
          consumed[s] = 0u;
          const int tn = t + S;
          if (tn < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int rows = min(T, nrows - tn * T);
            const unsigned bytes = static_cast<unsigned>(rows * lda * 8);
            reinterpret_cast<volatile int*>(stage_tile)[s] = tn;
            mbar_expect_tx(full + s, bytes);
            bulk_g2s(stages + static_cast<int64_t>(s) * sh.stage_bytes, a.A + (r_begin + static_cast<int64_t>(tn) * T) * lda,
                     bytes, full + s, pol);
          }
        }
      }
      if (lane < nu) {
        double rl = r[0];
#pragma unroll
        for (int u = 1; u < UNR; ++u)
          if (lane == u) rl = r[u];
        if (r_out) r_out[r_begin + k0 + lane] = rl;
        s_rr += rl * rl;
        s_bb += cb * cb;
        const double dd = rl - cp;
        s_dd += dd * dd;
        const double tt = ct - rl;
        s_tt += tt * tt;
      }
      cb = nb; cp = np; ct = nt;
      nb = fb; np = fp; nt = ft;
    }
    // fixed-order combination of the UNR lane partials
    s_rr = warp_sum(s_rr);
    s_dd = warp_sum(s_dd);
    s_tt = warp_sum(s_tt);
    s_bb = warp_sum(s_bb);
    if (lane == 0) {
      ssm[warp][0] = s_rr;
      ssm[warp][1] = r_prev ? s_dd : 0.0;
      ssm[warp][2] = r_true ? s_tt : 0.0;
      ssm[warp][3] = s_bb;
    }
  }
  __syncthreads();  // all tiles consumed: the ring is free for the reduction
  double* csm = reinterpret_cast<double*>(stages);
  if (warp < NCW) {
#pragma unroll
    for (int q = 0; q < CPL; ++q) csm[warp * NC + lane + 32 * q] = acc[q];
  }
  __syncthreads();
  double* out = a.part + static_cast<int64_t>(blockIdx.x) * (n + 4);
  for (int c = tid; c < n; c += THREADS) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < NCW; ++w) sum += csm[w * NC + c];
    out[c] = sum;
  }
  if (tid < 4) {
    double sum = 0.0;
    for (int w = 0; w < NCW; ++w) sum += ssm[w][tid];
    out[n + tid] = sum;
  }
#ifdef ITSK_TIMELINE
  if (tid == 0 && tl_slot >= 0 && tl_slot < TL_SLOTS) {
    atomicMin(&g_pass_tl[tl_slot][0], tl_t0);
    atomicMax(&g_pass_tl[tl_slot][1], gtime());
  }
#endif
  if (a.tickets) group_reduce(a, n);
#ifdef ITSK_TIMELINE
  if (tid == 0 && tl_slot >= 0 && tl_slot < TL_SLOTS) atomicMax(&g_pass_tl[tl_slot][2], gtime());
#endif
}

// ---------------------------------------------------------------------------
// Row groups (384 < n <= 2048; the C3 and C4 shapes): the 16 consumer warps
// form NG = 16 / GW groups of GW warps; group g owns batch t = g, g + NG, ...
// of RB = 4 consecutive rows (one stage of the ring, one bulk copy).  Inside
// a group every thread owns the column pairs {2t, 2t+1} + 64 GW j (j < 2),
// with x and its slice of c in registers (GW is the smallest power of two
// with 128 GW >= n).  Each thread reads its pairs of the 4 rows ONCE from
// shared memory (16-byte loads) into registers and releases the stage, so a
// row is read from shared memory once and x never is (the warp-per-row and
// warp-group kernels read the row twice and x from shared memory: ~2x the
// shared-memory traffic per byte of A).  Per batch: 4 partial dots per
// thread -> in-warp reduce-scatter (6 shuffles; lane l holds row l/8's warp
// sum) -> the GW warp partials per row in shared memory (double-buffered by
// the group's batch parity) -> ONE named barrier of the group -> every warp
// of the group sums the GW partials of the 4 rows in warp order (the same
// bits in every warp), r = b - dot -> c += r * row.  The group's first warp
// (lane u <-> row u) writes r and accumulates the norms.  The groups' c
// partials are summed in group order at the end; the norms likewise.
// The ring's stage count is a multiple of NG, so the batch a group waits for
// on a stage always follows that group's own previous batch there (no
// mbarrier phase aliasing without a stage-tag check).
// ---------------------------------------------------------------------------
constexpr int RW_NCW = 16, RW_RB = 4;

template <int GW, int CPP, bool ODD>
__global__ void __launch_bounds__(32 * RW_NCW, 1) k_pass_rows(PassArgs a, TmaShape sh) {
  constexpr int NG = RW_NCW / GW, GT = 32 * GW, RB = RW_RB;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  unsigned char* stages = smraw + 1024;
  __shared__ double dpart[NG][2][GW][RB];
  __shared__ __align__(16) double rsm[NG][2][RB];  // the batch's residuals, from the group's first warp
  __shared__ double ssm[NG][4];
  __shared__ int s_done;

  const double* r_true = a.r_true;
  const double* b = a.b;
  const double bscale = a.bscale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp / GW, gw = warp % GW, gt = tid - g * GT;  // group, warp / thread in group
  const int64_t n = a.n, lda = a.lda;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.x) * a.rows_per_cta;
  const int64_t r_end = min(a.m, r_begin + a.rows_per_cta);
  const int nrows = r_end > r_begin ? static_cast<int>(r_end - r_begin) : 0;
  const int S = sh.S;
  const int ntiles = (nrows + RB - 1) / RB;
  const int npre = min(S, ntiles);

  if (tid == 0) {
    for (int st = 0; st < S; ++st) mbar_init(full + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  // the ring's first S batches; batch t + S is issued into stage t % S by
  // the consuming group once all its warps passed the group barrier of
  // batch t (their values of the stage are in registers by then)
  const uint64_t pol = evict_first_policy();
  if (tid == 0) {
    for (int t = 0; t < npre; ++t) {
      const int rows = min(RB, nrows - t * RB);
      const unsigned bytes = static_cast<unsigned>(rows * lda * 8);
      mbar_expect_tx(full + t, bytes);
      bulk_g2s(stages + static_cast<int64_t>(t) * sh.stage_bytes, a.A + (r_begin + t * RB) * lda, bytes,
               full + t, pol);
    }
  }
  pdl_wait();

  const double* x;
  const double* r_prev;
  double* r_out;
  if (a.mode == 0) {
    x = a.x;
    r_prev = a.r_prev;
    r_out = a.r_out;
  } else {
    const LoopCtl* ctl = a.ctl;
    if (tid == 0) s_done = ctl->result.done;
    __syncthreads();
    if (s_done) {
      if (tid == 0)
        for (int t = 0; t < npre; ++t) mbar_wait(full + t, 0u);
      return;
    }
    const int64_t SL = ctl->r_slots;
    if (a.mode == 1) {
      const int64_t it = ctl->it;
      x = a.xs + (it + 1) * a.n;
      r_prev = a.rs + (it % SL) * a.m;
      r_out = a.rs + ((it + 1) % SL) * a.m;
    } else {
      x = a.xs;
      r_prev = nullptr;
      r_out = a.rs;
    }
  }

  double2 acc[CPP];
  int col[CPP];
#pragma unroll
  for (int j = 0; j < CPP; ++j) {
    acc[j] = make_double2(0.0, 0.0);
    col[j] = 2 * gt + 2 * GT * j;
  }

  {
    double2 xv[CPP];
#pragma unroll
    for (int j = 0; j < CPP; ++j) {
      const int c = col[j];
      xv[j].x = c < n ? x[c] : 0.0;
      xv[j].y = c + 1 < n ? x[c + 1] : 0.0;
    }
    // b / r_prev / r_true of the group's next batch (lane u <-> row u)
    const bool lead = lane < RB;
    auto fetch = [&](int t, double& fb, double& fp, double& ft) {
      const int k = t * RB + lane;
      const bool ok = lead && t < ntiles && k < nrows;
      const int64_t gi = r_begin + k;
      fb = ok ? b[gi] : 0.0;
      fp = (ok && gw == 0 && r_prev) ? r_prev[gi] : 0.0;
      ft = (ok && gw == 0 && r_true) ? r_true[gi] : 0.0;
    };
    double s_rr = 0.0, s_dd = 0.0, s_tt = 0.0, s_bb = 0.0;
    double cb = 0.0, cp = 0.0, ct = 0.0;  // used by the group's first warp only (it forms r)
    if (gw == 0) fetch(g, cb, cp, ct);
    // second-stage lane map: value i of lane l is warp (l % GW)'s partial of
    // row ((l / GW) % (RB / VPL)) * VPL + i
    constexpr int VPL = (GW * RB + 31) / 32;  // partials per lane
    constexpr int RPL = RB / VPL;              // row slots across the lanes
    // column validity is loop-invariant: masks computed once
    bool cok[CPP], cpad[CPP];
    int off[CPP];  // byte offset of the pair in a staged row (the first pair's when past n)
#pragma unroll
    for (int j = 0; j < CPP; ++j) {
      cok[j] = col[j] < n;
      cpad[j] = col[j] + 1 >= n;
      off[j] = 8 * (cok[j] ? col[j] : col[0]);
    }
    const int row_bytes = static_cast<int>(lda) * 8;
    uint32_t doff[CPP];
#pragma unroll
    for (int j = 0; j < CPP; ++j) doff[j] = static_cast<uint32_t>(off[j] - off[0]);
    // shared address of the thread's first pair in the group's current stage
    const uint32_t sa_stride = static_cast<uint32_t>(NG) * static_cast<uint32_t>(sh.stage_bytes);
    const uint32_t sa_wrap = static_cast<uint32_t>(S) * static_cast<uint32_t>(sh.stage_bytes);
    uint32_t sa = smem_u32(stages) + static_cast<uint32_t>(g) * static_cast<uint32_t>(sh.stage_bytes) +
                  static_cast<uint32_t>(off[0]);
    // stage index and mbarrier phase advance by NG per batch (S is a multiple
    // of NG): no integer division in the loop
    int st = g;
    unsigned ph = 0;
    for (int t = g, par = 0; t < ntiles; t += NG, par ^= 1) {
      double nb = 0.0, np = 0.0, nt = 0.0;
      if (gw == 0) fetch(t + NG, nb, np, nt);
      const int nu = min(RB, nrows - t * RB);
      mbar_wait(full + st, ph);
      const double* base = reinterpret_cast<const double*>(stages + static_cast<int64_t>(st) * sh.stage_bytes);
      double2 v[RB][CPP];
      if (nu == RB) {
        // a full batch: unconditional loads at per-thread byte offsets (a pair
        // past n re-reads the thread's first pair: its x is 0 and its c is
        // never written); only an odd n needs its pad column zeroed
        // 32-bit shared addresses: the thread's first pair in this stage (sa)
        // + row + pair offset — 7 adds per batch
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          const uint32_t ra = sa + static_cast<uint32_t>(u) * static_cast<uint32_t>(row_bytes);
#pragma unroll
          for (int j = 0; j < CPP; ++j) {
            double2 w;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y) : "r"(ra + doff[j]));
            if (ODD && cpad[j]) w.y = 0.0;
            v[u][j] = w;
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < RB; ++u)
#pragma unroll
          for (int j = 0; j < CPP; ++j) {
            double2 w = make_double2(0.0, 0.0);
            if (cok[j] && u < nu) {
              w = *reinterpret_cast<const double2*>(base + u * lda + col[j]);
              if (cpad[j]) w.y = 0.0;  // the pad column of an odd n
            }
            v[u][j] = w;
          }
      }
      double d[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        double e = 0.0;
#pragma unroll
        for (int j = 0; j < CPP; ++j) {
          e = fma(v[u][j].x, xv[j].x, e);
          e = fma(v[u][j].y, xv[j].y, e);
        }
        d[u] = e;
      }
      // in-warp reduce-scatter: lane l ends up with row l / 8's warp sum
      {
        const bool h4 = (lane & 16) != 0, h3 = (lane & 8) != 0;
        double k0 = h4 ? d[2] : d[0], k1 = h4 ? d[3] : d[1];
        const double e0 = h4 ? d[0] : d[2], e1 = h4 ? d[1] : d[3];
        k0 += __shfl_xor_sync(FULL, e0, 16);
        k1 += __shfl_xor_sync(FULL, e1, 16);
        double kk = h3 ? k1 : k0;
        kk += __shfl_xor_sync(FULL, h3 ? k0 : k1, 8);
        kk += __shfl_xor_sync(FULL, kk, 4);
        kk += __shfl_xor_sync(FULL, kk, 2);
        kk += __shfl_xor_sync(FULL, kk, 1);
        if ((lane & 7) == 0) dpart[g][par][gw][lane >> 3] = kk;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(GT) : "memory");
      // every warp of the group has its values of stage st: refill it.  By
      // the group's LAST warp: issued from lane 0 of the first warp, the
      // compiler merged this thread test with the first warp's branch below
      // and left lane 0 unreconverged, so every shuffle of the tree ran twice
      // on its divergent path (34 ms per C4 pass instead of 9)
      if (gw == GW - 1 && lane == 0 && t + S < ntiles) {
        const int tn = t + S;
        const int rows = min(RB, nrows - tn * RB);
        const unsigned bytes = static_cast<unsigned>(rows * lda * 8);
        mbar_expect_tx(full + st, bytes);
        bulk_g2s(stages + static_cast<int64_t>(st) * sh.stage_bytes, a.A + (r_begin + tn * RB) * lda, bytes,
                 full + st, pol);
      }
      // the group's GW partials per row, summed in a fixed tree by the
      // group's first warp, which hands r = b - dot of the 4 rows to the other
      // warps through shared memory (they wait on a second named barrier it
      // only arrives at; sixteen redundant copies of the tree were 2 of the
      // pass's ~19 instructions per element)
      double rv[RB];
      if (gw == 0) {
        double q[VPL];
        {
          const int w = lane % GW, r0 = ((lane / GW) % RPL) * VPL;
#pragma unroll
          for (int i = 0; i < VPL; ++i) q[i] = dpart[g][par][w][r0 + i];
        }
#pragma unroll
        for (int o = GW / 2; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < VPL; ++i) q[i] += __shfl_xor_sync(FULL, q[i], o);
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          const double dot = __shfl_sync(FULL, q[u % VPL], (u / VPL) * GW);
          rv[u] = u < nu ? bscale * __shfl_sync(FULL, cb, u) - dot : 0.0;
        }
        if constexpr (GW > 1) {
          if (lane == 0) {
#pragma unroll
            for (int u = 0; u < RB; u += 2)
              *reinterpret_cast<double2*>(&rsm[g][par][u]) = make_double2(rv[u], rv[u + 1]);
          }
          __syncwarp();
          asm volatile("bar.arrive %0, %1;" ::"r"(1 + NG + g), "r"(GT) : "memory");
        }
      } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + NG + g), "r"(GT) : "memory");
#pragma unroll
        for (int u = 0; u < RB; u += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(&rsm[g][par][u]);
          rv[u] = t2.x;
          rv[u + 1] = t2.y;
        }
      }
#pragma unroll
      for (int u = 0; u < RB; ++u)
#pragma unroll
        for (int j = 0; j < CPP; ++j) {
          acc[j].x = fma(rv[u], v[u][j].x, acc[j].x);
          acc[j].y = fma(rv[u], v[u][j].y, acc[j].y);
        }
      if (gw == 0 && lane < nu) {
        double rl = rv[0];
#pragma unroll
        for (int u = 1; u < RB; ++u)
          if (lane == u) rl = rv[u];
        if (r_out) r_out[r_begin + t * RB + lane] = rl;
        s_rr += rl * rl;
        s_bb += cb * cb;
        const double dd = rl - cp;
        s_dd += dd * dd;
        const double tt = ct - rl;
        s_tt += tt * tt;
      }
      cb = nb; cp = np; ct = nt;
      st += NG;
      sa += sa_stride;
      if (st >= S) {
        st -= S;
        sa -= sa_wrap;
        ph ^= 1u;
      }
    }
    if (gw == 0) {
      s_rr = warp_sum(s_rr);
      s_dd = warp_sum(s_dd);
      s_tt = warp_sum(s_tt);
      s_bb = warp_sum(s_bb);
      if (lane == 0) {
        ssm[g][0] = s_rr;
        ssm[g][1] = r_prev ? s_dd : 0.0;
        ssm[g][2] = r_true ? s_tt : 0.0;
        ssm[g][3] = s_bb;
      }
    }
  }
  __syncthreads();  // all stages consumed: the ring holds the groups' c partials
  double* out = a.part + static_cast<int64_t>(blockIdx.x) * (n + 4);
  if constexpr (NG == 1) {
    if (warp < RW_NCW) {
#pragma unroll
      for (int j = 0; j < CPP; ++j) {
        const int c = col[j];
        if (c < n) out[c] = acc[j].x;
        if (c + 1 < n) out[c + 1] = acc[j].y;
      }
    }
  } else {
    double* csm = reinterpret_cast<double*>(stages);  // NG x (2 GT CPP)
    constexpr int W = 2 * GT * CPP;
    if (warp < RW_NCW) {
#pragma unroll
      for (int j = 0; j < CPP; ++j) {
        csm[g * W + col[j]] = acc[j].x;
        csm[g * W + col[j] + 1] = acc[j].y;
      }
    }
    __syncthreads();
    for (int c = tid; c < n; c += 32 * RW_NCW) {
      double sum = 0.0;
#pragma unroll
      for (int gg = 0; gg < NG; ++gg) sum += csm[gg * W + c];
      out[c] = sum;
    }
  }
  if (tid < 4) {
    double sum = 0.0;
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) sum += ssm[gg][tid];
    out[n + tid] = sum;
  }
  if (a.tickets) group_reduce(a, n);
}

// ---------------------------------------------------------------------------
// Row slots (1408 < n <= 2048; the C4 shape).  The pass is HBM-bound, but the
// whole solve runs under the board's power cap and its time follows the SM
// clock: instructions per byte are what is left to save.  The row-group
// kernel above spends ~11.6 thread instructions per element at GW = 16
// (every thread holds 4 columns of 4 rows: 4 partial dots per thread to
// reduce-scatter, per-batch address arithmetic).  Here the 512 threads form 4
// slots of 128: a slot owns ONE row of the 4-row batch, a thread 8 column
// pairs {t + 128 k} of it — one partial dot per thread, a plain butterfly,
// 16-byte loads at immediate offsets from one address.  Rows are staged at a
// fixed 16 KB stride (one bulk copy per row, only the n columns: a wider lda
// costs no bandwidth); the ring is zeroed once, so the columns past n read
// zeros (their x is 0 and their c is never written).  Per batch: dot
// butterfly -> 16 warp partials -> barrier -> warp 0's lane u sums row u's 4
// partials in a fixed order, forms r = b - dot and hands it over through
// shared memory (a second barrier it only arrives at) -> c += r * row in the
// slot's registers.  The 4 slots' c partials are summed in slot order at the
// end.  10.5 thread instructions per element executed (ncu), 3 % faster than
// the row groups over sustained C4 passes (scripts/pass_sustained_ab.py).
// ---------------------------------------------------------------------------
constexpr int SL_T = 512, SL_RB = 4, SL_KP = 8, SL_ROW = 2048;  // threads, rows per batch, pairs per thread, staged row (doubles)
constexpr int SL_STAGE = SL_RB * SL_ROW * 8;                    // bytes per stage

template <bool ODD>
__global__ void __launch_bounds__(SL_T, 1) k_pass_slots(PassArgs a, TmaShape sh) {
  constexpr int RB = SL_RB, KP = SL_KP;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  unsigned char* stages = smraw + 1024;
  __shared__ __align__(16) double dpart[2][16];  // [batch parity][warp]: warp w holds row w / 4
  __shared__ __align__(16) double rsm[2][RB];    // the batch's residuals
  __shared__ double ssm[4];
  __shared__ int s_done;

  const double* r_true = a.r_true;
  const double* b = a.b;
  const double bscale = a.bscale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = tid >> 7, ts = tid & 127;
  const int64_t n = a.n, lda = a.lda;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.x) * a.rows_per_cta;
  const int64_t r_end = min(a.m, r_begin + a.rows_per_cta);
  const int nrows = r_end > r_begin ? static_cast<int>(r_end - r_begin) : 0;
  const int S = sh.S;
  const int ntiles = (nrows + RB - 1) / RB;
  const int npre = min(S, ntiles);

  // zero the ring (generic proxy) before the copies (async proxy) land in it
  {
    double2* z = reinterpret_cast<double2*>(stages);
    const int nz = S * (SL_STAGE / 16);
    for (int i = tid; i < nz; i += SL_T) z[i] = make_double2(0.0, 0.0);
  }
  if (tid == 0) {
    for (int st = 0; st < S; ++st) mbar_init(full + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  pdl_trigger();
  const uint64_t pol = evict_first_policy();
  const unsigned rowbytes = static_cast<unsigned>(((n + 1) & ~static_cast<int64_t>(1)) * 8);  // 16-byte multiple <= 8 lda
  auto issue = [&](int t, int st) {  // one thread: the rows of batch t into stage st
    const int rows = min(RB, nrows - t * RB);
    mbar_expect_tx(full + st, static_cast<unsigned>(rows) * rowbytes);
    for (int u = 0; u < rows; ++u)
      bulk_g2s(stages + static_cast<int64_t>(st) * SL_STAGE + u * (SL_ROW * 8), a.A + (r_begin + t * RB + u) * lda,
               rowbytes, full + st, pol);
  };
  if (tid == 0)
    for (int t = 0; t < npre; ++t) issue(t, t);
  pdl_wait();

  const double* x;
  const double* r_prev;
  double* r_out;
  if (a.mode == 0) {
    x = a.x;
    r_prev = a.r_prev;
    r_out = a.r_out;
  } else {
    const LoopCtl* ctl = a.ctl;
    if (tid == 0) s_done = ctl->result.done;
    __syncthreads();
    if (s_done) {
      if (tid == 0)
        for (int t = 0; t < npre; ++t) mbar_wait(full + t, 0u);
      return;
    }
    const int64_t SLOTS = ctl->r_slots;
    if (a.mode == 1) {
      const int64_t it = ctl->it;
      x = a.xs + (it + 1) * a.n;
      r_prev = a.rs + (it % SLOTS) * a.m;
      r_out = a.rs + ((it + 1) % SLOTS) * a.m;
    } else {
      x = a.xs;
      r_prev = nullptr;
      r_out = a.rs;
    }
  }

  // x (zero past n) in shared memory: with x, c and the row's values all in
  // registers the kernel spills at 512 threads; a second 16-byte shared load
  // per pair is cheaper than local memory
  double* xs = reinterpret_cast<double*>(stages + static_cast<int64_t>(S) * SL_STAGE);
  for (int c = tid; c < SL_ROW; c += SL_T) xs[c] = c < n ? x[c] : 0.0;
  __syncthreads();
  const uint32_t xa = smem_u32(xs) + static_cast<uint32_t>(ts) * 16u;
  double2 acc[KP];
  int padk = -1;  // the pair whose second column is the pad column of an odd n
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int c = 2 * (ts + 128 * k);
    acc[k] = make_double2(0.0, 0.0);
    if (ODD && c + 1 == n) padk = k;
  }
  // b / r_prev / r_true of the next batch, in warp 0 (lane u <-> row u)
  auto fetch = [&](int t, double& fb, double& fp, double& ft) {
    const int k = t * RB + lane;
    const bool ok = lane < RB && t < ntiles && k < nrows;
    const int64_t gi = r_begin + k;
    fb = ok ? b[gi] : 0.0;
    fp = (ok && r_prev) ? r_prev[gi] : 0.0;
    ft = (ok && r_true) ? r_true[gi] : 0.0;
  };
  double s_rr = 0.0, s_dd = 0.0, s_tt = 0.0, s_bb = 0.0;
  double cb = 0.0, cp = 0.0, ct = 0.0;
  if (warp == 0) fetch(0, cb, cp, ct);
  // shared address of the thread's first pair in the current stage
  uint32_t sa = smem_u32(stages) + static_cast<uint32_t>(slot) * (SL_ROW * 8) + static_cast<uint32_t>(ts) * 16u;
  int st = 0;
  unsigned ph = 0;
  for (int t = 0, par = 0; t < ntiles; ++t, par ^= 1) {
    double nb = 0.0, np = 0.0, nt = 0.0;
    if (warp == 0) fetch(t + 1, nb, np, nt);
    const int nu = min(RB, nrows - t * RB);
    mbar_wait(full + st, ph);
    double2 v[KP];
#define ITSK_SL_LD(K) \
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v[K].x), "=d"(v[K].y) : "r"(sa), "n"(2048 * K));
    ITSK_SL_LD(0) ITSK_SL_LD(1) ITSK_SL_LD(2) ITSK_SL_LD(3) ITSK_SL_LD(4) ITSK_SL_LD(5) ITSK_SL_LD(6) ITSK_SL_LD(7)
#undef ITSK_SL_LD
    static_assert(KP == 8, "eight pairs per thread");
    if (ODD) {
#pragma unroll
      for (int k = 0; k < KP; ++k)
        if (k == padk) v[k].y = 0.0;
    }
    // the thread's partial dot of its row: 4 chains, one fixed order
    double e[4] = {0.0, 0.0, 0.0, 0.0};
    {
      double2 xv[KP];
#define ITSK_SL_LDX(K) \
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(xv[K].x), "=d"(xv[K].y) : "r"(xa), "n"(2048 * K));
      ITSK_SL_LDX(0) ITSK_SL_LDX(1) ITSK_SL_LDX(2) ITSK_SL_LDX(3) ITSK_SL_LDX(4) ITSK_SL_LDX(5) ITSK_SL_LDX(6)
      ITSK_SL_LDX(7)
#undef ITSK_SL_LDX
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        e[k & 3] = fma(v[k].x, xv[k].x, e[k & 3]);
        e[k & 3] = fma(v[k].y, xv[k].y, e[k & 3]);
      }
    }
    double d = (e[0] + e[1]) + (e[2] + e[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(FULL, d, o);
    if (lane == 0) dpart[par][warp] = d;
    asm volatile("bar.sync 1, 512;" ::: "memory");
    // every thread has its values of stage st in registers: refill it (from the
    // last warp: see the note at the row-group kernel's refill)
    if (tid == SL_T - 32 && t + S < ntiles) issue(t + S, st);
    if (warp == 0) {
      if (lane < RB) {
        const double2 q0 = *reinterpret_cast<const double2*>(&dpart[par][4 * lane]);
        const double2 q1 = *reinterpret_cast<const double2*>(&dpart[par][4 * lane + 2]);
        const double dot = (q0.x + q0.y) + (q1.x + q1.y);
        const double rl = lane < nu ? bscale * cb - dot : 0.0;
        rsm[par][lane] = rl;
        if (lane < nu) {
          if (r_out) r_out[r_begin + t * RB + lane] = rl;
          s_rr += rl * rl;
          s_bb += cb * cb;
          const double dd = rl - cp;
          s_dd += dd * dd;
          const double tt = ct - rl;
          s_tt += tt * tt;
        }
      }
      cb = nb; cp = np; ct = nt;
      __syncwarp();
      asm volatile("bar.arrive 2, 512;" ::: "memory");
    } else {
      asm volatile("bar.sync 2, 512;" ::: "memory");
    }
    if (slot < nu) {  // (a slot past the last row holds an older batch's row)
      const double rv = rsm[par][slot];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        acc[k].x = fma(rv, v[k].x, acc[k].x);
        acc[k].y = fma(rv, v[k].y, acc[k].y);
      }
    }
    ++st;
    sa += SL_STAGE;
    if (st == S) {
      st = 0;
      sa -= static_cast<uint32_t>(S) * SL_STAGE;
      ph ^= 1u;
    }
  }
  if (warp == 0) {
    s_rr = warp_sum(s_rr);
    s_dd = warp_sum(s_dd);
    s_tt = warp_sum(s_tt);
    s_bb = warp_sum(s_bb);
    if (lane == 0) {
      ssm[0] = s_rr;
      ssm[1] = r_prev ? s_dd : 0.0;
      ssm[2] = r_true ? s_tt : 0.0;
      ssm[3] = s_bb;
    }
  }
  __syncthreads();  // all stages consumed: the ring holds the slots' c partials
  double* out = a.part + static_cast<int64_t>(blockIdx.x) * (n + 4);
  double* csm = reinterpret_cast<double*>(stages);  // RB x SL_ROW
#pragma unroll
  for (int k = 0; k < KP; ++k)
    *reinterpret_cast<double2*>(csm + slot * SL_ROW + 2 * (ts + 128 * k)) = acc[k];
  __syncthreads();
  for (int c = tid; c < n; c += SL_T) {
    double sum = 0.0;
#pragma unroll
    for (int g = 0; g < RB; ++g) sum += csm[g * SL_ROW + c];
    out[c] = sum;
  }
  if (tid < 4) out[n + tid] = ssm[tid];
  if (a.tickets) group_reduce(a, n);
}

// Fixed-order reduction of the per-CTA partials: one warp per output, lanes
// take CTAs strided by 32, then a fixed shuffle tree.
__global__ void k_finalize(const double* __restrict__ part, int grid, int64_t n, double* cs,
                           const LoopCtl* ctl) {
  if (ctl && ctl->result.done) return;
  const int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= n + 4) return;
  double s = 0.0;
  for (int g = lane; g < grid; g += 32) s += part[static_cast<int64_t>(g) * (n + 4) + c];
  s = warp_sum(s);
  if (lane == 0) cs[c] = s;
}

// Peer send for the passes without the in-kernel reduction (k_pass +
// k_finalize, rows not 16-byte aligned): the reduced partial, complete when
// this kernel starts, to every rank's receive buffer, then the flags.
__global__ void k_peer_send(const double* __restrict__ cs, int64_t n, const LoopCtl* ctl, int mode, PeerArgs pe) {
  if (ctl->result.done) return;
  const int64_t epoch = ctl->epoch_base + (mode == 2 ? 0 : ctl->it + 1);
  const int64_t w = peer_width(n);
  const int64_t slot = ((epoch & 1) * pe.size + pe.rank) * w;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
    const double v = c < n + 4 ? cs[c] : peer_ready_bit(pe);
    for (int r = 0; r < pe.size; ++r) pe.recv[r][slot + c] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (static_cast<int>(threadIdx.x) < pe.size)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pe.flags[threadIdx.x] + pe.rank),
                 "l"(static_cast<unsigned long long>(epoch))
                 : "memory");
}

template <int CPL>
size_t pass_smem() {
  return static_cast<size_t>(32 * CPL) * (1 + PASS_WARPS) * sizeof(double);
}

int cpl_for(int64_t n) {
  const int64_t need = (n + 31) / 32;
  int c = 1;
  while (c < need) c <<= 1;
  return c;
}

template <int CPL>
int blocks_per_sm() {
  static int cached = -1;
  if (cached < 0) {
    const size_t smem = pass_smem<CPL>();
    allow_max_smem(reinterpret_cast<const void*>(k_pass<CPL>));
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pass<CPL>, PASS_THREADS, smem) !=
            cudaSuccess ||
        nb < 1)
      nb = 1;
    cached = nb;
  }
  return cached;
}

int occupancy_for(int cpl) {
  switch (cpl) {
    case 1: return blocks_per_sm<1>();
    case 2: return blocks_per_sm<2>();
    case 4: return blocks_per_sm<4>();
    case 8: return blocks_per_sm<8>();
    case 16: return blocks_per_sm<16>();
    default: return blocks_per_sm<32>();
  }
}

template <int CPL>
int launch_cpl(const PassArgs& a, int grid, cudaStream_t s) {
  const size_t smem = pass_smem<CPL>();
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_pass<CPL>)));  // per device
  k_pass<CPL><<<grid, PASS_THREADS, smem, s>>>(a);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

constexpr int TMA_SMEM_BUDGET = 220 * 1024;

// columns per lane for the TMA path: exact multiples of 32 up to 8, then
// powers of two (ragged lanes are predicated off)
int tma_cpl(int64_t n) {
  const int64_t need = (n + 31) / 32;
  if (need <= 8) return static_cast<int>(std::max<int64_t>(1, need));
  if (need <= 16) return 16;
  if (need <= 32) return 32;
  return 64;
}

bool tma_eligible(const PassArgs& a) {
  // bulk copies need 16-byte aligned source rows
  return reinterpret_cast<uintptr_t>(a.A) % 16 == 0 && (a.lda % 2 == 0) && a.n <= 2048;
}

TmaShape tma_shape(int64_t lda, int cpl, int unr, int ncw) {
  TmaShape sh;
  const int64_t row_bytes = lda * 8;
  // ~16 KB (at least UNR rows) per bulk copy
  constexpr int64_t tile_target = 16384;
  int64_t T = std::max<int64_t>(1, (tile_target + row_bytes - 1) / row_bytes);
  T = ((T + unr - 1) / unr) * unr;
  sh.T = static_cast<int>(T);
  sh.stage_bytes = static_cast<int>(align_up(T * row_bytes, 128));
  const int xbytes = cpl > 8 ? 32 * cpl * 8 : 0;
  sh.S = std::min(24, (TMA_SMEM_BUDGET - 1024 - xbytes) / sh.stage_bytes);
  const int red = ncw * 32 * cpl * 8;  // final reduction reuses the ring
  while (sh.S * sh.stage_bytes < red) ++sh.S;
  return sh;
}

size_t tma_smem(const TmaShape& sh, int cpl) {
  return 1024 + (cpl > 8 ? 32 * cpl * 8 : 0) + static_cast<size_t>(sh.S) * sh.stage_bytes;
}

template <int CPL, int UNR, int NCW>
int launch_tma_u(const PassArgs& a0, int grid, cudaStream_t s) {
  PassArgs a = a0;
  const TmaShape sh = tma_shape(a.lda, CPL, UNR, NCW);
  // Row partition depends only on (m, grid) — not on lda or the tile size —
  // so the fixed-order reduction of c is the same for any leading dimension.
  a.rows_per_cta = align_up((a.m + grid - 1) / grid, 4);
  const size_t smem = tma_smem(sh, CPL);
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_pass_tma<CPL, UNR, NCW>)));
  ITSK_CUDA(launch_pdl(reinterpret_cast<const void*>(k_pass_tma<CPL, UNR, NCW>), dim3(grid), dim3(32 * NCW),
                       smem, s, a, sh));
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}


template <int GW, int CPP, bool ODD>
int launch_rows_p(const PassArgs& a0, int grid, cudaStream_t s) {
  constexpr int NG = RW_NCW / GW;
  PassArgs a = a0;
  TmaShape sh;
  sh.T = RW_RB;
  sh.stage_bytes = static_cast<int>(align_up(RW_RB * a.lda * 8, 128));
  // a multiple of NG stages (see the kernel), <= 32 mbarriers, and room for
  // the groups' c partials at the end
  int S = std::min(32, (TMA_SMEM_BUDGET - 1024) / sh.stage_bytes) / NG * NG;
  const int red = NG > 1 ? NG * 2 * 32 * GW * CPP * 8 : 0;
  while (S * sh.stage_bytes < red) S += NG;
  sh.S = std::max(NG, S);
  a.rows_per_cta = align_up((a.m + grid - 1) / grid, 4);
  const size_t smem = 1024 + static_cast<size_t>(sh.S) * sh.stage_bytes;
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_pass_rows<GW, CPP, ODD>)));
  ITSK_CUDA(launch_pdl(reinterpret_cast<const void*>(k_pass_rows<GW, CPP, ODD>), dim3(grid), dim3(32 * RW_NCW),
                       smem, s, a, sh));
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

template <int GW, int CPP>
int launch_rows(const PassArgs& a, int grid, cudaStream_t s) {
  return (a.n & 1) ? launch_rows_p<GW, CPP, true>(a, grid, s) : launch_rows_p<GW, CPP, false>(a, grid, s);
}

template <bool ODD>
int launch_slots_p(const PassArgs& a0, int grid, cudaStream_t s) {
  PassArgs a = a0;
  TmaShape sh;
  sh.T = SL_RB;
  sh.stage_bytes = SL_STAGE;
  sh.S = (TMA_SMEM_BUDGET - 1024 - SL_ROW * 8) / SL_STAGE;  // 3; a stage also holds the slots' c partials at the end
  a.rows_per_cta = align_up((a.m + grid - 1) / grid, 4);
  const size_t smem = 1024 + static_cast<size_t>(sh.S) * SL_STAGE + SL_ROW * 8;  // barriers | ring | x
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_pass_slots<ODD>)));
  ITSK_CUDA(launch_pdl(reinterpret_cast<const void*>(k_pass_slots<ODD>), dim3(grid), dim3(SL_T), smem, s, a, sh));
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

int launch_slots(const PassArgs& a, int grid, cudaStream_t s) {
  return (a.n & 1) ? launch_slots_p<true>(a, grid, s) : launch_slots_p<false>(a, grid, s);
}

template <int CPL>
int launch_tma(const PassArgs& a, int grid, cudaStream_t s) {
  // row groups where the group's 128 GW columns are mostly used (measured:
  // n = 500, 600, 1000, 2000 faster than the warp-per-row kernel; n = 200,
  // 300 slower, profiles/rd2_pass_rows_ab.txt)
  if (a.n > 384) {
    // row slots from n ~ 1400 (short runs, GB/s rows / slots: n = 1280 5024 / 4724, 1536 5223 / 5469,
    // 1792 5915 / 5971, 1920 5982 / 6157; sustained C4 passes under the power cap 10.40 / 10.07 ms)
    if (a.n > 1408) return launch_slots(a, grid, s);
    if (a.n > 1024) return launch_rows<16, 2>(a, grid, s);
    if (a.n > 512) return launch_rows<8, 2>(a, grid, s);
    return launch_rows<4, 2>(a, grid, s);
  }
  if constexpr (CPL <= 16) {
    return launch_tma_u<CPL, 4, 16>(a, grid, s);  // n <= 384: CPL <= 16
  } else {
    set_error("fused pass: no TMA variant for n = %lld", (long long)a.n);
    return ITSK_EINVAL;
  }
}

int tma_grid(int64_t m, int reserve = 0) {
  constexpr int per_sm = 1;
  int64_t g = static_cast<int64_t>(std::max(1, num_sms() - reserve)) * per_sm;
  const int64_t cap = (m + 7) / 8;
  if (g > cap) g = cap;
  return static_cast<int>(std::max<int64_t>(1, g));
}

}  // namespace

int pass_grid_v1(int64_t m, int64_t n) {
  const int cpl = cpl_for(n);
  int64_t g = static_cast<int64_t>(num_sms()) * occupancy_for(std::min(cpl, 32));
  const int64_t cap = (m + PASS_WARPS - 1) / PASS_WARPS;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

int pass_grid(int64_t m, int64_t n) { return std::max(pass_grid_v1(m, n), tma_grid(m)); }

int64_t pass_part_doubles(int64_t m, int64_t n) {
  return static_cast<int64_t>(pass_grid(m, n)) * (n + 4);
}

// rows of more than 1024 columns outside the staged kernels (k_pass_wide)
int launch_wide(PassArgs a, cudaStream_t s, int* grid_used) {
  int grid = num_sms() - a.sm_reserve;
  if (grid < 1) grid = 1;
  if (grid > a.m) grid = static_cast<int>(a.m);
  grid = std::min(grid, pass_grid(a.m, a.n));  // the partials buffer is sized for pass_grid CTAs
  *grid_used = grid;
  a.rows_per_cta = (a.m + grid - 1) / grid;
  if (a.n <= 4 * WIDE_THREADS) k_pass_wide<4><<<grid, WIDE_THREADS, 0, s>>>(a);
  else if (a.n <= 8 * WIDE_THREADS) k_pass_wide<8><<<grid, WIDE_THREADS, 0, s>>>(a);
  else if (a.n <= 16 * WIDE_THREADS) k_pass_wide<16><<<grid, WIDE_THREADS, 0, s>>>(a);
  else {
    set_error("fused pass: n=%lld is beyond the widest row kernel (8192 columns)", (long long)a.n);
    return ITSK_EINVAL;
  }
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

int launch_pass(const PassArgs& a0, cudaStream_t s, int* grid_used) {
  if (tma_eligible(a0)) {
    const int grid = tma_grid(a0.m, a0.sm_reserve);
    *grid_used = grid;
    switch (tma_cpl(a0.n)) {
      case 1: return launch_tma<1>(a0, grid, s);
      case 2: return launch_tma<2>(a0, grid, s);
      case 3: return launch_tma<3>(a0, grid, s);
      case 4: return launch_tma<4>(a0, grid, s);
      case 5: return launch_tma<5>(a0, grid, s);
      case 6: return launch_tma<6>(a0, grid, s);
      case 7: return launch_tma<7>(a0, grid, s);
      case 8: return launch_tma<8>(a0, grid, s);
      case 16: return launch_tma<16>(a0, grid, s);
      case 32: return launch_tma<32>(a0, grid, s);
      default: return launch_tma<64>(a0, grid, s);
    }
  }
  PassArgs a = a0;
  a.tickets = nullptr;  // the LDG variant leaves partials: finalize below when asked
  const int grid = pass_grid_v1(a.m, a.n);
  *grid_used = grid;
  a.rows_per_cta = (a.m + grid - 1) / grid;
  int rc;
  switch (cpl_for(a.n)) {
    case 1: rc = launch_cpl<1>(a, grid, s); break;
    case 2: rc = launch_cpl<2>(a, grid, s); break;
    case 4: rc = launch_cpl<4>(a, grid, s); break;
    case 8: rc = launch_cpl<8>(a, grid, s); break;
    case 16: rc = launch_cpl<16>(a, grid, s); break;
    case 32: rc = launch_cpl<32>(a, grid, s); break;
    default:
      rc = launch_wide(a, s, grid_used);
      break;
  }
  if (rc != ITSK_OK) return rc;
  const int grid_fin = *grid_used;
  if (rc == ITSK_OK && a0.tickets) rc = launch_finalize(a0.part, grid_fin, a0.n, a0.cs, a0.ctl, s);
  if (rc == ITSK_OK && a0.peer.size > 0 && a0.ctl) {
    k_peer_send<<<1, 256, 0, s>>>(a0.cs, a0.n, a0.ctl, a0.mode, a0.peer);
    count_launch();
    ITSK_CHECK_LAUNCH();
  }
  return rc;
}

// Groups of the in-kernel reduction of a loop pass (grid with `reserve` SMs
// left free), or 0 when the pass reduces through k_finalize instead (rows
// not 16-byte aligned, n > 2048): ITSK_LOOP_TAIL_SUMS needs the former.
int pass_tail_groups(const double* A, int64_t m, int64_t n, int64_t lda, int reserve) {
  PassArgs a{};
  a.A = A;
  a.n = n;
  a.lda = lda;
  if (!tma_eligible(a)) return 0;
  const int grid = tma_grid(m, reserve);
  int G = 0;
  pass_groups(m, n, &G);
  return (grid + G - 1) / G;
}

int pass_groups(int64_t m, int64_t n, int* group) {
  const int grid = pass_grid(m, n);
  int G = 1;
  while (G * G < grid) ++G;  // ~sqrt(grid): both levels read ~G partials per column
  if (group) *group = G;
  return (grid + G - 1) / G;
}

int launch_finalize(const double* part, int grid, int64_t n, double* cs, const LoopCtl* ctl,
                    cudaStream_t s) {
  // keep the max shared-memory carveout across the pass / finalize pair:
  // switching the L1/shared split between back-to-back kernels drains SMs
  ITSK_CUDA(func_attr_once(reinterpret_cast<const void*>(k_finalize),
                           cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  const int t = 256;
  k_finalize<<<static_cast<unsigned>(((n + 4) * 32 + t - 1) / t), t, 0, s>>>(part, grid, n, cs, ctl);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace itsk

using namespace itsk;

namespace {
// workspace of the stand-alone pass: partials | group partials | tickets
struct PassWs {
  double* part;
  double* gpart;
  unsigned* tickets;
  int ntickets, group;
  int64_t bytes;
};
PassWs pass_ws(void* ws, int64_t m, int64_t n) {
  Carver cv(ws, 1ll << 62);
  PassWs w;
  w.part = cv.take<double>(pass_part_doubles(m, n));
  const int ng = pass_groups(m, n, &w.group);
  w.gpart = cv.take<double>(static_cast<int64_t>(ng) * (n + 4));
  w.ntickets = ng + 1;
  w.tickets = cv.take<unsigned>(w.ntickets);
  w.bytes = cv.off + 256;
  return w;
}
}  // namespace

extern "C" int itsk_pass_workspace(int64_t m, int64_t n, int64_t* bytes) {
  ITSK_REQUIRE(bytes && m >= 1 && n >= 1, "bad pass shape");
  *bytes = pass_ws(nullptr, m, n).bytes;
  return ITSK_OK;
}

extern "C" int itsk_pass_workspace_init(void* ws, int64_t m, int64_t n, itsk_stream_t stream) {
  ITSK_REQUIRE(ws && m >= 1 && n >= 1, "bad pass shape");
  const PassWs w = pass_ws(ws, m, n);
  ITSK_CUDA(cudaMemsetAsync(w.tickets, 0, sizeof(unsigned) * w.ntickets, reinterpret_cast<cudaStream_t>(stream)));
  return ITSK_OK;
}

extern "C" int itsk_fused_pass(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                               const double* x, const double* r_prev, double* r_out,
                               const double* r_true, double* cs, void* ws, int64_t ws_bytes,
                               itsk_stream_t stream) {
  return itsk_fused_pass_ex(A, m, n, lda, b, 1.0, x, r_prev, r_out, r_true, cs, ws, ws_bytes, 0u, stream);
}

extern "C" int itsk_fused_pass_scaled(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                                      double bscale, const double* x, const double* r_prev, double* r_out,
                                      const double* r_true, double* cs, void* ws, int64_t ws_bytes,
                                      itsk_stream_t stream) {
  return itsk_fused_pass_ex(A, m, n, lda, b, bscale, x, r_prev, r_out, r_true, cs, ws, ws_bytes, 0u, stream);
}

extern "C" int itsk_fused_pass_ex(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                                  double bscale, const double* x, const double* r_prev, double* r_out,
                                  const double* r_true, double* cs, void* ws, int64_t ws_bytes,
                                  unsigned flags, itsk_stream_t stream) {
  ITSK_REQUIRE(A && b && x && cs && ws, "null pointer");
  ITSK_REQUIRE(m >= 1 && n >= 1 && lda >= n, "bad pass shape");
  ITSK_REQUIRE((flags & ~ITSK_PASS_WS_READY) == 0, "unknown pass flags");
  const PassWs w = pass_ws(ws, m, n);
  ITSK_REQUIRE(w.bytes <= ws_bytes, "pass workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PassArgs a{};
  a.A = A;
  a.m = m;
  a.n = n;
  a.lda = lda;
  a.b = b;
  a.x = x;
  a.r_prev = r_prev;
  a.r_out = r_out;
  a.r_true = r_true;
  a.part = w.part;
  a.mode = 0;
  a.bscale = bscale;
  // the same in-kernel reduction as the loop; its counters reset themselves,
  // so only a workspace not known to be initialised is cleared here
  a.tickets = w.tickets;
  a.gpart = w.gpart;
  a.cs = cs;
  a.group = w.group;
  if (!(flags & ITSK_PASS_WS_READY))
    ITSK_CUDA(cudaMemsetAsync(w.tickets, 0, sizeof(unsigned) * w.ntickets, s));
  int grid = 0;
  return launch_pass(a, s, &grid);
}

#ifdef ITSK_TIMELINE
extern "C" void itsk_pass_timeline_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, itsk::g_pass_tl, sizeof(itsk::g_pass_tl));
  unsigned long long z[itsk::TL_SLOTS][4];
  for (int i = 0; i < itsk::TL_SLOTS; ++i) {
    z[i][0] = ~0ull;
    z[i][1] = z[i][2] = z[i][3] = 0;
  }
  cudaMemcpyToSymbol(itsk::g_pass_tl, z, sizeof(z));
}
#endif
