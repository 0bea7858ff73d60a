// Householder QR of the augmented sketch [SA | Sb] (K2), panel / update split.
//
// Same algorithm and conventions as qr.cu (LAPACK dgeqr2 + dlarfb with the
// compact-WY factor of dlarft, dlarfg's beta = -sign(alpha) ||x||;
// /root/reference/pkg/src/itsketch/linalg.py:30-47 via dgeqrf), restructured
// for latency:
//
//   k_qr_panel   one thread-block cluster (<= 16 CTAs) factors the NB-wide
//                panel.  The CTAs' rows of the panel stay in shared memory;
//                each column costs ONE fused sweep over the rows (apply
//                reflector j and accumulate the partial sums of column j+1 in
//                the same pass), one __syncthreads and ONE cluster barrier
//                (each CTA pushes its record into every inbox through
//                distributed shared memory).  The panel ends with G = V'V on
//                DMMA tiles, summed over the cluster in rank order.
//   k_qr_y       Y_s = V_s' W2_s over the trailing columns: (column block x
//                row split) CTAs, cp.async double-buffered row chunks, DMMA.
//   k_qr_z       Z = T'Y without forming T: (T')^{-1} = diag(1/tau) +
//                strict_lower(G'), so z_i = tau_i (y_i - sum_{k<i} G_ki z_k)
//                (tau_i = 0 gives z_i = 0, as dlarft's zero column of T).
//   k_qr_apply   W2 -= V Z on (row block x column block) CTAs, DMMA.
//   k_qr_finish  R with diag(R) >= 0 (linalg.py:43-46) and z = (Q'Sb)[:n].
//
// Every cross-CTA sum runs in a fixed order: R is bitwise reproducible.
#include <cooperative_groups.h>
#include <cuda.h>  // green-context types (entry points fetched through the runtime)

#include <algorithm>
#include <cstdlib>

#include "itsk_common.cuh"
#include "itsk_kernels.cuh"

namespace cg = cooperative_groups;

namespace itsk {
namespace {

constexpr int QP_THREADS = 512;
constexpr int QP_WARPS = QP_THREADS / 32;
constexpr int UT = 64;        // update tile: 64 columns (and 64 rows in k_qr_apply)
constexpr int UTP = UT + 4;   // padded stride
constexpr int YRT = 32;       // row chunk of k_qr_y
constexpr int MAX_SPLIT = 48; // row splits of k_qr_y (partials summed by k_qr_z)
constexpr int MAX_C = 16;     // cluster size bound
constexpr int QP_RPT = 4;     // panel rows per thread bound (rows per CTA <= QP_RPT * QP_THREADS)
constexpr int NB_NEXT2 = 16;  // panel width of the streaming look-ahead (k_qr_next2)

__device__ __forceinline__ int64_t imin64(int64_t x, int64_t y) { return x < y ? x : y; }
__device__ __forceinline__ int64_t lo_of(int q, int P, int64_t len) {
  return (static_cast<int64_t>(q) * len) / P;
}
// D(8x8) += A(8x4) * B(4x8); fragments: a = A[g][t], b = B[t][g],
// d = D[g][2t + {0, 1}], g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int nbytes = valid ? 8 : 0;  // 0: zero-fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(nbytes) : "memory");
}
// 16 bytes, the first `src_bytes` (0, 8 or 16) from global, the rest zero
__device__ __forceinline__ void cp_async16z(double* dst, const double* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Distributed-shared-memory transactions: a remote 8-byte store that
// completes `bytes` on the destination CTA's mbarrier (no cluster barrier).
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(mbar)
               : "memory");
}
// The records land in this CTA's own shared memory (st.async with
// complete_tx on this CTA's mbarrier), so a CTA-scope acquire suffices; a
// cluster-scope acquire also invalidates L1 (CCTL.IVALL) at every column.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// V(r, c) of the panel starting at row k0: unit lower trapezoidal.
__device__ __forceinline__ double vval(double stored, int64_t r, int64_t k0, int c) {
  const int64_t jr = k0 + c;
  return r < jr ? 0.0 : (r == jr ? 1.0 : stored);
}

struct PanelArgs {
  double* W;
  int64_t d, ldw;
  int64_t k0;
  int kb;
  int64_t hmax;
  double* betas;  // global, n: R diagonal before the sign fix
  double* taus;   // global, n
  double* Gp;     // global, MAX_C x NB x NB: per-CTA partial V'V
  double* G;      // global, NB x NB: V'V of this panel
};

#ifdef ITSK_QR2_PROFILE
__device__ unsigned long long g_qr2_prof[12];
#define Q2P(i) do { if (threadIdx.x == 0 && q == 0) { long long _t = clock64(); _qa[i] += _t - _qt; _qt = _t; } } while (0)
#else
#define Q2P(i) do { } while (0)
#endif

template <int NB>
__global__ void __launch_bounds__(QP_THREADS, 1) k_qr_panel(PanelArgs a) {
  constexpr int PS = NB + 1;   // padded row stride (a wider pad would push C4's 1500-row panels out of shared memory)
  constexpr int REC = 2 * NB;  // [partial sums (NB) | owner's next pivot row (NB)]
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), q = static_cast<int>(cl.block_rank());
#ifdef ITSK_QR2_PROFILE
  long long _qt = clock64();
  long long _qa[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = a.k0, ldw = a.ldw;
  const int kb = a.kb;
  const int64_t len = a.d - k0;
  const int64_t lo = k0 + lo_of(q, C, len), hi = k0 + lo_of(q + 1, C, len);
  const int h = static_cast<int>(hi - lo);
  double* Ps = sm;                   // h x PS
  double* inbox = Ps + a.hmax * PS;  // 2 x C x REC (parity-buffered)
  double* red = inbox + 2 * C * REC; // QP_WARPS x NB
  double* taus = red + QP_WARPS * NB;
  double* betl = taus + NB;
  double* gbuf = betl + NB;  // (16 / (NB/8)^2) x NB x NB: G's row-split partials
  __shared__ int bnd[MAX_C + 1];  // row split of [k0, d) relative to k0 (no 64-bit divides later)
  __shared__ __align__(8) uint64_t mb[2];  // record arrivals, one mbarrier per inbox parity
  if (tid <= C) bnd[tid] = static_cast<int>(lo_of(tid, C, len));
  if (tid == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int cl_lane = lane < NB ? lane : NB - 1;  // NB = 16: upper half-warp mirrors

  // the panel's rows, all loads in flight (zero-filled past kb)
  for (int idx = tid; idx < h * NB; idx += QP_THREADS) {
    const int rr = idx / NB, c = idx - rr * NB;
    const bool ok = c < kb;
    cp_async8(Ps + rr * PS + c, a.W + (ok ? (lo + rr) * ldw + k0 + c : 0), ok);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  Q2P(7);

  // NB = 16 (the C4 shape, ~1500 rows per CTA): one sweep per column,
  // thread per row (rows tid, tid + 512, ...: a whole
  // row in one thread, no shuffles in the sweep): apply reflector jj
  // (row[c] += v_r temp_c for c > jj, v_r = row[jj] scal below the pivot, 1
  // on it) and accumulate the partial sums sum_{r > jj+1} a_{r,jj+1} a_{r,c}
  // of the next column in registers; a reduce-scatter across the warp puts
  // column c's warp sum in one lane (fixed order) -> red[warp][c].  Column
  // jj's v values are written back at the next sweep (every thread of the
  // CTA reads row[jj] in this one).  Only columns > jj are read or written.
  const int nrow_iter = (h + QP_THREADS - 1) / QP_THREADS;
  double vsave[QP_RPT];
  int vcol = -1;
  auto flush_v = [&]() {
    if (vcol < 0) return;
#pragma unroll
    for (int k = 0; k < QP_RPT; ++k) {
      const int r = tid + k * QP_THREADS;
      if (k < nrow_iter && r < h && lo + r > k0 + vcol) Ps[r * PS + vcol] = vsave[k];
    }
    vcol = -1;
  };
  __shared__ double s_temp[32];  // temp_c of the current reflector (lanes of warp 0 write it)
  auto sweep_t = [&](int jj, bool apply, double scal) {
    const int jn = jj + 1;
    const int jnc = jn < NB ? jn : 0;
    flush_v();
    double p[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) p[c] = 0.0;
    const int64_t jg = k0 + jj;
#pragma unroll
    for (int k = 0; k < QP_RPT; ++k) {
      const int r = tid + k * QP_THREADS;
      if (k >= nrow_iter || r >= h) break;
      const int64_t rg = lo + r;
      if (rg < jg) continue;  // rows above the pivot: final rows of R
      double* row = Ps + r * PS;
      const bool part = rg > jg + 1;  // below the next pivot
      double v = 1.0;
      if (apply && rg > jg) {
        v = row[jj] * scal;
        vsave[k] = v;
      }
      double xn = 0.0;
      if (jn < kb) {
        xn = row[jnc];
        if (apply) {
          xn = fma(v, s_temp[jnc], xn);
          row[jnc] = xn;
        }
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c < jn || c >= kb) continue;
        double x = xn;
        if (c != jn) {
          x = row[c];
          if (apply) {
            x = fma(v, s_temp[c], x);
            row[c] = x;
          }
        }
        if (part) p[c] = fma(xn, x, p[c]);
      }
    }
    if (apply) vcol = jj;
    Q2P(0);
    if (jn >= kb) return;  // last column: no record to exchange
    // reduce-scatter of p[0..NB) over the warp: halving steps at lane offsets
    // 16, 8, ... (NB = 32: lane l ends with column l; NB = 16: lanes 2c and
    // 2c+1 with column c), one fixed order for every column
    {
#pragma unroll
      for (int st = 0; (16 >> st) >= 32 / NB; ++st) {
        const int o = 16 >> st, half = NB >> (st + 1);
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int i2 = 0; i2 < half; ++i2) {
          const double keep = hi ? p[half + i2] : p[i2];
          const double send = hi ? p[i2] : p[half + i2];
          p[i2] = keep + __shfl_xor_sync(FULL, send, o);
        }
      }
#pragma unroll
      for (int o = 32 / NB / 2; o > 0; o >>= 1) p[0] += __shfl_xor_sync(FULL, p[0], o);
      if ((lane & (32 / NB - 1)) == 0) red[warp * NB + lane / (32 / NB)] = p[0];
    }
    __syncthreads();
    Q2P(1);
    const int buf = jn & 1;
    if (tid == 0)  // this CTA expects C records of (kb - jn) sums plus the owner's row
      mbar_expect_tx(&mb[buf], static_cast<unsigned>((C + 1) * (kb - jn) * 8));
    if (warp < C) {  // warp w delivers this CTA's record to CTA w
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (lane < kb) {
#pragma unroll
        for (int w = 0; w < QP_WARPS; w += 4) {
          s0 += red[w * NB + cl_lane];
          s1 += red[(w + 1) * NB + cl_lane];
          s2 += red[(w + 2) * NB + cl_lane];
          s3 += red[(w + 3) * NB + cl_lane];
        }
      }
      const int64_t jrn = k0 + jn;
      const bool own_next = jrn >= lo && jrn < hi;
      if (lane >= jn && lane < kb) {
        const uint32_t ib = mapa_u32(smem_u32(inbox + (buf * C + q) * REC + lane), warp);
        const uint32_t rb = mapa_u32(smem_u32(&mb[buf]), warp);
        st_async_f64(ib, (s0 + s1) + (s2 + s3), rb);
        if (own_next) st_async_f64(ib + NB * 8, Ps[(jrn - lo) * PS + lane], rb);
      }
    }
    Q2P(2);
    mbar_wait_cluster(&mb[buf], static_cast<unsigned>((jn >> 1) & 1));
    Q2P(3);
  };

  // NB = 32 (C2 / C3 shapes, <= ~600 rows per CTA): warp per row, lane per
  // column — measured faster there than thread per row (a 32-wide row in one
  // thread leaves half the threads idle and serialises the columns).
  // One sweep over the own rows (4 per step): apply reflector jj when `apply`
  // (lane c > jj: a_rc += v_r temp_c; lane jj stores v_r) and accumulate lane
  // c's partial sum_{r > j+1} a_{r,jj+1} a_{r,c} for the next column; then
  // every CTA's record goes to every inbox and the cluster synchronises.
  auto sweep_w = [&](int jj, bool apply, double scal, double temp) {
    const int jn = jj + 1;
    const int jl = static_cast<int>(k0 + jj - lo);  // local index of row j (may be outside [0,h))
    const int jnl = jl + 1;
    // lane predicates are loop-invariant: lanes with temp == 0 rewrite their
    // value unchanged, lanes < jn accumulate partials nobody reads
    const bool l_v = apply && lane == jj;
    const bool l_st = lane < NB;
    const int jsrc = jn < NB ? jn : 0;
    const int jcol = jj < 0 ? 0 : jj;
    double p0 = 0.0, p1 = 0.0;
    // rows j and j+1: updated, not part of the next column's sums
    if (apply) {
#pragma unroll
      for (int sr0 = 0; sr0 < 2; ++sr0) {
        const int sr = jl + sr0;
        if (sr >= 0 && sr < h && (sr & (QP_WARPS - 1)) == warp) {
          double* row = Ps + sr * PS;
          const double v = row[cl_lane];
          const double vr = sr0 == 0 ? 1.0 : row[jcol] * scal;
          double v2 = fma(vr, temp, v);
          if (l_v && sr0 == 1) v2 = vr;
          if (l_st) row[lane] = v2;
        }
      }
    }
    // bulk rows r > j+1 owned by this warp (rr = warp mod QP_WARPS)
    const int start = jnl + 1 > 0 ? jnl + 1 : 0;
    int rr = start + ((warp - start) & (QP_WARPS - 1));
    if (apply) {
      for (; rr + 3 * QP_WARPS < h; rr += 4 * QP_WARPS) {
        double v[4], x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double* row = Ps + (rr + u * QP_WARPS) * PS;
          v[u] = row[cl_lane];
          x[u] = row[jcol];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double vr = x[u] * scal;
          double v2 = fma(vr, temp, v[u]);
          v2 = l_v ? vr : v2;
          if (l_st) Ps[(rr + u * QP_WARPS) * PS + lane] = v2;
          const double xn = __shfl_sync(FULL, v2, jsrc);
          if (u & 1) p1 = fma(xn, v2, p1); else p0 = fma(xn, v2, p0);
        }
      }
      for (; rr < h; rr += QP_WARPS) {
        double* row = Ps + rr * PS;
        const double vr = row[jcol] * scal;
        double v2 = fma(vr, temp, row[cl_lane]);
        v2 = l_v ? vr : v2;
        if (l_st) row[lane] = v2;
        const double xn = __shfl_sync(FULL, v2, jsrc);
        p0 = fma(xn, v2, p0);
      }
    } else {
      for (; rr + 3 * QP_WARPS < h; rr += 4 * QP_WARPS) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double v = Ps[(rr + u * QP_WARPS) * PS + cl_lane];
          const double xn = __shfl_sync(FULL, v, jsrc);
          if (u & 1) p1 = fma(xn, v, p1); else p0 = fma(xn, v, p0);
        }
      }
      for (; rr < h; rr += QP_WARPS) {
        const double v = Ps[rr * PS + cl_lane];
        const double xn = __shfl_sync(FULL, v, jsrc);
        p0 = fma(xn, v, p0);
      }
    }
    Q2P(0);
    if (jn >= kb) return;  // last column: no record to exchange
    if (lane < NB) red[warp * NB + lane] = p0 + p1;
    __syncthreads();
    Q2P(1);
    const int buf = jn & 1;
    if (tid == 0)  // this CTA expects C records of (kb - jn) sums plus the owner's row
      mbar_expect_tx(&mb[buf], static_cast<unsigned>((C + 1) * (kb - jn) * 8));
    if (warp < C) {  // warp w delivers this CTA's record to CTA w
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (lane < kb) {
#pragma unroll
        for (int w = 0; w < QP_WARPS; w += 4) {
          s0 += red[w * NB + lane];
          s1 += red[(w + 1) * NB + lane];
          s2 += red[(w + 2) * NB + lane];
          s3 += red[(w + 3) * NB + lane];
        }
      }
      const int64_t jrn = k0 + jn;
      const bool own_next = jrn >= lo && jrn < hi;
      if (lane >= jn && lane < kb) {
        const uint32_t ib = mapa_u32(smem_u32(inbox + (buf * C + q) * REC + lane), warp);
        const uint32_t rb = mapa_u32(smem_u32(&mb[buf]), warp);
        st_async_f64(ib, (s0 + s1) + (s2 + s3), rb);
        if (own_next) st_async_f64(ib + NB * 8, Ps[(jrn - lo) * PS + lane], rb);
      }
    }
    Q2P(2);
    mbar_wait_cluster(&mb[buf], static_cast<unsigned>((jn >> 1) & 1));
    Q2P(3);
  };

  cl.sync();  // bnd, and every CTA's mbarriers initialised before any remote transaction
  if constexpr (NB == 16) sweep_t(-1, false, 0.0);  // partial sums of column 0
  else sweep_w(-1, false, 0.0, 0.0);
  int own = 0;
  for (int jj = 0; jj < kb; ++jj) {
    const int buf = jj & 1;
    while (own + 1 < C && bnd[own + 1] <= jj) ++own;  // owner of row k0 + jj
    // warp 0 forms the dlarfg coefficients from the inbox (fixed order) and
    // publishes tau, scal and temp_c; the other warps wait at the barrier
    // (sixteen redundant copies of the sqrt/divide chain were slower)
    __shared__ double s_coef[2];
    if (warp == 0) {
      double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0;
      const double* ib = inbox + buf * C * REC + cl_lane;
#pragma unroll
      for (int t = 0; t < MAX_C; t += 4) {
        if (t < C) S0 += ib[t * REC];
        if (t + 1 < C) S1 += ib[(t + 1) * REC];
        if (t + 2 < C) S2 += ib[(t + 2) * REC];
        if (t + 3 < C) S3 += ib[(t + 3) * REC];
      }
      const double S = (S0 + S1) + (S2 + S3);
      const double arow = ib[own * REC + NB];
      const double xn2 = __shfl_sync(FULL, S, jj);
      const double alpha = __shfl_sync(FULL, arow, jj);
      double beta, tau, scal;
      if (xn2 == 0.0) {  // dlarfg: H = I
        tau = 0.0;
        beta = alpha;
        scal = 1.0;
      } else {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      s_temp[lane] = (lane > jj && lane < kb) ? -tau * (arow + scal * S) : 0.0;
      if (lane == 0) {
        taus[jj] = tau;
        betl[jj] = beta;
        s_coef[0] = tau;
        s_coef[1] = scal;
      }
    }
    __syncthreads();
    const double tau = s_coef[0], scal = s_coef[1];
    Q2P(4);
    if constexpr (NB == 16) sweep_t(jj, tau != 0.0, scal);
    else sweep_w(jj, tau != 0.0, scal, s_temp[lane]);
  }
  flush_v();
  __syncthreads();
  Q2P(5);
  // write the panel back (R rows above the diagonal, v below), betas, taus
  for (int idx = tid; idx < h * NB; idx += QP_THREADS) {
    const int rr = idx / NB, c = idx - rr * NB;
    if (c < kb) a.W[(lo + rr) * ldw + k0 + c] = Ps[rr * PS + c];
  }
  if (q == 0)
    for (int c = tid; c < kb; c += QP_THREADS) {
      a.betas[k0 + c] = betl[c];
      a.taus[k0 + c] = taus[c];
    }
  Q2P(8);
  // G_q = V_own' V_own on DMMA tiles, to global: NT = (NB/8)^2 tiles, each
  // over KS = 16 / NT row splits (every warp busy; 4 interleaved chains per
  // warp), the splits summed in a fixed order through shared memory
  {
    constexpr int GT = NB / 8, NT = GT * GT, KS = QP_WARPS / NT;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int tile = warp % NT, ks = warp / NT;
    const int mt = tile / GT, nt = tile - mt * GT;
    const int ci = mt * 8 + g4, ck = nt * 8 + g4;
    const int groups = (h + 3) / 4;
    const int gb0 = (ks * groups) / KS * 4, gb1 = min(h, ((ks + 1) * groups) / KS * 4);
    double e0[4] = {0.0, 0.0, 0.0, 0.0}, e1[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r0 = gb0; r0 < gb1; r0 += 16) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + 4 * u + t4;
        const bool ok = r < gb1;
        const double av = ok ? vval(Ps[r * PS + ci], lo + r, k0, ci) : 0.0;
        const double bv = ok ? vval(Ps[r * PS + ck], lo + r, k0, ck) : 0.0;
        dmma(e0[u], e1[u], av, bv);
      }
    }
    const double g0 = (e0[0] + e0[1]) + (e0[2] + e0[3]);
    const double g1 = (e1[0] + e1[1]) + (e1[2] + e1[3]);
    double* gp = a.Gp + static_cast<int64_t>(q) * NB * NB;
    if constexpr (KS == 1) {
      gp[ci * NB + nt * 8 + 2 * t4] = g0;
      gp[ci * NB + nt * 8 + 2 * t4 + 1] = g1;
    } else {
      double* gb = gbuf + ks * NB * NB;
      gb[ci * NB + nt * 8 + 2 * t4] = g0;
      gb[ci * NB + nt * 8 + 2 * t4 + 1] = g1;
      __syncthreads();
      for (int e = tid; e < NB * NB; e += QP_THREADS) {
        double sum = 0.0;
#pragma unroll
        for (int k = 0; k < KS; ++k) sum += gbuf[k * NB * NB + e];
        gp[e] = sum;
      }
    }
  }
  Q2P(9);
  cl.sync();
  Q2P(10);
  // G = sum_t G_t in rank order; element e summed by CTA e % C (all C
  // partial loads in flight before the adds: one L2 round trip, not C)
  for (int e = q + C * tid; e < NB * NB; e += C * QP_THREADS) {
    double v[MAX_C];
#pragma unroll
    for (int t = 0; t < MAX_C; ++t) v[t] = t < C ? __ldcg(a.Gp + static_cast<int64_t>(t) * NB * NB + e) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < MAX_C; ++t)
      if (t < C) s += v[t];
    a.G[e] = s;
  }
  Q2P(6);
#ifdef ITSK_QR2_PROFILE
  if (threadIdx.x == 0 && q == 0)
    for (int i = 0; i < 12; ++i) atomicAdd(&g_qr2_prof[i], static_cast<unsigned long long>(_qa[i]));
#endif
}

struct UpdArgs {
  double* W;
  int64_t d, ldw, k0;
  int kb;
  int64_t c0, Nt;     // trailing columns [c0, c0 + Nt)
  double* Yp;         // S x NB x ldy partial Y
  double* Z;          // NB x ldy
  int64_t ldy;
  int S;
  const double* G;    // NB x NB
  const double* taus; // global, indexed k0 + i
};

// Y_s = V_s' W2_s  (M = NB reflectors, N = UT columns, K = rows of split s)
template <int NB>
__global__ void __launch_bounds__(256) k_qr_y(UpdArgs a) {
  constexpr int MT = NB / 8, NT = UT / 8;
  constexpr int TPW = (MT * NT + 7) / 8;  // tiles per warp (8 warps)
  constexpr int VS = NB + 4;              // strides = 4 mod 16: conflict-free DMMA fragments
  constexpr int WS = UT + 4;
  extern __shared__ __align__(16) double ysm[];
  double* Vt = ysm;                  // 2 x YRT x VS
  double* Wt = Vt + 2 * YRT * VS;    // 2 x YRT x WS
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int64_t cb = static_cast<int64_t>(blockIdx.x) * UT;
  const int cw = static_cast<int>(imin64(UT, a.Nt - cb));
  const int64_t len = a.d - a.k0;
  const int64_t rlo = a.k0 + lo_of(blockIdx.y, a.S, len), rhi = a.k0 + lo_of(blockIdx.y + 1, a.S, len);
  const int nchunks = static_cast<int>((rhi - rlo + YRT - 1) / YRT);
  auto load = [&](int ch, int st) {
    const int64_t r0 = rlo + static_cast<int64_t>(ch) * YRT;
    double* vt = Vt + st * YRT * VS;
    double* wt = Wt + st * YRT * WS;
    for (int idx = tid; idx < YRT * NB; idx += 256) {
      const int rr = idx / NB, c = idx - rr * NB;
      const int64_t r = r0 + rr;
      const bool ok = r < rhi && c < a.kb;
      cp_async8(vt + rr * VS + c, a.W + (ok ? r * a.ldw + a.k0 + c : 0), ok);
    }
    for (int idx = tid; idx < YRT * UT; idx += 256) {
      const int rr = idx / UT, c = idx - rr * UT;
      const int64_t r = r0 + rr;
      const bool ok = r < rhi && c < cw;
      cp_async8(wt + rr * WS + c, a.W + (ok ? r * a.ldw + a.c0 + cb + c : 0), ok);
    }
    cp_commit();
  };
  double d0[TPW], d1[TPW];
#pragma unroll
  for (int u = 0; u < TPW; ++u) d0[u] = d1[u] = 0.0;
  if (nchunks > 0) load(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch & 1;
    if (ch + 1 < nchunks) {
      load(ch + 1, st ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int64_t r0 = rlo + static_cast<int64_t>(ch) * YRT;
    const double* vt = Vt + st * YRT * VS;
    const double* wt = Wt + st * YRT * WS;
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      const int T = warp * TPW + u;
      if (T < MT * NT) {
        const int mt = T / NT, nt = T - mt * NT;
        const int ci = mt * 8 + g4;
#pragma unroll
        for (int k = 0; k < YRT; k += 4) {
          const double av = vval(vt[(k + t4) * VS + ci], r0 + k + t4, a.k0, ci);
          dmma(d0[u], d1[u], av, wt[(k + t4) * WS + nt * 8 + g4]);
        }
      }
    }
    __syncthreads();  // stage st is refilled by the next iteration's load
  }
  double* Y = a.Yp + static_cast<int64_t>(blockIdx.y) * NB * a.ldy;
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int T = warp * TPW + u;
    if (T < MT * NT) {
      const int mt = T / NT, nt = T - mt * NT;
      const int i = mt * 8 + g4, c = nt * 8 + t4 * 2;
      if (c < cw) Y[i * a.ldy + cb + c] = d0[u];
      if (c + 1 < cw) Y[i * a.ldy + cb + c + 1] = d1[u];
    }
  }
}

// Z = T' sum_s Y_s for UT columns: z_i = tau_i (y_i - sum_{k<i} G_ki z_k)
template <int NB>
__global__ void __launch_bounds__(256) k_qr_z(UpdArgs a) {
  __shared__ double Ys[NB][UT + 1];
  __shared__ double Gs[NB][NB + 1];
  __shared__ double ts[NB];
  const int tid = threadIdx.x;
  const int64_t cb = static_cast<int64_t>(blockIdx.x) * UT;
  const int cw = static_cast<int>(imin64(UT, a.Nt - cb));
  for (int idx = tid; idx < NB * UT; idx += 256) {
    const int i = idx / UT, c = idx - i * UT;
    double s = 0.0;
    if (i < a.kb && c < cw) {
      // all S partial loads in flight at once, summed in split order
      const double* yp = a.Yp + static_cast<int64_t>(i) * a.ldy + cb + c;
      const int64_t stride = static_cast<int64_t>(NB) * a.ldy;
      double v[MAX_SPLIT];
#pragma unroll
      for (int sp = 0; sp < MAX_SPLIT; ++sp) v[sp] = sp < a.S ? yp[sp * stride] : 0.0;
#pragma unroll
      for (int sp = 0; sp < MAX_SPLIT; ++sp) s += v[sp];
    }
    Ys[i][c] = s;
  }
  for (int idx = tid; idx < NB * NB; idx += 256) Gs[idx / NB][idx % NB] = a.G[idx];
  if (tid < NB) ts[tid] = tid < a.kb ? a.taus[a.k0 + tid] : 0.0;
  __syncthreads();
  if (tid < cw) {
    const int c = tid;
    for (int i = 0; i < a.kb; ++i) {
      double s0 = 0.0, s1 = 0.0;
      int k = 0;
      for (; k + 1 < i; k += 2) {
        s0 = fma(Gs[k][i], Ys[k][c], s0);
        s1 = fma(Gs[k + 1][i], Ys[k + 1][c], s1);
      }
      if (k < i) s0 = fma(Gs[k][i], Ys[k][c], s0);
      Ys[i][c] = ts[i] * (Ys[i][c] - (s0 + s1));  // row i of Z overwrites row i of Y
    }
    for (int i = 0; i < a.kb; ++i) a.Z[i * a.ldy + cb + c] = Ys[i][c];
  }
}

// W2 -= V Z on a 64-row x 64-column tile
template <int NB>
__global__ void __launch_bounds__(256) k_qr_apply(UpdArgs a) {
  constexpr int NT = UT / 8;  // 64 output tiles, 8 per warp
  __shared__ double Zs[NB][UTP];
  __shared__ double Vs[UT][NB + 4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int64_t r0 = a.k0 + static_cast<int64_t>(blockIdx.x) * UT;
  const int rh = static_cast<int>(imin64(UT, a.d - r0));
  const int64_t cb = static_cast<int64_t>(blockIdx.y) * UT;
  const int cw = static_cast<int>(imin64(UT, a.Nt - cb));
  for (int idx = tid; idx < NB * UT; idx += 256) {
    const int i = idx / UT, c = idx - i * UT;
    Zs[i][c] = (i < a.kb && c < cw) ? a.Z[i * a.ldy + cb + c] : 0.0;
  }
  for (int idx = tid; idx < UT * NB; idx += 256) {
    const int rr = idx / NB, c = idx - rr * NB;
    const int64_t r = r0 + rr;
    Vs[rr][c] = (rr < rh && c < a.kb) ? vval(a.W[r * a.ldw + a.k0 + c], r, a.k0, c) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int T = warp * 8 + u;
    const int mt = T / NT, nt = T - mt * NT;
    const int rr = mt * 8 + g4, c = nt * 8 + t4 * 2;
    double* wp = a.W + (r0 + rr) * a.ldw + a.c0 + cb + c;
    const bool rok = rr < rh;
    double d0 = (rok && c < cw) ? wp[0] : 0.0;
    double d1 = (rok && c + 1 < cw) ? wp[1] : 0.0;
#pragma unroll
    for (int k = 0; k < NB; k += 4) dmma(d0, d1, -Vs[mt * 8 + g4][k + t4], Zs[k + t4][nt * 8 + g4]);
    if (rok) {
      if (c < cw) wp[0] = d0;
      if (c + 1 < cw) wp[1] = d1;
    }
  }
}

// Look-ahead update of the NEXT panel's columns [c0, c0 + nb2) by the
// panel just factored, in one cluster launch (the same row split as
// k_qr_panel): each CTA stages its rows of V and of the block, forms its
// partial Y = V'W2 on DMMA tiles, the partials are summed through distributed
// shared memory in rank order (every CTA redundantly, so all hold the same
// Y), Z = T'Y by substitution with G and tau, and W2 -= V Z.  The rest of
// the trailing matrix is updated by k_qr_y / k_qr_z / k_qr_apply on a side
// stream while the next panel is factored.
#ifdef ITSK_QRNEXT_PROBE
__device__ unsigned long long g_qn_prof[8];
#define QNP(i) do { if (threadIdx.x == 0 && q == 0) { long long _t = clock64(); atomicAdd(&g_qn_prof[i], (unsigned long long)(_t - _qt)); _qt = _t; } } while (0)
#else
#define QNP(i) do { } while (0)
#endif

// DMMA fragments read a[g][t] / b[t][g] from row-major shared tiles: a row
// stride = 4 (mod 16) doubles puts the 16 lanes of each half-warp (g, t in
// 0..3) on 16 distinct 8-byte banks (a +1 pad gives 4-way conflicts).
template <int NB>
__global__ void __launch_bounds__(QP_THREADS, 1) k_qr_next(UpdArgs a, int64_t hmax) {
  constexpr int VS = NB + 4, BS = 36;
#ifdef ITSK_QRNEXT_PROBE
  long long _qt = clock64();
#endif
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), q = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int64_t k0 = a.k0, ldw = a.ldw;
  const int64_t len = a.d - k0;
  const int64_t lo = k0 + lo_of(q, C, len), hi = k0 + lo_of(q + 1, C, len);
  const int h = static_cast<int>(hi - lo);
  const int hp = (h + 7) & ~7;
  const int hz = (h + 15) & ~15;           // rows staged (zero-filled past h)
  const int nb2 = static_cast<int>(a.Nt);  // <= 32
  double* Vs = sm;                      // (hmax + 16) x VS
  double* Bs = Vs + (hmax + 16) * VS;   // (hmax + 16) x BS
  double* Yq = Bs + (hmax + 16) * BS;   // 32 x BS: this CTA's partial
  double* Ys = Yq + 32 * BS;            // 32 x BS: the sum, then Z
  double* Gs = Ys + 32 * BS;            // NB x VS
  double* ts = Gs + NB * VS;            // NB
  double* Yo = ts + NB;                 // NB x 32: the elements this CTA owns, summed
  // rows staged with cp.async (all loads in flight; zero-fill past h / kb /
  // nb2), then V's unit lower trapezoid fixed up on the rows k0 .. k0+kb-1
  for (int idx = tid; idx < hz * 32; idx += QP_THREADS) {
    const int rr = idx >> 5, c = idx & 31;
    const int64_t r = lo + rr;
    if (c < NB) {
      const bool ok = rr < h && c < a.kb;
      cp_async8(Vs + rr * VS + c, a.W + (ok ? r * ldw + k0 + c : 0), ok);
    }
    const bool okb = rr < h && c < nb2;
    cp_async8(Bs + rr * BS + c, a.W + (okb ? r * ldw + a.c0 + c : 0), okb);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  if (lo < k0 + a.kb)
    for (int idx = tid; idx < NB * NB; idx += QP_THREADS) {
      const int rr = idx / NB, c = idx - rr * NB;
      const int64_t r = lo + rr;
      if (rr < h && c < a.kb && r <= k0 + c) Vs[rr * VS + c] = (r == k0 + c) ? 1.0 : 0.0;
    }
  for (int idx = tid; idx < NB * NB; idx += QP_THREADS) Gs[(idx / NB) * VS + idx % NB] = a.G[idx];
  if (tid < NB) ts[tid] = tid < a.kb ? a.taus[k0 + tid] : 0.0;
  __syncthreads();
  QNP(0);
  // partial Y (NB x 32): warp -> 8x8 tile (NB/8 x 4 tiles over 16 warps);
  // the row sum runs in 4 interleaved DMMA chains (a dependent DMMA costs
  // ~300 cycles: one chain over all rows was most of this kernel's time)
  constexpr int MT = NB / 8;
  if (warp < MT * 4) {
    const int mt = warp >> 2, nt = warp & 3;
    double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
    const int hp16 = (hp + 15) & ~15;  // rows beyond hp are zero-filled below
    for (int k = 0; k < hp16; k += 16) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k + 4 * u + t4;
        dmma(d0[u], d1[u], Vs[kk * VS + mt * 8 + g4], Bs[kk * BS + nt * 8 + g4]);
      }
    }
    Yq[(mt * 8 + g4) * BS + nt * 8 + 2 * t4] = (d0[0] + d0[1]) + (d0[2] + d0[3]);
    Yq[(mt * 8 + g4) * BS + nt * 8 + 2 * t4 + 1] = (d1[0] + d1[1]) + (d1[2] + d1[3]);
  }
  QNP(1);
  cl.sync();
  QNP(5);
  // sum of the C partials in rank order: reduce-scatter (CTA q sums the
  // elements e = q (mod C) over all ranks, all remote loads in flight), then
  // all-gather from the owners
  for (int e = q + C * tid; e < NB * 32; e += C * QP_THREADS) {
    const uint32_t la = smem_u32(Yq + (e >> 5) * BS + (e & 31));
    double v[MAX_C];
#pragma unroll
    for (int t = 0; t < MAX_C; ++t) {
      v[t] = 0.0;
      if (t < C) asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v[t]) : "r"(mapa_u32(la, t)) : "memory");
    }
    double sum = 0.0;
#pragma unroll
    for (int t = 0; t < MAX_C; ++t)
      if (t < C) sum += v[t];
    Yo[e] = sum;
  }
  cl.sync();
  for (int e = tid; e < NB * 32; e += QP_THREADS) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(mapa_u32(smem_u32(Yo + e), e % C)) : "memory");
    Ys[(e >> 5) * BS + (e & 31)] = v;
  }
  __syncthreads();
  QNP(2);
  // Z = T'Y: z_i = tau_i (y_i - sum_{k<i} G_ki z_k).  Warp per column, lane
  // j carries t_j = y_j - sum_{k<i} G_kj z_k; step i: z_i = tau_i t_i (lane
  // i), broadcast, lanes j > i subtract G_ij z_i.
  // two columns per warp, their chains interleaved
  // lane j's column of G and its tau in registers: the chain is shuffle +
  // FMA only (the same products: lane i forms tau_i t_i)
  double gcol[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) gcol[i] = Gs[i * VS + (lane < NB ? lane : 0)];
  const double mytau = ts[lane < NB ? lane : 0];
  for (int c = warp; c < nb2; c += 2 * QP_WARPS) {
    const int c2 = c + QP_WARPS;
    const bool two = c2 < nb2;
    double t = lane < a.kb ? Ys[lane * BS + c] : 0.0;
    double u = (two && lane < a.kb) ? Ys[lane * BS + c2] : 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (i >= a.kb) break;
      const double g = gcol[i];
      const double zi = __shfl_sync(FULL, mytau * t, i);
      const double wi = __shfl_sync(FULL, mytau * u, i);
      if (lane == i) {
        t = zi;
        u = wi;
      } else if (lane > i) {
        t = fma(-g, zi, t);
        u = fma(-g, wi, u);
      }
    }
    Ys[lane * BS + c] = lane < a.kb ? t : 0.0;
    if (two) Ys[lane * BS + c2] = lane < a.kb ? u : 0.0;
  }
  __syncthreads();
  QNP(3);
  // W2 -= V Z: (hp/8) x 4 tiles of 8x8; a warp's tiles advance together
  // through k so their DMMA chains interleave
  const int ntile = (hp >> 3) * 4;
  constexpr int TW = 8;  // tiles per warp per round
  for (int T0 = warp * TW; T0 < ntile; T0 += QP_WARPS * TW) {
    double d0[TW], d1[TW];
#pragma unroll
    for (int u = 0; u < TW; ++u) {
      const int T = T0 + u;
      const int rr = (T >> 2) * 8 + g4, c = (T & 3) * 8 + 2 * t4;
      d0[u] = T < ntile ? Bs[rr * BS + c] : 0.0;
      d1[u] = T < ntile ? Bs[rr * BS + c + 1] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NB; k += 4) {
#pragma unroll
      for (int u = 0; u < TW; ++u) {
        const int T = T0 + u < ntile ? T0 + u : 0;
        const int rr = (T >> 2) * 8 + g4;
        dmma(d0[u], d1[u], -Vs[rr * VS + k + t4], Ys[(k + t4) * BS + (T & 3) * 8 + g4]);
      }
    }
#pragma unroll
    for (int u = 0; u < TW; ++u) {
      const int T = T0 + u;
      const int rr = (T >> 2) * 8 + g4, c = (T & 3) * 8 + 2 * t4;
      if (T < ntile && rr < h) {
        double* wp = a.W + (lo + rr) * ldw + a.c0 + c;
        if (c < nb2) wp[0] = d0[u];
        if (c + 1 < nb2) wp[1] = d1[u];
      }
    }
  }
  cl.sync();  // no CTA exits while another may still read its Yo
  QNP(4);
}

// Streaming look-ahead (16-wide panels at C4 sizes, where k_qr_next's
// whole-slice staging does not fit): the same update of the next panel's
// nb2 <= NB columns by the panel just factored, in one cluster launch with
// the panel's row split, but the CTA's rows pass through a double-buffered
// cp.async ring of NX_RC-row chunks twice: pass 1 accumulates the partial
// Y = V'B on DMMA tiles (16 warps = 4 tiles x 4 row slices, 4 interleaved
// chains each, the slices summed in a fixed order), the partials are summed
// over the cluster in rank order (DSMEM), Z = T'Y by substitution with G and
// tau; pass 2 re-streams the chunks and stores B - V Z.  V and B are
// L2-resident (just written by the panel and the previous updates).
constexpr int NX_RC = 128;   // rows per chunk
constexpr int NX_ST = 4;     // ring stages (3 chunks, ~120 KB, in flight per SM)
constexpr int NX_S = NB_NEXT2 + 4;

template <int NB>
__global__ void __launch_bounds__(QP_THREADS, 1) k_qr_next2(UpdArgs a) {
  static_assert(NB == NB_NEXT2, "k_qr_next2 is instantiated for 16-wide panels");
  extern __shared__ __align__(16) double sm[];
#ifdef ITSK_QRNEXT_PROBE
  long long _qt = clock64();
#endif
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), q = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int64_t k0 = a.k0, ldw = a.ldw;
  const int64_t len = a.d - k0;
  const int64_t lo = k0 + lo_of(q, C, len), hi = k0 + lo_of(q + 1, C, len);
  const int h = static_cast<int>(hi - lo);
  const int nb2 = static_cast<int>(a.Nt);
  const int kb = a.kb;
  double* Vs = sm;                          // NX_ST x NX_RC x NX_S
  double* Bs = Vs + NX_ST * NX_RC * NX_S;   // NX_ST x NX_RC x NX_S
  double* Yk = Bs + NX_ST * NX_RC * NX_S;   // 4 slices x NB x NB
  double* Yq = Yk + 4 * NB * NB;            // NB x NB: this CTA's partial
  double* Ys = Yq + NB * NB;                // NB x NB: the sum, then Z
  double* Yo = Ys + NB * NB;                // NB x NB: elements this CTA owns, summed
  const int nch = (h + NX_RC - 1) / NX_RC;
  // 16-byte copies where W's rows are 16-byte aligned (even ldw; k0, c0 are
  // multiples of 16), a partial pair zero-filled by the source size
  const bool vec16 = (ldw & 1) == 0 && (reinterpret_cast<uintptr_t>(a.W) & 15) == 0;
  auto load = [&](int ch) {
    const int st = ch % NX_ST;
    double* vs = Vs + st * NX_RC * NX_S;
    double* bs = Bs + st * NX_RC * NX_S;
    const int r0 = ch * NX_RC;
    if (vec16) {
      for (int idx = tid; idx < NX_RC * (NB / 2); idx += QP_THREADS) {
        const int rr = idx / (NB / 2), c = 2 * (idx - rr * (NB / 2));
        const int64_t r = lo + r0 + rr;
        const bool rok = r0 + rr < h;
        const int sv = rok ? 8 * max(0, min(2, kb - c)) : 0;
        const int sb = rok ? 8 * max(0, min(2, nb2 - c)) : 0;
        cp_async16z(vs + rr * NX_S + c, a.W + (sv ? r * ldw + k0 + c : 0), sv);
        cp_async16z(bs + rr * NX_S + c, a.W + (sb ? r * ldw + a.c0 + c : 0), sb);
      }
      return;
    }
    for (int idx = tid; idx < NX_RC * NB; idx += QP_THREADS) {
      const int rr = idx / NB, c = idx - rr * NB;
      const int64_t r = lo + r0 + rr;
      const bool okv = r0 + rr < h && c < kb;
      cp_async8(vs + rr * NX_S + c, a.W + (okv ? r * ldw + k0 + c : 0), okv);
      const bool okb = r0 + rr < h && c < nb2;
      cp_async8(bs + rr * NX_S + c, a.W + (okb ? r * ldw + a.c0 + c : 0), okb);
    }
  };
  // V(r, c) with the unit-diagonal fix (rows of the panel's top triangle)
  auto vfix = [&](double v, int64_t r, int c) { return vval(v, r, k0, c); };
  // ---- pass 1: Y partial ----
  const int tile = warp & 3, slice = warp >> 2;  // 4 tiles (NB/8)^2, 4 row slices of each chunk
  const int mt = tile >> 1, nt = tile & 1;
  double e0[4] = {0.0, 0.0, 0.0, 0.0}, e1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int ch = 0; ch < NX_ST - 1; ++ch) {
    if (ch < nch) load(ch);
    cp_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    cp_wait<NX_ST - 2>();
    __syncthreads();
    if (ch + NX_ST - 1 < nch) load(ch + NX_ST - 1);
    cp_commit();
    const int st = ch % NX_ST;
    const double* vs = Vs + st * NX_RC * NX_S;
    const double* bs = Bs + st * NX_RC * NX_S;
    const int r0 = ch * NX_RC;
    // slice `slice` takes rows [slice * 32, slice * 32 + 32) of the chunk
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const int rr = slice * 32 + u * 8 + kk + t4;
        const int64_t r = lo + r0 + rr;
        const double av = vfix(vs[rr * NX_S + mt * 8 + g4], r, mt * 8 + g4);
        const double bv = bs[rr * NX_S + nt * 8 + g4];
        dmma(e0[u], e1[u], av, bv);
      }
    }
  }
  cp_wait<0>();
  __syncthreads();
  QNP(0);
  {
    double* yk = Yk + slice * NB * NB;
    yk[(mt * 8 + g4) * NB + nt * 8 + 2 * t4] = (e0[0] + e0[1]) + (e0[2] + e0[3]);
    yk[(mt * 8 + g4) * NB + nt * 8 + 2 * t4 + 1] = (e1[0] + e1[1]) + (e1[2] + e1[3]);
  }
  __syncthreads();
  for (int e = tid; e < NB * NB; e += QP_THREADS)
    Yq[e] = (Yk[e] + Yk[NB * NB + e]) + (Yk[2 * NB * NB + e] + Yk[3 * NB * NB + e]);
  cl.sync();
  QNP(1);
  // the C partials summed in rank order: CTA q sums the elements e = q mod C
  // over all ranks, then every CTA gathers the owners' sums
  for (int e = q + C * tid; e < NB * NB; e += C * QP_THREADS) {
    const uint32_t la = smem_u32(Yq + e);
    double v[MAX_C];
#pragma unroll
    for (int t = 0; t < MAX_C; ++t) {
      v[t] = 0.0;
      if (t < C) asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v[t]) : "r"(mapa_u32(la, t)) : "memory");
    }
    double sum = 0.0;
#pragma unroll
    for (int t = 0; t < MAX_C; ++t)
      if (t < C) sum += v[t];
    Yo[e] = sum;
  }
  cl.sync();
  for (int e = tid; e < NB * NB; e += QP_THREADS) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(mapa_u32(smem_u32(Yo + e), e % C)) : "memory");
    Ys[e] = v;
  }
  __syncthreads();
  QNP(2);
  // Z = T'Y: warp c < nb2 handles column c; lane j carries t_j
  if (warp < nb2) {
    const int c = warp;
    const int jl = lane < NB ? lane : 0;
    double t = lane < kb ? Ys[jl * NB + c] : 0.0;
    const double mytau = lane < kb ? a.taus[k0 + jl] : 0.0;
    // lane j's column of G in registers, all loads in flight before the chain
    double gcol[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) gcol[i] = a.G[i * NB + jl];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (i >= kb) break;
      const double g = gcol[i];
      const double zi = __shfl_sync(FULL, mytau * t, i);
      if (lane == i) t = zi;
      else if (lane > i) t = fma(-g, zi, t);
    }
    __syncwarp();
    if (lane < NB) Ys[jl * NB + c] = lane < kb ? t : 0.0;
  }
  __syncthreads();
  QNP(3);
  // ---- pass 2: B -= V Z, chunk by chunk ----
#pragma unroll
  for (int ch = 0; ch < NX_ST - 1; ++ch) {
    if (ch < nch) load(ch);
    cp_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    cp_wait<NX_ST - 2>();
    __syncthreads();
    if (ch + NX_ST - 1 < nch) load(ch + NX_ST - 1);
    cp_commit();
    const int st = ch % NX_ST;
    const double* vs = Vs + st * NX_RC * NX_S;
    const double* bs = Bs + st * NX_RC * NX_S;
    const int r0 = ch * NX_RC;
    // NX_RC x NB output = (NX_RC / 8) x 2 tiles of 8x8: one row tile per warp, both column tiles
    {
      const int rt = warp;  // 16 warps x 8 rows = NX_RC
      const int rr = rt * 8 + g4;
      const int64_t r = lo + r0 + rr;
      double d[2][2];
#pragma unroll
      for (int ct = 0; ct < 2; ++ct) {
        d[ct][0] = bs[rr * NX_S + ct * 8 + 2 * t4];
        d[ct][1] = bs[rr * NX_S + ct * 8 + 2 * t4 + 1];
      }
#pragma unroll
      for (int k = 0; k < NB; k += 4) {
        const int rk = rt * 8 + g4;
        const double av = -vfix(vs[rk * NX_S + k + t4], lo + r0 + rk, k + t4);
#pragma unroll
        for (int ct = 0; ct < 2; ++ct) dmma(d[ct][0], d[ct][1], av, Ys[(k + t4) * NB + ct * 8 + g4]);
      }
      if (r0 + rr < h) {
#pragma unroll
        for (int ct = 0; ct < 2; ++ct) {
          const int c = ct * 8 + 2 * t4;
          double* wp = a.W + r * ldw + a.c0 + c;
          if (c < nb2) wp[0] = d[ct][0];
          if (c + 1 < nb2) wp[1] = d[ct][1];
        }
      }
    }
  }
  cp_wait<0>();
  QNP(4);
  cl.sync();  // no CTA exits while another may still read its Yo
  QNP(5);
}

size_t next2_smem() {
  return static_cast<size_t>(2 * NX_ST * NX_RC * NX_S + 4 * NB_NEXT2 * NB_NEXT2 + 3 * NB_NEXT2 * NB_NEXT2) * 8;
}

size_t next_smem(int64_t hmax, int nb) {
  return static_cast<size_t>((hmax + 16) * (nb + 4) + (hmax + 16) * 36 + 2 * 32 * 36 + nb * (nb + 4) + nb +
                             nb * 32) * 8;
}

// R (sign-fixed upper triangle) and z = sign-fixed Q'Sb (linalg.py:43-46).
__global__ void k_qr_finish(const double* W, int64_t n, int64_t ldw, int64_t N, const double* betas,
                            double* R, double* z, int* singular) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int64_t i = e / n, c = e - i * n;
  const double bi = betas[i];
  const double sg = bi < 0.0 ? -1.0 : 1.0;
  const double rv = (c < i) ? 0.0 : (c == i ? sg * bi : sg * W[i * ldw + c]);
  R[e] = rv;
  // bit 1: a non-finite entry of R or z — the reference's triangular solves
  // refuse those (scipy solve_triangular's check_finite, linalg.py:59-68)
  bool bad = !isfinite(rv);
  if (c == 0) {
    if (z && N > n) {
      const double zv = sg * W[i * ldw + n];
      z[i] = zv;
      bad = bad || !isfinite(zv);
    }
    if (bi == 0.0) atomicOr(singular, 1);
  }
  if (bad) atomicOr(singular, 2);
}

// Side stream and events of the look-ahead (per device, created once).
bool lookahead_enabled() { return true; }

// Side streams (per device, created once): 0 = the look-ahead's rest of the
// trailing matrix, 1 = the far updates, 2 = the critical path (panels, their
// block updates, the next block's far update) at the highest priority, so
// the panel chain's CTAs are scheduled ahead of the overlapping far GEMMs.
int side_stream(cudaStream_t* out, int which = 0) {
  static cudaStream_t st[64][3] = {};
  int dev = 0;
  ITSK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || which < 0 || which > 2) return ITSK_EINVAL;
  if (!st[dev][which]) {
    int lo = 0, hi = 0;
    ITSK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ITSK_CUDA(cudaStreamCreateWithPriority(&st[dev][which], cudaStreamNonBlocking, which == 2 ? hi : lo));
  }
  *out = st[dev][which];
  return ITSK_OK;
}

// SM partition of the two-level QR (green contexts): the panel chain (one
// 16-CTA cluster at a time, ~200 KB of shared memory per CTA, and the
// one-CTA T recurrence) on a partition of QG_SMS SMs, every GEMM-shaped
// update on the rest.  Sharing all SMs, the chain's big-CTA kernels waited
// for SMs to drain of the far GEMMs' CTAs (up to ~0.5 ms per outer block).
// The partition changes no operation order (splits follow the device's SM
// count): results are bitwise the same with it or without (ITSK_QR_GREEN=0).
constexpr unsigned QG_SMS = 16;
struct QrGreen {
  bool ok = false;
  cudaStream_t chain = nullptr;  // the panel chain (highest priority)
  cudaStream_t upd = nullptr;    // the outer block's Gram / near update (highest priority)
  cudaStream_t side = nullptr;   // the look-ahead's rest of the block (highest priority: the next
                                 // panel's look-ahead waits for it)
  cudaStream_t far = nullptr;    // the far rest (lowest priority: due a block later)
  cudaStream_t nearY = nullptr;  // the near update's Y = V'W, beside the Gram and T (highest priority)
};

QrGreen make_qr_green(int dev) {
  QrGreen g;
  auto entry = [](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPointByVersion(name, fn, CUDART_VERSION, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess && *fn != nullptr;
  };
  decltype(&cuDeviceGet) p_dev_get = nullptr;
  decltype(&cuDeviceGetDevResource) p_get_res = nullptr;
  decltype(&cuDevSmResourceSplitByCount) p_split = nullptr;
  decltype(&cuDevResourceGenerateDesc) p_desc = nullptr;
  decltype(&cuGreenCtxCreate) p_create = nullptr;
  decltype(&cuGreenCtxStreamCreate) p_stream = nullptr;
  if (!entry("cuDeviceGet", reinterpret_cast<void**>(&p_dev_get)) ||
      !entry("cuDeviceGetDevResource", reinterpret_cast<void**>(&p_get_res)) ||
      !entry("cuDevSmResourceSplitByCount", reinterpret_cast<void**>(&p_split)) ||
      !entry("cuDevResourceGenerateDesc", reinterpret_cast<void**>(&p_desc)) ||
      !entry("cuGreenCtxCreate", reinterpret_cast<void**>(&p_create)) ||
      !entry("cuGreenCtxStreamCreate", reinterpret_cast<void**>(&p_stream)))
    return g;
  CUdevice cd;
  if (p_dev_get(&cd, dev) != CUDA_SUCCESS) return g;
  CUdevResource all, part, rest;
  if (p_get_res(cd, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return g;
  unsigned np = 1;
  if (p_split(&part, &np, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, QG_SMS) != CUDA_SUCCESS ||
      np != 1 || part.sm.smCount < QG_SMS || rest.sm.smCount < 64)
    return g;
  CUdevResourceDesc da, db;
  CUgreenCtx ga, gb;
  if (p_desc(&da, &part, 1) != CUDA_SUCCESS || p_desc(&db, &rest, 1) != CUDA_SUCCESS) return g;
  if (p_create(&ga, da, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      p_create(&gb, db, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return g;
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return g;
  CUstream c0, c1, c2, c3, c4;
  if (p_stream(&c0, ga, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS ||
      p_stream(&c1, gb, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS ||
      p_stream(&c2, gb, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS ||
      p_stream(&c3, gb, CU_STREAM_NON_BLOCKING, lo) != CUDA_SUCCESS ||
      p_stream(&c4, gb, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS)
    return g;
  g.nearY = reinterpret_cast<cudaStream_t>(c4);
  g.chain = reinterpret_cast<cudaStream_t>(c0);
  g.upd = reinterpret_cast<cudaStream_t>(c1);
  g.side = reinterpret_cast<cudaStream_t>(c2);
  g.far = reinterpret_cast<cudaStream_t>(c3);
  g.ok = true;
  return g;
}

// per device, created once (nullptr streams when green contexts are
// unavailable or ITSK_QR_GREEN=0: the shared-SM path)
QrGreen qr_green() {
  static QrGreen g[64];
  static bool tried[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return QrGreen{};
  if (const char* e = getenv("ITSK_QR_GREEN"))
    if (atoi(e) == 0) return QrGreen{};
  if (!tried[dev]) {
    tried[dev] = true;
    g[dev] = make_qr_green(dev);
    cudaGetLastError();  // a failed probe leaves no sticky error behind
    if (getenv("ITSK_QR_GREEN_VERBOSE"))
      fprintf(stderr, "itsk: QR SM partition on device %d: %s\n", dev, g[dev].ok ? "on" : "unavailable");
  }
  return g[dev];
}

cudaError_t pooled_event(int which, cudaEvent_t* out) {
  static cudaEvent_t ev[64][12] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!ev[dev][which]) {
    e = cudaEventCreateWithFlags(&ev[dev][which], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  *out = ev[dev][which];
  return cudaSuccess;
}

// kernel-argument array for cudaLaunchKernelExC (one by-value struct)
struct ArgPack {
  void* p[1];
};
inline void** args_of(PanelArgs& pa) {
  static thread_local ArgPack ap;
  ap.p[0] = &pa;
  return ap.p;
}

size_t y_smem(int nb) { return static_cast<size_t>(2 * YRT * (nb + 4) + 2 * YRT * (UT + 4)) * 8; }

}  // namespace

// ---------------------------------------------------------------------------
QrV2Plan qr_v2_plan(int64_t d, int64_t n) {
  QrV2Plan p{};
  p.C = static_cast<int>(std::min<int64_t>(MAX_C, std::max<int64_t>(1, d / 64)));
  p.hmax = (d + p.C - 1) / p.C + 1;
  const int64_t N = n + 1;
  for (int nb : {32, 16}) {
    const int ks = QP_WARPS / ((nb / 8) * (nb / 8));
    const int64_t doubles = p.hmax * (nb + 1) + 2 * p.C * 2 * nb + QP_WARPS * nb + 2 * nb + (ks > 1 ? ks * nb * nb : 0);
    if (doubles * 8 <= 225 * 1024 && p.hmax <= QP_RPT * QP_THREADS) {
      p.NB = nb;
      p.smem = static_cast<size_t>(doubles * 8);
      break;
    }
  }
  p.ldy = N;
  // Yp (MAX_SPLIT x 32 x N) | Z (32 x N) | betas (n) | taus (n) | Gp (MAX_C x 32 x 32) | G (32 x 32 per panel:
  // the side-stream update of panel k reads its G while panel k+1 writes its own)
  const int64_t npan = (n + 15) / 16;
  p.ws_doubles = static_cast<int64_t>(MAX_SPLIT + 1) * 32 * N + 2 * n + (MAX_C + npan) * 32 * 32 + 64;
  // two-level blocking (n >= 3 outer blocks): per outer block its Gram matrix
  // G_B (QR_OB^2), and two sets of far-update buffers (Yp, Z: the next
  // block's columns on the main stream, the rest on a side stream)
  p.two_level = n >= 3 * QR_OB;
  if (p.two_level) {
    const int64_t nblk = (n + QR_OB - 1) / QR_OB;
    p.far_off = p.ws_doubles;
    p.ws_doubles += nblk * QR_OB * QR_OB + 2 * (qr_far_yp_doubles() + static_cast<int64_t>(QR_OB) * N) +
                    qr_far_yp_doubles();
    // the look-ahead without k_qr_next: a second Yp / Z set for the next
    // panel's update on the main stream
    p.next_off = p.ws_doubles;
    p.ws_doubles += static_cast<int64_t>(MAX_SPLIT + 1) * 32 * N;
  }
  return p;
}

int launch_qr_v2(double* W, int64_t d, int64_t n, int64_t ldw, int64_t N, double* R, double* z,
                 int* singular, double* ws, const QrV2Plan& P, cudaStream_t s_caller) {
  // the factorisation runs on the high-priority stream, joined to the
  // caller's stream at both ends
  cudaStream_t s = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  const QrGreen gr = P.two_level ? qr_green() : QrGreen{};
  {
    int rc = gr.ok ? ITSK_OK : side_stream(&s, 2);
    if (rc) return rc;
    if (gr.ok) s = gr.chain;
    ITSK_CUDA(pooled_event(4, &ev_in));
    ITSK_CUDA(pooled_event(5, &ev_out));
    ITSK_CUDA(cudaEventRecord(ev_in, s_caller));
    ITSK_CUDA(cudaStreamWaitEvent(s, ev_in, 0));
  }
  double* Yp = ws;
  double* Z = Yp + static_cast<int64_t>(MAX_SPLIT) * 32 * N;
  double* betas = Z + 32 * N;
  double* taus = betas + n;
  double* Gp = taus + n;
  double* G = Gp + MAX_C * 32 * 32;
  ITSK_CUDA(cudaMemsetAsync(singular, 0, sizeof(int), s));
  const void* kp = P.NB == 32 ? reinterpret_cast<const void*>(k_qr_panel<32>)
                              : reinterpret_cast<const void*>(k_qr_panel<16>);
  const void* ky = P.NB == 32 ? reinterpret_cast<const void*>(k_qr_y<32>)
                              : reinterpret_cast<const void*>(k_qr_y<16>);
  const void* kn = P.NB == 32 ? reinterpret_cast<const void*>(k_qr_next<32>)
                              : reinterpret_cast<const void*>(k_qr_next<16>);
  ITSK_CUDA(allow_max_smem(kp));
  ITSK_CUDA(allow_max_smem(ky));
  ITSK_CUDA(allow_max_smem(kn));
  ITSK_CUDA(func_attr_once(kp, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  ITSK_CUDA(func_attr_once(kn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_qr_next2<NB_NEXT2>)));
  ITSK_CUDA(func_attr_once(reinterpret_cast<const void*>(k_qr_next2<NB_NEXT2>),
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const int nsm = num_sms();
  const size_t ysm = y_smem(P.NB);
  const size_t nsmem = next_smem(P.hmax, P.NB);
  // look-ahead: the next panel's columns are updated right after the panel
  // (k_qr_next, critical path); the rest of the trailing matrix on a side
  // stream, overlapping the next panel.  Ordering: rest(k) before next(k+1)
  // (which updates columns rest(k) covered), rest(k) after panel(k).
  // k_qr_next (one cluster kernel) when its shared memory fits; else, in
  // two-level mode, the next panel's columns through the regular update
  // kernels on the critical path (own Yp / Z) and the rest beside them
  const bool ahead_k = nsmem <= 220 * 1024 && lookahead_enabled();
  const bool ahead = ahead_k || (P.two_level && lookahead_enabled());
  cudaStream_t side = nullptr;
  if (ahead) {
    int rc = gr.ok ? ITSK_OK : side_stream(&side);
    if (rc) return rc;
    if (gr.ok) side = gr.side;
  }
  cudaEvent_t ev_main = nullptr, ev_side = nullptr;
  if (ahead || P.two_level) {
    ITSK_CUDA(pooled_event(0, &ev_main));
    ITSK_CUDA(pooled_event(1, &ev_side));
    ITSK_CUDA(cudaEventRecord(ev_main, s));  // the side streams start after prior work on s
    if (ahead) ITSK_CUDA(cudaStreamWaitEvent(side, ev_main, 0));
  }
  // Y = V'W2 (row splits), Z = T'Y, W2 -= V Z for the columns of `u`
  auto launch_update = [&](UpdArgs u, int64_t rows, cudaStream_t st) {
    const int64_t ncb = (u.Nt + UT - 1) / UT;
    int S = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(MAX_SPLIT, (2 * nsm) / ncb)));
    S = static_cast<int>(std::min<int64_t>(S, std::max<int64_t>(1, rows / (2 * YRT))));
    u.S = S;
    dim3 gy(static_cast<unsigned>(ncb), static_cast<unsigned>(S));
    dim3 ga(static_cast<unsigned>((rows + UT - 1) / UT), static_cast<unsigned>(ncb));
    if (P.NB == 32) {
      k_qr_y<32><<<gy, 256, ysm, st>>>(u);
      k_qr_z<32><<<static_cast<unsigned>(ncb), 256, 0, st>>>(u);
      k_qr_apply<32><<<ga, 256, 0, st>>>(u);
    } else {
      k_qr_y<16><<<gy, 256, ysm, st>>>(u);
      k_qr_z<16><<<static_cast<unsigned>(ncb), 256, 0, st>>>(u);
      k_qr_apply<16><<<ga, 256, 0, st>>>(u);
    }
    count_launch(3);
  };
  bool side_busy = false;
  // Two-level blocking (P.two_level, n >= 3 QR_OB): the panels' updates stay
  // inside their outer block of QR_OB columns; when a block is done, its
  // reflectors update the far columns in one compact-WY step (qr_far.cu):
  // the next block's columns on s (its panels need them), the rest on a
  // second side stream, overlapping the next block's panels.  Ordering: the
  // far update of block B+1's next block waits for block B's far rest.
  const bool two = P.two_level;
  cudaStream_t side_far = nullptr;
  // ev_far: the previous block's far update of the NEXT block's columns (the
  // near update waits only for those); ev_far_all: all of its far work
  cudaEvent_t ev_g = nullptr, ev_far = nullptr, ev_far_all = nullptr;
  bool far_busy = false;
  double* Gfar = ws + P.far_off;
  double* Ypf[3] = {nullptr, nullptr, nullptr};
  double* Zf[2] = {nullptr, nullptr};
  // green partition: the Gram and near update on `upd` (GEMM partition),
  // handed over to and from the chain through ev_s2u / ev_u2s
  cudaStream_t upd = nullptr, upy = nullptr;
  cudaEvent_t ev_s2u = nullptr, ev_u2s = nullptr, ev_y = nullptr;
  if (two) {
    int rc = gr.ok ? ITSK_OK : side_stream(&side_far, 1);
    if (rc) return rc;
    if (gr.ok) {
      side_far = gr.far;
      upd = gr.upd;
      upy = gr.nearY;
      ITSK_CUDA(pooled_event(7, &ev_s2u));
      ITSK_CUDA(pooled_event(8, &ev_u2s));
      ITSK_CUDA(pooled_event(9, &ev_y));
    }
    ITSK_CUDA(pooled_event(2, &ev_g));
    ITSK_CUDA(pooled_event(3, &ev_far));
    ITSK_CUDA(pooled_event(6, &ev_far_all));
    ITSK_CUDA(cudaStreamWaitEvent(side_far, ev_main, 0));
    const int64_t nblk = (n + QR_OB - 1) / QR_OB;
    Ypf[0] = Gfar + nblk * QR_OB * QR_OB;
    Zf[0] = Ypf[0] + qr_far_yp_doubles();
    Ypf[1] = Zf[0] + static_cast<int64_t>(QR_OB) * N;
    Zf[1] = Ypf[1] + qr_far_yp_doubles();
    Ypf[2] = Zf[1] + static_cast<int64_t>(QR_OB) * N;  // the Gram's partials (beside the near Y)
  }
  for (int64_t k0 = 0; k0 < n; k0 += P.NB) {
    const int kb = static_cast<int>(std::min<int64_t>(P.NB, n - k0));
    // columns the panel's own update covers: its outer block (two-level; the
    // last block also covers the rhs column) or all
    const int64_t blk0 = two ? (k0 / QR_OB) * QR_OB : 0;
    const int64_t horizon = (two && blk0 + QR_OB < n) ? blk0 + QR_OB : N;
    if (two && k0 == blk0 && horizon == N && far_busy) {
      // the last block's updates reach the rhs column, which the previous
      // block's far rest may still be updating
      ITSK_CUDA(cudaStreamWaitEvent(s, ev_far_all, 0));
      far_busy = false;
    }
    double* Gk = G + (k0 / P.NB) * 32 * 32;
    PanelArgs pa;
    pa.W = W;
    pa.d = d;
    pa.ldw = ldw;
    pa.k0 = k0;
    pa.kb = kb;
    pa.hmax = P.hmax;
    pa.betas = betas;
    pa.taus = taus;
    pa.Gp = Gp;
    pa.G = Gk;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.C);
    cfg.blockDim = dim3(QP_THREADS);
    cfg.dynamicSmemBytes = P.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ITSK_CUDA(cudaLaunchKernelExC(&cfg, kp, args_of(pa)));
    count_launch();
    const int64_t c0 = k0 + kb, Nt = horizon - c0;
    if (two && c0 == horizon && horizon < N) {
      // the outer block [blk0, horizon) is factored: its far update
      const int ob = static_cast<int>(horizon - blk0);
      double* Gb = Gfar + (blk0 / QR_OB) * QR_OB * QR_OB;
      // green: the Gram on u and the near update's Y on upy (both need only
      // V), T on the chain stream; then Z and the apply on u
      const cudaStream_t u = upd ? upd : s;
      const int64_t nn = std::min<int64_t>(QR_OB, N - horizon);
      if (upd) {
        ITSK_CUDA(cudaEventRecord(ev_s2u, s));
        ITSK_CUDA(cudaStreamWaitEvent(u, ev_s2u, 0));
        ITSK_CUDA(cudaStreamWaitEvent(upy, ev_s2u, 0));
        if (far_busy) ITSK_CUDA(cudaStreamWaitEvent(upy, ev_far, 0));  // the previous block's update of these columns
        int rc = launch_qr_far_update(W, d, ldw, blk0, ob, horizon, nn, Gb, taus, Ypf[0], Zf[0], upy, 1);
        if (rc) return rc;
        ITSK_CUDA(cudaEventRecord(ev_y, upy));
      }
      int rc = launch_qr_far_gram(W, d, ldw, blk0, ob, taus, Ypf[upd ? 2 : 0], Gb, u, s, ev_u2s);
      if (rc) return rc;
      ITSK_CUDA(cudaEventRecord(ev_g, s));
      if (upd) {
        ITSK_CUDA(cudaStreamWaitEvent(u, ev_g, 0));
        ITSK_CUDA(cudaStreamWaitEvent(u, ev_y, 0));
        rc = launch_qr_far_update(W, d, ldw, blk0, ob, horizon, nn, Gb, taus, Ypf[0], Zf[0], u, 2);
      } else {
        if (far_busy) ITSK_CUDA(cudaStreamWaitEvent(u, ev_far, 0));  // the previous block's update of these columns
        rc = launch_qr_far_update(W, d, ldw, blk0, ob, horizon, nn, Gb, taus, Ypf[0], Zf[0], u);
      }
      if (rc) return rc;
      if (upd) {  // the next block's panels need it
        ITSK_CUDA(cudaEventRecord(ev_u2s, u));
        ITSK_CUDA(cudaStreamWaitEvent(s, ev_u2s, 0));
      }
      if (N - horizon > nn) {
        // the far rest on the side stream, the block after next first: the
        // next block's own near update waits only for that part (stream order
        // keeps every later column's updates in block order)
        const int64_t f0 = horizon + nn, nf = N - f0, n1 = std::min<int64_t>(QR_OB, nf);
        if (upd) {  // its Y needs only V: started before T
          ITSK_CUDA(cudaStreamWaitEvent(side_far, ev_s2u, 0));
          rc = launch_qr_far_update(W, d, ldw, blk0, ob, f0, n1, Gb, taus, Ypf[1], Zf[1], side_far, 1);
          if (rc) return rc;
          ITSK_CUDA(cudaStreamWaitEvent(side_far, ev_g, 0));
          rc = launch_qr_far_update(W, d, ldw, blk0, ob, f0, n1, Gb, taus, Ypf[1], Zf[1], side_far, 2);
        } else {
          ITSK_CUDA(cudaStreamWaitEvent(side_far, ev_g, 0));
          rc = launch_qr_far_update(W, d, ldw, blk0, ob, f0, n1, Gb, taus, Ypf[1], Zf[1], side_far);
        }
        if (rc) return rc;
        ITSK_CUDA(cudaEventRecord(ev_far, side_far));
        if (nf > n1) {
          rc = launch_qr_far_update(W, d, ldw, blk0, ob, f0 + n1, nf - n1, Gb, taus, Ypf[1], Zf[1], side_far);
          if (rc) return rc;
        }
        ITSK_CUDA(cudaEventRecord(ev_far_all, side_far));
        far_busy = true;
      } else {
        far_busy = false;
      }
      continue;
    }
    if (Nt <= 0) continue;
    UpdArgs ua;
    ua.W = W;
    ua.d = d;
    ua.ldw = ldw;
    ua.k0 = k0;
    ua.kb = kb;
    ua.c0 = c0;
    ua.Nt = Nt;
    ua.Yp = Yp;
    ua.Z = Z;
    ua.ldy = P.ldy;
    ua.G = Gk;
    ua.taus = taus;
    const int64_t rows = d - k0;
    cudaStream_t us = s;  // stream of the bulk update
    if (ahead) {
      ITSK_CUDA(cudaEventRecord(ev_main, s));  // panel(k) done
      // the next panel's block on s (after rest(k-1) finished on the side stream)
      if (side_busy) ITSK_CUDA(cudaStreamWaitEvent(s, ev_side, 0));
      UpdArgs un = ua;
      const int64_t nb2 = std::min<int64_t>(P.NB, Nt);
      un.Nt = nb2;
      if (ahead_k) {
        cudaLaunchConfig_t nc = cfg;
        nc.dynamicSmemBytes = nsmem;
        void* nargs[] = {&un, const_cast<int64_t*>(&P.hmax)};
        ITSK_CUDA(cudaLaunchKernelExC(&nc, kn, nargs));
        count_launch();
      } else if (P.NB == NB_NEXT2) {
        cudaLaunchConfig_t nc = cfg;
        nc.dynamicSmemBytes = next2_smem();
        void* nargs[] = {&un};
        ITSK_CUDA(cudaLaunchKernelExC(&nc, reinterpret_cast<const void*>(k_qr_next2<NB_NEXT2>), nargs));
        count_launch();
      } else {
        un.Yp = ws + P.next_off;
        un.Z = un.Yp + static_cast<int64_t>(MAX_SPLIT) * 32 * N;
        launch_update(un, rows, s);
        ITSK_CHECK_LAUNCH();
      }
      if (Nt == nb2) continue;
      ua.c0 = c0 + nb2;
      ua.Nt = Nt - nb2;
      // rest(k) on the side stream once panel(k) is done (beside next(k))
      ITSK_CUDA(cudaStreamWaitEvent(side, ev_main, 0));
      us = side;
    }
    launch_update(ua, rows, us);
    ITSK_CHECK_LAUNCH();
    if (ahead) {
      ITSK_CUDA(cudaEventRecord(ev_side, side));
      side_busy = true;
    }
  }
  if (ahead && side_busy) ITSK_CUDA(cudaStreamWaitEvent(s, ev_side, 0));
  if (two && far_busy) ITSK_CUDA(cudaStreamWaitEvent(s, ev_far_all, 0));
  // the finish is n^2 elementwise work: on the GEMM partition when green
  cudaStream_t fs = s;
  if (upd) {
    ITSK_CUDA(cudaEventRecord(ev_s2u, s));
    ITSK_CUDA(cudaStreamWaitEvent(upd, ev_s2u, 0));
    fs = upd;
  }
  k_qr_finish<<<static_cast<unsigned>((n * n + 255) / 256), 256, 0, fs>>>(W, n, ldw, N, betas, R, z, singular);
  count_launch();
  ITSK_CHECK_LAUNCH();
  ITSK_CUDA(cudaEventRecord(ev_out, fs));
  ITSK_CUDA(cudaStreamWaitEvent(s_caller, ev_out, 0));
  return ITSK_OK;
}

}  // namespace itsk

#ifdef ITSK_QRNEXT_PROBE
extern "C" void itsk_qrnext_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, itsk::g_qn_prof, sizeof(unsigned long long) * 8);
}
#endif

#ifdef ITSK_QR2_PROFILE
extern "C" void itsk_qr2_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, itsk::g_qr2_prof, sizeof(unsigned long long) * 12);
  unsigned long long z[12] = {0};
  cudaMemcpyToSymbol(itsk::g_qr2_prof, z, sizeof(z));
}
#endif
