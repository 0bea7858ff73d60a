// Device-resident refinement loop (K5): _run_refinement
// (/root/reference/pkg/src/itsketch/solvers.py:270-320).
//
// One iteration = two kernels:
//   fused pass  r = b - A x, c = A'r and the norms (solvers.py:299-302,
//               :343); the pass also sums its per-CTA partials (last CTA of
//               each group, then the last group, in a fixed order: PassArgs)
//   k_tail      one CTA: the control step (divergence guard :302-305,
//               _record :241-256, stopping rule + extra_iters countdown
//               :308-318) and, unless the loop stopped, the next iterate:
//               d = R^{-1}R^{-T} c (:294, :339-340) and
//               x+ = x + d | x + alpha d + beta (x - x-) (:295-298).
// All loop state (iteration counter, guard history, countdown, stop reason)
// lives in a LoopCtl block in device memory, so the whole loop runs as one
// CUDA graph whose WHILE conditional node is cleared by k_tail — no host
// round trip per iteration.  For multi-GPU the host calls step_pre (pass +
// local partial sums), sums p->cs across ranks (the only collective), then
// step_post (control + next iterate, replicated).
#include <algorithm>

#include "itsk_common.cuh"
#include "itsk_dense.cuh"
#include "itsk_trsv_cluster.cuh"
#include "itsk_kernels.cuh"

namespace itsk {
namespace {


__global__ void k_loop_init(LoopCtl* ctl, int64_t m, int64_t n, int64_t max_iters,
                            int64_t extra_iters, int variant, int r_slots, int has_truth,
                            int has_xtrue, double alpha, double beta, double u, double gamma,
                            double rho, double truth_beta, int64_t epoch_base) {
  ctl->m = m;
  ctl->n = n;
  ctl->max_iters = max_iters;
  ctl->extra_iters = extra_iters;
  ctl->variant = variant;
  ctl->r_slots = r_slots;
  ctl->has_truth = has_truth;
  ctl->has_xtrue = has_xtrue;
  ctl->alpha = alpha;
  ctl->beta = beta;
  ctl->u = u;
  ctl->gamma = gamma;
  ctl->rho = rho;
  ctl->truth_beta = truth_beta;
  ctl->it = 0;
  ctl->countdown = -1;
  ctl->nhist = 0;
  ctl->eval_next = 1;
  ctl->resolve = 0;
  ctl->epoch_base = epoch_base;
  for (int i = 0; i < 8; ++i) ctl->hist[i] = 0.0;
  ctl->lo = INFINITY;
  ctl->xtnorm = 0.0;
  ctl->result.iterations = 0;
  ctl->result.stop_reason = ITSK_STOP_MAX_ITERS;
  ctl->result.done = 0;
  ctl->result.sol_slot = 0;
  ctl->result.bnorm2 = 0.0;
}

// ||x||^2 with the per-thread order of control_step's fused loop (explicit
// FMA), so a replayed rule sees the same bits as a live one.
__device__ double xnorm2_of(const double* x, int64_t n, double* red) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = __fma_rn(x[i], x[i], s);
  return block_sum(s, red);
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// should_stop (solvers.py:174-192, evaluated left to right) and the
// extra_iters countdown (:306-316) for the iterates k = ctl->eval_next..last
// in order.  Called by every thread of the CTA (the norms of earlier iterates
// are block sums); the iterate `last` uses the caller's values.  Returns the
// iterate the reference stops at, or -1.
__device__ int64_t replay_rule(const LoopPtrs& p, LoopCtl* ctl, int64_t last, double last_xnorm2,
                               double last_change, double last_resnorm, double* red) {
  __shared__ int64_t s_stop;
  const int64_t n = ctl->n, K = ctl->max_iters + 1;
  const double normest = __ldcg(p.normest), condest = __ldcg(p.condest);
  if (threadIdx.x == 0) s_stop = -1;
  __syncthreads();
  for (int64_t k = ctl->eval_next; k <= last; ++k) {
    const double xn2 = (k == last) ? last_xnorm2 : xnorm2_of(p.xs + k * n, n, red);
    if (threadIdx.x == 0) {
      const double change = (k == last) ? last_change : p.trace[2 * K + k - 1];
      const double resnorm = (k == last) ? last_resnorm : p.trace[3 * K + k];
      if (ctl->countdown < 0) {
        const double bound = ctl->u * (ctl->gamma * normest * sqrt(xn2) + ctl->rho * condest * resnorm);
        if (change <= bound) ctl->countdown = static_cast<int32_t>(ctl->extra_iters);
      }
      if (ctl->countdown >= 0) {
        if (ctl->countdown == 0) s_stop = k;
        else ctl->countdown -= 1;
      }
    }
    __syncthreads();
    if (s_stop >= 0) break;
  }
  if (threadIdx.x == 0) ctl->eval_next = static_cast<int32_t>(last + 1);
  const int64_t r = s_stop;
  __syncthreads();
  return r;
}

// Guard + record + stopping rule.  begin == 1 records iterate 0 only.
// Called by every thread of the tail CTA with `ctl` a shared-memory copy of
// the loop state; returns the (CTA-uniform) done flag.  With deferred
// estimates (p.est_ready) the rule is evaluated only once they are ready,
// replaying the iterates recorded meanwhile (replay_rule); a loop that ends
// first (guard, max_iters) is settled by k_loop_finish.
__device__ int control_step(const LoopPtrs& p, LoopCtl* ctl, int begin) {
  __shared__ double red[DENSE_THREADS / 32];
  __shared__ int s_done, s_eval;
  __shared__ double s_change, s_resnorm;
  const int64_t n = ctl->n, it = ctl->it;
  const int64_t K = ctl->max_iters + 1;
  const int64_t xi = begin ? 0 : it + 1;
  const double* x = p.xs + xi * n;
  // the pass's scalars, loaded before the block sums (one L2 round trip
  // overlapped with them instead of after)
  double rr = 0.0, dd = 0.0, tt = 0.0, bb = 0.0;
  if (threadIdx.x == 0) {
    rr = p.cs[n];
    dd = p.cs[n + 1];
    tt = p.cs[n + 2];
    bb = p.cs[n + 3];
  }
  double sx = 0.0, sf = 0.0, st = 0.0;
  int fin = 1;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = x[i];
    sx = __fma_rn(v, v, sx);
    fin &= isfinite(v) ? 1 : 0;
    if (ctl->has_xtrue) {
      const double e = p.x_true[i] - v;
      sf += e * e;
      if (begin) st += p.x_true[i] * p.x_true[i];
    }
  }
  const double xnorm2 = block_sum(sx, red);
  const double fe2 = block_sum(sf, red);
  const double xt2 = block_sum(st, red);
  const int all_fin = __syncthreads_and(fin);
  if (threadIdx.x == 0) {
    const double resnorm = sqrt(rr);
    double* fe = p.trace;
    double* re = p.trace + K;
    double* ch = p.trace + 2 * K;
    double* rn = p.trace + 3 * K;
    if (begin) {
      ctl->xtnorm = sqrt(xt2);
      ctl->result.bnorm2 = bb;
    }
    const int64_t rec = begin ? 0 : it + 1;
    if (ctl->has_xtrue) fe[rec] = sqrt(fe2) / ctl->xtnorm;
    if (ctl->has_truth)
      re[rec] = ctl->truth_beta > 0 ? sqrt(tt) / ctl->truth_beta : resnorm / sqrt(ctl->result.bnorm2);
    rn[rec] = resnorm;
    int done = 0, eval = 0;
    // deferred estimates: evaluable once ready — on several ranks once ready
    // on every rank (the ready bits summed by the peer exchange), so all
    // ranks evaluate the rule at the same iteration and stop together
    const bool ready = p.est_ready == nullptr ||
                       (p.peer.size > 0 ? p.cs[n + 4] == static_cast<double>(p.peer.size)
                                        : ld_acquire_u64(p.est_ready) != 0);
    if (begin) {
      ctl->result.iterations = 0;
      ctl->result.sol_slot = 0;
      if (ctl->max_iters == 0) {
        done = 1;
        ctl->result.stop_reason = ITSK_STOP_MAX_ITERS;
      }
    } else {
      const double change = sqrt(dd);
      ch[it] = change;
      // _DivergenceGuard.diverged (solvers.py:230-238)
      bool diverged = !(isfinite(resnorm) && all_fin);
      if (!diverged) {
        ctl->hist[ctl->nhist % 8] = resnorm;
        ctl->nhist += 1;
        ctl->lo = fmin(ctl->lo, resnorm);
        if (ctl->nhist > 5) {
          const bool growing = resnorm > ctl->hist[(ctl->nhist - 6) % 8];
          diverged = growing && resnorm > 1.0e4 * ctl->lo;
        }
      }
      if (diverged) {
        done = 1;
        ctl->result.stop_reason = ITSK_STOP_DIVERGED;
        ctl->result.iterations = static_cast<int32_t>(it + 1);
        ctl->result.sol_slot = static_cast<int32_t>(it + 1);
        if (!ready) ctl->resolve = 1;
      } else {
        ctl->it = static_cast<int32_t>(it + 1);
        eval = ready ? 1 : 0;
        s_change = change;
        s_resnorm = resnorm;
      }
    }
    ctl->result.done = done;
    s_done = done;
    s_eval = eval;
  }
  __syncthreads();
  if (begin || s_done) return s_done;
  const int64_t nit = it + 1;
  const int64_t stop = s_eval ? replay_rule(p, ctl, nit, xnorm2, s_change, s_resnorm, red) : -1;
  if (threadIdx.x == 0) {
    int done = 0;
    if (stop >= 0) {
      done = 1;
      ctl->result.stop_reason = ITSK_STOP_RULE;
      ctl->result.iterations = static_cast<int32_t>(stop);
      ctl->result.sol_slot = static_cast<int32_t>(stop);
    } else {
      ctl->result.iterations = static_cast<int32_t>(nit);
      ctl->result.sol_slot = static_cast<int32_t>(nit);
      if (nit >= ctl->max_iters) {
        done = 1;
        ctl->result.stop_reason = ITSK_STOP_MAX_ITERS;
        if (!s_eval) ctl->resolve = 1;
      }
    }
    ctl->result.done = done;
    s_done = done;
  }
  __syncthreads();
  return s_done;
}

// Settles a loop that ended before its deferred estimates were ready
// (itsk_loop_finish; stream-ordered after the estimates): the rule replayed
// over the iterates it did not see; a stop it finds comes before the guard's
// or max_iters' (solvers.py:300-318: the rule of iterate k is checked before
// iterate k+1 runs, and at max_iters before the loop exits).
__global__ void __launch_bounds__(DENSE_THREADS) k_loop_finish(LoopPtrs p) {
  __shared__ double red[DENSE_THREADS / 32];
  constexpr int CTL_WORDS = sizeof(LoopCtl) / 8;
  __shared__ LoopCtl s_ctl;
  if (threadIdx.x < CTL_WORDS)
    reinterpret_cast<uint64_t*>(&s_ctl)[threadIdx.x] = reinterpret_cast<const uint64_t*>(p.ctl)[threadIdx.x];
  __syncthreads();
  LoopCtl* ctl = &s_ctl;
  if (!ctl->resolve) return;
  const int64_t n = ctl->n, K = ctl->max_iters + 1;
  const int64_t last = ctl->it;  // the last iterate that passed the guard
  const double xn2 = xnorm2_of(p.xs + last * n, n, red);
  const int64_t stop = last >= ctl->eval_next
                           ? replay_rule(p, ctl, last, xn2, p.trace[2 * K + last - 1], p.trace[3 * K + last], red)
                           : -1;
  if (threadIdx.x == 0) {
    if (stop >= 0) {
      ctl->result.stop_reason = ITSK_STOP_RULE;
      ctl->result.iterations = static_cast<int32_t>(stop);
      ctl->result.sol_slot = static_cast<int32_t>(stop);
    }
    ctl->resolve = 0;
  }
  __syncthreads();
  if (threadIdx.x < CTL_WORDS)
    reinterpret_cast<uint64_t*>(p.ctl)[threadIdx.x] = reinterpret_cast<const uint64_t*>(&s_ctl)[threadIdx.x];
}

__global__ void k_flag_store(uint64_t* flag, uint64_t value) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

// Peer exchange, receiving side (itsk_peer_params): wait until every rank's
// partial of this epoch has landed, then p.cs = sum over ranks in rank order
// (identical bytes on every rank).  A rank that never arrives (a failed peer)
// traps after 60 s instead of hanging the GPU.
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ void peer_gather(const LoopPtrs& p, int64_t epoch_base, int64_t it_epoch) {
  const PeerArgs& pe = p.peer;
  const uint64_t epoch = static_cast<uint64_t>(epoch_base + it_epoch);
  const uint64_t* fl = pe.flags[pe.rank];
  if (static_cast<int>(threadIdx.x) < pe.size) {
    uint64_t t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys_u64(fl + threadIdx.x) < epoch) {
      __nanosleep(64);
      uint64_t t = 0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 60ull * 1000000000ull) asm volatile("trap;");
    }
  }
  __syncthreads();
  const int64_t w = peer_width(p.n);  // c, the norms and the ready bits (their sum: ranks ready)
  const double* rv = pe.recv[pe.rank] + (epoch & 1) * pe.size * w;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
    double s = __ldcg(rv + c);
    for (int r = 1; r < pe.size; ++r) s += __ldcg(rv + r * w + c);
    p.cs[c] = s;
  }
  __syncthreads();
}

// ITSK_LOOP_TAIL_SUMS: the last level of the pass's reduction, moved here
// (the pass's grid has completed): even groups into s0, odd groups into s1,
// then s0 + s1 — group_reduce's order, so cs has the same bits.
__device__ void tail_group_sum(const LoopPtrs& p) {
  const int64_t w = p.n + 4;
  const int ne = (p.ng + 1) / 2, no = p.ng / 2;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
    double v[16];
    double s0 = 0.0, s1 = 0.0;
    for (int g0 = 0; g0 < ne; g0 += 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = g0 + k < ne ? __ldcg(p.gpart + (2 * (g0 + k)) * w + c) : 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (g0 + k < ne) s0 += v[k];
    }
    for (int g0 = 0; g0 < no; g0 += 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = g0 + k < no ? __ldcg(p.gpart + (2 * (g0 + k) + 1) * w + c) : 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (g0 + k < no) s1 += v[k];
    }
    p.cs[c] = s0 + s1;
  }
  __syncthreads();
}

enum : int { TAIL_CONTROL = 2, TAIL_STEP = 4, TAIL_BEGIN = 8 };

// The serial tail of an iteration on one CTA (see the file comment).
#ifdef ITSK_TAIL_PROBE
__device__ unsigned long long g_tail_prof[16];
#define TP(i) do { if (threadIdx.x == 0) { long long _t = clock64(); atomicAdd(&g_tail_prof[i], (unsigned long long)(_t - _tp)); _tp = _t; } } while (0)
#else
#define TP(i) do { } while (0)
#endif

#ifdef ITSK_TIMELINE
// [slot][0] entry, [1] after the dependency wait, [2] after control, [3] after
// R'y = c, [4] after R x = y, [5] end
__device__ unsigned long long g_tail_tl[TL_SLOTS][8];
#define TL(i) do { if (threadIdx.x == 0 && tl_slot >= 0 && tl_slot < TL_SLOTS) g_tail_tl[tl_slot][i] = gtime(); } while (0)
#else
#define TL(i) do { } while (0)
#endif

template <bool PACKED>
__global__ void __launch_bounds__(DENSE_THREADS) k_tail(LoopPtrs p, int flags, int grid,
                                                        cudaGraphConditionalHandle h, int use_cond) {
#ifdef ITSK_TIMELINE
  const unsigned long long tl_t0 = gtime();
  int tl_slot = -1;
#endif
#ifdef ITSK_TAIL_PROBE
  long long _tp = clock64();
  if (threadIdx.x == 0) atomicAdd(&g_tail_prof[15], 1ull);
#endif
  // Programmatic dependent launch: let the next pass start streaming A, and
  // stage R (written long before) while the preceding pass finishes; the
  // pass's outputs and the loop state are read after griddepcontrol.wait.
  pdl_trigger();
  extern __shared__ double sm[];
  const int64_t n = p.n;
  double* v = sm;
  if (PACKED && (flags & TAIL_STEP)) {
    if (p.Rp) stage_packed_bulk(p.Rp, n, sm, p.rp_inv != 0); else stage_packed(p.R, n, sm);
    v = sm + (p.rp_inv ? rp_doubles(n) : packed_doubles(n));
  }
  pdl_wait();
  // the loop state in shared memory: the control step's scalar bookkeeping
  // would otherwise be a chain of dependent L2 round trips
  constexpr int CTL_WORDS = sizeof(LoopCtl) / 8;
  static_assert(sizeof(LoopCtl) % 8 == 0 && CTL_WORDS <= DENSE_THREADS, "LoopCtl copy");
  __shared__ LoopCtl s_ctl;
  if (threadIdx.x < CTL_WORDS)
    reinterpret_cast<uint64_t*>(&s_ctl)[threadIdx.x] = reinterpret_cast<const uint64_t*>(p.ctl)[threadIdx.x];
  __syncthreads();
  LoopCtl* ctl = &s_ctl;
  if (p.ng > 0 && !ctl->result.done) tail_group_sum(p);
  if (p.peer.size > 0 && !ctl->result.done)
    peer_gather(p, ctl->epoch_base, (flags & TAIL_BEGIN) ? 0 : ctl->it + 1);
  // c for the solves, staged now: its loads overlap the control step
  if ((flags & TAIL_STEP) && !ctl->result.done)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] = p.cs[i];
  TP(0);
#ifdef ITSK_TIMELINE
  tl_slot = (flags & TAIL_BEGIN) ? 0 : static_cast<int>(ctl->it) + 1;
  if (threadIdx.x == 0 && tl_slot < TL_SLOTS) g_tail_tl[tl_slot][0] = tl_t0;
#endif
  TL(1);
  if (ctl->result.done) {
    if (use_cond && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
    return;
  }
  if (flags & TAIL_CONTROL) {
    const int done = control_step(p, ctl, (flags & TAIL_BEGIN) ? 1 : 0);
    TP(2);
    TL(2);
    if (threadIdx.x < CTL_WORDS)
      reinterpret_cast<uint64_t*>(p.ctl)[threadIdx.x] = reinterpret_cast<const uint64_t*>(&s_ctl)[threadIdx.x];
    if (done) {
      if (use_cond && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
      return;
    }
  }
  if (!(flags & TAIL_STEP)) return;
  // d = R^{-1} R^{-T} c in shared memory (R staged above), then x_{it+1}
  __shared__ double red_s[64 * (DENSE_THREADS / 32)];
  __syncthreads();
  TP(3);
  if (PACKED) {
    const RPacked R(sm, n);
    const DiagInv inv = diag_inv_at(sm, n, p.rp_inv != 0);
    trsv_t_inplace(R, n, v, red_s, inv);
    TP(4);
    TL(3);
    trsv_n_inplace(R, n, v, red_s, inv);
    TP(5);
    TL(4);
  } else {
    const RGlobal R(p.R, n);
    trsv_t_inplace(R, n, v, red_s);
    trsv_n_inplace(R, n, v, red_s);
  }
  // x_{i+1} in the reference's exact operation order (no FMA contraction)
  const int64_t it = ctl->it;
  const double* x = p.xs + it * n;
  const double* xp = p.xs + (it > 0 ? it - 1 : 0) * n;
  double* xn = p.xs + (it + 1) * n;
  const double alpha = ctl->alpha, beta = ctl->beta;
  const bool basic = ctl->variant == ITSK_VARIANT_BASIC;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double xi = x[i], di = v[i];
    if (basic) {
      xn[i] = __dadd_rn(xi, di);
    } else {
      const double t = __dadd_rn(xi, __dmul_rn(alpha, di));
      xn[i] = __dadd_rn(t, __dmul_rn(beta, __dsub_rn(xi, xp[i])));
    }
  }
  __syncthreads();
  TP(6);
  TL(5);
}

// Large n (R's triangle beyond shared memory, n <= TCL_NMAX): the tail on a
// cluster of TCL_NC CTAs.  CTA 0 runs the control step exactly as k_tail
// (the same 512-thread block sums, so a replayed stopping rule sees the same
// bits); after a cluster barrier every CTA takes its share of the
// triangular-solve pair (itsk_trsv_cluster.cuh) and the owner of each
// 32-row block writes that block of x_{it+1} in the reference's operation
// order.
__global__ void __launch_bounds__(DENSE_THREADS, 1) k_tail_cl(LoopPtrs p, int flags,
                                                             cudaGraphConditionalHandle h, int use_cond) {
  namespace cg = cooperative_groups;
  pdl_trigger();
  extern __shared__ __align__(16) double sm_cl[];
  cg::cluster_group cl = cg::this_cluster();
  const int q = static_cast<int>(cl.block_rank());
  pdl_wait();
  constexpr int CTL_WORDS = sizeof(LoopCtl) / 8;
  __shared__ LoopCtl s_ctl;
  if (q == 0) {
    if (threadIdx.x < CTL_WORDS)
      reinterpret_cast<uint64_t*>(&s_ctl)[threadIdx.x] = reinterpret_cast<const uint64_t*>(p.ctl)[threadIdx.x];
    __syncthreads();
    LoopCtl* ctl = &s_ctl;
    if (!ctl->result.done) {
      if (p.ng > 0) tail_group_sum(p);
      if (p.peer.size > 0) peer_gather(p, ctl->epoch_base, (flags & TAIL_BEGIN) ? 0 : ctl->it + 1);
      int done = 0;
      if (flags & TAIL_CONTROL) {
        done = control_step(p, ctl, (flags & TAIL_BEGIN) ? 1 : 0);
        if (threadIdx.x < CTL_WORDS)
          reinterpret_cast<uint64_t*>(p.ctl)[threadIdx.x] = reinterpret_cast<const uint64_t*>(&s_ctl)[threadIdx.x];
      }
      if (done && use_cond && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
    } else if (use_cond && threadIdx.x == 0) {
      cudaGraphSetConditional(h, 0);
    }
    __threadfence();
  }
  cl.sync();  // the loop state CTA 0 wrote is visible to the cluster
  const LoopCtl* g = p.ctl;
  if (__ldcg(&g->result.done) || !(flags & TAIL_STEP)) return;
  const int64_t n = p.n;
  const int64_t it = __ldcg(&g->it);
  const double* x = p.xs + it * n;
  const double* xp = p.xs + (it > 0 ? it - 1 : 0) * n;
  double* xn = p.xs + (it + 1) * n;
  const double alpha = __ldcg(&g->alpha), beta = __ldcg(&g->beta);
  const bool basic = __ldcg(&g->variant) == ITSK_VARIANT_BASIC;
  trsv_pair_cluster(p.R, p.Rp, static_cast<int>(n), p.cs, sm_cl, [&](int b, int lane, double di) {
    const int64_t i = 32 * b + lane;
    const double xi = x[i];
    if (basic) {
      xn[i] = __dadd_rn(xi, di);
    } else {
      const double t = __dadd_rn(xi, __dmul_rn(alpha, di));
      xn[i] = __dadd_rn(t, __dmul_rn(beta, __dsub_rn(xi, xp[i])));
    }
  });
}

// The cluster pair alone: d = R^{-1} R^{-T} c (itsk_trsv_pair_cl, tests).
__global__ void __launch_bounds__(DENSE_THREADS, 1) k_trsv_pair_cl(const double* R, const double* Rp, int64_t n,
                                                                  const double* c, double* d) {
  extern __shared__ __align__(16) double sm_cl[];
  trsv_pair_cluster(R, Rp, static_cast<int>(n), c, sm_cl, [&](int b, int lane, double v) { d[32 * b + lane] = v; });
}

bool tail_on_cluster(int64_t n) { return !use_packed(n, n + 32) && n <= TCL_NMAX; }

cudaError_t launch_cluster_pdl(const void* func, int64_t n, cudaStream_t s, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(TCL_NC);
  cfg.blockDim = dim3(DENSE_THREADS);
  cfg.dynamicSmemBytes = tcl_smem_bytes(n);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = TCL_NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelExC(&cfg, func, args);
}

struct LoopLayout {
  LoopCtl* ctl;
  double* step;
  double* part;
  double* gpart;
  unsigned* tickets;
  int ntickets;
  int group;
  int64_t bytes;
};

LoopLayout loop_layout(void* ws, int64_t m, int64_t n) {
  Carver cv(ws, 1ll << 62);
  LoopLayout L;
  L.ctl = cv.take<LoopCtl>(1);
  L.step = cv.take<double>(n + 32);
  L.part = cv.take<double>(pass_part_doubles(m, n));
  const int ng = pass_groups(m, n, &L.group);
  L.gpart = cv.take<double>(static_cast<int64_t>(ng) * (n + 4));
  L.ntickets = ng + 1;
  L.tickets = cv.take<unsigned>(L.ntickets);
  L.bytes = cv.off + 256;
  return L;
}

int check_params(const itsk_loop_params* p) {
  ITSK_REQUIRE(p, "null params");
  ITSK_REQUIRE(p->m >= 1 && p->n >= 1 && (p->csr || p->lda >= p->n), "bad loop shape");
  ITSK_REQUIRE(p->max_iters >= 0 && p->extra_iters >= 0, "bad iteration counts");
  ITSK_REQUIRE(p->r_slots == 2 || p->r_slots >= p->max_iters + 1, "r_slots must be 2 or max_iters+1");
  ITSK_REQUIRE((p->A || p->csr) && p->b && p->R && p->normest && p->condest && p->xs && p->rs && p->trace &&
                   p->cs && p->ws,
               "null pointer in loop params");
  ITSK_REQUIRE(p->n <= 6000, "loop: n too large for the single-CTA solves");
  if (p->peer) {
    const itsk_peer_params* g = p->peer;
    ITSK_REQUIRE(g->size >= 1 && g->size <= ITSK_MAX_PEERS && g->rank >= 0 && g->rank < g->size &&
                     g->epoch_base >= 1,
                 "bad peer params (size %d, rank %d, epoch_base %lld)", g->size, g->rank,
                 (long long)g->epoch_base);
    for (int r = 0; r < g->size; ++r) ITSK_REQUIRE(g->recv[r] && g->flags[r], "null peer buffer of rank %d", r);
    ITSK_REQUIRE(!p->csr, "peer exchange: dense A only");
  }
  ITSK_REQUIRE(!p->est_ready || p->r_slots == p->max_iters + 1,
               "deferred estimates need every residual kept (r_slots == max_iters + 1)");
  int64_t need = loop_layout(nullptr, p->m, p->n).bytes;
  ITSK_REQUIRE(need <= p->ws_bytes, "loop workspace too small");
  return ITSK_OK;
}

int loop_sm_reserve();

PeerArgs peer_args(const itsk_loop_params* p) {
  PeerArgs g;
  if (!p->peer) return g;
  g.rank = p->peer->rank;
  g.size = p->peer->size;
  g.epoch_base = p->peer->epoch_base;
  g.est_ready = p->est_ready;
  for (int r = 0; r < ITSK_MAX_PEERS; ++r) {
    g.recv[r] = p->peer->recv[r];
    g.flags[r] = p->peer->flags[r];
  }
  return g;
}

LoopPtrs make_ptrs(const itsk_loop_params* p) {
  LoopLayout L = loop_layout(p->ws, p->m, p->n);
  LoopPtrs q;
  q.A = p->A;
  q.b = p->b;
  q.R = p->R;
  q.Rp = p->Rp;
  q.x_true = p->x_true;
  q.r_true = p->r_true;
  q.normest = p->normest;
  q.condest = p->condest;
  q.est_ready = p->est_ready;
  q.peer = peer_args(p);
  {
    const LoopLayout L = loop_layout(p->ws, p->m, p->n);
    const int ng = ((p->opts & ITSK_LOOP_TAIL_SUMS) && !p->peer && !p->csr)
                       ? pass_tail_groups(p->A, p->m, p->n, p->lda, loop_sm_reserve())
                       : 0;
    q.gpart = ng > 0 ? L.gpart : nullptr;
    q.ng = ng;
  }
  q.xs = p->xs;
  q.rs = p->rs;
  q.trace = p->trace;
  q.cs = p->cs;
  q.step = L.step;
  q.part = L.part;
  q.ctl = L.ctl;
  q.lda = p->lda;
  q.n = p->n;
  q.rp_inv = (p->Rp != nullptr && use_packed_inv(p->n, p->n + 32)) ? 1 : 0;
  return q;
}

// SMs the loop's passes leave free: the tail CTA (which the next pass
// overlaps under programmatic dependent launch) and the deferred estimates
// (condest's 2-CTA cluster, normest) running beside the first iterations.
// A pass CTA that finds no free SM would wait for them.
int loop_sm_reserve() { return 4; }

PassArgs pass_args(const itsk_loop_params* p, const LoopPtrs& q, int mode) {
  PassArgs a{};
  a.A = p->A;
  a.m = p->m;
  a.n = p->n;
  a.lda = p->lda;
  a.b = p->b;
  a.r_true = p->r_true;
  a.part = q.part;
  a.ctl = q.ctl;
  a.xs = p->xs;
  a.rs = p->rs;
  a.mode = mode;
  // the pass reduces its partials into p->cs itself
  const LoopLayout L = loop_layout(p->ws, p->m, p->n);
  a.tickets = L.tickets;
  a.gpart = L.gpart;
  a.cs = p->cs;
  a.group = L.group;
  a.sm_reserve = loop_sm_reserve();
  a.peer = q.peer;
  a.tail_sums = q.ng > 0 ? 1 : 0;
  return a;
}

// the loop's pass: the dense fused pass, or the CSR row / CSC chunk passes
int loop_pass(const itsk_loop_params* p, const LoopPtrs& q, int mode, cudaStream_t s, int* grid) {
  if (p->csr) {
    *grid = 0;
    return launch_csr_pass(reinterpret_cast<const CsrPlan*>(p->csr), p->b, 1.0, nullptr, nullptr, nullptr,
                           p->r_true, p->cs, q.ctl, p->xs, p->rs, mode, s);
  }
  return launch_pass(pass_args(p, q, mode), s, grid);
}

int reset_tickets(const itsk_loop_params* p, cudaStream_t s) {
  const LoopLayout L = loop_layout(p->ws, p->m, p->n);
  ITSK_CUDA(cudaMemsetAsync(L.tickets, 0, sizeof(unsigned) * L.ntickets, s));
  return ITSK_OK;
}

bool trsv_packed(int64_t n) { return use_packed(n, n + 32); }

size_t trsv_smem(int64_t n) {
  // sized for the extended layout when it fits (k_step_trsv stages it iff Rp is set)
  const int64_t tri = use_packed_inv(n, n + 32) ? rp_doubles(n) : packed_doubles(n);
  return static_cast<size_t>((trsv_packed(n) ? tri : 0) + n + 32) * sizeof(double);
}

int enqueue_tail(const itsk_loop_params* p, const LoopPtrs& q, int flags, int grid, cudaStream_t s,
                 cudaGraphConditionalHandle cond = cudaGraphConditionalHandle{}, int use_cond = 0) {
  if (tail_on_cluster(p->n)) {
    (void)grid;
    LoopPtrs qq = q;
    void* args[] = {&qq, &flags, &cond, &use_cond};
    ITSK_CUDA(launch_cluster_pdl(reinterpret_cast<const void*>(k_tail_cl), p->n, s, args));
    count_launch();
    ITSK_CHECK_LAUNCH();
    return ITSK_OK;
  }
  const size_t smem = (flags & TAIL_STEP) ? trsv_smem(p->n) : 0;
  const void* fn = trsv_packed(p->n) ? reinterpret_cast<const void*>(k_tail<true>)
                                     : reinterpret_cast<const void*>(k_tail<false>);
  ITSK_CUDA(launch_pdl(fn, dim3(1), dim3(DENSE_THREADS), smem, s, q, flags, grid, cond, use_cond));
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

int prepare_attrs(int64_t n) {
  (void)n;
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_tail<true>)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_tail<false>)));
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_tail_cl)));
  ITSK_CUDA(func_attr_once(reinterpret_cast<const void*>(k_tail_cl), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return ITSK_OK;
}

int loop_unroll() { return 2; }  // two iterations per graph body: every other boundary keeps PDL

struct GraphHandle {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

}  // namespace
}  // namespace itsk

using namespace itsk;

#ifdef ITSK_TIMELINE
extern "C" void itsk_tail_timeline_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, itsk::g_tail_tl, sizeof(itsk::g_tail_tl));
  unsigned long long z[itsk::TL_SLOTS][8] = {};
  cudaMemcpyToSymbol(itsk::g_tail_tl, z, sizeof(z));
}
#endif

#ifdef ITSK_TAIL_PROBE
extern "C" void itsk_tail_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, itsk::g_tail_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(itsk::g_tail_prof, z, sizeof(z));
}
#endif

extern "C" int itsk_loop_workspace(int64_t m, int64_t n, int64_t* bytes) {
  ITSK_REQUIRE(bytes && m >= 1 && n >= 1, "bad loop shape");
  *bytes = loop_layout(nullptr, m, n).bytes;
  return ITSK_OK;
}

extern "C" int itsk_loop_result_ptr(const itsk_loop_params* p, itsk_loop_result** out) {
  ITSK_REQUIRE(p && out && p->ws, "null pointer");
  *out = &loop_layout(p->ws, p->m, p->n).ctl->result;
  return ITSK_OK;
}

extern "C" int itsk_loop_begin_local(const itsk_loop_params* p, itsk_stream_t stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if ((rc = prepare_attrs(p->n))) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  LoopPtrs q = make_ptrs(p);
  k_loop_init<<<1, 1, 0, s>>>(q.ctl, p->m, p->n, p->max_iters, p->extra_iters, p->variant,
                              p->r_slots, p->has_truth, p->x_true != nullptr, p->alpha, p->beta,
                              p->u, p->gamma, p->rho, p->truth_beta, p->peer ? p->peer->epoch_base : 0);
  count_launch();
  ITSK_CHECK_LAUNCH();
  if ((rc = reset_tickets(p, s))) return rc;
  int grid = 0;
  return loop_pass(p, q, 2, s, &grid);
}

extern "C" int itsk_loop_begin_finish(const itsk_loop_params* p, itsk_stream_t stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if ((rc = prepare_attrs(p->n))) return rc;
  LoopPtrs q = make_ptrs(p);
  return enqueue_tail(p, q, TAIL_CONTROL | TAIL_BEGIN | TAIL_STEP, 0, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int itsk_loop_begin(const itsk_loop_params* p, itsk_stream_t stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if ((rc = prepare_attrs(p->n))) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  LoopPtrs q = make_ptrs(p);
  k_loop_init<<<1, 1, 0, s>>>(q.ctl, p->m, p->n, p->max_iters, p->extra_iters, p->variant,
                              p->r_slots, p->has_truth, p->x_true != nullptr, p->alpha, p->beta,
                              p->u, p->gamma, p->rho, p->truth_beta, p->peer ? p->peer->epoch_base : 0);
  count_launch();
  ITSK_CHECK_LAUNCH();
  if ((rc = reset_tickets(p, s))) return rc;
  int grid = 0;
  rc = loop_pass(p, q, 2, s, &grid);
  if (rc) return rc;
  return enqueue_tail(p, q, TAIL_CONTROL | TAIL_BEGIN | TAIL_STEP, grid, s);
}

// local half of an iteration: the pass over this rank's rows and its partial sums
extern "C" int itsk_loop_step_pre(const itsk_loop_params* p, itsk_stream_t stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if ((rc = prepare_attrs(p->n))) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  LoopPtrs q = make_ptrs(p);
  int grid = 0;
  return loop_pass(p, q, 1, s, &grid);
}

// replicated half: control step and the next iterate
extern "C" int itsk_loop_step_post(const itsk_loop_params* p, itsk_stream_t stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if ((rc = prepare_attrs(p->n))) return rc;
  LoopPtrs q = make_ptrs(p);
  return enqueue_tail(p, q, TAIL_CONTROL | TAIL_STEP, 0, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int itsk_loop_graph_create(const itsk_loop_params* p, itsk_stream_t stream,
                                      void** handle) {
  (void)stream;
  int rc = check_params(p);
  if (rc) return rc;
  ITSK_REQUIRE(handle, "null handle");
  if ((rc = prepare_attrs(p->n))) return rc;
  pass_grid(p->m, p->n);  // warm the occupancy cache outside capture
  LoopPtrs q = make_ptrs(p);
  GraphHandle* gh = new GraphHandle();
  cudaStream_t cap = nullptr;
  auto fail = [&](int code) {
    if (cap) cudaStreamDestroy(cap);
    if (gh->exec) cudaGraphExecDestroy(gh->exec);
    if (gh->graph) cudaGraphDestroy(gh->graph);
    delete gh;
    return code;
  };
  if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess ||
      cudaGraphCreate(&gh->graph, 0) != cudaSuccess) {
    set_error("graph create failed");
    return fail(ITSK_ECUDA);
  }
  cudaGraphConditionalHandle cond;
  cudaError_t e = cudaGraphConditionalHandleCreate(&cond, gh->graph, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = cond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  if (e == cudaSuccess) e = cudaGraphAddNode(&node, gh->graph, nullptr, 0, &np);
  if (e != cudaSuccess) {
    set_error("conditional node: %s", cudaGetErrorString(e));
    return fail(ITSK_ECUDA);
  }
  cudaGraph_t body = np.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) {
    set_error("capture begin: %s", cudaGetErrorString(e));
    return fail(ITSK_ECUDA);
  }
  // The body holds `unroll` iterations: a kernel boundary inside the body
  // keeps programmatic dependent launch (the next pass streams A while the
  // tail runs), the WHILE node's re-launch between bodies does not.  Once the
  // loop is done the remaining kernels of the body are no-ops.
  int grid = 0;
  for (int u = 0; u < loop_unroll() && rc == ITSK_OK; ++u) {
    rc = loop_pass(p, q, 1, cap, &grid);
    if (rc == ITSK_OK) rc = enqueue_tail(p, q, TAIL_CONTROL | TAIL_STEP, grid, cap, cond, 1);
  }
  cudaGraph_t captured = body;
  e = cudaStreamEndCapture(cap, &captured);
  if (rc != ITSK_OK) return fail(rc);
  if (e != cudaSuccess) {
    set_error("capture end: %s", cudaGetErrorString(e));
    return fail(ITSK_ECUDA);
  }
  e = cudaGraphInstantiate(&gh->exec, gh->graph, 0);
  if (e != cudaSuccess) {
    set_error("graph instantiate: %s", cudaGetErrorString(e));
    return fail(ITSK_ECUDA);
  }
  cudaStreamDestroy(cap);
  *handle = gh;
  return ITSK_OK;
}

extern "C" int itsk_loop_finish(const itsk_loop_params* p, itsk_stream_t stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!p->est_ready) return ITSK_OK;
  LoopPtrs q = make_ptrs(p);
  k_loop_finish<<<1, DENSE_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(q);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

extern "C" int itsk_trsv_pair_cl(const double* R, const double* Rp, int64_t n, const double* c, double* d,
                                 itsk_stream_t stream) {
  ITSK_REQUIRE(R && c && d && n >= 1 && n <= TCL_NMAX, "cluster TRSV pair: bad arguments (n <= %d)", TCL_NMAX);
  const void* fn = reinterpret_cast<const void*>(k_trsv_pair_cl);
  ITSK_CUDA(allow_max_smem(fn));
  ITSK_CUDA(func_attr_once(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(TCL_NC);
  cfg.blockDim = dim3(DENSE_THREADS);
  cfg.dynamicSmemBytes = tcl_smem_bytes(n);
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = TCL_NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&R, &Rp, &n, &c, &d};
  ITSK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

extern "C" int itsk_flag_store(uint64_t* flag, uint64_t value, itsk_stream_t stream) {
  ITSK_REQUIRE(flag, "null flag");
  k_flag_store<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flag, value);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

extern "C" int itsk_loop_graph_launch(void* handle, itsk_stream_t stream) {
  ITSK_REQUIRE(handle, "null handle");
  GraphHandle* gh = static_cast<GraphHandle*>(handle);
  ITSK_CUDA(cudaGraphLaunch(gh->exec, reinterpret_cast<cudaStream_t>(stream)));
  return ITSK_OK;
}

extern "C" void itsk_loop_graph_destroy(void* handle) {
  if (!handle) return;
  GraphHandle* gh = static_cast<GraphHandle*>(handle);
  if (gh->exec) cudaGraphExecDestroy(gh->exec);
  if (gh->graph) cudaGraphDestroy(gh->graph);
  delete gh;
}
