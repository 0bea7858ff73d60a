// Internal declarations shared by the .cu files (not part of the C ABI).
#pragma once
#include "itsk_common.cuh"

namespace itsk {

// Device-resident loop control block (lives in the loop workspace).
struct LoopCtl {
  // constants (written by k_loop_init)
  int64_t m, n, max_iters, extra_iters;
  int32_t variant, r_slots, has_truth, has_xtrue;
  double alpha, beta, u, gamma, rho, truth_beta;
  // state
  int32_t it;         // completed iterations; current iterate is xs[it]
  int32_t countdown;  // -1 == None (solvers.py:292)
  int32_t nhist;      // divergence-guard history length
  int32_t eval_next;  // first iterate whose stopping rule is not yet evaluated (deferred estimates)
  double hist[8];     // ring of the last 6 residual norms (solvers.py:223-238)
  double lo;          // running minimum
  double xtnorm;      // ||x_true||
  int32_t resolve;    // loop ended before the deferred estimates were ready
  int32_t pad1;
  int64_t epoch_base; // peer exchange: epoch of the begin pass (written per loop, read by the graph's kernels)
  itsk_loop_result result;
};

// Peer exchange of the loop's partial sums (itsk_peer_params); size == 0: off.
struct PeerArgs {
  int rank = 0, size = 0;
  int64_t epoch_base = 0;
  double* recv[ITSK_MAX_PEERS] = {};
  uint64_t* flags[ITSK_MAX_PEERS] = {};
  // deferred estimates: the sender's local ready flag travels with its
  // partial (element n + 4), so all ranks see the same sum of ready bits
  const uint64_t* est_ready = nullptr;
};

// width of one rank's record in the peer receive buffers: c (n), the four
// norms, the ready bit
__host__ __device__ inline int64_t peer_width(int64_t n) { return n + 5; }

// the sender's ready bit (1.0 when the estimates are not deferred)
__device__ __forceinline__ double peer_ready_bit(const PeerArgs& pe) {
  if (!pe.est_ready) return 1.0;
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(pe.est_ready) : "memory");
  return v != 0 ? 1.0 : 0.0;
}

// Pointers the per-iteration kernels resolve from ctl->it.
struct LoopPtrs {
  const double* A;
  const double* b;
  const double* R;
  const double* Rp;  // packed upper triangle or nullptr
  const double* x_true;
  const double* r_true;
  const double* normest;
  const double* condest;
  const uint64_t* est_ready;  // nullptr: the estimates are ready
  PeerArgs peer;
  const double* gpart;  // tail_sums: the pass's group partials (ng x (n+4)), summed by the tail
  int ng;               // 0: the pass reduced into cs itself
  double* xs;
  double* rs;
  double* trace;
  double* cs;
  double* step;  // n: R^{-1}R^{-T} c
  double* part;  // pass partials
  LoopCtl* ctl;
  int64_t lda;
  int64_t n;
  int rp_inv;  // Rp carries the diagonal-block inverses and the TRSV kernel stages them
};

int launch_trsv_pair_device(const double* R, int64_t n, const double* c, double* y,
                            cudaStream_t s);

// Fused pass.  When ctl != nullptr the x / r_prev / r_out pointers are
// resolved on the device from ctl->it (graph-capturable loop body) and the
// kernel is a no-op once ctl->result.done is set.
struct PassArgs {
  const double* A;
  int64_t m, n, lda;
  const double* b;
  const double* x;
  const double* r_prev;
  double* r_out;
  const double* r_true;
  double* part;  // grid x (n + 4)
  int64_t rows_per_cta;
  // loop mode
  const LoopCtl* ctl;
  const double* xs;
  double* rs;
  int mode;  // 0 = explicit pointers, 1 = loop step (x = xs[it+1]), 2 = loop begin (x = xs[0])
  // in-kernel reduction (optional): when `tickets` is set the pass itself
  // sums the per-CTA partials into `cs` — the last CTA of each group of
  // `group` CTAs sums its group into gpart, the last group sums the groups,
  // both in CTA / group order (deterministic); tickets self-reset.
  unsigned* tickets;  // ceil(grid / group) + 1 counters, zero before first use
  double* gpart;      // ceil(grid / group) x (n + 4)
  double* cs;         // n + 4
  int group;
  double bscale = 1.0;  // r = bscale * b - A x (LSQR: u_{k+1} beta = A y - alpha u_k)
  int sm_reserve = 0;   // SMs left free for kernels running beside the pass (the loop's estimates and tail)
  int tail_sums = 0;    // loop: stop after the group level; the tail sums the groups (ITSK_LOOP_TAIL_SUMS)
  PeerArgs peer;        // loop mode: send the reduced partial to every rank
};

// counters / group partials needed by the in-kernel reduction of a pass
int pass_groups(int64_t m, int64_t n, int* group);
int pass_tail_groups(const double* A, int64_t m, int64_t n, int64_t lda, int reserve);

int pass_grid(int64_t m, int64_t n);
int64_t pass_part_doubles(int64_t m, int64_t n);
int launch_pass(const PassArgs& a, cudaStream_t s, int* grid_used);
int launch_finalize(const double* part, int grid, int64_t n, double* cs, const LoopCtl* ctl,
                    cudaStream_t s);

// Sparse CSR A (sparse.cu): the pass over a plan, explicit pointers (mode 0)
// or loop mode (x / r slots from ctl, as PassArgs)
struct CsrPlan;
int launch_csr_pass(const CsrPlan* P, const double* b, double bscale, const double* x, const double* r_prev,
                    double* r_out, const double* r_true, double* cs, const LoopCtl* ctl, const double* xs,
                    double* rs, int mode, cudaStream_t s);

// Panel / update split QR (qr2.cu), the default path of itsk_qr_aug.
struct QrV2Plan {
  int C;             // cluster size of the panel kernel
  int NB;            // panel width (32, or 16 when 32 does not fit), 0 = unusable
  int64_t hmax;      // rows per CTA bound
  size_t smem;       // panel kernel dynamic shared memory
  int64_t ldy;       // leading dimension of the partial Y buffers
  int64_t ws_doubles;
  bool two_level;    // outer blocks of QR_OB columns with a far update (qr_far.cu)
  int64_t far_off;   // offset (doubles) of the far-update buffers
  int64_t next_off;  // offset of the next-panel update's Yp / Z (look-ahead without k_qr_next)
};
QrV2Plan qr_v2_plan(int64_t d, int64_t n);
// Far update of the two-level blocked QR (qr_far.cu): the compact-WY T of an
// outer block (from G = V'V), and W_far -= V T' V' W_far for the far columns
// [c0, c0+Nf) (G then holds T).
constexpr int QR_OB = 128;          // outer block width
constexpr int FAR_YP_TILES = 320;   // Yp capacity: splits x 64-column tiles
int64_t qr_far_yp_doubles();
// G = V'V on s; T (one CTA) on t_stream (nullptr: s), after s through ev_handoff
int launch_qr_far_gram(double* W, int64_t d, int64_t ldw, int64_t b0, int ob, const double* taus, double* Yp,
                       double* G, cudaStream_t s, cudaStream_t t_stream = nullptr, cudaEvent_t ev_handoff = nullptr);
// parts: 1 = Y = V'W_far only (needs V, not T), 2 = Z = T'Y and W_far -= V Z
// (after part 1 on the same buffers), 3 = both
int launch_qr_far_update(double* W, int64_t d, int64_t ldw, int64_t b0, int ob, int64_t c0, int64_t Nf,
                         const double* G, const double* taus, double* Yp, double* Z, cudaStream_t s,
                         int parts = 3);
int launch_qr_v2(double* W, int64_t d, int64_t n, int64_t ldw, int64_t N, double* R, double* z,
                 int* singular, double* ws, const QrV2Plan& P, cudaStream_t s);



}  // namespace itsk
