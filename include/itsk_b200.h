/*
 * itsk_b200.h — C ABI of the B200-native iterative-sketching least-squares
 * path (libitsk_b200.so, sm_100a).
 *
 * The reference (arXiv 2311.04362 package `itsketch`) is pure Python: its
 * drop-in boundary is the function API
 *   iterative_sketching(a, b, cfg, truth) -> SolveResult
 * (/root/reference/pkg/src/itsketch/solvers.py:323-345), which calls the
 * pieces below.  Each entry point names the reference routine it replaces.
 * The Python host layer (paper_2311_04362_b200/) binds these with ctypes and
 * mirrors the reference's Python API; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer (cudaMalloc / torch CUDA
 *     tensor) unless documented otherwise; matrices are row-major fp64 with an
 *     explicit leading dimension (elements), as numpy C-order arrays are;
 *   - every call is asynchronous on `stream` unless documented otherwise;
 *   - return value: ITSK_OK or an ITSK_E* status; itsk_last_error() gives a
 *     thread-local message.  No C++ exception crosses the ABI;
 *   - no global mutable state besides the launch counter and the per-thread
 *     error string: calls on different streams/workspaces are independent.
 */
#ifndef ITSK_B200_H_
#define ITSK_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* itsk_stream_t; /* == cudaStream_t */

enum {
  ITSK_OK = 0,
  ITSK_EINVAL = 1,    /* bad argument; maps to ValueError        */
  ITSK_ESINGULAR = 2, /* exact zero on diag(R); SingularMatrixError (linalg.py:17-18,54-55) */
  ITSK_ECUDA = 3,     /* CUDA runtime error                       */
  ITSK_ENODEV = 4     /* no sm_100 device                         */
};

enum { ITSK_VARIANT_BASIC = 0, ITSK_VARIANT_WEIGHTED = 1 };

enum { /* SolveTrace.stop_reason (solvers.py:72) */
  ITSK_STOP_MAX_ITERS = 0,
  ITSK_STOP_RULE = 1,
  ITSK_STOP_DIVERGED = 2
};

const char* itsk_last_error(void);
int itsk_version(void);
/* 0 if device `dev` is an sm_100 part this library was built for. */
int itsk_device_check(int dev);
/* Number of kernels launched through this library so far (process-wide). */
int64_t itsk_launch_count(void);

/* ----------------------------------------------------------------------
 * Sparse sign embedding pattern — replaces sparse_sign_new
 * (embed.py:83-99) with _distinct_rows (embed.py:28-42): the exact numpy
 * Generator(PCG64) stream (32-bit buffered Lemire draws, whole-column
 * redraws of columns holding a repeat, then choice([-1,1]) signs),
 * generated on the device by jump-ahead.  pcg[0..3] = state_hi, state_lo,
 * inc_hi, inc_lo of default_rng(seed).bit_generator.state.
 * Outputs: rows/neg in the reference's (m, zeta) order; sk_ptr/sk_src the
 * same pattern grouped by sketch row (CSR of S), sources ascending, sign in
 * bit 31.  Synchronises `stream` (the redraw loop is data dependent).
 * -------------------------------------------------------------------- */
int itsk_pattern_workspace(int64_t d, int64_t m, int64_t zeta, int64_t* bytes);
int itsk_sparse_sign_pattern(int64_t d, int64_t m, int64_t zeta, const uint64_t pcg[4],
                             int has_uint32, uint32_t uinteger, uint32_t* rows,
                             uint8_t* neg, uint32_t* sk_ptr, uint32_t* sk_src, void* ws,
                             int64_t ws_bytes, itsk_stream_t stream);

/* CSR (grouped by sketch row, sources ascending) of a contiguous slice of
 * the pattern: rows/neg point at entry row0*zeta of the full (m, zeta)
 * arrays, m is the slice length; sources are slice-local.  Used by each rank
 * of a row-sharded solve for its own block of columns of S. */
int itsk_pattern_csr(const uint32_t* rows, const uint8_t* neg, int64_t m, int64_t zeta, int64_t d,
                     uint32_t* sk_ptr, uint32_t* sk_src, void* ws, int64_t ws_bytes,
                     itsk_stream_t stream);

/* ----------------------------------------------------------------------
 * S·[A | b] — replaces SparseSignEmbedding.apply_dense / apply_vec
 * (embed.py:62-74 → scipy csc_matvecs), called from sketch_and_solve
 * (solvers.py:207-208).  SAb is d x (n + (b != NULL)), leading dim ldw.
 * Summation order equals the reference's (ascending source row, product
 * rounded before the add), so SAb is bitwise identical to scipy's.
 * For a row shard (multi-GPU) pass the shard's rows and its own CSR
 * (itsk_pattern_csr); the per-rank partial sketches are then summed.
 * m < 2^31 and n <= lda < 2^31 (ITSK_EINVAL otherwise).
 * -------------------------------------------------------------------- */
int itsk_sketch(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                const uint32_t* sk_ptr, const uint32_t* sk_src, int64_t d, int64_t zeta,
                double* SAb, int64_t ldw, itsk_stream_t stream);
/* The same sum restricted to the source rows [row0, row1), continuing from
 * SAb's current values when `accumulate` is set: windows taken in row order
 * give the bitwise result of one itsk_sketch call, so A can be sketched
 * chunk by chunk while it is still being copied to the device. A points to
 * row 0 (only rows row0..row1-1 are read). */
int itsk_sketch_rows(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                     const uint32_t* sk_ptr, const uint32_t* sk_src, int64_t d, int64_t zeta,
                     double* SAb, int64_t ldw, int64_t row0, int64_t row1, int accumulate,
                     itsk_stream_t stream);

/* ----------------------------------------------------------------------
 * Householder QR of the d x n sketch with the reflectors also applied to
 * column n (Sb) — replaces householder_qr_econ (linalg.py:30-47, LAPACK
 * dgeqrf+dorgqr, diag(R) >= 0) and Q'·Sb (solvers.py:209).  W (d x (n+1),
 * ldw) is overwritten.  R: n x n row-major (ld n), upper, diag >= 0.
 * z = (Q'Sb)[:n] with the same sign fix.  Returns ITSK_ESINGULAR (after
 * synchronising) if some R_kk == 0, like _check_square_upper.
 * -------------------------------------------------------------------- */
int itsk_qr_workspace(int64_t d, int64_t n, int64_t* bytes);
/* Row blocks of the factorisation: 1 = one Householder QR (W then holds the
 * reflectors below the diagonal); more for a d beyond one factorisation's
 * range (~50000 rows): TSQR over blocks of <= 24000 rows — each block with
 * its share of the rhs column, then the stacked [R_i | z_i] — which returns
 * the R and z of the whole matrix and leaves no single set of reflectors. */
int itsk_qr_row_blocks(int64_t d, int64_t n, int64_t* blocks);
int itsk_qr_aug(double* W, int64_t d, int64_t n, int64_t ldw, double* R, double* z,
                void* ws, int64_t ws_bytes, itsk_stream_t stream);
/* The same without the host round trip: the factorisation's flags are
 * copied to the device int *singular on the stream — bit 0: an exact zero on
 * diag(R) (the caller raises SingularMatrixError when it reads the flag with
 * its results); bit 1: a non-finite entry in R or z (the reference's
 * triangular solves refuse those: scipy solve_triangular's check_finite,
 * linalg.py:59-68 -> ValueError).  itsk_qr_aug itself returns NaNs like
 * LAPACK's QR (linalg.py:42) and reports only the zero pivot. */
int itsk_qr_aug_async(double* W, int64_t d, int64_t n, int64_t ldw, double* R, double* z, void* ws,
                      int64_t ws_bytes, int* singular, itsk_stream_t stream);

/* tri_solve_upper (linalg.py:59-62, trans=0: R y = c) and
 * tri_solve_upper_transpose (linalg.py:65-68, trans=1: R' y = c). */
int itsk_trsv(const double* R, int64_t n, const double* c, double* y, int trans,
              itsk_stream_t stream);
/* solve_step (solvers.py:339-340): y = R^{-1} R^{-T} c. */
/* itsk_trsv with R staged from itsk_pack_upper's layout Rp (one bulk copy;
 * the diagonal-block inverses applied where well conditioned — the loop
 * tail's arithmetic).  Used for x0 = R^-1 z and LSQR's solves. */
int itsk_trsv_rp(const double* R, const double* Rp, int64_t n, const double* c, double* y, int trans,
                 itsk_stream_t stream);
/* The loop's solve pair d = R^{-1} R^{-T} c (solvers.py:339-340) on a
 * 16-CTA thread-block cluster: 32-row blocks owned round robin, each
 * block's chain warp waits for its predecessor's values (pushed through
 * distributed shared memory), helper warps add the older terms; fixed-order
 * sums (reproducible).  n <= 4096.  Rp: itsk_pack_upper's layout (its
 * diagonal-block inverses) or NULL.  The loop tail uses the same code when
 * R's triangle does not fit one CTA's shared memory. */
int itsk_trsv_pair_cl(const double* R, const double* Rp, int64_t n, const double* c, double* d,
                      itsk_stream_t stream);
int itsk_trsv_pair(const double* R, int64_t n, const double* c, double* y, double* tmp,
                   itsk_stream_t stream);

/* Packed form of R for the single-CTA R kernels, which bulk-copy it into
 * shared memory in one shot: the upper triangle by rows (row i holds
 * R[i][i..n), padded to 16 bytes), then the inverses of the 32x32 diagonal
 * blocks (packed the same way) and each block's 1-norm condition number.
 * The substitutions multiply by a block inverse when that block is well
 * conditioned (kappa_1 <= 1e4) and run the scalar chain otherwise. */
int itsk_pack_upper_doubles(int64_t n, int64_t* doubles);
int itsk_pack_upper(const double* R, int64_t n, double* Rp, itsk_stream_t stream);

/* rand_power_norm_est (linalg.py:79-105) with the start vector v0 (host
 * numpy default_rng(seed).standard_normal(n)), `steps` power steps; the
 * result is written to *out (device scalar).  Rp: itsk_pack_upper(R) or NULL. */
int itsk_normest(const double* R, int64_t n, const double* v0, int64_t steps, double* out,
                 const double* Rp, itsk_stream_t stream);
/* cond_est (linalg.py:108-113): sigma_max/sigma_min of R from Lanczos on
 * R'R and on R^{-1}R^{-T}, stopped when the extreme Ritz values settle to
 * 1e-13; *out (device).  Rp: packed R or NULL. */
int itsk_condest_workspace(int64_t n, int64_t* doubles);
int itsk_condest(const double* R, int64_t n, const double* v0, double* out, const double* Rp,
                 itsk_stream_t stream);
/* The same estimate with the (R'R)^{-1} Lanczos run on X = R^{-1} (formed
 * once into ws, itsk_condest_workspace doubles) by matrix-vector products
 * instead of two triangular solves per step. */
int itsk_condest_ws(const double* R, int64_t n, const double* v0, double* out, const double* Rp,
                    double* ws, int64_t ws_doubles, itsk_stream_t stream);

/* ----------------------------------------------------------------------
 * The fused pass of the refinement loop (solvers.py:290,299,343 — r = b-Ax
 * and A'r — plus the norms of solvers.py:300-302 and _record's RE):
 *   r = b - A x;  c = A' r;
 *   scal = [|r|^2, |r - r_prev|^2, |r_true - r|^2, |b|^2]
 * in one streaming read of A.  r_prev, r_out, r_true may be NULL.  Per-CTA
 * partials go to the workspace and are summed in a fixed order
 * (deterministic) into cs = [c(n) | scal(4)].
 * -------------------------------------------------------------------- */
int itsk_pass_workspace(int64_t m, int64_t n, int64_t* bytes);
int itsk_fused_pass(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                    const double* x, const double* r_prev, double* r_out,
                    const double* r_true, double* cs, void* ws, int64_t ws_bytes,
                    itsk_stream_t stream);
/* The same pass with r = bscale * b - A x: one LSQR bidiagonalisation step
 * beta' u' = A R^{-1} v - alpha u in one sweep over A (b = beta u, x = -R^{-1} v,
 * bscale = -alpha / beta), c = A' (beta' u') alongside (solvers.py:455-461). */
int itsk_fused_pass_scaled(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                           double bscale, const double* x, const double* r_prev, double* r_out,
                           const double* r_true, double* cs, void* ws, int64_t ws_bytes,
                           itsk_stream_t stream);

/* Pass flags.  ITSK_PASS_WS_READY: the workspace's reduction counters are
 * zero — set by itsk_pass_workspace_init once, and left so by every pass that
 * completes — so the per-call reset (a memset on the stream, which also stops
 * a programmatic-dependent-launch overlap with the previous pass) is skipped. */
#define ITSK_PASS_WS_READY 1u
int itsk_pass_workspace_init(void* ws, int64_t m, int64_t n, itsk_stream_t stream);
int itsk_fused_pass_ex(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                       double bscale, const double* x, const double* r_prev, double* r_out,
                       const double* r_true, double* cs, void* ws, int64_t ws_bytes,
                       unsigned flags, itsk_stream_t stream);

/* ----------------------------------------------------------------------
 * Sparse CSR A (embed.py:76-80 apply_sparse; solvers.py:195-196 and the
 * loop's a @ x / a.T @ r on a scipy CSR matrix, section 3.5).
 * A plan keeps the caller's CSR arrays (row_ptr m+1, col nnz, val nnz; device
 * pointers that must outlive the plan) and builds, once, the CSC copy and
 * the chunk table of the A'r pass.  itsk_csr_sketch is bitwise scipy's S·A;
 * itsk_csr_pass writes cs = [A'r | |r|^2, |r - r_prev|^2, |r_true - r|^2,
 * |b|^2] like itsk_fused_pass (r = bscale*b - A x bitwise scipy's).
 * -------------------------------------------------------------------- */
typedef struct itsk_csr_plan itsk_csr_plan;
int itsk_csr_plan_create(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t m,
                         int64_t n, int64_t nnz, itsk_stream_t stream, itsk_csr_plan** plan);
void itsk_csr_plan_destroy(itsk_csr_plan* plan);
int itsk_csr_shape(const itsk_csr_plan* plan, int64_t* m, int64_t* n, int64_t* nnz);
int itsk_csr_sketch(const itsk_csr_plan* plan, const double* b, const uint32_t* sk_ptr,
                    const uint32_t* sk_src, int64_t d, int64_t zeta, double* SAb, int64_t ldw,
                    itsk_stream_t stream);
int itsk_csr_pass(const itsk_csr_plan* plan, const double* b, double bscale, const double* x,
                  const double* r_prev, double* r_out, const double* r_true, double* cs,
                  itsk_stream_t stream);

/* ----------------------------------------------------------------------
 * Device-resident refinement loop (_run_refinement, solvers.py:270-320).
 * State, constants and trace live in device memory; the loop runs as one
 * CUDA graph with a conditional WHILE node (no host round trip per
 * iteration), or step-wise for multi-GPU (collective between pre and post).
 * -------------------------------------------------------------------- */
/* Peer-memory exchange of the loop's per-iteration partial sums (the
 * allreduce of [c | norms] over NVLink without NCCL): each rank's pass, after
 * its in-kernel reduction, stores its partial into every rank's receive
 * buffer (peer-mapped pointers, e.g. torch symmetric memory) and raises its
 * flag there with the exchange's epoch; each rank's tail waits for all flags
 * of that epoch and sums the partials in rank order — the same bytes on
 * every rank.  recv[r]: rank r's buffer of 2 x size x (n+5) doubles (epoch
 * parity x source rank; per source: c, the 4 norms and the sender's
 * deferred-estimate ready bit, so every rank takes the same decision of
 * when the stopping rule becomes evaluable); flags[r]: rank r's size uint64
 * flags, zero before the first exchange.  Exchanges of one loop use epochs epoch_base ..
 * epoch_base + max_iters; the next loop on the same buffers starts above. */
#define ITSK_MAX_PEERS 8
typedef struct itsk_peer_params {
  int32_t rank, size;
  int64_t epoch_base;
  double* recv[ITSK_MAX_PEERS];
  uint64_t* flags[ITSK_MAX_PEERS];
} itsk_peer_params;

typedef struct itsk_loop_params {
  int64_t m, n, lda;        /* local rows on this rank */
  int64_t max_iters, extra_iters;
  int32_t variant;          /* ITSK_VARIANT_* (solvers.py:295-298)           */
  int32_t r_slots;          /* rows of rs: max_iters+1 (keep all) or 2       */
  double alpha, beta;       /* _update_coeffs (solvers.py:259-267)           */
  double u, gamma, rho;     /* should_stop (solvers.py:174-192)              */
  double truth_beta;        /* Truth.beta; RE = |r*-r|/beta, or |r|/|b| if 0 */
  int32_t has_truth;
  const double* A;
  const double* b;
  const double* R;          /* n x n, ld n                                   */
  const double* Rp;         /* itsk_pack_upper(R) or NULL                    */
  const double* x_true;     /* n, nullable                                   */
  const double* r_true;     /* m (local), nullable                           */
  const double* normest;    /* device scalars from itsk_normest/itsk_condest */
  const double* condest;
  double* xs;               /* (max_iters+1) x n, xs[0] = x0 on entry        */
  double* rs;               /* r_slots x m                                   */
  double* trace;            /* 4 x (max_iters+1): fe, re, change, |r|        */
  double* cs;               /* n + 8: reduced [c | scal]; the collective's buffer */
  void* ws;                 /* itsk_loop_workspace bytes                     */
  int64_t ws_bytes;
  const struct itsk_csr_plan* csr; /* sparse A (A, lda unused) or NULL        */
  /* Deferred estimates (nullable).  When set, normest/condest may still be
   * running on another stream while the loop starts: the tail evaluates the
   * stopping rule only once *est_ready != 0 (store it with itsk_flag_store
   * after both estimates, on their stream), replaying the rule over the
   * iterations already recorded; itsk_loop_finish, enqueued after the
   * estimates, settles a loop that ended (guard / max_iters) before they
   * were ready.  Requires r_slots == max_iters + 1 (the stop may move back
   * to an earlier, still-held iterate).  With a peer exchange the rule becomes
   * evaluable once the flag is set on EVERY rank (each rank's ready bit
   * travels with its partial), so all ranks stop at the same iteration; a
   * host-collective (step_pre / allreduce / step_post) loop over several
   * ranks must not defer. */
  const uint64_t* est_ready;
  /* Peer-memory exchange (nullable): with it the sharded loop needs no host
   * collective — itsk_loop_begin / the loop graph run it end to end. */
  const itsk_peer_params* peer;
  /* ITSK_LOOP_TAIL_SUMS: the pass leaves the last level of its [c | norms]
   * reduction to the tail kernel (cs is complete only after the tail: not
   * with a host collective between step_pre and step_post). */
  uint32_t opts;
} itsk_loop_params;
#define ITSK_LOOP_TAIL_SUMS 1u

typedef struct itsk_loop_result { /* read back with one D2H copy */
  int32_t iterations;  /* len(iterates) - 1                       */
  int32_t stop_reason; /* ITSK_STOP_*                             */
  int32_t done;
  int32_t sol_slot;    /* xs row holding SolveResult.solution     */
  double bnorm2;
  double pad[3];
} itsk_loop_result;

int itsk_loop_workspace(int64_t m, int64_t n, int64_t* bytes);
/* Writes constants, r0 = b - A x0 (fused pass), records iterate 0 and
 * forms x1.  For multi-GPU call itsk_loop_begin_local, allreduce p->cs,
 * then itsk_loop_begin_finish. */
int itsk_loop_begin(const itsk_loop_params* p, itsk_stream_t stream);
int itsk_loop_begin_local(const itsk_loop_params* p, itsk_stream_t stream);
int itsk_loop_begin_finish(const itsk_loop_params* p, itsk_stream_t stream);
/* One iteration, split around the collective: pre = fused pass over the
 * local rows + partial sums into p->cs; post = guard, stopping rule, trace
 * and (unless stopped) the next iterate (two TRSVs + update).  Both are
 * no-ops once the loop is done. */
int itsk_loop_step_pre(const itsk_loop_params* p, itsk_stream_t stream);
int itsk_loop_step_post(const itsk_loop_params* p, itsk_stream_t stream);
/* Whole loop as a CUDA graph (conditional WHILE); the handle caches the
 * instantiated graph for repeated solves on the same buffers. */
int itsk_loop_graph_create(const itsk_loop_params* p, itsk_stream_t stream, void** handle);
int itsk_loop_graph_launch(void* handle, itsk_stream_t stream);
void itsk_loop_graph_destroy(void* handle);
/* Settles the deferred stopping rule (est_ready set): replays the rule over
 * the iterations the loop ran before the estimates were ready and moves the
 * stop back to where the reference would have stopped (solvers.py:306-316).
 * A no-op otherwise.  Enqueue after the loop and after the estimates. */
int itsk_loop_finish(const itsk_loop_params* p, itsk_stream_t stream);
/* *flag = value with release semantics (the estimates' ready flag). */
int itsk_flag_store(uint64_t* flag, uint64_t value, itsk_stream_t stream);
/* sizeof(itsk_loop_params) (0), sizeof(itsk_loop_result) (1),
 * sizeof(itsk_peer_params) (2) as compiled into the library; -1 otherwise. */
int64_t itsk_struct_size(int which);
/* Device pointer of the itsk_loop_result inside the loop workspace. */
int itsk_loop_result_ptr(const itsk_loop_params* p, itsk_loop_result** out);

#ifdef __cplusplus
}
#endif
#endif /* ITSK_B200_H_ */
