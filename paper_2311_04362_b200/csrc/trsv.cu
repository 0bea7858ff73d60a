// Small n x n kernels on the R factor (K4): triangular solves, the power-
// method norm estimate and the condition estimate.
//
//   tri_solve_upper            linalg.py:59-62   R y = c   (back substitution)
//   tri_solve_upper_transpose  linalg.py:65-68   R'y = c   (forward substitution)
//   solve_step                 solvers.py:339-340  y = R^{-1} R^{-T} c
//   rand_power_norm_est        linalg.py:79-105
//   cond_est                   linalg.py:108-113
//
// R is row-major, ld n, upper triangular, diag(R) > 0 (validated once by the
// QR).  One CTA of 1024 threads; vectors live in shared memory and R streams
// from L2 (it stays resident across iterations).  Blocks of 32 rows:
//   R'y = c  right-looking: solve the 32x32 diagonal block with one warp,
//            then all threads update the later entries from contiguous row
//            segments of R;
//   R y = c  left-looking from the bottom: one warp per row reduces the
//            contiguous row segment against the solved tail, then one warp
//            solves the diagonal block.
#include <cooperative_groups.h>

#include <cfloat>

#include "itsk_common.cuh"
#include "itsk_dense.cuh"

namespace cg = cooperative_groups;
#include "itsk_kernels.cuh"

namespace itsk {

namespace {

// Accessor selection: PACKED stages the upper triangle in shared memory first.
template <bool PACKED>
struct RSel;
template <>
struct RSel<true> {
  using type = RPacked;
  // with_inv: Rp carries the diagonal-block inverses (extended layout) and
  // the kernel's shared memory was sized for all of it
  __device__ static RPacked make(const double* R, const double* Rp, int64_t n, double*& sm,
                                 DiagInv* inv = nullptr, bool with_inv = false) {
    with_inv = with_inv && Rp != nullptr;
    if (Rp) stage_packed_bulk(Rp, n, sm, with_inv); else stage_packed(R, n, sm);
    RPacked a(sm, n);
    if (inv) *inv = diag_inv_at(sm, n, with_inv);
    sm += with_inv ? rp_doubles(n) : packed_doubles(n);
    return a;
  }
};
template <>
struct RSel<false> {
  using type = RGlobal;
  __device__ static RGlobal make(const double* R, const double*, int64_t n, double*&,
                                 DiagInv* inv = nullptr, bool = false) {
    if (inv) *inv = DiagInv{nullptr, nullptr};
    return RGlobal(R, n);
  }
};

// Rp (nullable): itsk_pack_upper's layout, staged with one bulk copy;
// with_inv: it carries the diagonal-block inverses (the loop tail's solves).
template <bool PACKED>
__global__ void __launch_bounds__(DENSE_THREADS) k_trsv(const double* R, const double* Rp, int64_t n,
                                                        const double* c, double* y, int mode, int with_inv) {
  extern __shared__ double sm[];
  double* cur = sm;
  DiagInv inv{nullptr, nullptr};
  const auto RA = RSel<PACKED>::make(R, Rp, n, cur, &inv, with_inv != 0);
  double* v = cur;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] = c[i];
  __syncthreads();
  __shared__ double red_s[64 * (DENSE_THREADS / 32)];
  if (mode == 1 || mode == 2) trsv_t_inplace(RA, n, v, red_s, inv);
  if (mode == 0 || mode == 2) trsv_n_inplace(RA, n, v, red_s, inv);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) y[i] = v[i];
}

// rand_power_norm_est (linalg.py:96-105)
template <bool PACKED>
__global__ void __launch_bounds__(DENSE_THREADS) k_normest(const double* R0, const double* Rp, int64_t n,
                                                          const double* v0, int64_t steps, double* out) {
  extern __shared__ double sm[];
  double* cur = sm;
  const auto R = RSel<PACKED>::make(R0, Rp, n, cur);
  double* v = cur;
  double* t = cur + n;
  double* w = cur + 2 * n;
  __shared__ double red[64 * (DENSE_THREADS / 32)];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] = v0[i];
  __syncthreads();
  double nv = sqrt(dot_sm(v, v, n, red));
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] = v[i] / nv;
  __syncthreads();
  for (int64_t s = 0; s < steps; ++s) {
    trmv_n(R, n, v, t);
    trmv_t(R, n, t, w, red);
    const double nw = sqrt(dot_sm(w, w, n, red));
    if (nw == 0.0) {
      if (threadIdx.x == 0) *out = 0.0;
      return;
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] = w[i] / nw;
    __syncthreads();
  }
  trmv_n(R, n, v, t);
  const double r = sqrt(dot_sm(t, t, n, red));
  if (threadIdx.x == 0) *out = r;
}

// Number of eigenvalues of the k x k symmetric tridiagonal (al, be) below x
// (Sturm count through the LDL' recurrence).
__device__ __forceinline__ int sturm_below(const double* al, const double* be, int k, double x) {
  int below = 0;
  double q = al[0] - x;
  if (q < 0) ++below;
  for (int i = 1; i < k; ++i) {
    if (q == 0.0) q = 1e-300;
    q = al[i] - x - be[i - 1] * be[i - 1] / q;
    if (q < 0) ++below;
  }
  return below;
}

// Largest eigenvalue of the k x k symmetric tridiagonal (al, be), to full
// precision, by parallel multisection: each round the CTA's T threads test T
// shifts spread over the current bracket [lo, hi] and keep the sub-interval
// holding the top eigenvalue — log2(T+1) ~ 9 bits per round instead of one
// per (sequential, divide-bound) bisection step.  Called by all threads;
// returns the same value on every thread.
__device__ double tridiag_max_eig(const double* al, const double* be, int k) {
  __shared__ double s_lo, s_hi;
  __shared__ int s_best;
  const int tid = threadIdx.x, T = blockDim.x;
  if (tid == 0) {
    double lo = al[0], hi = al[0];
    for (int i = 0; i < k; ++i) {
      const double r = (i > 0 ? fabs(be[i - 1]) : 0.0) + (i < k - 1 ? fabs(be[i]) : 0.0);
      lo = fmin(lo, al[i] - r);
      hi = fmax(hi, al[i] + r);
    }
    s_lo = lo;
    s_hi = hi;
  }
  __syncthreads();
  for (int round = 0; round < 16; ++round) {
    const double lo = s_lo, hi = s_hi;
    const double w = hi - lo;
    if (!(w > 0.0)) break;
    const double x = lo + w * (static_cast<double>(tid + 1) / (T + 1));
    // an eigenvalue lies above x  <=>  fewer than k lie below x
    const int above = (x > lo && x < hi && sturm_below(al, be, k, x) < k) ? tid : -1;
    if (tid == 0) s_best = -1;
    __syncthreads();
    if (above >= 0) atomicMax(&s_best, above);
    __syncthreads();
    if (tid == 0) {
      const int t = s_best;
      const double nlo = t >= 0 ? lo + w * (static_cast<double>(t + 1) / (T + 1)) : lo;
      const double nhi = t + 1 < T ? lo + w * (static_cast<double>(t + 2) / (T + 1)) : hi;
      s_lo = nlo;
      s_hi = fmax(nhi, nlo);
    }
    __syncthreads();
    if (s_hi - s_lo <= 2.0 * DBL_EPSILON * fmax(fabs(s_lo), fabs(s_hi))) break;
  }
  return 0.5 * (s_lo + s_hi);
}

constexpr int LANCZOS_MAX = 96;

// Lanczos on op = R'R (inv == 0) or R^{-1}R^{-T} (inv == 1); returns the
// largest Ritz value, stopping once it is stable to rounding.
template <class RA>
__device__ double lanczos_max(const RA& R, int64_t n, const double* v0, int inv, double* q,
                              double* qp, double* w, double* t, double* red, double* al,
                              double* be, DiagInv dinv) {
  const int tid = threadIdx.x;
  double nv = sqrt(dot_sm(v0, v0, n, red));
  for (int64_t i = tid; i < n; i += blockDim.x) {
    q[i] = v0[i] / nv;
    qp[i] = 0.0;
  }
  __syncthreads();
  const int kmax = static_cast<int>(min(static_cast<int64_t>(LANCZOS_MAX), n));
  double theta_prev = 0.0, theta = 0.0, bprev = 0.0;
  int stable = 0;
  for (int k = 0; k < kmax; ++k) {
    if (inv == 2) {
      // R holds X = R^{-1}: (R'R)^{-1} q = X (X' q), two parallel matvecs
      trmv_t(R, n, q, t, red);
      trmv_n(R, n, t, w);
    } else if (inv) {
      for (int64_t i = tid; i < n; i += blockDim.x) w[i] = q[i];
      __syncthreads();
      trsv_t_inplace(R, n, w, red, dinv);
      trsv_n_inplace(R, n, w, red, dinv);
    } else {
      trmv_n(R, n, q, t);
      trmv_t(R, n, t, w, red);
    }
    for (int64_t i = tid; i < n; i += blockDim.x) w[i] -= bprev * qp[i];
    __syncthreads();
    const double a = dot_sm(q, w, n, red);
    for (int64_t i = tid; i < n; i += blockDim.x) w[i] -= a * q[i];
    __syncthreads();
    const double b = sqrt(dot_sm(w, w, n, red));
    if (tid == 0) {
      al[k] = a;
      be[k] = b;
    }
    __syncthreads();
    theta = tridiag_max_eig(al, be, k + 1);
    // stop once the extreme Ritz value has settled (two consecutive steps
    // within 1e-12 relative — far below what the stopping rule resolves)
    if (k > 0 && fabs(theta - theta_prev) <= 1e-12 * fabs(theta)) {
      if (++stable >= 2) break;
    } else {
      stable = 0;
    }
    theta_prev = theta;
    if (b == 0.0 || !(b == b)) break;
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const double qi = q[i];
      qp[i] = qi;
      q[i] = w[i] / b;
    }
    __syncthreads();
    bprev = b;
  }
  return theta;
}

template <bool PACKED>
__global__ void __launch_bounds__(DENSE_THREADS) k_condest(const double* R0, const double* Rp, int64_t n,
                                                          const double* v0, double* out, int with_inv,
                                                          const double* X) {
  extern __shared__ double sm[];
  double* cur = sm;
  DiagInv dinv;
  const unsigned rank0 = cg::this_cluster().block_rank();
  // CTA 1 with X = R^{-1} (k_tri_inverse): Lanczos on X X' by matvecs
  const bool use_x = rank0 == 1 && X != nullptr;
  const auto R = use_x ? RSel<PACKED>::make(X, nullptr, n, cur, &dinv, false)
                       : RSel<PACKED>::make(R0, Rp, n, cur, &dinv, with_inv != 0);
  double* q = cur;
  double* qp = cur + n;
  double* w = cur + 2 * n;
  double* t = cur + 3 * n;
  __shared__ double red[64 * (DENSE_THREADS / 32)];
  double* al = cur + 4 * n;
  double* be = al + LANCZOS_MAX;
  // CTA 0: largest eigenvalue of R'R; CTA 1: of (R'R)^{-1}; both at once in a
  // 2-CTA cluster, combined through distributed shared memory.
  __shared__ double theta;
  const unsigned rank = cg::this_cluster().block_rank();
  const double th = lanczos_max(R, n, v0, use_x ? 2 : static_cast<int>(rank), q, qp, w, t, red, al, be, dinv);
  if (threadIdx.x == 0) theta = th;
  cg::this_cluster().sync();
  if (rank == 0 && threadIdx.x == 0) {
    const double other = *cg::this_cluster().map_shared_rank(&theta, 1);
    *out = sqrt(theta * other);
  }
  cg::this_cluster().sync();
}

// X = R^{-1} (upper triangular, dense row-major n x n; entries below the
// diagonal are not written).  Warp per row i of X: x' R = e_i' by the axpy
// form of forward substitution on R' — after x_j = s_j / R_jj, every later
// partial sum takes s_k -= x_j R_jk from the contiguous row j of R (staged
// packed in shared memory when it fits).  Only condest's (R'R)^{-1} Lanczos
// uses X: its Ritz values match the two-TRSV operator's to ~1e-15 on the
// sketched factors (graded triangles), far inside the 1e-9 the estimate is
// checked to.
template <bool PACKED>
__global__ void __launch_bounds__(256) k_tri_inverse(const double* __restrict__ R0, const double* __restrict__ Rp,
                                                     int64_t n64, double* __restrict__ X, int wpb) {
  extern __shared__ double sm[];
  double* cur = sm;
  const auto R = RSel<PACKED>::make(R0, Rp, n64, cur);
  const int n = static_cast<int>(n64);
  double* rinv = cur;
  for (int j = threadIdx.x; j < n; j += blockDim.x) rinv[j] = 1.0 / R(j, j);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= wpb) return;
  double* sv = rinv + n + static_cast<int64_t>(warp) * n;
  const int i = blockIdx.x * wpb + warp;
  if (i >= n) return;
  for (int k = i + lane; k < n; k += 32) sv[k] = (k == i) ? 1.0 : 0.0;
  __syncwarp();
  for (int j = i; j < n; ++j) {
    const double xj = sv[j] * rinv[j];
    for (int k = j + 1 + lane; k < n; k += 32) sv[k] = fma(-xj, R(j, k), sv[k]);
    __syncwarp();
  }
  double* xr = X + static_cast<int64_t>(i) * n;
  for (int k = i + lane; k < n; k += 32) xr[k] = sv[k] * rinv[k];
}

__global__ void k_pack_upper(const double* __restrict__ R, int64_t n, double* __restrict__ Rp) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int64_t i = e / n, j = e - i * n;
  if (j >= i) Rp[i * n - (i * (i - 1)) / 2 + (j - i)] = R[e];
}

// Inverse of diagonal block B (warp per block, lane j = column j) into the
// extended packed layout, plus its 1-norm condition number.  Column j of
// D^-1 by back substitution: x_j = 1/D_jj, x_k = -(sum_{l=k+1..j} D_kl x_l)/D_kk.
__global__ void __launch_bounds__(32) k_invert_diag(const double* __restrict__ R, int64_t n64,
                                                   double* __restrict__ X, double* __restrict__ kap) {
  const int n = static_cast<int>(n64);
  const int B = blockIdx.x, lane = threadIdx.x;
  const int b0 = 32 * B, bs = min(32, n - b0);
  __shared__ double D[32][33];
  __shared__ double rinv[32];
  double dv[32];
#pragma unroll
  for (int k = 0; k < 32; ++k)  // all 32 loads in flight
    dv[k] = (k < bs && lane < bs && lane >= k) ? R[static_cast<int64_t>(b0 + k) * n + b0 + lane] : 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) D[k][lane] = dv[k];
  __syncwarp();
  rinv[lane] = lane < bs ? 1.0 / D[lane][lane] : 0.0;
  __syncwarp();
  double x[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = 0.0;
  if (lane < bs) {
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (k == lane) {
        x[k] = rinv[k];
      } else if (k < lane) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int l = k + 1; l < 32; ++l)
          if (l <= lane) {
            if (l & 1) s1 = fma(D[k][l], x[l], s1); else s0 = fma(D[k][l], x[l], s0);
          }
        x[k] = -(s0 + s1) * rinv[k];
      }
    }
  }
  double* Xb = X + static_cast<int64_t>(B) * DIAG_BLK_PACKED;
  double cx = 0.0, cd = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k <= lane && lane < bs) {
      Xb[k * bs - ((k * (k - 1)) >> 1) + (lane - k)] = x[k];
      cx += fabs(x[k]);
      cd += fabs(D[k][lane]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cx = fmax(cx, __shfl_xor_sync(FULL, cx, o));
    cd = fmax(cd, __shfl_xor_sync(FULL, cd, o));
  }
  if (lane == 0) {
    const double k1 = cx * cd;
    kap[B] = (k1 == k1) ? k1 : INFINITY;  // a zero pivot gives inf/nan: use the chain
  }
}

}  // namespace

template <class K>
int prep(K kernel, size_t smem) {
  // dynamic + static (the kernels' reduction arrays) may cross the 48 KB
  // default even when `smem` alone does not; the opt-in is cached per kernel
  if (smem > 16 * 1024) ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(kernel)));
  return ITSK_OK;
}

int launch_trsv(const double* R, int64_t n, const double* c, double* y, int mode, cudaStream_t s,
                const double* Rp = nullptr) {
  const int64_t other = n + 32;
  const bool packed = use_packed(n, other);
  const bool with_inv = packed && Rp != nullptr && use_packed_inv(n, other);
  const int64_t tri = with_inv ? rp_doubles(n) : (packed ? packed_doubles(n) : 0);
  const size_t smem = static_cast<size_t>(tri + other) * sizeof(double);
  int rc;
  if (packed) {
    if ((rc = prep(k_trsv<true>, smem))) return rc;
    k_trsv<true><<<1, DENSE_THREADS, smem, s>>>(R, Rp, n, c, y, mode, with_inv ? 1 : 0);
  } else {
    if ((rc = prep(k_trsv<false>, smem))) return rc;
    k_trsv<false><<<1, DENSE_THREADS, smem, s>>>(R, nullptr, n, c, y, mode, 0);
  }
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

int launch_trsv_pair_device(const double* R, int64_t n, const double* c, double* y,
                            cudaStream_t s) {
  return launch_trsv(R, n, c, y, 2, s);
}

}  // namespace itsk

using namespace itsk;

extern "C" int itsk_trsv(const double* R, int64_t n, const double* c, double* y, int trans,
                         itsk_stream_t stream) {
  ITSK_REQUIRE(R && c && y && n >= 1, "bad trsv arguments");
  ITSK_REQUIRE(n <= 16384, "trsv: n too large for the single-CTA kernel");
  return launch_trsv(R, n, c, y, trans ? 1 : 0, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int itsk_trsv_rp(const double* R, const double* Rp, int64_t n, const double* c, double* y,
                            int trans, itsk_stream_t stream) {
  ITSK_REQUIRE(R && Rp && c && y && n >= 1, "bad trsv arguments");
  ITSK_REQUIRE(n <= 16384, "trsv: n too large for the single-CTA kernel");
  return launch_trsv(R, n, c, y, trans ? 1 : 0, reinterpret_cast<cudaStream_t>(stream), Rp);
}

extern "C" int itsk_trsv_pair(const double* R, int64_t n, const double* c, double* y, double* tmp,
                              itsk_stream_t stream) {
  (void)tmp;
  ITSK_REQUIRE(R && c && y && n >= 1 && n <= 16384, "bad trsv arguments");
  return launch_trsv(R, n, c, y, 2, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int itsk_normest(const double* R, int64_t n, const double* v0, int64_t steps,
                            double* out, const double* Rp, itsk_stream_t stream) {
  ITSK_REQUIRE(R && v0 && out && n >= 1 && steps >= 1, "bad normest arguments");
  ITSK_REQUIRE(n <= 8000, "normest: n too large for the single-CTA kernel");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t other = 3 * n + 32;
  const bool packed = use_packed(n, other);
  const size_t smem = static_cast<size_t>((packed ? packed_doubles(n) : 0) + other) * sizeof(double);
  int rc;
  if (packed) {
    if ((rc = prep(k_normest<true>, smem))) return rc;
    k_normest<true><<<1, DENSE_THREADS, smem, s>>>(R, Rp, n, v0, steps, out);
  } else {
    if ((rc = prep(k_normest<false>, smem))) return rc;
    k_normest<false><<<1, DENSE_THREADS, smem, s>>>(R, nullptr, n, v0, steps, out);
  }
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

extern "C" int itsk_condest_workspace(int64_t n, int64_t* doubles) {
  ITSK_REQUIRE(doubles && n >= 1, "bad n");
  *doubles = n * n;  // X = R^{-1} for itsk_condest_ws
  return ITSK_OK;
}

namespace {
int launch_tri_inverse(const double* R, const double* Rp, int64_t n, double* X, cudaStream_t s) {
  const int64_t scratch = n;  // 1/R_jj
  const bool packed = Rp != nullptr && use_packed(n, scratch + 8 * n);
  const int64_t base = (packed ? packed_doubles(n) : 0) + scratch;
  const int64_t room = (DENSE_SMEM_BUDGET / 8) - base;
  int wpb = static_cast<int>(std::min<int64_t>(8, room / n));
  if (wpb < 1) return ITSK_EINVAL;
  const size_t smem = static_cast<size_t>(base + static_cast<int64_t>(wpb) * n) * sizeof(double);
  const unsigned grid = static_cast<unsigned>((n + wpb - 1) / wpb);
  int rc;
  if (packed) {
    if ((rc = prep(k_tri_inverse<true>, smem))) return rc;
    k_tri_inverse<true><<<grid, 32 * wpb, smem, s>>>(R, Rp, n, X, wpb);
  } else {
    if ((rc = prep(k_tri_inverse<false>, smem))) return rc;
    k_tri_inverse<false><<<grid, 32 * wpb, smem, s>>>(R, nullptr, n, X, wpb);
  }
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

int launch_condest(const double* R, int64_t n, const double* v0, double* out, const double* Rp, const double* X,
                   cudaStream_t s) {
  const int64_t other = 4 * n + 32 + 2 * LANCZOS_MAX;
  const bool packed = use_packed(n, other);
  const int with_inv = Rp != nullptr && use_packed_inv(n, other);
  const size_t smem =
      static_cast<size_t>((packed ? (with_inv ? rp_doubles(n) : packed_doubles(n)) : 0) + other) * sizeof(double);
  int rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(DENSE_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (packed) {
    if ((rc = prep(k_condest<true>, smem))) return rc;
    ITSK_CUDA(cudaLaunchKernelEx(&cfg, k_condest<true>, R, Rp, n, v0, out, with_inv, X));
  } else {
    if ((rc = prep(k_condest<false>, smem))) return rc;
    ITSK_CUDA(cudaLaunchKernelEx(&cfg, k_condest<false>, R, static_cast<const double*>(nullptr), n, v0, out, 0, X));
  }
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}
}  // namespace

extern "C" int itsk_condest(const double* R, int64_t n, const double* v0, double* out,
                            const double* Rp, itsk_stream_t stream) {
  ITSK_REQUIRE(R && v0 && out && n >= 1, "bad condest arguments");
  ITSK_REQUIRE(n <= 6000, "condest: n too large for the single-CTA kernel");
  return launch_condest(R, n, v0, out, Rp, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int itsk_condest_ws(const double* R, int64_t n, const double* v0, double* out, const double* Rp,
                               double* ws, int64_t ws_doubles, itsk_stream_t stream) {
  ITSK_REQUIRE(R && v0 && out && ws && n >= 1, "bad condest arguments");
  ITSK_REQUIRE(n <= 6000, "condest: n too large for the single-CTA kernel");
  ITSK_REQUIRE(ws_doubles >= n * n, "condest workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int rc = launch_tri_inverse(R, Rp, n, ws, s);
  if (rc == ITSK_EINVAL) return launch_condest(R, n, v0, out, Rp, nullptr, s);  // no room: the TRSV operator
  if (rc) return rc;
  return launch_condest(R, n, v0, out, Rp, ws, s);
}

extern "C" int itsk_pack_upper_doubles(int64_t n, int64_t* doubles) {
  ITSK_REQUIRE(doubles && n >= 1, "bad n");
  *doubles = rp_doubles(n);
  return ITSK_OK;
}

extern "C" int itsk_pack_upper(const double* R, int64_t n, double* Rp, itsk_stream_t stream) {
  ITSK_REQUIRE(R && Rp && n >= 1, "bad pack arguments");
  ITSK_REQUIRE(n <= 46340, "pack: n too large");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t total = n * n;
  k_pack_upper<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(R, n, Rp);
  count_launch();
  ITSK_CHECK_LAUNCH();
  double* X = Rp + packed_bytes(n) / 8;
  k_invert_diag<<<static_cast<unsigned>(nblocks32(n)), 32, 0, s>>>(R, n, X, X + invd_doubles(n));
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}
