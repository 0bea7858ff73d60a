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
      const double r = bj - dot;
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

__global__ void k_finalize(const double* __restrict__ part, int grid, int64_t n, double* cs,
                           const LoopCtl* ctl) {
  if (ctl && ctl->result.done) return;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n + 4) return;
  double s = 0.0;
  for (int g = 0; g < grid; ++g) s += part[static_cast<int64_t>(g) * (n + 4) + c];
  cs[c] = s;
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
    cudaFuncSetAttribute(k_pass<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
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
  blocks_per_sm<CPL>();  // sets the smem attribute once
  k_pass<CPL><<<grid, PASS_THREADS, smem, s>>>(a);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace

int pass_grid(int64_t m, int64_t n) {
  const int cpl = cpl_for(n);
  int64_t g = static_cast<int64_t>(num_sms()) * occupancy_for(cpl);
  const int64_t cap = (m + PASS_WARPS - 1) / PASS_WARPS;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

int64_t pass_part_doubles(int64_t m, int64_t n) {
  return static_cast<int64_t>(pass_grid(m, n)) * (n + 4);
}

int launch_pass(const PassArgs& a0, cudaStream_t s) {
  PassArgs a = a0;
  const int grid = pass_grid(a.m, a.n);
  a.rows_per_cta = (a.m + grid - 1) / grid;
  switch (cpl_for(a.n)) {
    case 1: return launch_cpl<1>(a, grid, s);
    case 2: return launch_cpl<2>(a, grid, s);
    case 4: return launch_cpl<4>(a, grid, s);
    case 8: return launch_cpl<8>(a, grid, s);
    case 16: return launch_cpl<16>(a, grid, s);
    case 32: return launch_cpl<32>(a, grid, s);
    default:
      set_error("fused pass: n=%lld exceeds the register-resident row limit (1024)",
                (long long)a.n);
      return ITSK_EINVAL;
  }
}

int launch_finalize(const double* part, int grid, int64_t n, double* cs, const LoopCtl* ctl,
                    cudaStream_t s) {
  const int t = 128;
  k_finalize<<<static_cast<unsigned>((n + 4 + t - 1) / t), t, 0, s>>>(part, grid, n, cs, ctl);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace itsk

using namespace itsk;

extern "C" int itsk_pass_workspace(int64_t m, int64_t n, int64_t* bytes) {
  ITSK_REQUIRE(bytes && m >= 1 && n >= 1, "bad pass shape");
  *bytes = pass_part_doubles(m, n) * static_cast<int64_t>(sizeof(double)) + 256;
  return ITSK_OK;
}

extern "C" int itsk_fused_pass(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                               const double* x, const double* r_prev, double* r_out,
                               const double* r_true, double* cs, void* ws, int64_t ws_bytes,
                               itsk_stream_t stream) {
  ITSK_REQUIRE(A && b && x && cs && ws, "null pointer");
  ITSK_REQUIRE(m >= 1 && n >= 1 && lda >= n, "bad pass shape");
  ITSK_REQUIRE(pass_part_doubles(m, n) * 8 <= ws_bytes, "pass workspace too small");
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
  a.part = static_cast<double*>(ws);
  a.mode = 0;
  int rc = launch_pass(a, s);
  if (rc) return rc;
  return launch_finalize(a.part, pass_grid(m, n), n, cs, nullptr, s);
}
