// Single-CTA dense kernels on the n x n R factor, shared (inline) by the
// stand-alone entry points (trsv.cu) and the loop body (loop.cu).
//
// R: row-major, ld n, upper triangular.  Vectors live in shared memory.
// When the packed upper triangle fits (n <= ~220 for 190 KB), it is staged
// once per kernel into shared memory (RPacked); otherwise R is read from L2
// (RGlobal).  The substitution chains keep the 32x32 diagonal block of the
// current step in registers, so each of the n sequential steps costs a
// divide, a shuffle and an FMA — no memory round trip.
#pragma once
#include "itsk_common.cuh"

namespace itsk {

#ifdef ITSK_DENSE_PROBE
__device__ long long g_probe[8];
#endif

// 512 threads: the register-resident 32x32 diagonal block needs > 64 regs/thread.
constexpr int DENSE_THREADS = 512;

// Index math is 32-bit throughout (n <= 16384 is enforced by the entry points).
struct RGlobal {
  const double* __restrict__ R;
  int nn;
  __device__ __forceinline__ RGlobal(const double* r, int64_t n) : R(r), nn(static_cast<int>(n)) {}
  __device__ __forceinline__ double operator()(int i, int j) const { return R[i * nn + j]; }
  // incremental addressing: element index; (i, j) -> (i + 1, j) adds rstep(i)
  __device__ __forceinline__ int addr(int i, int j) const { return i * nn + j; }
  __device__ __forceinline__ int rstep(int) const { return nn; }
  __device__ __forceinline__ double ld(int a) const { return R[a]; }
};

// upper triangle packed by rows: row i holds R[i][i..n) starting at
// off(i) = i*n - i(i-1)/2; the accessor subtracts i from a per-row base.
struct RPacked {
  uint32_t base;  // shared-window address of the packed triangle
  int nn;
  __device__ __forceinline__ RPacked(const double* P, int64_t n)
      : base(static_cast<uint32_t>(__cvta_generic_to_shared(P))), nn(static_cast<int>(n)) {}
  __device__ __forceinline__ double operator()(int i, int j) const {
    const uint32_t off = static_cast<uint32_t>(i * nn - ((i * (i - 1)) >> 1) + (j - i));
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + off * 8u));  // read-only data: no volatile
    return v;
  }
  // incremental addressing: shared-window byte address; (i, j) -> (i + 1, j)
  // adds rstep(i) = (n - i - 1) * 8
  __device__ __forceinline__ uint32_t addr(int i, int j) const {
    return base + static_cast<uint32_t>(i * nn - ((i * (i - 1)) >> 1) + (j - i)) * 8u;
  }
  __device__ __forceinline__ uint32_t rstep(int i) const { return static_cast<uint32_t>(nn - i - 1) * 8u; }
  __device__ __forceinline__ double ld(uint32_t a) const {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
  }
};

__host__ __device__ __forceinline__ int64_t packed_doubles(int64_t n) { return n * (n + 1) / 2; }

__device__ __forceinline__ void stage_packed(const double* __restrict__ R, int64_t n, double* P) {
  // one flat sweep over R so every thread keeps several independent loads in
  // flight; consecutive threads read consecutive elements
  const int nn = static_cast<int>(n * n), ni = static_cast<int>(n);
#pragma unroll 4
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int i = e / ni, j = e - i * ni;
    const double v = R[e];
    if (j >= i) P[i * ni - ((i * (i - 1)) >> 1) + (j - i)] = v;
  }
  __syncthreads();
}

// Packed upper triangle in global memory (itsk_pack_upper) -> shared memory
// with ONE bulk copy (the row-by-row gather from the dense R is latency bound).
__host__ __device__ __forceinline__ int64_t packed_bytes(int64_t n) {
  return (packed_doubles(n) * 8 + 15) / 16 * 16;
}

// Extended packed layout written by itsk_pack_upper (all offsets in doubles):
//   [0, P0)          upper triangle packed by rows, P0 = packed_bytes(n)/8
//   [P0, P0 + XD)    inverses of the 32x32 diagonal blocks, block B at
//                    P0 + 528 B, packed by rows like the triangle (a partial
//                    last block holds bs(bs+1)/2 entries)
//   [P0 + XD, +nblk) kappa_1 of each diagonal block (||D||_1 ||D^-1||_1)
// A kernel may stage the whole layout or only its first P0 doubles.
constexpr int DIAG_BLK_PACKED = 528;  // 32 * 33 / 2
// Blocks whose 1-norm condition number exceeds this use the substitution
// chain; better-conditioned ones multiply by the stored inverse (forward
// error kappa(D) u either way, and R's diagonal blocks of the sketched
// problems are well conditioned: kappa(D_B) ~ kappa(R)^(32/n)).
constexpr double INVD_COND_MAX = 1.0e4;

__host__ __device__ __forceinline__ int64_t invd_doubles(int64_t n) {
  const int64_t rem = n % 32;
  return (n / 32) * DIAG_BLK_PACKED + rem * (rem + 1) / 2;
}
__host__ __device__ __forceinline__ int64_t nblocks32(int64_t n) { return (n + 31) / 32; }
__host__ __device__ __forceinline__ int64_t rp_doubles(int64_t n) {
  return (packed_bytes(n) / 8 + invd_doubles(n) + nblocks32(n) + 1) / 2 * 2;
}

// Diagonal-block inverses in shared memory (X == nullptr: not available).
struct DiagInv {
  const double* X;
  const double* kap;
  __device__ __forceinline__ bool use(int B) const { return X != nullptr && kap[B] <= INVD_COND_MAX; }
  __device__ __forceinline__ const double* blk(int B) const { return X + B * DIAG_BLK_PACKED; }
};

__device__ __forceinline__ DiagInv diag_inv_at(const double* P, int64_t n, bool with_inv) {
  DiagInv d;
  d.X = with_inv ? P + packed_bytes(n) / 8 : nullptr;
  d.kap = with_inv ? d.X + invd_doubles(n) : nullptr;
  return d;
}

__device__ __forceinline__ void stage_packed_bulk(const double* Rp, int64_t n, double* P, bool with_inv = false) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned bytes = static_cast<unsigned>(with_inv ? rp_doubles(n) * 8 : packed_bytes(n));
    mbar_expect_tx(&bar, bytes);
    bulk_g2s_plain(P, Rp, bytes, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
}

// The kernels below need a scratch area `red` of at least
// 64 * (blockDim.x / 32) doubles in shared memory.

// Software-pipelined blocked substitution (32-wide blocks).  While warp 0
// runs the sequential chain of block I, the other warps already accumulate
// into block I+1 (I-1 for the back solve) the contributions of every block
// that is final; warp 0 then adds only the neighbouring block's 32x32 product
// before starting the next chain.  Per step the chain costs one multiply by
// the precomputed 1/R_kk, one shuffle and one FMA (dtrsv divides; y*(1/d)
// differs from y/d by at most one rounding — the solve stays backward
// stable).  All sums run in a fixed order: results are reproducible.

// y := R^{-T} y   (forward substitution)
template <class RA>
__device__ __forceinline__ void trsv_t_inplace(const RA& R, int n64, double* y, double* red,
                                               DiagInv inv = DiagInv{nullptr, nullptr}) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  // helper warps: those not sharing warp 0's scheduler (warp % 4 != 0), so
  // the sequential block chain of warp 0 issues without competition
  const int nw = blockDim.x >> 5, nh = nw - (nw >> 2);
  const int hidx = warp - (warp >> 2) - 1;
  const int nblk = static_cast<int>((n + 31) / 32);
  // vectors, partials and block inverses all live in shared memory: let the
  // compiler emit LDS/STS instead of generic loads
  if (!__isShared(y) || !__isShared(red)) __builtin_unreachable();
  if (inv.X != nullptr && !__isShared(inv.X)) __builtin_unreachable();
  for (int I = 0; I < nblk; ++I) {
    const int b0 = 32 * I;
    if (warp == 0) {
#ifdef ITSK_DENSE_PROBE
      long long _c0 = clock64();
#endif
      const int bs = static_cast<int>(min(32, n - b0));
      const int jl = min(b0 + lane, n - 1);
      // contributions of blocks < I-1 (helpers, previous step) and of block I-1
      // contributions of blocks < I-1 (helper partials, fixed order)
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (I >= 2) {
        const double* pb = red + (I & 1) * 32 * nw + lane;
#pragma unroll
        for (int w = 1; w < DENSE_THREADS / 32; w += 4) {
          s1 += pb[w * 32];
          if (w + 1 < DENSE_THREADS / 32) s2 += pb[(w + 1) * 32];
          if (w + 2 < DENSE_THREADS / 32) s3 += pb[(w + 2) * 32];
          if (w + 3 < DENSE_THREADS / 32) s0 += pb[(w + 3) * 32];
        }
      }
#ifdef ITSK_DENSE_PROBE
      const double _sdep = s0 + s1 + s2 + s3;
      __syncwarp();
      long long _ca = clock64() + (_sdep == 12345.0 ? 1 : 0);
#endif
      if (I >= 1) {
        // block I-1's rows (final) into block I, two rounds of 16 independent
        // loads feeding 4 FMA chains
        const int pb0 = b0 - 32;
        auto ad = R.addr(pb0, jl);
#pragma unroll
        for (int h2 = 0; h2 < 32; h2 += 16) {
          double rv[16], yv[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            rv[k] = R.ld(ad);
            ad += R.rstep(pb0 + h2 + k);
            yv[k] = y[pb0 + h2 + k];
          }
#pragma unroll
          for (int k = 0; k < 16; k += 4) {
            s0 = fma(rv[k], yv[k], s0);
            s1 = fma(rv[k + 1], yv[k + 1], s1);
            s2 = fma(rv[k + 2], yv[k + 2], s2);
            s3 = fma(rv[k + 3], yv[k + 3], s3);
          }
        }
      }
      const double s = (s0 + s1) + (s2 + s3);
      const double yv = y[jl];
      double yi = (lane < bs) ? yv - s : 0.0;
#ifdef ITSK_DENSE_PROBE
      __syncwarp();
      long long _c1 = clock64() + (yi == 12345.0 ? 1 : 0);
      if (lane == 0) { g_probe[2] += _ca - _c0; g_probe[3] += _c1 - _ca; }
#endif
      if (inv.use(I)) {
        // y_B = X' t with X = D^-1 packed by rows: lane i sums X[k][i] t_k, k <= i
        const double* X = inv.blk(I);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int off = lane;  // X[k][lane] at off(k) + lane - k, off(k+1) - off(k) = bs - k
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          const double t0 = __shfl_sync(FULL, yi, k), t1 = __shfl_sync(FULL, yi, k + 1);
          const double t2 = __shfl_sync(FULL, yi, k + 2), t3 = __shfl_sync(FULL, yi, k + 3);
          const int o0 = off, o1 = o0 + bs - k - 1, o2 = o1 + bs - k - 2, o3 = o2 + bs - k - 3;
          off = o3 + bs - k - 4;
          if (k < lane + 1 && lane < bs) a0 = fma(X[o0], t0, a0);
          if (k + 1 < lane + 1 && lane < bs) a1 = fma(X[o1], t1, a1);
          if (k + 2 < lane + 1 && lane < bs) a2 = fma(X[o2], t2, a2);
          if (k + 3 < lane + 1 && lane < bs) a3 = fma(X[o3], t3, a3);
        }
        yi = (a0 + a1) + (a2 + a3);
      } else {
        double col[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const double v = R(min(b0 + k, n - 1), jl);
          col[k] = (k < lane && lane < bs) ? v : 0.0;
        }
        const double dg = R(jl, jl);
        const double rinv = (lane < bs) ? 1.0 / dg : 0.0;
        // straight-line chain: for k >= bs the step is a no-op (lane k holds 0,
        // col[k] == 0), so no per-step branch / reconvergence is needed
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          if (lane == k) yi *= rinv;
          const double yk = __shfl_sync(FULL, yi, k);
          yi = fma(-col[k], yk, yi);  // col[k] == 0 for lanes <= k
        }
      }
#ifdef ITSK_DENSE_PROBE
      __syncwarp();
      long long _c2 = clock64();
      if (lane == 0) { g_probe[0] += _c1 - _c0; g_probe[1] += _c2 - _c1; }
#endif
      if (lane < bs) y[b0 + lane] = yi;
    } else if (I + 1 < nblk) {
      // helpers: rows [0, b0) (blocks < I, final) into block I+1
      double acc = 0.0;
      if (warp & 3) {
        const int t0 = b0 + 32;
        const int jl = min(t0 + lane, n - 1);
        const int k_lo = (b0 * hidx) / nh, k_hi = (b0 * (hidx + 1)) / nh;
        for (int k = k_lo; k < k_hi; ++k) acc = fma(R(k, jl), y[k], acc);
      }
      red[((I + 1) & 1) * 32 * nw + warp * 32 + lane] = acc;
    }
    __syncthreads();
  }
}

// x := R^{-1} x   (back substitution, blocks from the bottom)
template <class RA>
__device__ __forceinline__ void trsv_n_inplace(const RA& R, int n64, double* x, double* red,
                                               DiagInv inv = DiagInv{nullptr, nullptr}) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  const int nw = blockDim.x >> 5, nh = nw - (nw >> 2);  // helpers: warp % 4 != 0 (see trsv_t_inplace)
  const int hidx = warp - (warp >> 2) - 1;
  const int nblk = static_cast<int>((n + 31) / 32);
  if (!__isShared(x) || !__isShared(red)) __builtin_unreachable();
  if (inv.X != nullptr && !__isShared(inv.X)) __builtin_unreachable();
  for (int I = nblk - 1; I >= 0; --I) {
    const int b0 = 32 * I;
    const int be = min(b0 + 32, n);
    const int bs = static_cast<int>(be - b0);
    if (warp == 0) {
      const int il = min(b0 + lane, n - 1);
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (I + 1 < nblk) s0 = red[(I & 1) * 32 * nw + lane];  // columns beyond block I+1 (helpers)
      if (I + 1 < nblk) {  // block I+1's contribution: row il, columns [be, be+32)
        const int cb = be;
        const int cw = static_cast<int>(min(32, n - cb));
#pragma unroll
        for (int h2 = 0; h2 < 32; h2 += 16) {
          double rv[16], xv[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int kk = h2 + k;
            const int cc = min(cb + kk, n - 1);
            rv[k] = kk < cw ? R(il, cc) : 0.0;
            xv[k] = x[cc];
          }
#pragma unroll
          for (int k = 0; k < 16; k += 4) {
            s1 = fma(rv[k], xv[k], s1);
            s2 = fma(rv[k + 1], xv[k + 1], s2);
            s3 = fma(rv[k + 2], xv[k + 2], s3);
            s0 = fma(rv[k + 3], xv[k + 3], s0);
          }
        }
      }
      const double s = (s0 + s1) + (s2 + s3);
      const double xv = x[il];
      double t = (lane < bs) ? xv - s : 0.0;
      if (inv.use(I)) {
        // x_B = X t: lane i sums X[i][k] t_k over k >= i (row i of the packed block)
        const double* Xr = inv.blk(I) + (lane * bs - ((lane * (lane - 1)) >> 1)) - lane;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          const double t0 = __shfl_sync(FULL, t, k), t1 = __shfl_sync(FULL, t, k + 1);
          const double t2 = __shfl_sync(FULL, t, k + 2), t3 = __shfl_sync(FULL, t, k + 3);
          if (k >= lane && k < bs) a0 = fma(Xr[k], t0, a0);
          if (k + 1 >= lane && k + 1 < bs) a1 = fma(Xr[k + 1], t1, a1);
          if (k + 2 >= lane && k + 2 < bs) a2 = fma(Xr[k + 2], t2, a2);
          if (k + 3 >= lane && k + 3 < bs) a3 = fma(Xr[k + 3], t3, a3);
        }
        t = (lane < bs) ? (a0 + a1) + (a2 + a3) : 0.0;
      } else {
        double row[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const double v = R(il, min(b0 + k, n - 1));
          row[k] = (k > lane && k < bs) ? v : 0.0;
        }
        const double dg = R(il, il);
        const double rinv = (lane < bs) ? 1.0 / dg : 0.0;
#pragma unroll
        for (int k = 31; k >= 0; --k) {  // no-op steps for k >= bs (see trsv_t_inplace)
          if (lane == k) t *= rinv;
          const double xk = __shfl_sync(FULL, t, k);
          t = fma(-row[k], xk, t);  // row[k] == 0 for lanes >= k
        }
      }
      if (lane < bs) x[b0 + lane] = t;
    } else if (I >= 1 && (warp & 3)) {
      // helpers: columns [be + 32, n) (blocks > I+1, final) into the rows of block I-1
      const int tb0 = b0 - 32;
      const int c0 = be;  // blocks > I are final
      for (int rr = hidx; rr < 32; rr += nh) {
        const int i = tb0 + rr;
        double acc = 0.0;
        for (int j = c0 + lane; j < n; j += 32) acc = fma(R(i, j), x[j], acc);
        acc = warp_sum(acc);
        if (lane == 0) red[((I - 1) & 1) * 32 * nw + rr] = acc;
      }
    }
    __syncthreads();
  }
}

// out := R v  (upper): 4 rows per warp at a time, reductions interleaved
template <class RA>
__device__ __forceinline__ void trmv_n(const RA& R, int n64, const double* v, double* out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  const int nw = blockDim.x >> 5;
  for (int i0 = 4 * warp; i0 < n; i0 += 4 * nw) {
    double s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s[u] = 0.0;
      const int i = i0 + u;
      if (i < n)
        for (int j = i + lane; j < n; j += 32) s[u] = fma(R(i, j), v[j], s[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += __shfl_xor_sync(FULL, s[u], o);
    if (lane < 4 && i0 + lane < n) {
      double r = s[0];
#pragma unroll
      for (int u = 1; u < 4; ++u)
        if (lane == u) r = s[u];
      out[i0 + lane] = r;
    }
  }
  __syncthreads();
}

// out := R' v : a warp owns a 32-column block (lane = column j) and runs the
// rows i <= j of that block down two interleaved chains (even / odd i), so
// there is no cross-warp reduction and one barrier at the end.  Row segments
// are contiguous (conflict-free), v[i] is a broadcast.
template <class RA>
__device__ __forceinline__ void trmv_t(const RA& R, int n64, const double* v, double* out,
                                       double* red) {
  (void)red;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(n64);
  const int nw = blockDim.x >> 5;
  const int nblk = (n + 31) / 32;
  // heaviest blocks (the last ones) first
  for (int bb = warp; bb < nblk; bb += nw) {
    const int b = nblk - 1 - bb;
    const int j = 32 * b + lane;
    const int jj = min(j, n - 1);
    double a0 = 0.0, a1 = 0.0;
    int i = 0;
    for (; i + 1 <= jj; i += 2) {
      a0 = fma(R(i, jj), v[i], a0);
      a1 = fma(R(i + 1, jj), v[i + 1], a1);
    }
    if (i == jj) a0 = fma(R(i, jj), v[i], a0);
    if (j < n) out[j] = a0 + a1;
  }
  __syncthreads();
}

__device__ __forceinline__ double dot_sm(const double* a, const double* b, int64_t n, double* red) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += a[i] * b[i];
  return block_sum(s, red);
}

// Shared-memory budget of the single-CTA R kernels.
constexpr int64_t DENSE_SMEM_BUDGET = 200 * 1024;

__host__ __device__ __forceinline__ bool use_packed(int64_t n, int64_t other_doubles) {
  return (packed_doubles(n) + other_doubles) * 8 <= DENSE_SMEM_BUDGET;
}

// the extended layout (triangle + diagonal-block inverses) fits as well
__host__ __device__ __forceinline__ bool use_packed_inv(int64_t n, int64_t other_doubles) {
  return (rp_doubles(n) + other_doubles) * 8 <= DENSE_SMEM_BUDGET;
}

}  // namespace itsk
