// The loop's triangular-solve pair d = R^{-1} R^{-T} c (solvers.py:339-340,
// linalg.py:59-68) on a cluster of TCL_NC CTAs, for large n (C4: n = 2000,
// where one CTA streaming R's 16 MB triangle from L2 spent ~0.6 ms per pair).
//
// R is split in 32-wide blocks, block b owned by CTA b % TCL_NC (round
// robin: the late, expensive blocks spread over the cluster).  Forward
// substitution R^T y = c, per owned block b:
//     y_b = D_b^{-T} (c_b - sum_{j<b} R_{j,b}^T y_j)
// The chain warp of b prefetches R_{b-1,b} (the last term) into registers,
// waits for y_{b-1}, adds that term to the helper warps' partial sums of the
// terms j <= b-2, solves the diagonal block (its stored inverse, or a
// register substitution chain when the block is ill conditioned), and
// pushes y_b into every CTA's shared memory: every lane sends its value to
// each CTA with st.async, which completes 8 bytes of the block's mbarrier
// there — the waiters' try_wait wakes when all 256 bytes have landed (no
// release fence behind 32 remote stores, no polled flag).  Helper warps take the terms j <= b-2 of every
// owned block, j = h, h + NH, ... ascending: the R block is loaded before
// y_j arrives, so a term is added ~a hundred cycles after its y_j lands.
// Backward substitution R x = y mirrors it from the last block down.  Every
// sum runs in a fixed order (helper partials in ascending j, combined in
// helper order), so d is reproducible bit for bit.
#pragma once
#include <cooperative_groups.h>

#include "itsk_common.cuh"
#include "itsk_dense.cuh"

namespace itsk {

constexpr int TCL_NC = 16;         // CTAs per cluster (non-portable size)
constexpr int TCL_KO_MAX = 8;      // owned 32-blocks per CTA: n <= TCL_NC * TCL_KO_MAX * 32 = 4096
constexpr int TCL_NMAX = TCL_NC * TCL_KO_MAX * 32;
constexpr int TCL_DS = 33;         // padded stride of the staged diagonal inverses

__host__ __device__ __forceinline__ int tcl_ko(int64_t n) {
  return static_cast<int>((nblocks32(n) + TCL_NC - 1) / TCL_NC);
}

// dynamic shared memory of the cluster pair (doubles, then words)
__host__ __device__ __forceinline__ size_t tcl_smem_bytes(int64_t n) {
  const int64_t nb = nblocks32(n), ko = tcl_ko(n), nh = 16 - ko;
  const int64_t dbl = 2 * nb * 32 + nh * ko * 32 * 2 + ko * 32 * TCL_DS + 2 * nb /* mbarriers */;
  const int64_t words = 2 * ko + ko;
  return static_cast<size_t>(dbl * 8 + words * 4 + 64);
}

__device__ __forceinline__ uint32_t tcl_mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// 8 bytes into a CTA of the cluster, counted on that CTA's mbarrier when they land
__device__ __forceinline__ void tcl_st_async(uint32_t a, double v, uint32_t bar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(a),
               "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tcl_wait_count(const unsigned* p, unsigned target) {
  while (*reinterpret_cast<const volatile unsigned*>(p) < target) __nanosleep(20);
  __threadfence_block();
}

struct TclShared {
  double* yv;       // n (+pad): y of every block, as it lands
  double* xv;       // n: x of every block
  double* acc;      // NH x KO x 2 x 32: helper partials (forward, backward)
  double* dinv;     // KO x 32 x TCL_DS: the owned blocks' diagonal inverses (dense)
  uint64_t* rdyF;   // nb mbarriers: y_b landed here (256 bytes each, phase 0)
  uint64_t* rdyB;   // nb mbarriers: x_b landed here
  unsigned* cntF;   // KO: helper terms added (forward)
  unsigned* cntB;   // KO: helper terms added (backward)
  int* dok;         // KO: the stored inverse is usable
};

__device__ __forceinline__ TclShared tcl_carve(void* base, int64_t n) {
  const int nb = static_cast<int>(nblocks32(n)), ko = tcl_ko(n), nh = 16 - ko;
  TclShared s;
  double* d = static_cast<double*>(base);
  s.yv = d;
  s.xv = s.yv + nb * 32;
  s.acc = s.xv + nb * 32;
  s.dinv = s.acc + nh * ko * 64;
  s.rdyF = reinterpret_cast<uint64_t*>(s.dinv + ko * 32 * TCL_DS);
  s.rdyB = s.rdyF + nb;
  unsigned* w = reinterpret_cast<unsigned*>(s.rdyB + nb);
  s.cntF = w;
  s.cntB = s.cntF + ko;
  s.dok = reinterpret_cast<int*>(s.cntB + ko);
  return s;
}

// One call per CTA of the cluster (512 threads each).  c: global (n).
// Emit(b, lane, value) receives d of block b's row 32 b + lane from the
// owner's chain warp (lane < block size).  Rp: itsk_pack_upper's layout
// (for the diagonal inverses and their kappa), or nullptr (substitution).
template <class Emit>
__device__ void trsv_pair_cluster(const double* __restrict__ R, const double* __restrict__ Rp, int n,
                                  const double* __restrict__ c, void* smem, Emit emit) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int q = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = static_cast<int>(nblocks32(n)), ko = tcl_ko(n), nh = 16 - ko;
  TclShared S = tcl_carve(smem, n);
  // ---- setup: flags / counters zero, the owned diagonal inverses staged ----
  for (int i = tid; i < nb; i += blockDim.x) {
    // one arrival (this thread's, with the 256 bytes every block publishes:
    // lanes past a short last block send zeros) arms phase 0 of each barrier
    mbar_init(&S.rdyF[i], 1);
    mbar_init(&S.rdyB[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&S.rdyF[i], 256);
    mbar_expect_tx(&S.rdyB[i], 256);
  }
  if (tid < ko) {
    S.cntF[tid] = 0u;
    S.cntB[tid] = 0u;
  }
  for (int i = tid; i < nh * ko * 64; i += blockDim.x) S.acc[i] = 0.0;
  const double* X = Rp ? Rp + packed_bytes(n) / 8 : nullptr;
  const double* kap = Rp ? X + invd_doubles(n) : nullptr;
  for (int k = warp; k < ko; k += 16) {
    const int b = q + TCL_NC * k;
    double* Dk = S.dinv + k * 32 * TCL_DS;
    if (b < nb) {
      const int bs = min(32, n - 32 * b);
      const bool ok = X != nullptr && kap[b] <= INVD_COND_MAX;
      if (lane == 0) S.dok[k] = ok ? 1 : 0;
      if (ok) {
        // packed by rows: row r holds X[r][r..bs) at off(r) = r bs - r(r-1)/2
        const double* Xb = X + static_cast<int64_t>(DIAG_BLK_PACKED) * b;
        for (int r = 0; r < 32; ++r) {
          const int off = r * bs - ((r * (r - 1)) >> 1);
          Dk[r * TCL_DS + lane] = (r < bs && lane >= r && lane < bs) ? Xb[off + lane - r] : 0.0;
        }
      }
    }
  }
  cl.sync();  // every CTA's barriers armed before any remote store
  const uint32_t yv_a = smem_u32(S.yv), xv_a = smem_u32(S.xv);
  const uint32_t rf_a = smem_u32(S.rdyF), rb_a = smem_u32(S.rdyB);

  // publish the 32 values of block b (val in lane i) into every CTA's vec:
  // lane i sends its value to each CTA and counts it on that CTA's barrier b
  auto publish = [&](int b, double val, uint32_t vec_a, uint32_t bar_a) {
    const uint32_t va = vec_a + static_cast<uint32_t>(32 * b + lane) * 8u, ba = bar_a + 8u * b;
#pragma unroll
    for (int r = 0; r < TCL_NC; ++r) tcl_st_async(tcl_mapa(va, r), val, tcl_mapa(ba, r));
  };

  // ================= forward: R^T y = c =================
  if (warp < ko) {
    const int k = warp, b = q + TCL_NC * k;
    if (b < nb) {
      const int b0 = 32 * b, bs = min(32, n - b0);
      const int col = b0 + min(lane, bs - 1);
      // the last term's block R_{b-1,b}: column `col`, rows of block b-1
      double rb[32];
      if (b >= 1) {
#pragma unroll
        for (int t = 0; t < 32; ++t) rb[t] = R[static_cast<int64_t>(b0 - 32 + t) * n + col];
      }
      const double cb = c[col];
      // helper terms j <= b-2
      if (b >= 2) tcl_wait_count(&S.cntF[k], static_cast<unsigned>(b - 1));
      double s = 0.0;
      for (int h = 0; h < nh; ++h) s += S.acc[(h * ko + k) * 64 + lane];
      if (b >= 1) {
        mbar_wait(&S.rdyF[b - 1], 0);
        const double* yp = S.yv + b0 - 32;
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          t0 = fma(rb[t], yp[t], t0);
          t1 = fma(rb[t + 1], yp[t + 1], t1);
        }
        s += t0 + t1;
      }
      double t = lane < bs ? cb - s : 0.0;
      double y;
      if (S.dok[k]) {
        // y_i = sum_{r <= i} X[r][i] t_r
        const double* Dk = S.dinv + k * 32 * TCL_DS;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int r = 0; r < 32; r += 2) {
          a0 = fma(Dk[r * TCL_DS + lane], __shfl_sync(FULL, t, r), a0);
          a1 = fma(Dk[(r + 1) * TCL_DS + lane], __shfl_sync(FULL, t, r + 1), a1);
        }
        y = lane < bs ? a0 + a1 : 0.0;
      } else {
        // substitution with D_b's column `col` in registers
        double dc[32];
#pragma unroll
        for (int r = 0; r < 32; ++r)
          dc[r] = (r < lane && lane < bs && r < bs) ? R[static_cast<int64_t>(b0 + r) * n + col] : 0.0;
        const double rinv = lane < bs ? 1.0 / R[static_cast<int64_t>(col) * n + col] : 0.0;
        y = t;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          if (lane == r) y *= rinv;
          const double yr = __shfl_sync(FULL, y, r);
          y = fma(-dc[r], yr, y);
        }
      }
      publish(b, y, yv_a, rf_a);
    }
  } else {
    // helpers: terms j <= b-2 of the owned blocks, j = h, h + NH, ...
    const int h = warp - ko;
    for (int j = h; j < nb; j += nh) {
      for (int k = 0; k < ko; ++k) {
        const int b = q + TCL_NC * k;
        if (b >= nb || b < j + 2) continue;
        const int b0 = 32 * b, bs = min(32, n - b0);
        const int col = b0 + min(lane, bs - 1);
        double rv[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) rv[t] = R[static_cast<int64_t>(32 * j + t) * n + col];
        mbar_wait(&S.rdyF[j], 0);
        const double* yp = S.yv + 32 * j;
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          t0 = fma(rv[t], yp[t], t0);
          t1 = fma(rv[t + 1], yp[t + 1], t1);
        }
        double* ap = S.acc + (h * ko + k) * 64 + lane;
        *ap += t0 + t1;
        __syncwarp();
        __threadfence_block();
        if (lane == 0) atomicAdd(&S.cntF[k], 1u);
      }
    }
  }
  cl.sync();  // y complete everywhere; the forward counters / partials are done with

  // ================= backward: R x = y =================
  if (warp < ko) {
    const int k = warp, b = q + TCL_NC * k;
    if (b < nb) {
      const int b0 = 32 * b, bs = min(32, n - b0);
      const int row = b0 + min(lane, bs - 1);
      // the last term's block R_{b,b+1}: row `row`, columns of block b+1
      double rb[32];
      const int nb1 = b + 1 < nb ? min(32, n - b0 - 32) : 0;
#pragma unroll
      for (int t = 0; t < 32; ++t) rb[t] = t < nb1 ? R[static_cast<int64_t>(row) * n + b0 + 32 + t] : 0.0;
      mbar_wait(&S.rdyF[b], 0);  // this CTA's own copy of y_b (sent like the others)
      const double yb = S.yv[row];
      const int after = nb - 2 - b;  // helper terms j >= b+2
      if (after > 0) tcl_wait_count(&S.cntB[k], static_cast<unsigned>(after));
      double s = 0.0;
      for (int hh = 0; hh < nh; ++hh) s += S.acc[(hh * ko + k) * 64 + 32 + lane];
      if (nb1 > 0) {
        mbar_wait(&S.rdyB[b + 1], 0);
        const double* xp = S.xv + b0 + 32;
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          t0 = fma(rb[t], xp[t], t0);
          t1 = fma(rb[t + 1], xp[t + 1], t1);
        }
        s += t0 + t1;
      }
      double t = lane < bs ? yb - s : 0.0;
      double x;
      if (S.dok[k]) {
        // x_i = sum_{r >= i} X[i][r] t_r
        const double* Dk = S.dinv + k * 32 * TCL_DS;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int r = 0; r < 32; r += 2) {
          a0 = fma(Dk[lane * TCL_DS + r], __shfl_sync(FULL, t, r), a0);
          a1 = fma(Dk[lane * TCL_DS + r + 1], __shfl_sync(FULL, t, r + 1), a1);
        }
        x = lane < bs ? a0 + a1 : 0.0;
      } else {
        double dr[32];
#pragma unroll
        for (int r = 0; r < 32; ++r)
          dr[r] = (r > lane && r < bs && lane < bs) ? R[static_cast<int64_t>(row) * n + b0 + r] : 0.0;
        const double rinv = lane < bs ? 1.0 / R[static_cast<int64_t>(row) * n + row] : 0.0;
        x = t;
#pragma unroll
        for (int r = 31; r >= 0; --r) {
          if (lane == r) x *= rinv;
          const double xr = __shfl_sync(FULL, x, r);
          x = fma(-dr[r], xr, x);
        }
      }
      publish(b, x, xv_a, rb_a);
      if (lane < bs) emit(b, lane, x);
    }
  } else {
    // helpers: terms j >= b+2 of the owned blocks, j = nb-1-h, nb-1-h-NH, ... descending
    const int h = warp - ko;
    for (int j = nb - 1 - h; j >= 0; j -= nh) {
      for (int k = 0; k < ko; ++k) {
        const int b = q + TCL_NC * k;
        if (b >= nb || j < b + 2) continue;
        const int b0 = 32 * b, bs = min(32, n - b0);
        const int row = b0 + min(lane, bs - 1);
        const int js = min(32, n - 32 * j);
        double rv[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) rv[t] = t < js ? R[static_cast<int64_t>(row) * n + 32 * j + t] : 0.0;
        mbar_wait(&S.rdyB[j], 0);
        const double* xp = S.xv + 32 * j;
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          t0 = fma(rv[t], xp[t], t0);
          t1 = fma(rv[t + 1], xp[t + 1], t1);
        }
        double* ap = S.acc + (h * ko + k) * 64 + 32 + lane;
        *ap += t0 + t1;
        __syncwarp();
        __threadfence_block();
        if (lane == 0) atomicAdd(&S.cntB[k], 1u);
      }
    }
  }
  // every block's values have landed here (asynchronous stores complete only
  // on the barriers), then: no CTA exits while another may still store into it
  for (int i = tid; i < 2 * nb; i += blockDim.x) mbar_wait(&S.rdyF[i], 0);  // rdyB follows rdyF
  cl.sync();
}

}  // namespace itsk
