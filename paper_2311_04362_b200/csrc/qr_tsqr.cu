// Communication-avoiding Householder QR of the augmented sketch [SA | Sb]
// inside one thread-block cluster (the cluster path of K2).
//
// Same contract as qr.cu (householder_qr_econ, linalg.py:30-47, and Q'Sb,
// solvers.py:209), different schedule.  The column-by-column algorithm needs
// one cluster-wide exchange per column (n of them); here every 32-wide panel
// costs one local QR per CTA plus a log2(C)-level reduction tree (TSQR /
// CAQR, Demmel et al.):
//
//   1. each CTA factors the panel rows it owns (Householder, shared memory,
//      no cross-CTA traffic) and applies its reflectors to its own trailing
//      rows (compact-WY, DMMA tiles);
//   2. pairs of CTAs merge their 32x32 R factors: the stacked 64x32 matrix is
//      factored and its reflectors are applied to the two CTAs' top trailing
//      rows; after log2(C) levels CTA 0 holds the panel's final R rows;
//   3. CTA 0 retires those rows (they are rows k0..k0+kb-1 of R, and their Sb
//      entries are z = Q'Sb); all other rows stay active for the next panel.
//
// Householder QR is backward stable in any such order, so R matches LAPACK's
// to rounding (tests/test_gpu_parity.py).  All reductions run in a fixed
// order: the result is bitwise reproducible.
#include <cooperative_groups.h>

#include <algorithm>

#include "itsk_common.cuh"
#include "itsk_kernels.cuh"

namespace cg = cooperative_groups;

namespace itsk {
namespace {

constexpr int TB = 32;             // panel width
constexpr int TP = TB + 1;         // padded row stride of panel-shaped smem blocks
constexpr int TT = 512;            // threads per CTA
constexpr int TW = TT / 32;
constexpr int RTL = 32;            // row tile of the trailing updates
constexpr int CBL = 64;            // column chunk of the trailing updates
constexpr int CBLP = CBL + 4;      // padded stride of staged tiles

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = valid ? 8 : 0;  // src-size 0 zero-fills the destination
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct TsqrArgs {
  double* W;
  int64_t d, n, ldw, N;
  double* R;
  double* z;
  int* singular;
  int64_t hmax;
};

// Row map of a block of up to two contiguous row segments (local rows, or the
// stacked tops of a tree pair): row i -> global row.
struct RowMap {
  int64_t a0, b0;  // starts of segment 0 / 1
  int na;          // rows in segment 0
  __device__ __forceinline__ int64_t operator()(int i) const { return i < na ? a0 + i : b0 + (i - na); }
};

// In-place Householder QR of the m x kb block A (smem, stride TP):
// R in the upper triangle (diag = beta, LAPACK dlarfg sign), reflectors
// below the diagonal (unit diagonal implicit), taus[0..min(m,kb)).
__device__ void smem_qr(double* A, int m, int kb, double* taus, double* wv, double* tv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nref = min(m, kb);
  for (int jj = 0; jj < nref; ++jj) {
    const int ncol = kb - jj;
    // S_c = sum_{r>jj} A[r][jj] A[r][jj+c]  (c = 0 gives ||x||^2); two columns per warp
    const int c0 = warp, c1 = warp + TW;
    if (c0 < ncol) {
      double s0 = 0.0, s1 = 0.0;
      for (int r = jj + 1 + lane; r < m; r += 32) {
        const double* row = A + r * TP + jj;
        const double xr = row[0];
        s0 = fma(xr, row[c0], s0);
        if (c1 < ncol) s1 = fma(xr, row[c1], s1);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(FULL, s0, o);
        s1 += __shfl_xor_sync(FULL, s1, o);
      }
      if (lane == 0) {
        wv[c0] = s0;
        if (c1 < ncol) wv[c1] = s1;
      }
    }
    __syncthreads();
    const double xn2 = wv[0];
    const double alpha = A[jj * TP + jj];
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
    // temp_c = -tau * v'a_c,  v'a_c = a_jc + scal * S_c
    if (tid > 0 && tid < ncol) tv[tid] = -tau * (A[jj * TP + jj + tid] + scal * wv[tid]);
    if (tid == 0) taus[jj] = tau;
    __syncthreads();
    if (tid == 0) A[jj * TP + jj] = beta;
    if (tau != 0.0) {
      const int cc = lane;
      for (int r = jj + warp; r < m; r += TW) {
        double* row = A + r * TP + jj;
        const double vr = (r == jj) ? 1.0 : row[0] * scal;
        if (cc > 0 && cc < ncol) row[cc] += vr * tv[cc];
        __syncwarp();
        if (lane == 0 && r != jj) row[0] = vr;
      }
    }
    __syncthreads();
  }
}

// V element (r, c) of reflector block A (m x kb, stride TP): unit lower trapezoid.
__device__ __forceinline__ double vget(const double* A, int r, int c, int m, int kb) {
  const double v = A[min(r, m - 1) * TP + min(c, kb - 1)];
  return (r >= m || c >= kb || r < c) ? 0.0 : (r == c ? 1.0 : v);
}

// T (kb x kb, stride TB) of the compact WY form (dlarft forward/columnwise)
// from the reflectors in A (m x kb) and taus.  G = V'V on DMMA tiles.
__device__ void build_t(const double* A, int m, int kb, const double* taus, double* Gs, double* Ts) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  {  // G: 16 tiles of 8x8, one per warp
    const int mt = warp >> 2, nt = warp & 3;
    double d0 = 0.0, d1 = 0.0;
    for (int k = 0; k < m; k += 4) {
      const double av = vget(A, k + t4, mt * 8 + g4, m, kb);
      const double bv = vget(A, k + t4, nt * 8 + g4, m, kb);
      dmma(d0, d1, av, bv);
    }
    const int r = mt * 8 + g4, c = nt * 8 + t4 * 2;
    Gs[r * TB + c] = d0;
    Gs[r * TB + c + 1] = d1;
  }
  __syncthreads();
  if (warp == 0) {
    for (int i = 0; i < kb; ++i) {
      const double ti = taus[i];
      const double g = (lane < i) ? -ti * Gs[lane * TB + i] : 0.0;
      double acc = 0.0;
      for (int l = 0; l < i; ++l) {
        const double gl = __shfl_sync(FULL, g, l);
        if (lane <= l) acc += Ts[lane * TB + l] * gl;
      }
      if (lane < i) Ts[lane * TB + i] = (ti == 0.0) ? 0.0 : acc;
      if (lane == i) Ts[i * TB + i] = ti;
      if (lane > i) Ts[lane * TB + i] = 0.0;
      __syncwarp();
    }
    for (int i = kb; i < TB; ++i) Ts[lane * TB + i] = 0.0;
  }
  __syncthreads();
}

// X <- (I - V T V')' X = X - V T' (V' X) for the global rows map(0..m) and
// columns [c_beg, c_end) of W, V = reflectors in A (m x kb).  Tiles of X are
// staged with double-buffered cp.async; products on DMMA tiles.
__device__ void apply_qt(const TsqrArgs& a, const RowMap& map, int m, int64_t c_beg, int64_t c_end,
                         const double* A, int kb, const double* Ts, double* tile /* 2 x RTL x CBLP */,
                         double* Zs /* TB x CBLP */) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  double* W = a.W;
  const int64_t ldw = a.ldw;
  const int ntile = (m + RTL - 1) / RTL;
  for (int64_t cb = c_beg; cb < c_end; cb += CBL) {
    const int cw = static_cast<int>(min(static_cast<int64_t>(CBL), c_end - cb));
    auto stage = [&](int t, int bf) {
      double* dst = tile + bf * RTL * CBLP;
      for (int idx = tid; idx < RTL * CBL; idx += TT) {
        const int rr = idx / CBL, c = idx % CBL;
        const int r = t * RTL + rr;
        const bool ok = r < m && c < cw;
        cp_async8(dst + rr * CBLP + c, ok ? W + map(r) * ldw + cb + c : W, ok);
      }
      cp_commit();
    };
    // (1) Y = V'X  (32 x cw): 32 output tiles, two per warp
    double y0[2] = {0.0, 0.0}, y1[2] = {0.0, 0.0};
    stage(0, 0);
    for (int t = 0; t < ntile; ++t) {
      if (t + 1 < ntile) {
        stage(t + 1, (t + 1) & 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      const double* tb = tile + (t & 1) * RTL * CBLP;
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const int T = warp * 2 + tt;
        const int mt = T >> 3, nt = T & 7;
#pragma unroll
        for (int k = 0; k < RTL; k += 4) {
          const int r = t * RTL + k + t4;
          const double av = vget(A, r, mt * 8 + g4, m, kb);
          const double bv = tb[(k + t4) * CBLP + nt * 8 + g4];
          dmma(y0[tt], y1[tt], av, bv);
        }
      }
      __syncthreads();
    }
    // (2) Z = T'Y via shared memory
    double* Ys = tile;  // reuse the first tile buffer
#pragma unroll
    for (int tt = 0; tt < 2; ++tt) {
      const int T = warp * 2 + tt;
      const int mt = T >> 3, nt = T & 7;
      Ys[(mt * 8 + g4) * CBLP + nt * 8 + t4 * 2] = y0[tt];
      Ys[(mt * 8 + g4) * CBLP + nt * 8 + t4 * 2 + 1] = y1[tt];
    }
    __syncthreads();
    for (int idx = tid; idx < TB * CBL; idx += TT) {
      const int jj = idx / CBL, c = idx % CBL;
      double s = 0.0;
      for (int kk = 0; kk <= jj; ++kk) s += Ts[kk * TB + jj] * Ys[kk * CBLP + c];
      Zs[jj * CBLP + c] = s;
    }
    __syncthreads();
    // (3) X -= V Z, row tile by row tile
    stage(0, 0);
    for (int t = 0; t < ntile; ++t) {
      if (t + 1 < ntile) {
        stage(t + 1, (t + 1) & 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      const double* tb = tile + (t & 1) * RTL * CBLP;
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const int T = warp * 2 + tt;  // 4 (rows) x 8 (cols) tiles of 8x8
        const int mt = T >> 3, nt = T & 7;
        const int rr = mt * 8 + g4, c = nt * 8 + t4 * 2;
        double d0 = tb[rr * CBLP + c], d1 = tb[rr * CBLP + c + 1];
#pragma unroll
        for (int k = 0; k < TB; k += 4) {
          const double av = -vget(A, t * RTL + mt * 8 + g4, k + t4, m, kb);
          const double bv = Zs[(k + t4) * CBLP + nt * 8 + g4];
          dmma(d0, d1, av, bv);
        }
        const int r = t * RTL + rr;
        if (r < m) {
          double* wp = W + map(r) * ldw + cb + c;
          if (c < cw) wp[0] = d0;
          if (c + 1 < cw) wp[1] = d1;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(TT, 1) k_qr_tsqr(TsqrArgs a) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), p = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x;
  const int64_t d = a.d, n = a.n, ldw = a.ldw, N = a.N;
  double* W = a.W;
  const int64_t lo = (static_cast<int64_t>(p) * d) / C, hi = (static_cast<int64_t>(p + 1) * d) / C;
  double* Ps = sm;                            // hmax x TP: active rows of the panel
  double* Sk = Ps + a.hmax * TP;              // 2TB x TP: stacked R pair (tree)
  double* Gs = Sk + 2 * TB * TP;              // TB x TB
  double* Ts = Gs + TB * TB;                  // TB x TB
  double* taus = Ts + TB * TB;                // TB
  double* wv = taus + TB;                     // TB
  double* tv = wv + TB;                       // TB
  double* tile = tv + TB;                     // 2 x RTL x CBLP
  double* Zs = tile + 2 * RTL * CBLP;         // TB x CBLP

  for (int64_t k0 = 0; k0 < n; k0 += TB) {
    const int kb = static_cast<int>(min(static_cast<int64_t>(TB), n - k0));
    const int64_t ra = (p == 0) ? lo + k0 : lo;  // CTA 0 retired its first k0 rows
    const int na = static_cast<int>(hi - ra);
    // ---- 1. local QR of the owned panel rows --------------------------------
    for (int idx = tid; idx < na * TB; idx += TT) {
      const int rr = idx / TB, c = idx % TB;
      Ps[rr * TP + c] = (c < kb) ? W[(ra + rr) * ldw + k0 + c] : 0.0;
    }
    __syncthreads();
    smem_qr(Ps, na, kb, taus, wv, tv);
    const int64_t ct0 = k0 + kb;
    if (ct0 < N) {
      build_t(Ps, na, kb, taus, Gs, Ts);
      const RowMap own{ra, 0, na};
      apply_qt(a, own, na, ct0, N, Ps, kb, Ts, tile, Zs);
    }
    // ---- 2. reduction tree over the CTAs' R factors -------------------------
    for (int s = 1; s < C; s <<= 1) {
      cl.sync();  // partner's R (smem) and top rows (global) are complete
      if ((p % (2 * s)) == 0 && p + s < C) {
        const int q = p + s;
        const int64_t ra_q = (static_cast<int64_t>(q) * d) / C;
        const double* Pq = cl.map_shared_rank(Ps, q);
        // stack [R_p ; R_q]: rows 0..kb-1 from this CTA, kb..2kb-1 from the partner
        for (int idx = tid; idx < 2 * kb * TB; idx += TT) {
          const int rr = idx / TB, c = idx % TB;
          const int br = rr < kb ? rr : rr - kb;
          const double src = rr < kb ? Ps[br * TP + c] : Pq[br * TP + c];
          Sk[rr * TP + c] = (c >= br && c < kb) ? src : 0.0;
        }
        __syncthreads();
        smem_qr(Sk, 2 * kb, kb, taus, wv, tv);
        // merged R back into this CTA's top rows
        for (int idx = tid; idx < kb * TB; idx += TT) {
          const int rr = idx / TB, c = idx % TB;
          if (c >= rr) Ps[rr * TP + c] = Sk[rr * TP + c];
        }
        if (ct0 < N) {
          build_t(Sk, 2 * kb, kb, taus, Gs, Ts);
          const RowMap pair{ra, ra_q, kb};
          apply_qt(a, pair, 2 * kb, ct0, N, Sk, kb, Ts, tile, Zs);
        }
        __syncthreads();
      }
    }
    cl.sync();
    // ---- 3. CTA 0 retires the panel's R rows ---------------------------------
    if (p == 0) {
      const int64_t rbase = lo + k0;
      for (int64_t idx = tid; idx < static_cast<int64_t>(kb) * n; idx += TT) {
        const int i = static_cast<int>(idx / n);
        const int64_t c = idx % n;
        const double dg = Ps[i * TP + i];
        const double sg = dg < 0.0 ? -1.0 : 1.0;
        double v;
        if (c < k0 + i) v = 0.0;
        else if (c < k0 + kb) v = sg * Ps[i * TP + (c - k0)];
        else v = sg * W[(rbase + i) * ldw + c];
        a.R[(k0 + i) * n + c] = v;
      }
      for (int i = tid; i < kb; i += TT) {
        const double dg = Ps[i * TP + i];
        const double sg = dg < 0.0 ? -1.0 : 1.0;
        if (a.z && N > n) a.z[k0 + i] = sg * W[(rbase + i) * ldw + n];
        if (dg == 0.0) atomicOr(a.singular, 1);
      }
    }
    __syncthreads();
  }
  cl.sync();
}

size_t tsqr_smem_doubles(int64_t hmax) {
  return static_cast<size_t>(hmax * TP + 2 * TB * TP + 2 * TB * TB + 3 * TB + 2 * RTL * CBLP + TB * CBLP);
}

}  // namespace

// Cluster size for the TSQR path, 0 if it does not apply: every CTA needs at
// least one panel of rows, CTA 0 must hold all n rows of R, and the owned
// panel rows must fit in shared memory.
int qr_tsqr_plan(int64_t d, int64_t n, size_t* smem) {
  for (int C = 16; C >= 2; C >>= 1) {
    const int64_t hmin = d / C;
    const int64_t hmax = (d + C - 1) / C + 1;
    const size_t sb = tsqr_smem_doubles(hmax) * sizeof(double);
    if (hmin >= std::max<int64_t>(n, TB) && sb <= 220 * 1024) {
      *smem = sb;
      return C;
    }
  }
  return 0;
}

int launch_qr_tsqr(double* W, int64_t d, int64_t n, int64_t ldw, int64_t N, double* R, double* z,
                   int* singular, int C, size_t smem, cudaStream_t s) {
  TsqrArgs a;
  a.W = W;
  a.d = d;
  a.n = n;
  a.ldw = ldw;
  a.N = N;
  a.R = R;
  a.z = z;
  a.singular = singular;
  a.hmax = (d + C - 1) / C + 1;
  ITSK_CUDA(allow_max_smem(reinterpret_cast<const void*>(k_qr_tsqr)));
  ITSK_CUDA(func_attr_once(reinterpret_cast<const void*>(k_qr_tsqr),
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(TT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ITSK_CUDA(cudaLaunchKernelEx(&cfg, k_qr_tsqr, a));
  count_launch();
  return ITSK_OK;
}

}  // namespace itsk
