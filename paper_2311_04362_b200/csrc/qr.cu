// Householder QR of the augmented sketch [SA | Sb] (K2).
//
// Replaces householder_qr_econ (/root/reference/pkg/src/itsketch/linalg.py:30-47,
// LAPACK dgeqrf + dorgqr, then diag(R) >= 0) and the x0 right-hand side
// Q'·Sb (solvers.py:209).  Blocked right-looking Householder (LAPACK
// dgeqr2/dlarft/dlarfb semantics, dlarfg's beta = -sign(alpha)*||x||), run as
// ONE cooperative kernel: every CTA owns a contiguous block of rows of W for
// the whole factorisation; column norms and reflector products are reduced
// across CTAs with fixed-order sums (deterministic, identical on every CTA)
// between software grid barriers.  Q is never formed: the reflectors are
// applied to the Sb column like any other trailing column, which yields
// z = (Q'Sb)[:n] directly.  The trailing update W -= V (T'(V'W)) of each
// 32-wide panel is computed per CTA on its own rows.
#include <cooperative_groups.h>

#include "itsk_common.cuh"

namespace itsk {
namespace {

constexpr int NB = 32;
constexpr int QR_THREADS = 256;
constexpr int YCH = 64;  // Y columns reduced per smem chunk

struct QrArgs {
  double* W;
  int64_t d, n, ldw, N;  // N = n + 1 columns (last is Sb) or n
  double* R;
  double* z;
  double* part1;  // 2 x P
  double* part2;  // P x NB
  double* part3;  // P x NB x ld3
  double* Zg;     // NB x N
  double* betas;  // n
  double* taus;   // n
  unsigned* bar;
  int* singular;
  int64_t hmax;
  int64_t ld3;
};

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__global__ void __launch_bounds__(QR_THREADS) k_qr(QrArgs a) {
  extern __shared__ double sm[];
  const int P = gridDim.x, p = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = QR_THREADS / 32;
  const int64_t d = a.d, n = a.n, ldw = a.ldw, N = a.N;
  double* W = a.W;
  const int64_t lo = (static_cast<int64_t>(p) * d) / P;
  const int64_t hi = (static_cast<int64_t>(p + 1) * d) / P;
  double* Vs = sm;                   // hmax x NB
  double* Ts = Vs + a.hmax * NB;     // NB x NB
  double* Gs = Ts + NB * NB;         // NB x NB
  double* red = Gs + NB * NB;        // 32
  double* wv = red + 32;             // NB
  double* Ys = wv + NB;              // NB x YCH
  __shared__ double s_tau[NB];

  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int kb = static_cast<int>(min(static_cast<int64_t>(NB), n - k0));
    // ---------------- panel: unblocked Householder (dgeqr2) ----------------
    for (int jj = 0; jj < kb; ++jj) {
      const int64_t j = k0 + jj;
      const int64_t rs = max(lo, j + 1);
      double ss = 0.0;
      for (int64_t r = rs + tid; r < hi; r += QR_THREADS) {
        const double v = W[r * ldw + j];
        ss += v * v;
      }
      ss = block_sum(ss, red);
      // part1 is double-buffered by column parity: without a barrier between
      // B(j) and A(j+1) (tau == 0), a fast CTA must not overwrite the slot a
      // slow CTA is still summing.
      double* part1 = a.part1 + (j & 1) * P;
      if (tid == 0) part1[p] = ss;
      grid_barrier(a.bar);
      double t = 0.0;
      for (int q = tid; q < P; q += QR_THREADS) t += ldcg(part1 + q);
      const double xn2 = block_sum(t, red);
      const double alpha = ldcg(W + j * ldw + j);
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
      if (tid == 0) s_tau[jj] = tau;
      if (tid == 0 && p == 0) {
        a.betas[j] = beta;
        a.taus[j] = tau;
      }
      if (xn2 != 0.0)
        for (int64_t r = rs + tid; r < hi; r += QR_THREADS) W[r * ldw + j] *= scal;
      __syncthreads();
      const int ncp = static_cast<int>(k0 + kb - j - 1);
      if (ncp > 0 && tau != 0.0) {
        const int64_t r0 = max(lo, j);
        for (int cc = warp; cc < ncp; cc += nwarp) {
          const int64_t c = j + 1 + cc;
          double acc = 0.0;
          for (int64_t r = r0 + lane; r < hi; r += 32) {
            const double v = (r == j) ? 1.0 : W[r * ldw + j];
            acc += v * W[r * ldw + c];
          }
          acc = warp_sum(acc);
          if (lane == 0) a.part2[static_cast<int64_t>(p) * NB + cc] = acc;
        }
        grid_barrier(a.bar);
        for (int cc = warp; cc < ncp; cc += nwarp) {
          double s = 0.0;
          for (int q = lane; q < P; q += 32) s += ldcg(a.part2 + static_cast<int64_t>(q) * NB + cc);
          s = warp_sum(s);
          if (lane == 0) wv[cc] = s;
        }
        __syncthreads();
        const int64_t nr = hi > r0 ? hi - r0 : 0;
        for (int64_t idx = tid; idx < nr * ncp; idx += QR_THREADS) {
          const int64_t r = r0 + idx / ncp;
          const int cc = static_cast<int>(idx % ncp);
          const double v = (r == j) ? 1.0 : W[r * ldw + j];
          const double temp = -tau * wv[cc];
          W[r * ldw + j + 1 + cc] += v * temp;
        }
      }
      // W[j][j] keeps alpha (other CTAs may still be reading it when there is
      // no barrier after B); R's diagonal comes from betas[] at the end.
      __syncthreads();
    }
    // ---------------- trailing update: W -= V T' V' W (dlarft + dlarfb) ------
    const int64_t ct0 = k0 + kb;
    const int64_t Nt = N - ct0;
    if (Nt <= 0) continue;
    const int64_t rlo = max(lo, k0);
    const int64_t hv = hi > rlo ? hi - rlo : 0;
    for (int64_t idx = tid; idx < hv * NB; idx += QR_THREADS) {
      const int64_t rr = idx / NB;
      const int jj = static_cast<int>(idx % NB);
      const int64_t r = rlo + rr;
      double v = 0.0;
      if (jj < kb) v = (r < k0 + jj) ? 0.0 : (r == k0 + jj ? 1.0 : W[r * ldw + k0 + jj]);
      Vs[idx] = v;
    }
    __syncthreads();
    // partial [G | Y] = V_own' [V_own | W_own(:, ct0:)]
    const int64_t ncols3 = kb + Nt;
    for (int64_t cidx = tid; cidx < ncols3; cidx += QR_THREADS) {
      double acc[NB];
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) acc[jj] = 0.0;
      for (int64_t rr = 0; rr < hv; ++rr) {
        const double x = (cidx < kb) ? Vs[rr * NB + cidx] : W[(rlo + rr) * ldw + ct0 + cidx - kb];
        const double* vrow = Vs + rr * NB;
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) acc[jj] = fma(vrow[jj], x, acc[jj]);
      }
      double* dst = a.part3 + static_cast<int64_t>(p) * NB * a.ld3 + cidx;
#pragma unroll
      for (int jj = 0; jj < NB; ++jj)
        if (jj < kb) dst[jj * a.ld3] = acc[jj];
    }
    grid_barrier(a.bar);
    // every CTA: G (fixed order) and T
    for (int idx = tid; idx < kb * kb; idx += QR_THREADS) {
      const int jj = idx / kb, kk = idx % kb;
      double s = 0.0;
      for (int q = 0; q < P; ++q) s += ldcg(a.part3 + (static_cast<int64_t>(q) * NB + jj) * a.ld3 + kk);
      Gs[jj * NB + kk] = s;
    }
    __syncthreads();
    if (warp == 0) {  // dlarft, forward / columnwise, lane k owns row k of T
      for (int i = 0; i < kb; ++i) {
        const double ti = s_tau[i];
        double g = (lane < i) ? -ti * Gs[lane * NB + i] : 0.0;
        // T(0:i, i) = T(0:i, 0:i) * g   (upper triangular T)
        double acc = 0.0;
        for (int l = 0; l < i; ++l) {
          const double gl = __shfl_sync(FULL, g, l);
          if (lane <= l) acc += Ts[lane * NB + l] * gl;
        }
        if (lane < i) Ts[lane * NB + i] = (ti == 0.0) ? 0.0 : acc;
        if (lane == i) Ts[i * NB + i] = ti;
        if (lane > i && lane < NB) Ts[lane * NB + i] = 0.0;
        __syncwarp();
      }
    }
    __syncthreads();
    // Y slice of this CTA -> Z = T' Y  (global, NB x N)
    const int64_t c_lo = (static_cast<int64_t>(p) * Nt) / P;
    const int64_t c_hi = (static_cast<int64_t>(p + 1) * Nt) / P;
    for (int64_t cb = c_lo; cb < c_hi; cb += YCH) {
      const int w = static_cast<int>(min(static_cast<int64_t>(YCH), c_hi - cb));
      for (int idx = tid; idx < kb * w; idx += QR_THREADS) {
        const int jj = idx / w, cc = idx % w;
        double s = 0.0;
        for (int q = 0; q < P; ++q)
          s += ldcg(a.part3 + (static_cast<int64_t>(q) * NB + jj) * a.ld3 + kb + cb + cc);
        Ys[jj * YCH + cc] = s;
      }
      __syncthreads();
      for (int idx = tid; idx < kb * w; idx += QR_THREADS) {
        const int jj = idx / w, cc = idx % w;
        double s = 0.0;
        for (int kk = 0; kk <= jj; ++kk) s += Ts[kk * NB + jj] * Ys[kk * YCH + cc];
        a.Zg[jj * N + cb + cc] = s;
      }
      __syncthreads();
    }
    grid_barrier(a.bar);
    for (int64_t c = tid; c < Nt; c += QR_THREADS) {
      double zc[NB];
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) zc[jj] = (jj < kb) ? ldcg(a.Zg + jj * N + c) : 0.0;
      for (int64_t rr = 0; rr < hv; ++rr) {
        double* wp = W + (rlo + rr) * ldw + ct0 + c;
        double acc = *wp;
        const double* vrow = Vs + rr * NB;
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) acc = fma(-vrow[jj], zc[jj], acc);
        *wp = acc;
      }
    }
    // The next panel's first grid barrier orders these writes before any
    // cross-CTA read; own-row reads only need the CTA barrier.
    __syncthreads();
  }
  grid_barrier(a.bar);
  // R = sign-fixed upper triangle, z = sign-fixed Q'Sb (linalg.py:43-46)
  const int64_t gtid = static_cast<int64_t>(p) * QR_THREADS + tid;
  const int64_t gstride = static_cast<int64_t>(P) * QR_THREADS;
  for (int64_t idx = gtid; idx < n * n; idx += gstride) {
    const int64_t i = idx / n, c = idx % n;
    const double bi = ldcg(a.betas + i);
    const double sg = bi < 0.0 ? -1.0 : 1.0;
    a.R[idx] = (c < i) ? 0.0 : (c == i ? sg * bi : sg * ldcg(W + i * ldw + c));
  }
  for (int64_t i = gtid; i < n; i += gstride) {
    const double bi = ldcg(a.betas + i);
    const double sg = bi < 0.0 ? -1.0 : 1.0;
    if (a.z && N > n) a.z[i] = sg * ldcg(W + i * ldw + n);
    if (bi == 0.0) atomicOr(a.singular, 1);
  }
}

struct QrLayout {
  int P;
  int64_t hmax, ld3;
  size_t smem;
  int64_t bytes;
  unsigned* bar;
  int* singular;
  double *part1, *part2, *part3, *Zg, *betas, *taus;
};

int qr_grid(int64_t d) {
  const int sms = num_sms();
  int64_t P = (d + 15) / 16;  // >= 16 rows per CTA
  if (P > sms) P = sms;
  if (P < 1) P = 1;
  return static_cast<int>(P);
}

QrLayout qr_layout(void* ws, int64_t d, int64_t n, int has_rhs) {
  QrLayout L;
  L.P = qr_grid(d);
  const int64_t N = n + (has_rhs ? 1 : 0);
  L.hmax = (d + L.P - 1) / L.P + 1;
  L.ld3 = NB + N;
  L.smem = static_cast<size_t>(L.hmax * NB + 2 * NB * NB + 32 + NB + NB * YCH) * sizeof(double);
  Carver cv(ws, 1ll << 62);
  L.bar = cv.take<unsigned>(64);
  L.singular = cv.take<int>(64);
  L.part1 = cv.take<double>(2 * L.P);
  L.part2 = cv.take<double>(static_cast<int64_t>(L.P) * NB);
  L.part3 = cv.take<double>(static_cast<int64_t>(L.P) * NB * L.ld3);
  L.Zg = cv.take<double>(NB * N);
  L.betas = cv.take<double>(n);
  L.taus = cv.take<double>(n);
  L.bytes = cv.off + 256;
  return L;
}

}  // namespace
}  // namespace itsk

using namespace itsk;

extern "C" int itsk_qr_workspace(int64_t d, int64_t n, int64_t* bytes) {
  ITSK_REQUIRE(bytes && d >= n && n >= 1, "need d >= n >= 1");
  *bytes = qr_layout(nullptr, d, n, 1).bytes;
  return ITSK_OK;
}

extern "C" int itsk_qr_aug(double* W, int64_t d, int64_t n, int64_t ldw, double* R, double* z,
                           void* ws, int64_t ws_bytes, itsk_stream_t stream) {
  ITSK_REQUIRE(W && R && ws, "null pointer");
  ITSK_REQUIRE(n >= 1 && d >= n, "need m >= n, got %lld x %lld", (long long)d, (long long)n);
  const int has_rhs = z != nullptr;
  ITSK_REQUIRE(ldw >= n + has_rhs, "bad leading dimension");
  QrLayout L = qr_layout(ws, d, n, has_rhs);
  ITSK_REQUIRE(L.bytes <= ws_bytes, "qr workspace too small (%lld < %lld)", (long long)ws_bytes,
               (long long)L.bytes);
  ITSK_REQUIRE(L.smem <= 200 * 1024, "qr: too many rows per CTA");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ITSK_CUDA(cudaMemsetAsync(L.bar, 0, 512, s));
  QrArgs a;
  a.W = W;
  a.d = d;
  a.n = n;
  a.ldw = ldw;
  a.N = n + has_rhs;
  a.R = R;
  a.z = z;
  a.part1 = L.part1;
  a.part2 = L.part2;
  a.part3 = L.part3;
  a.Zg = L.Zg;
  a.betas = L.betas;
  a.taus = L.taus;
  a.bar = L.bar;
  a.singular = L.singular;
  a.hmax = L.hmax;
  a.ld3 = L.ld3;
  ITSK_CUDA(cudaFuncSetAttribute(k_qr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(L.smem)));
  void* args[] = {&a};
  ITSK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_qr), dim3(L.P),
                                        dim3(QR_THREADS), args, L.smem, s));
  count_launch();
  int singular = 0;
  ITSK_CUDA(cudaMemcpyAsync(&singular, L.singular, sizeof(int), cudaMemcpyDeviceToHost, s));
  ITSK_CUDA(cudaStreamSynchronize(s));
  if (singular) {
    set_error("zero diagonal entry in triangular factor");
    return ITSK_ESINGULAR;
  }
  return ITSK_OK;
}
