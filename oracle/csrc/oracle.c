/* CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/itsketch_oracle.py).
 *
 * oracle_sketch_apply: restates scipy 1.18.1 `_sparsetools.csc_matvecs`, the
 *   routine behind SparseSignEmbedding.apply_dense
 *   (/root/reference/pkg/src/itsketch/embed.py:62-67): for every column j of
 *   the d x m CSC matrix S in ascending order and each of its zeta stored
 *   entries, y[row, :] += val * x[j, :], product rounded before the add.
 *   Built with -ffp-contract=off so no FMA changes the rounding.
 * oracle_sketch_apply_csr: the same for a CSR A — scipy's S_csc @ A.tocsc()
 *   (embed.py:76-80, csr_matmat on the transposes) adds, per output entry,
 *   fl(s * a_jc) over the sources j ascending (stored order inside a row),
 *   i.e. the dense sum with the zero entries of A skipped.
 * oracle_pcg64_words: the 32-bit word stream numpy's Generator(PCG64) feeds
 *   its bounded-integer sampler (embed.py:89-91), for pinning the GPU stream.
 */
#include <stdint.h>

void oracle_sketch_apply(int64_t m, int64_t k, int64_t zeta, const int64_t* rows,
                         const double* vals, const double* x, double* y) {
  for (int64_t j = 0; j < m; ++j) {
    const double* xj = x + j * k;
    for (int64_t t = 0; t < zeta; ++t) {
      const double v = vals[j * zeta + t];
      double* yi = y + rows[j * zeta + t] * k;
      for (int64_t c = 0; c < k; ++c) {
        double prod = v * xj[c];
        yi[c] = yi[c] + prod;
      }
    }
  }
}

void oracle_sketch_apply_csr(int64_t m, int64_t n, int64_t zeta, const int64_t* rows, const double* vals,
                             const int64_t* row_ptr, const int32_t* col, const double* val, double* y) {
  for (int64_t j = 0; j < m; ++j) {
    for (int64_t t = 0; t < zeta; ++t) {
      const double v = vals[j * zeta + t];
      double* yi = y + rows[j * zeta + t] * n;
      for (int64_t e = row_ptr[j]; e < row_ptr[j + 1]; ++e) {
        double prod = val[e] * v;
        yi[col[e]] = yi[col[e]] + prod;
      }
    }
  }
}

typedef unsigned __int128 u128;
static const u128 kMult = (((u128)0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;

static inline uint64_t pcg_out(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

void oracle_pcg64_words(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                        int has32, uint32_t pending, int64_t count, uint32_t* out) {
  u128 s = (((u128)s_hi) << 64) | s_lo;
  u128 inc = (((u128)i_hi) << 64) | i_lo;
  int64_t k = 0;
  if (has32 && count > 0) out[k++] = pending;
  while (k < count) {
    s = s * kMult + inc;
    uint64_t v = pcg_out(s);
    out[k++] = (uint32_t)v;
    if (k < count) out[k++] = (uint32_t)(v >> 32);
  }
}
