// Sparse sign embedding pattern on the device.
//
// Replaces sparse_sign_new / _distinct_rows
// (/root/reference/pkg/src/itsketch/embed.py:28-42, 83-99).  The reference
// draws, from one numpy Generator(PCG64) seeded with `rng_seed`:
//   rows  = integers(0, d, (m, zeta))        (32-bit buffered Lemire draws)
//   while some column j holds a repeated row: rows[bad] = integers(0, d, (nbad, zeta))
//   signs = choice([-1., 1.], (m, zeta))     (== integers(0, 2), no rejection)
// All three consume one stream of 32-bit words (low half of each 64-bit PCG
// output first, the other half buffered in the generator and carried across
// calls).  Here every thread jumps ahead (LCG advance, O(log k)) to its own
// chunk of that word stream; the rare Lemire rejections are resolved with a
// prefix sum over per-chunk reject counts, so the output is bit-identical to
// numpy's sequential loop.
#include <algorithm>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "itsk_common.cuh"

namespace itsk {
namespace {

typedef unsigned __int128 u128;
constexpr int CH = 64;  // words per thread chunk

__device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return (static_cast<u128>(hi) << 64) | lo;
}
__device__ __forceinline__ u128 pcg_mult() {
  return mk128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull);
}
__device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t x = static_cast<uint64_t>(s >> 64) ^ static_cast<uint64_t>(s);
  const unsigned rot = static_cast<unsigned>(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
// State after `delta` LCG steps (Brown's jump-ahead).
__device__ u128 pcg_advance(u128 s, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

// The affine map of `delta` LCG steps: state -> mult * state + plus.
struct Jump {
  u128 mult, plus;
};
__device__ Jump pcg_jump(u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return Jump{acc_mult, acc_plus};
}

struct Stream {
  uint64_t s_hi, s_lo, i_hi, i_lo;
  uint32_t pending;
  int has;  // numpy's has_uint32 at stream start
};

// Sequential reader of 32-bit words starting at absolute word index `w`.
struct WordCursor {
  u128 s, inc;
  uint64_t buf;
  int half;  // 1 when the high half of `buf` is the next word
  uint32_t pending;
  int use_pending;

  __device__ WordCursor(const Stream& st, uint64_t w) {
    inc = mk128(st.i_hi, st.i_lo);
    const u128 s0 = mk128(st.s_hi, st.s_lo);
    use_pending = (st.has && w == 0);
    pending = st.pending;
    const uint64_t k = (st.has && w > 0) ? w - 1 : (st.has ? 0 : w);
    // base word k lives in output k>>1 (after (k>>1)+1 steps), half k&1.
    const uint64_t o = k >> 1;
    s = pcg_advance(s0, inc, o);  // state before producing output o
    half = 0;
    buf = 0;
    if (!use_pending && (k & 1)) {
      s = s * pcg_mult() + inc;
      buf = pcg_output(s);
      half = 1;
    }
  }
  // From the state before output k >> 1 (k = the word index, has_uint32
  // already accounted for): no jump-ahead here.
  __device__ WordCursor(u128 s_before, u128 inc_, uint64_t k) : inc(inc_), pending(0), use_pending(0) {
    s = s_before;
    half = 0;
    buf = 0;
    if (k & 1) {
      s = s * pcg_mult() + inc;
      buf = pcg_output(s);
      half = 1;
    }
  }
  __device__ __forceinline__ uint32_t next() {
    if (use_pending) {
      use_pending = 0;
      return pending;
    }
    if (half) {
      half = 0;
      return static_cast<uint32_t>(buf >> 32);
    }
    s = s * pcg_mult() + inc;
    buf = pcg_output(s);
    half = 1;
    return static_cast<uint32_t>(buf);
  }
};

__device__ __forceinline__ bool lemire_accept(uint32_t w, uint32_t bound, uint32_t thr,
                                              uint32_t* out) {
  const uint64_t prod = static_cast<uint64_t>(w) * bound;
  *out = static_cast<uint32_t>(prod >> 32);
  return static_cast<uint32_t>(prod) >= thr;
}

__global__ void k_lemire_count(Stream st, const uint64_t* w0p, uint64_t nwords, uint32_t bound,
                               uint32_t thr, uint32_t* counts, uint64_t nchunks) {
  const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t w0 = *w0p;  // stream position stays on the device: no host round trip
  if (c == 0) counts[nchunks] = 0;  // so the scan's last slot is the total
  if (c >= nchunks) return;
  const uint64_t beg = c * CH;
  const uint64_t len = min(static_cast<uint64_t>(CH), nwords - beg);
  uint32_t acc = 0;
  if (thr != 0) {
    WordCursor cur(st, w0 + beg);
    for (uint64_t i = 0; i < len; ++i) {
      uint32_t v;
      acc += lemire_accept(cur.next(), bound, thr, &v) ? 1u : 0u;
    }
  } else {
    acc = static_cast<uint32_t>(len);
  }
  counts[c] = acc;
}

// Emits accepted draws; draw q goes to dst[map(q)] where map is identity
// (mode 0) or the q-th slot of the redrawn columns (mode 1).  Writes the
// absolute word index following draw N-1 to *end_word.
__global__ void k_lemire_emit(Stream st, const uint64_t* w0p, uint64_t nwords, uint32_t bound,
                              uint32_t thr, const uint32_t* scanned, uint64_t nchunks,
                              uint64_t N, uint32_t* dst, const uint32_t* bad_cols,
                              int64_t zeta, uint64_t* end_word) {
  const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t w0 = *w0p;
  // too few accepted words in the margin: k_redraw draws the rest
  if (c >= nchunks) return;
  uint64_t q = scanned[c];
  if (q >= N) return;
  const uint64_t beg = c * CH;
  const uint64_t len = min(static_cast<uint64_t>(CH), nwords - beg);
  WordCursor cur(st, w0 + beg);
  for (uint64_t i = 0; i < len && q < N; ++i) {
    uint32_t v;
    if (!lemire_accept(cur.next(), bound, thr, &v)) continue;
    uint64_t pos = q;
    if (bad_cols) pos = static_cast<uint64_t>(bad_cols[q / zeta]) * zeta + (q % zeta);
    dst[pos] = v;
    if (q == N - 1) *end_word = w0 + beg + i + 1;
    ++q;
  }
}

// The first draw (dst[q] = draw q): a warp's 32 chunks emit one contiguous
// range of draws, so they are staged in shared memory and written out
// coalesced (each lane's own draws are 64 consecutive words, strided 64
// apart across the warp, when stored directly).
constexpr int EM_WARPS = 4;
__global__ void __launch_bounds__(32 * EM_WARPS) k_lemire_emit_first(
    Stream st, const uint64_t* w0p, uint64_t nwords, uint32_t bound, uint32_t thr, const uint32_t* scanned,
    uint64_t nchunks, uint64_t N, uint32_t* dst, uint64_t* end_word) {
  __shared__ uint32_t stage[EM_WARPS][32 * CH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t w0 = *w0p;
  const uint64_t cw0 = c - lane;  // first chunk of the warp
  if (cw0 >= nchunks) return;     // warp-uniform
  const uint64_t cw1 = min(cw0 + 32, nchunks);
  const uint64_t qw0 = scanned[cw0];
  const uint64_t qw1 = min(static_cast<uint64_t>(scanned[cw1]), N);  // scanned[nchunks] = total
  uint32_t* sg = stage[warp];
  if (c < nchunks) {
    uint64_t q = scanned[c];
    if (q < N) {
      const uint64_t beg = c * CH;
      const uint64_t len = min(static_cast<uint64_t>(CH), nwords - beg);
      WordCursor cur(st, w0 + beg);
      for (uint64_t i = 0; i < len && q < N; ++i) {
        uint32_t v;
        if (!lemire_accept(cur.next(), bound, thr, &v)) continue;
        sg[q - qw0] = v;
        if (q == N - 1) *end_word = w0 + beg + i + 1;
        ++q;
      }
    }
  }
  __syncwarp();
  for (uint64_t q = qw0 + lane; q < qw1; q += 32) dst[q] = sg[q - qw0];
}

// choice([-1., 1.]) → integers(0, 2): neg = (w >> 31) == 0, one word each.
__global__ void k_signs(Stream st, const uint64_t* w0p, uint64_t N, uint8_t* neg) {
  const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t w0 = *w0p;
  const uint64_t beg = c * CH;
  if (beg >= N) return;
  const uint64_t len = min(static_cast<uint64_t>(CH), N - beg);
  WordCursor cur(st, w0 + beg);
  if (len == CH && (reinterpret_cast<uintptr_t>(neg) & 15) == 0) {
    // a full chunk: the 64 sign bytes packed in registers, four 16-byte stores
    // (byte stores strided 64 bytes across the warp were most of the time)
    static_assert(CH == 64, "k_signs packs 64 bytes");
    uint64_t pk[8];
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) {
      uint64_t v = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) v |= static_cast<uint64_t>((cur.next() >> 31) == 0 ? 1 : 0) << (8 * b);
      pk[w8] = v;
    }
    uint4* dst = reinterpret_cast<uint4*>(neg + beg);  // beg % 64 == 0; neg is 16-byte aligned
#pragma unroll
    for (int q = 0; q < 4; ++q)
      dst[q] = make_uint4(static_cast<uint32_t>(pk[2 * q]), static_cast<uint32_t>(pk[2 * q] >> 32),
                          static_cast<uint32_t>(pk[2 * q + 1]), static_cast<uint32_t>(pk[2 * q + 1] >> 32));
    return;
  }
  for (uint64_t i = 0; i < len; ++i) neg[beg + i] = (cur.next() >> 31) == 0 ? 1 : 0;
}

__global__ void k_tile_rows(uint32_t* rows, int64_t m, int64_t zeta) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e < m * zeta) rows[e] = static_cast<uint32_t>(e % zeta);
}

// Flags columns (rows of the (m, zeta) array) holding a repeated value,
// restricted to `cols` when non-null (only redrawn columns can change).
__global__ void k_flag_dupes(const uint32_t* rows, int64_t zeta, const uint32_t* cols,
                             int64_t ncols, uint32_t* flags) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= ncols) return;
  const int64_t j = cols ? cols[q] : q;
  const uint32_t* r = rows + j * zeta;
  uint32_t bad = 0;
  for (int64_t a = 1; a < zeta && !bad; ++a) {
    const uint32_t ra = r[a];
    for (int64_t b = 0; b < a; ++b)
      if (r[b] == ra) {
        bad = 1;
        break;
      }
  }
  flags[q] = bad;
}

__global__ void k_compact(const uint32_t* flags, const uint32_t* scanned, const uint32_t* cols,
                          int64_t ncols, uint32_t* out, uint32_t* total) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= ncols) return;
  if (flags[q]) out[scanned[q]] = cols ? cols[q] : static_cast<uint32_t>(q);
  if (q == ncols - 1) *total = scanned[q] + flags[q];
}

// ---------------------------------------------------------------------------
// Redraw rounds on one CTA (no host round trip).  After the parallel first
// draw and the parallel duplicate scan of all m columns, the reference's
// while loop (embed.py:37-42) redraws only the bad columns, in ascending
// column order, each round from the stream position where the previous one
// ended; after the first round a few hundred or thousand columns remain, so
// one CTA runs every further round: words drawn in tiles (thread t takes
// RD_W consecutive words, a block scan of the accept counts places the
// draws in stream order), then the redrawn columns re-checked and compacted
// in order.  The same code finishes the first draw if its word margin ran
// short (draws total..N-1, then a full duplicate scan).
constexpr int RD_T = 1024;
constexpr int RD_W = 4;
constexpr double RD_PAR_MIN = 65536.0;  // redraw rounds with more draws run as parallel kernels

// Exclusive prefix sum over the CTA in thread order; *tot = the CTA total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* tot) {
  __shared__ uint32_t wsum[RD_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = wsum[lane];
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    wsum[lane] = wi - w;
    if (lane == 31) *tot = wi;
  }
  __syncthreads();
  const uint32_t r = wsum[warp] + inc - v;
  __syncthreads();  // wsum is reused by the next call
  return r;
}

// Draws `count` Lemire values from word position `pos` on; draw q goes to
// rows[q0 + q] (cols == nullptr) or to column cols[q / zeta], slot q % zeta.
// Returns (every thread) the position after the last accepted word.
// Per-thread jump-ahead, set up once per kernel: a thread's words of a tile
// start RD_W * tid words (2 * tid outputs, RD_W even) after the tile's, and
// consecutive tiles are RD_T * RD_W words apart — so only the first tile of
// each call needs a (one-thread) jump from the stream origin, every other
// cursor is one affine step from a shared base state (the full per-thread
// 128-bit jump-ahead per tile was most of this kernel's time).
struct RedrawJumps {
  Jump mine;  // 2 * tid outputs
  Jump tile;  // RD_T * RD_W / 2 outputs
};

__device__ uint64_t draw_seq(const Stream& st, const RedrawJumps& jp, uint64_t pos, uint64_t count,
                             uint32_t bound, uint32_t thr, uint32_t* rows, uint64_t q0, const uint32_t* cols,
                             int64_t zeta) {
  static_assert(RD_W % 2 == 0, "thread word offsets must keep the tile's word parity");
  __shared__ uint32_t s_tot;
  __shared__ uint64_t s_end;
  __shared__ uint64_t s_base[2];
  const u128 inc = mk128(st.i_hi, st.i_lo);
  // word index k of `pos` (numpy's buffered half-word consumed first when has)
  const uint64_t k0 = st.has ? pos - 1 : pos;  // pos > 0 in every call
  if (threadIdx.x == 0) {
    const u128 b = pcg_advance(mk128(st.s_hi, st.s_lo), inc, k0 >> 1);  // state before output k0 >> 1
    s_base[0] = static_cast<uint64_t>(b >> 64);
    s_base[1] = static_cast<uint64_t>(b);
  }
  __syncthreads();
  u128 base_state = mk128(s_base[0], s_base[1]);
  uint64_t done = 0;
  while (done < count) {
    const uint64_t base = pos + static_cast<uint64_t>(threadIdx.x) * RD_W;
    WordCursor cur(jp.mine.mult * base_state + jp.mine.plus, inc, (st.has ? base - 1 : base));
    uint32_t v[RD_W];
    unsigned acc = 0, cnt = 0;
#pragma unroll
    for (int i = 0; i < RD_W; ++i) {
      if (lemire_accept(cur.next(), bound, thr, &v[i])) {
        acc |= 1u << i;
        ++cnt;
      }
    }
    const uint32_t ex = block_excl_scan(cnt, &s_tot);
    uint64_t q = done + ex;
#pragma unroll
    for (int i = 0; i < RD_W; ++i) {
      if (!(acc >> i & 1u)) continue;
      if (q < count) {
        const uint64_t at = cols ? static_cast<uint64_t>(cols[q / zeta]) * zeta + (q % zeta) : q0 + q;
        rows[at] = v[i];
        if (q == count - 1) s_end = base + i + 1;
      }
      ++q;
    }
    __syncthreads();
    const uint64_t tot = s_tot;
    if (done + tot >= count) {
      pos = s_end;
      done = count;
    } else {
      pos += static_cast<uint64_t>(RD_T) * RD_W;
      done += tot;
      base_state = jp.tile.mult * base_state + jp.tile.plus;
    }
    __syncthreads();
  }
  return pos;
}

// Columns of `in` (all columns 0..nin-1 when in == nullptr) holding a
// repeated row, compacted in order into `out`; returns their number.
__device__ uint32_t flag_compact(const uint32_t* rows, int64_t zeta, const uint32_t* in, uint32_t nin,
                                 uint32_t* out) {
  __shared__ uint32_t s_tot;
  uint32_t nout = 0;
  for (uint32_t c0 = 0; c0 < nin; c0 += RD_T) {
    const uint32_t q = c0 + threadIdx.x;
    uint32_t j = 0, bad = 0;
    if (q < nin) {
      j = in ? in[q] : q;
      const uint32_t* r = rows + static_cast<int64_t>(j) * zeta;
      for (int64_t a = 1; a < zeta && !bad; ++a) {
        const uint32_t ra = r[a];
        for (int64_t b = 0; b < a; ++b)
          if (r[b] == ra) {
            bad = 1;
            break;
          }
      }
    }
    const uint32_t ex = block_excl_scan(bad, &s_tot);
    if (bad) out[nout + ex] = j;
    nout += s_tot;
  }
  return nout;
}

// first != 0: continues from the parallel first draw (slots[0] = position
// before it, *pos_in = after it unless its margin ran short, which this
// kernel then completes); first == 0: continues after host-driven parallel
// rounds (*pos_in = position, bad_a = the current bad list).  The final
// position goes to slots[0] for k_signs.
__global__ void __launch_bounds__(RD_T, 1) k_redraw(Stream st, uint32_t bound, uint32_t thr, uint64_t N,
                                                    uint32_t* rows, int64_t m, int64_t zeta,
                                                    const uint32_t* scanned1, uint64_t nchunks1,
                                                    uint64_t nwords1, uint64_t* slots, const uint64_t* pos_in,
                                                    uint32_t* bad_a, uint32_t* bad_b, const uint32_t* nbad1,
                                                    int first) {
  const u128 inc = mk128(st.i_hi, st.i_lo);
  RedrawJumps jp;
  jp.mine = pcg_jump(inc, static_cast<uint64_t>(threadIdx.x) * (RD_W / 2));
  jp.tile = pcg_jump(inc, static_cast<uint64_t>(RD_T) * RD_W / 2);
  const uint64_t total1 = first ? scanned1[nchunks1] : N;
  uint64_t pos;
  uint32_t nbad;
  uint32_t* cur = bad_a;
  uint32_t* nxt = bad_b;
  if (total1 < N) {
    pos = draw_seq(st, jp, slots[0] + nwords1, N - total1, bound, thr, rows, total1, nullptr, zeta);
    nbad = flag_compact(rows, zeta, nullptr, static_cast<uint32_t>(m), cur);
  } else {
    pos = *pos_in;
    nbad = *nbad1;
  }
  while (nbad > 0) {
    pos = draw_seq(st, jp, pos, static_cast<uint64_t>(nbad) * zeta, bound, thr, rows, 0, cur, zeta);
    nbad = flag_compact(rows, zeta, cur, nbad, nxt);
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) slots[0] = pos;
}

__global__ void k_pack_src(const uint8_t* neg, int64_t m, int64_t zeta, uint32_t* vals) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e < m * zeta)
    vals[e] = static_cast<uint32_t>(e / zeta) | (static_cast<uint32_t>(neg[e]) << 31);
}

__global__ void k_row_ptr(const uint32_t* keys, int64_t nnz, int64_t d, uint32_t* ptr) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i > d) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < static_cast<uint32_t>(i)) lo = mid + 1; else hi = mid;
  }
  ptr[i] = static_cast<uint32_t>(lo);
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

struct PatternWs {
  uint32_t* counts;    // nchunks + 1
  uint32_t* scanned;   // nchunks + 1
  uint32_t* flags;     // m
  uint32_t* fscan;     // m
  uint32_t* bad_a;     // m
  uint32_t* bad_b;     // m
  uint32_t* keys_out;  // m*zeta
  uint32_t* vals_in;   // m*zeta
  uint64_t* scalars;   // [end_word, nbad(u32 as u64), ...]
  void* cub_tmp;
  size_t cub_bytes;
  uint64_t chunk_cap;
};

int64_t max_words(int64_t N) {
  // Lemire rejection probability is < bound / 2^32; allow a 0.2% + 4096
  // margin and fall back to a second, exact pass if it is ever exceeded.
  return N + N / 512 + 4096;
}

size_t cub_bytes_needed(int64_t m, int64_t zeta) {
  const int64_t nnz = m * zeta;
  const int64_t nchunks = max_words(nnz) / CH + 2;
  size_t a = 0, b = 0, c = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, static_cast<int>(nnz));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                static_cast<int>(nchunks));
  cub::DeviceScan::ExclusiveSum(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                static_cast<int>(m));
  return std::max(a, std::max(b, c));
}

int64_t carve(Carver& cv, PatternWs& w, int64_t m, int64_t zeta) {
  const int64_t nnz = m * zeta;
  const int64_t nchunks = max_words(nnz) / CH + 2;
  w.chunk_cap = static_cast<uint64_t>(nchunks);
  w.counts = cv.take<uint32_t>(nchunks + 1);
  w.scanned = cv.take<uint32_t>(nchunks + 1);
  w.flags = cv.take<uint32_t>(m + 1);
  w.fscan = cv.take<uint32_t>(m + 1);
  w.bad_a = cv.take<uint32_t>(m + 1);
  w.bad_b = cv.take<uint32_t>(m + 1);
  w.keys_out = cv.take<uint32_t>(nnz);
  w.vals_in = cv.take<uint32_t>(nnz);
  w.scalars = cv.take<uint64_t>(8);
  w.cub_bytes = cub_bytes_needed(m, zeta);
  w.cub_tmp = cv.take<char>(static_cast<int64_t>(w.cub_bytes));
  return cv.off;
}

// Group the (m, zeta) pattern by sketch row, keeping source order ascending
// (stable LSD sort of entries enumerated column-major == ascending j).
int build_csr(const uint32_t* rows, const uint8_t* neg, int64_t m, int64_t zeta, int64_t d,
              uint32_t* sk_ptr, uint32_t* sk_src, PatternWs& w, cudaStream_t s) {
  const int64_t nnz = m * zeta;
  k_pack_src<<<blocks_for(nnz, 256), 256, 0, s>>>(neg, m, zeta, w.vals_in);
  count_launch();
  int end_bit = 1;
  while ((1ll << end_bit) < d) ++end_bit;
  size_t tb = w.cub_bytes;
  ITSK_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, rows, w.keys_out, w.vals_in, sk_src,
                                            static_cast<int>(nnz), 0, end_bit, s));
  count_launch(end_bit <= 8 ? 2 : 4);
  k_row_ptr<<<blocks_for(d + 1, 256), 256, 0, s>>>(w.keys_out, nnz, d, sk_ptr);
  count_launch();
  ITSK_CHECK_LAUNCH();
  return ITSK_OK;
}

}  // namespace
}  // namespace itsk

using namespace itsk;

extern "C" int itsk_pattern_workspace(int64_t d, int64_t m, int64_t zeta, int64_t* bytes) {
  ITSK_REQUIRE(bytes && d >= 1 && m >= 1 && zeta >= 1 && zeta <= d, "bad pattern shape");
  Carver cv(nullptr, 0);
  PatternWs w;
  *bytes = carve(cv, w, m, zeta) + 256;
  return ITSK_OK;
}

extern "C" int itsk_sparse_sign_pattern(int64_t d, int64_t m, int64_t zeta, const uint64_t pcg[4],
                                        int has_uint32, uint32_t uinteger, uint32_t* rows,
                                        uint8_t* neg, uint32_t* sk_ptr, uint32_t* sk_src,
                                        void* ws, int64_t ws_bytes, itsk_stream_t stream) {
  ITSK_REQUIRE(d >= 1 && m >= 1, "d and m must be >= 1");
  ITSK_REQUIRE(zeta >= 1 && zeta <= d, "need 1 <= zeta <= d, got zeta=%lld, d=%lld",
               (long long)zeta, (long long)d);
  ITSK_REQUIRE(d <= 0xFFFFFFFFll && m < (1ll << 31) && m * zeta < (1ll << 32),
               "pattern too large for 32-bit indices");
  ITSK_REQUIRE(rows && neg && pcg, "null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Carver cv(ws, ws_bytes);
  PatternWs w;
  carve(cv, w, m, zeta);
  ITSK_REQUIRE(cv.ok(), "pattern workspace too small");
  Stream st{pcg[0], pcg[1], pcg[2], pcg[3], uinteger, has_uint32 ? 1 : 0};
  const int64_t nnz = m * zeta;
  // stream position on the device: slots[0] before / after all row draws,
  // slots[1] after the first draw (the host never waits on the pattern)
  uint64_t* slots = w.scalars + 2;
  ITSK_CUDA(cudaMemsetAsync(w.scalars, 0, 8 * sizeof(uint64_t), s));
  if (zeta == d) {  // np.tile(np.arange(d), (m, 1)): no draws
    k_tile_rows<<<blocks_for(nnz, 256), 256, 0, s>>>(rows, m, zeta);
    count_launch();
    ITSK_CHECK_LAUNCH();
  } else {
    // first draw, all m*zeta values in parallel (embed.py:36): per-chunk
    // accept counts, their scan, emission in stream order
    const uint32_t bound = static_cast<uint32_t>(d);
    const uint32_t thr = static_cast<uint32_t>((0x100000000ull - bound) % bound);
    uint64_t nwords = static_cast<uint64_t>(max_words(nnz));
    // test hook: a short first-draw margin exercises k_redraw's completion path
    if (const char* e = getenv("ITSK_PATTERN_WORDS_DIV")) nwords = std::max<uint64_t>(1, nwords / std::max(1, atoi(e)));
    const uint64_t nchunks = (nwords + CH - 1) / CH;
    k_lemire_count<<<blocks_for(nchunks, 256), 256, 0, s>>>(st, slots, nwords, bound, thr, w.counts, nchunks);
    count_launch();
    size_t tb = w.cub_bytes;
    ITSK_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.counts, w.scanned, static_cast<int>(nchunks + 1), s));
    count_launch();
    k_lemire_emit_first<<<blocks_for(nchunks, 32 * EM_WARPS), 32 * EM_WARPS, 0, s>>>(
        st, slots, nwords, bound, thr, w.scanned, nchunks, static_cast<uint64_t>(nnz), rows, slots + 1);
    count_launch();
    // duplicate scan of every column, compacted in column order (embed.py:38-40)
    k_flag_dupes<<<blocks_for(m, 256), 256, 0, s>>>(rows, zeta, nullptr, m, w.flags);
    count_launch();
    tb = w.cub_bytes;
    ITSK_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.flags, w.fscan, static_cast<int>(m), s));
    count_launch();
    uint32_t* nbad_dev = reinterpret_cast<uint32_t*>(w.scalars + 1);
    k_compact<<<blocks_for(m, 256), 256, 0, s>>>(w.flags, w.fscan, nullptr, m, w.bad_a, nbad_dev);
    count_launch();
    // Further rounds (embed.py:41).  When many columns are expected to hold a
    // repeat (small d, large zeta: C5's d = 4n points redraw a quarter of the
    // columns), the big rounds run as parallel draws with the host reading
    // each round's count; the tail of small rounds — all of them at C1..C4 —
    // runs on one CTA with no host round trip.
    uint32_t* cur = w.bad_a;
    uint32_t* nxt = w.bad_b;
    uint64_t* pin = slots + 1;
    uint64_t* pout = slots + 2;
    int first = 1;
    double keep = 1.0;  // expected fraction of columns without a repeat
    for (int64_t k = 1; k < zeta; ++k) keep *= 1.0 - static_cast<double>(k) / static_cast<double>(d);
    if (static_cast<double>(m) * (1.0 - keep) * static_cast<double>(zeta) > RD_PAR_MIN) {
      uint64_t hs[2];
      uint32_t tot1 = 0;
      ITSK_CUDA(cudaMemcpyAsync(&tot1, w.scanned + nchunks, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      ITSK_CUDA(cudaMemcpyAsync(hs, w.scalars, sizeof(hs), cudaMemcpyDeviceToHost, s));
      ITSK_CUDA(cudaStreamSynchronize(s));
      uint32_t nbad = static_cast<uint32_t>(hs[1]);
      if (tot1 >= static_cast<uint64_t>(nnz)) {  // else k_redraw completes the short first draw
        first = 0;
        while (static_cast<uint64_t>(nbad) * zeta > RD_PAR_MIN) {
          const uint64_t N = static_cast<uint64_t>(nbad) * zeta;
          uint64_t nw = static_cast<uint64_t>(max_words(static_cast<int64_t>(N)));
          for (;;) {  // a short margin (never seen in practice) retries with more words
            const uint64_t nch = (nw + CH - 1) / CH;
            ITSK_REQUIRE(nch <= w.chunk_cap, "pattern: redraw margin exceeds the workspace");
            k_lemire_count<<<blocks_for(nch, 256), 256, 0, s>>>(st, pin, nw, bound, thr, w.counts, nch);
            count_launch();
            tb = w.cub_bytes;
            ITSK_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.counts, w.scanned, static_cast<int>(nch + 1), s));
            count_launch();
            k_lemire_emit<<<blocks_for(nch, 256), 256, 0, s>>>(st, pin, nw, bound, thr, w.scanned, nch, N, rows,
                                                                 cur, zeta, pout);
            count_launch();
            uint32_t tot = 0;
            ITSK_CUDA(cudaMemcpyAsync(&tot, w.scanned + nch, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
            ITSK_CUDA(cudaStreamSynchronize(s));
            if (tot >= N) break;
            nw = nw * 2 + 65536;
          }
          k_flag_dupes<<<blocks_for(nbad, 256), 256, 0, s>>>(rows, zeta, cur, nbad, w.flags);
          count_launch();
          tb = w.cub_bytes;
          ITSK_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.flags, w.fscan, static_cast<int>(nbad), s));
          count_launch();
          k_compact<<<blocks_for(nbad, 256), 256, 0, s>>>(w.flags, w.fscan, cur, nbad, nxt, nbad_dev);
          count_launch();
          ITSK_CHECK_LAUNCH();
          ITSK_CUDA(cudaMemcpyAsync(hs, w.scalars, sizeof(hs), cudaMemcpyDeviceToHost, s));
          ITSK_CUDA(cudaStreamSynchronize(s));
          nbad = static_cast<uint32_t>(hs[1]);
          std::swap(cur, nxt);
          std::swap(pin, pout);
        }
      }
    }
    k_redraw<<<1, RD_T, 0, s>>>(st, bound, thr, static_cast<uint64_t>(nnz), rows, m, zeta, w.scanned, nchunks,
                                nwords, slots, pin, cur, nxt, nbad_dev, first);
    count_launch();
    ITSK_CHECK_LAUNCH();
  }
  k_signs<<<blocks_for((nnz + CH - 1) / CH, 256), 256, 0, s>>>(st, slots, nnz, neg);
  count_launch();
  ITSK_CHECK_LAUNCH();
  if (sk_ptr && sk_src) {
    int rc2 = build_csr(rows, neg, m, zeta, d, sk_ptr, sk_src, w, s);
    if (rc2) return rc2;
  }
  return ITSK_OK;
}

extern "C" int itsk_pattern_csr(const uint32_t* rows, const uint8_t* neg, int64_t m, int64_t zeta,
                                int64_t d, uint32_t* sk_ptr, uint32_t* sk_src, void* ws,
                                int64_t ws_bytes, itsk_stream_t stream) {
  ITSK_REQUIRE(rows && neg && sk_ptr && sk_src && ws, "null pointer");
  ITSK_REQUIRE(d >= 1 && m >= 1 && zeta >= 1 && m < (1ll << 31) && m * zeta < (1ll << 31),
               "bad pattern slice");
  Carver cv(ws, ws_bytes);
  PatternWs w;
  carve(cv, w, m, zeta);
  ITSK_REQUIRE(cv.ok(), "pattern workspace too small");
  return build_csr(rows, neg, m, zeta, d, sk_ptr, sk_src, w, reinterpret_cast<cudaStream_t>(stream));
}
