// tm_ingest.cu — transaction-log ingestion on the GPU.
//
// Replaces txgraph.parse_transactions (txgraph.py:253-314) + build_graph
// (:317-354) for the data rows of a delimited log (the host resolves the
// header row against the ColumnMapping, _resolve_columns :207-234):
//
//   1. rows        csv.reader splits records at '\n', '\r\n' or a lone '\r'
//                  (no quoted fields here).  Two passes over 4 KiB tiles:
//                  terminator counts per tile, a scan, then each tile writes
//                  its terminator offsets — coalesced 16-byte loads.
//   2. edges       blank rows ([] or one whitespace-only field, :285-286)
//                  are skipped but still counted in line numbers: a keep
//                  flag per row and a scan give each record its edge id.
//   3. fields      one thread per row splits it at the delimiter and runs
//                  the reference's per-row checks in the reference's order:
//                  column count (:289-290), timestamp = int() or strptime
//                  with the mapping's format (:237-247), negative (:294),
//                  amount = float() (:296), currency strip (:299), label
//                  sets (:300-308).  The first failing row wins (atomicMin).
//   4. ids         node keys (bank, account) — or the account alone when
//                  the bank column is unmapped — are hashed (64 bit) in the
//                  order node_of sees them (src then dst per row, :275-282).
//                  A stable radix sort of (hash, position), run heads, and
//                  a scan over first-occurrence flags give dense ids in
//                  FIRST-SEEN order; adjacent equal hashes are compared byte
//                  by byte, so a collision is reported, never merged.  The
//                  currency vocabulary (build_graph :341-345) is the same
//                  computation over one key per edge.
//
// Floats: float() is correctly rounded; decimal literals with <= 19
// significant digits are converted exactly — 128-bit integer arithmetic for
// decimal exponents in [-22, 19] (all practical amounts), multi-limb
// arithmetic beyond, inf / 0.0 outside the double range.  Results that
// would be subnormal are TM_PARSE_UNSUPPORTED.  Inputs
// that Python accepts but this parser does not (quoted fields, longer
// mantissas, '_' digit separators, timestamps beyond int64) fail loudly with
// TM_PARSE_UNSUPPORTED — there is no CPU fallback.
#include <vector>

#include "tm_internal.cuh"

struct tm_ingest {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n_rows = 0, n_edges = 0, n_nodes = 0, n_cur = 0;
  tmb::DevBuf src, dst, time, amount, currency, label;
  tmb::DevBuf vocab_off;    // int64 [n_cur + 1] byte offsets of the vocabulary strings
  tmb::DevBuf vocab_bytes;  // the strings in code (first-seen) order
};

namespace tmb {
namespace {

constexpr int kTileThreads = 256;
constexpr int kTileBytes = kTileThreads * 16;

__device__ __forceinline__ bool is_term(const char *__restrict__ b, int64_t len, int64_t i) {
  const char c = b[i];
  return c == '\n' || (c == '\r' && (i + 1 >= len || b[i + 1] != '\n'));
}

// per-thread terminator count of bytes [t0, t0 + 16); quotes flagged
__device__ __forceinline__ int count16(const char *__restrict__ b, int64_t len, int64_t t0,
                                       unsigned *quote) {
  int n = 0;
  bool q = false;
  if (t0 + 16 <= len && ((reinterpret_cast<uintptr_t>(b + t0) & 15) == 0)) {
    const uint4 w = *reinterpret_cast<const uint4 *>(b + t0);
    const char *c = reinterpret_cast<const char *>(&w);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const char x = c[k];
      const char nx = k + 1 < 16 ? c[k + 1] : (t0 + 16 < len ? b[t0 + 16] : 0);
      n += (x == '\n') || (x == '\r' && (t0 + k + 1 >= len || nx != '\n'));
      q |= x == '"';
    }
  } else {
    for (int64_t i = t0; i < t0 + 16 && i < len; ++i) {
      n += is_term(b, len, i);
      q |= b[i] == '"';
    }
  }
  if (q) atomicOr(quote, 1u);
  return n;
}

__global__ void __launch_bounds__(kTileThreads) k_term_count(const char *__restrict__ b, int64_t len,
                                                             unsigned long long *__restrict__ counts,
                                                             unsigned *quote) {
  const int64_t t0 = (int64_t)blockIdx.x * kTileBytes + (int64_t)threadIdx.x * 16;
  int n = count16(b, len, t0, quote);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  __shared__ int ws[kTileThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int i = 0; i < kTileThreads / 32; ++i) s += ws[i];
    counts[blockIdx.x] = (unsigned long long)s;
  }
}

__global__ void __launch_bounds__(kTileThreads) k_term_write(const char *__restrict__ b, int64_t len,
                                                             const unsigned long long *__restrict__ offs,
                                                             int64_t *__restrict__ rend) {
  const int64_t t0 = (int64_t)blockIdx.x * kTileBytes + (int64_t)threadIdx.x * 16;
  int n = 0;
  for (int64_t i = t0; i < t0 + 16 && i < len; ++i) n += is_term(b, len, i);
  // block exclusive scan of n
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __shared__ int ws[kTileThreads / 32];
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < warp; ++i) base += ws[i];
  int64_t k = (int64_t)offs[blockIdx.x] + base + incl - n;
  for (int64_t i = t0; i < t0 + 16 && i < len; ++i)
    if (is_term(b, len, i)) rend[k++] = i;
}

// ------------------------------------------------------------ row helpers

struct Row {
  int64_t s, e;  // content [s, e), terminator excluded
};

__device__ __forceinline__ Row row_at(const char *__restrict__ b, int64_t len,
                                      const int64_t *__restrict__ rend, int64_t r) {
  Row w;
  w.s = r == 0 ? 0 : rend[r - 1] + 1;
  w.e = rend[r];
  if (w.e < len && b[w.e] == '\n' && w.e > w.s && b[w.e - 1] == '\r') w.e -= 1;
  return w;
}

// Python str.isspace() characters in UTF-8: byte length of the one starting
// at i (forward) or ending at e (backward), 0 if none
__device__ __forceinline__ bool ascii_ws(unsigned char c) {
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}
__device__ __forceinline__ bool ws3(unsigned char a, unsigned char b1, unsigned char c) {
  if (a == 0xE1) return b1 == 0x9A && c == 0x80;                       // U+1680
  if (a == 0xE2 && b1 == 0x80) return c <= 0x8A || c == 0xA8 || c == 0xA9 || c == 0xAF;  // U+2000-200A, 2028/9, 202F
  if (a == 0xE2 && b1 == 0x81) return c == 0x9F;                       // U+205F
  if (a == 0xE3) return b1 == 0x80 && c == 0x80;                       // U+3000
  return false;
}
__device__ __forceinline__ int ws_fwd(const unsigned char *p, int64_t i, int64_t e) {
  const unsigned char c = p[i];
  if (ascii_ws(c)) return 1;
  if (c == 0xC2 && i + 1 < e && (p[i + 1] == 0x85 || p[i + 1] == 0xA0)) return 2;
  if (c >= 0xE1 && c <= 0xE3 && i + 2 < e && ws3(c, p[i + 1], p[i + 2])) return 3;
  return 0;
}
__device__ __forceinline__ int ws_back(const unsigned char *p, int64_t s, int64_t e) {
  if (ascii_ws(p[e - 1])) return 1;
  if (e - 2 >= s && p[e - 2] == 0xC2 && (p[e - 1] == 0x85 || p[e - 1] == 0xA0)) return 2;
  if (e - 3 >= s && ws3(p[e - 3], p[e - 2], p[e - 1])) return 3;
  return 0;
}
__device__ __forceinline__ void strip(const unsigned char *p, int64_t &s, int64_t &e) {
  int k;
  while (s < e && (k = ws_fwd(p, s, e)) > 0) s += k;
  while (e > s && (k = ws_back(p, s, e)) > 0) e -= k;
}

// blank row: [] or a single field that strips to nothing (txgraph.py:285-286)
__device__ __forceinline__ bool blank_row(const unsigned char *p, Row w, char delim) {
  for (int64_t i = w.s; i < w.e; ++i)
    if (p[i] == (unsigned char)delim) return false;
  int64_t s = w.s, e = w.e;
  strip(p, s, e);
  return s == e;
}

__global__ void k_keep(const char *__restrict__ b, int64_t len, const int64_t *__restrict__ rend,
                       int64_t n_rows, char delim, uint32_t *__restrict__ keep) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  keep[r] = blank_row(reinterpret_cast<const unsigned char *>(b), row_at(b, len, rend, r), delim) ? 0u : 1u;
}

// ------------------------------------------------------------ numbers

constexpr int kOk = TM_PARSE_OK, kUnsup = TM_PARSE_UNSUPPORTED;

// int(text) for stripped text: [+-] digits with single '_' between digits.
// 0 ok, 1 not an int, kUnsup beyond int64
__device__ int parse_int(const unsigned char *p, int64_t s, int64_t e, int64_t &out) {
  if (s >= e) return 1;
  bool neg = false;
  if (p[s] == '+' || p[s] == '-') {
    neg = p[s] == '-';
    ++s;
  }
  if (s >= e) return 1;
  unsigned __int128 v = 0;
  bool prev_digit = false, big = false;
  for (int64_t i = s; i < e; ++i) {
    const unsigned char c = p[i];
    if (c >= '0' && c <= '9') {
      v = v * 10 + (c - '0');
      if (v > ((unsigned __int128)1 << 64)) big = true, v = (unsigned __int128)1 << 64;
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < e && p[i + 1] >= '0' && p[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return 1;
    }
  }
  if (big || v > (unsigned __int128)INT64_MAX + (neg ? 1 : 0)) return kUnsup;
  out = neg ? (int64_t)(0 - (uint64_t)v) : (int64_t)(uint64_t)v;
  return 0;
}

__device__ __forceinline__ int bitlen128(unsigned __int128 x) {
  const uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
  return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

__device__ __forceinline__ unsigned __int128 pow10_128(int k) {
  unsigned __int128 r = 1;
  for (int i = 0; i < k; ++i) r *= 10;
  return r;
}

// Wide path of float(): w * 10^q for exponents the 128-bit path cannot hold,
// with little-endian 32-bit limbs (1088 bits: |q| <= 330 with 19 digits).
// Rare (only exotic literals take it), so it is plain schoolbook code.
constexpr int kLimbs = 34;
struct Big {
  uint32_t d[kLimbs];
  int n;  // limbs in use
};
__device__ void big_set(Big &x, uint64_t v) {
  x.d[0] = (uint32_t)v;
  x.d[1] = (uint32_t)(v >> 32);
  x.n = x.d[1] ? 2 : (x.d[0] ? 1 : 0);
}
__device__ bool big_mul(Big &x, uint32_t m) {
  uint64_t carry = 0;
  for (int i = 0; i < x.n; ++i) {
    const uint64_t t = (uint64_t)x.d[i] * m + carry;
    x.d[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) {
    if (x.n == kLimbs) return false;
    x.d[x.n++] = (uint32_t)carry;
  }
  return true;
}
__device__ bool big_pow5(Big &x, int n) {  // x *= 5^n
  while (n > 0) {
    const int k = n < 13 ? n : 13;
    uint32_t f = 1;
    for (int i = 0; i < k; ++i) f *= 5;
    if (!big_mul(x, f)) return false;
    n -= k;
  }
  return true;
}
__device__ int big_bitlen(const Big &x) { return x.n ? 32 * (x.n - 1) + 32 - __clz(x.d[x.n - 1]) : 0; }
__device__ bool big_bit(const Big &x, int b) { return b >= 0 && (b >> 5) < x.n && ((x.d[b >> 5] >> (b & 31)) & 1); }
__device__ bool big_any_below(const Big &x, int b) {  // any bit in [0, b)
  for (int i = 0; i < x.n && 32 * i < b; ++i) {
    const int hi = b - 32 * i;
    const uint32_t mask = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1);
    if (x.d[i] & mask) return true;
  }
  return false;
}
__device__ uint32_t big_limb_shifted(const Big &x, int i, int sh) {  // limb i of x << sh
  const int q = sh >> 5, r = sh & 31;
  const int j = i - q;
  const uint32_t lo = (j >= 0 && j < x.n) ? x.d[j] : 0;
  const uint32_t lo2 = (j - 1 >= 0 && j - 1 < x.n) ? x.d[j - 1] : 0;
  return r ? (lo << r) | (lo2 >> (32 - r)) : lo;
}
__device__ bool big_shl(Big &x, int sh) {
  const int nb = big_bitlen(x) + sh;
  const int n = (nb + 31) >> 5;
  if (n > kLimbs) return false;
  uint32_t t[kLimbs];
  for (int i = 0; i < n; ++i) t[i] = big_limb_shifted(x, i, sh);
  for (int i = 0; i < n; ++i) x.d[i] = t[i];
  x.n = n;
  while (x.n && !x.d[x.n - 1]) --x.n;
  return true;
}
// R -= B << sh if R >= B << sh; returns whether it subtracted
__device__ bool big_try_sub(Big &R, const Big &B, int sh) {
  const int bl = big_bitlen(B) + sh, rl = big_bitlen(R);
  if (bl > rl) return false;
  const int n = R.n;
  if (bl == rl) {
    for (int i = n - 1; i >= 0; --i) {
      const uint32_t a = R.d[i], b = big_limb_shifted(B, i, sh);
      if (a != b) {
        if (a < b) return false;
        break;
      }
    }
  }
  int64_t borrow = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t t = (int64_t)R.d[i] - big_limb_shifted(B, i, sh) - borrow;
    R.d[i] = (uint32_t)t;
    borrow = t < 0 ? 1 : 0;
  }
  while (R.n && !R.d[R.n - 1]) --R.n;
  return true;
}
// round m (53 significant bits wanted) given the dropped-bit summary
__device__ double round_pack(uint64_t m, bool half_bit, bool below, int ex, bool &ok) {
  if (half_bit && (below || (m & 1))) {
    if (++m == (1ull << 53)) m >>= 1, ++ex;
  }
  ok = ex >= -1074;  // normal result (no double rounding into subnormals)
  return ldexp((double)m, ex);
}
// w * 10^q correctly rounded, or false (outside the normal range)
__device__ bool wide_decimal(uint64_t w, int q, double &out) {
  Big N;
  big_set(N, w);
  bool ok = true;
  if (q >= 0) {
    if (!big_pow5(N, q)) return false;
    const int L = big_bitlen(N);
    if (L <= 53) {
      uint64_t m = (uint64_t)N.d[0] | (N.n > 1 ? (uint64_t)N.d[1] << 32 : 0);
      out = ldexp((double)m, q);
      return true;
    }
    const int sft = L - 53;
    uint64_t m = 0;
    for (int b = 0; b < 53; ++b) m |= (uint64_t)big_bit(N, sft + b) << b;
    out = round_pack(m, big_bit(N, sft - 1), big_any_below(N, sft - 1), sft + q, ok);
    return ok;
  }
  const int n = -q;
  Big B;
  big_set(B, 1);
  if (!big_pow5(B, n)) return false;
  const int k = 54 + big_bitlen(B) - (64 - __clzll((long long)w));
  if (k < 0 || !big_shl(N, k)) return false;
  uint64_t Q = 0;
  for (int i = 56; i >= 0; --i)
    if (big_try_sub(N, B, i)) Q |= 1ull << i;
  const int sft = (64 - __clzll((long long)Q)) - 53;
  const uint64_t m = Q >> sft;
  const bool half_bit = (Q >> (sft - 1)) & 1;
  const bool below = (Q & ((1ull << (sft - 1)) - 1)) != 0 || N.n != 0;
  out = round_pack(m, half_bit, below, sft - k - n, ok);
  return ok;
}

__device__ __forceinline__ bool ieq(unsigned char c, char lower) { return (c | 0x20) == lower; }

// float(text): 0 ok, TM_PARSE_AMOUNT invalid, kUnsup outside the exact path
__device__ int parse_float(const unsigned char *p, int64_t s, int64_t e, double &out) {
  strip(p, s, e);
  if (s >= e) return TM_PARSE_AMOUNT;
  bool neg = false;
  if (p[s] == '+' || p[s] == '-') {
    neg = p[s] == '-';
    ++s;
  }
  const int64_t n = e - s;
  // inf / infinity / nan (case-insensitive)
  if (n == 3 && ieq(p[s], 'i') && ieq(p[s + 1], 'n') && ieq(p[s + 2], 'f')) {
    out = neg ? -INFINITY : INFINITY;
    return kOk;
  }
  if (n == 8) {
    const char *w = "infinity";
    bool ok = true;
    for (int k = 0; k < 8; ++k) ok &= ieq(p[s + k], w[k]);
    if (ok) {
      out = neg ? -INFINITY : INFINITY;
      return kOk;
    }
  }
  if (n == 3 && ieq(p[s], 'n') && ieq(p[s + 1], 'a') && ieq(p[s + 2], 'n')) {
    out = copysign(NAN, neg ? -1.0 : 1.0);
    return kOk;
  }
  uint64_t w = 0;
  int nd = 0;          // significant digits kept in w
  int q = 0;           // decimal exponent of w
  int zeros = 0;       // pending zeros after the last nonzero kept digit
  bool any = false, dot = false, inexact = false;
  int64_t i = s;
  for (; i < e; ++i) {
    const unsigned char c = p[i];
    if (c >= '0' && c <= '9') {
      any = true;
      if (dot) --q;
      if (c == '0') {
        if (nd > 0) ++zeros;
        continue;
      }
      // a nonzero digit: flush pending zeros into w
      if (nd + zeros + 1 > 19) {
        inexact = true;
        break;
      }
      for (int z = 0; z < zeros; ++z) w *= 10;
      nd += zeros;
      zeros = 0;
      w = w * 10 + (c - '0');
      ++nd;
    } else if (c == '.' && !dot) {
      dot = true;
    } else {
      break;
    }
  }
  if (inexact) return kUnsup;
  if (!any) return TM_PARSE_AMOUNT;
  q += zeros;  // trailing zeros of the mantissa become exponent
  if (i < e) {
    if (p[i] == '_') return kUnsup;
    if (p[i] != 'e' && p[i] != 'E') return TM_PARSE_AMOUNT;
    ++i;
    bool eneg = false;
    if (i < e && (p[i] == '+' || p[i] == '-')) {
      eneg = p[i] == '-';
      ++i;
    }
    if (i >= e) return TM_PARSE_AMOUNT;
    int x = 0;
    for (; i < e; ++i) {
      const unsigned char c = p[i];
      if (c == '_') return kUnsup;
      if (c < '0' || c > '9') return TM_PARSE_AMOUNT;
      if (x < 100000) x = x * 10 + (c - '0');
    }
    q += eneg ? -x : x;
  }
  if (w == 0) {
    out = neg ? -0.0 : 0.0;
    return kOk;
  }
  double v;
  const int mag = q + nd;  // w * 10^q lies in [10^(mag-1), 10^mag)
  if (mag > 310) {         // beyond DBL_MAX: float() gives inf
    out = neg ? -INFINITY : INFINITY;
    return kOk;
  }
  if (mag < -330) {        // below the smallest subnormal / 2: 0.0
    out = neg ? -0.0 : 0.0;
    return kOk;
  }
  if (q > 38 || q < -22 ||
      (q >= 0 && bitlen128(pow10_128(q)) + (64 - __clzll((long long)w)) > 127)) {
    double v;
    if (!wide_decimal(w, q, v)) return kUnsup;
    out = neg ? -v : v;
    return kOk;
  }
  if (q >= 0) {
    const unsigned __int128 P = pow10_128(q);
    const unsigned __int128 N = (unsigned __int128)w * P;
    const int L = bitlen128(N);
    if (L <= 53) {
      v = (double)(uint64_t)N;
    } else {
      const int sft = L - 53;
      uint64_t m = (uint64_t)(N >> sft);
      const unsigned __int128 dropped = N & ((((unsigned __int128)1) << sft) - 1);
      const unsigned __int128 half = ((unsigned __int128)1) << (sft - 1);
      int ex = sft;
      if (dropped > half || (dropped == half && (m & 1))) {
        if (++m == (1ull << 53)) m >>= 1, ++ex;
      }
      v = ldexp((double)m, ex);
    }
  } else {
    const unsigned __int128 D = pow10_128(-q);
    const int bw = 64 - __clzll((long long)w);
    const int k = 54 + bitlen128(D) - bw;  // numerator has 54 + bitlen(D) <= 128 bits
    const unsigned __int128 Nn = (unsigned __int128)w << k;
    const unsigned __int128 Q = Nn / D;
    const bool sticky = (Nn % D) != 0;
    const int sft = bitlen128(Q) - 53;  // 1 or 2
    uint64_t m = (uint64_t)(Q >> sft);
    const uint64_t dropped = (uint64_t)Q & ((1ull << sft) - 1), half = 1ull << (sft - 1);
    int ex = sft - k;
    if (dropped > half || (dropped == half && (sticky || (m & 1)))) {
      if (++m == (1ull << 53)) m >>= 1, ++ex;
    }
    v = ldexp((double)m, ex);
  }
  out = neg ? -v : v;
  return kOk;
}

// ------------------------------------------------------------ strptime

__device__ __forceinline__ bool dig(unsigned char c) { return c >= '0' && c <= '9'; }

// candidate matches of one directive at p[i..e), in the regex's alternative
// order (_strptime.TimeRE): returns the byte length of alternative `alt` and
// its value, or 0 when that alternative does not match
__device__ int fmt_alt(int op, int alt, const unsigned char *p, int64_t i, int64_t e, int &val) {
  const int64_t left = e - i;
  const unsigned char a = left > 0 ? p[i] : 0, b = left > 1 ? p[i + 1] : 0;
  switch (op) {
    case TM_FMT_Y:  // \d\d\d\d
      if (alt == 0 && left >= 4 && dig(a) && dig(b) && dig(p[i + 2]) && dig(p[i + 3])) {
        val = (a - '0') * 1000 + (b - '0') * 100 + (p[i + 2] - '0') * 10 + (p[i + 3] - '0');
        return 4;
      }
      return 0;
    case TM_FMT_y:  // \d\d
      if (alt == 0 && left >= 2 && dig(a) && dig(b)) {
        val = (a - '0') * 10 + (b - '0');
        return 2;
      }
      return 0;
    case TM_FMT_m:  // 1[0-2]|0[1-9]|[1-9]
      if (alt == 0 && left >= 2 && a == '1' && b >= '0' && b <= '2') return val = 10 + (b - '0'), 2;
      if (alt == 1 && left >= 2 && a == '0' && b >= '1' && b <= '9') return val = b - '0', 2;
      if (alt == 2 && left >= 1 && a >= '1' && a <= '9') return val = a - '0', 1;
      return 0;
    case TM_FMT_d:  // 3[0-1]|[1-2]\d|0[1-9]|[1-9]| [1-9]
      if (alt == 0 && left >= 2 && a == '3' && (b == '0' || b == '1')) return val = 30 + (b - '0'), 2;
      if (alt == 1 && left >= 2 && (a == '1' || a == '2') && dig(b)) return val = (a - '0') * 10 + (b - '0'), 2;
      if (alt == 2 && left >= 2 && a == '0' && b >= '1' && b <= '9') return val = b - '0', 2;
      if (alt == 3 && left >= 1 && a >= '1' && a <= '9') return val = a - '0', 1;
      if (alt == 4 && left >= 2 && a == ' ' && b >= '1' && b <= '9') return val = b - '0', 2;
      return 0;
    case TM_FMT_H:  // 2[0-3]|[0-1]\d|\d
      if (alt == 0 && left >= 2 && a == '2' && b >= '0' && b <= '3') return val = 20 + (b - '0'), 2;
      if (alt == 1 && left >= 2 && (a == '0' || a == '1') && dig(b)) return val = (a - '0') * 10 + (b - '0'), 2;
      if (alt == 2 && left >= 1 && dig(a)) return val = a - '0', 1;
      return 0;
    case TM_FMT_M:  // [0-5]\d|\d
      if (alt == 0 && left >= 2 && a >= '0' && a <= '5' && dig(b)) return val = (a - '0') * 10 + (b - '0'), 2;
      if (alt == 1 && left >= 1 && dig(a)) return val = a - '0', 1;
      return 0;
    case TM_FMT_S:  // 6[0-1]|[0-5]\d|\d
      if (alt == 0 && left >= 2 && a == '6' && (b == '0' || b == '1')) return val = 60 + (b - '0'), 2;
      if (alt == 1 && left >= 2 && a >= '0' && a <= '5' && dig(b)) return val = (a - '0') * 10 + (b - '0'), 2;
      if (alt == 2 && left >= 1 && dig(a)) return val = a - '0', 1;
      return 0;
    default: return 0;
  }
}
__device__ __forceinline__ int fmt_nalt(int op) {
  switch (op) {
    case TM_FMT_m: case TM_FMT_H: case TM_FMT_S: return 3;
    case TM_FMT_d: return 5;
    case TM_FMT_M: return 2;
    default: return 1;
  }
}

__device__ __forceinline__ int64_t days_from_civil(int64_t y, int m, int d) {
  y -= m <= 2;
  const int64_t era = (y >= 0 ? y : y - 399) / 400;
  const int64_t yoe = y - era * 400;
  const int64_t doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
  const int64_t doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + doe - 719468;
}

// datetime.strptime(text, fmt) -> epoch seconds (UTC): the FIRST match of
// the directive regex in backtracking order must consume the whole text
// (re.match + "unconverted data remains"), then datetime() validates.
__device__ bool strptime_epoch(const tm_csv_mapping &m, const unsigned char *p, int64_t s, int64_t e,
                               int64_t &out) {
  int64_t pos[TM_FMT_MAX + 1];
  int alt[TM_FMT_MAX + 1], val[TM_FMT_MAX];
  const int n = m.n_fmt;
  int k = 0;
  pos[0] = s;
  alt[0] = 0;
  bool matched = false;
  while (true) {
    if (k == n) {
      matched = true;
      break;
    }
    const int op = m.fmt_op[k];
    const int64_t i = pos[k];
    // alternatives of op k, from alt[k] on, in regex order
    int len = 0;
    if (op == TM_FMT_LIT) {
      if (alt[k] == 0 && i < e) {
        const unsigned char c = p[i], want = (unsigned char)m.fmt_arg[k];
        const bool letter = (want | 0x20) >= 'a' && (want | 0x20) <= 'z';
        if (c == want || (letter && (c | 0x20) == (want | 0x20))) len = 1;
      }
      if (!len) alt[k] = 1;
    } else if (op == TM_FMT_SPACE) {
      // \s+ is greedy: alternative a keeps (run - a) whitespace characters
      int64_t ends[64];
      int run = 0, w;
      int64_t j = i;
      while (j < e && run < 64 && (w = ws_fwd(p, j, e)) > 0) {
        j += w;
        ends[run++] = j;
      }
      if (alt[k] < run) len = (int)(ends[run - 1 - alt[k]] - i);
      else alt[k] = run;
    } else {
      const int na = fmt_nalt(op);
      while (alt[k] < na && (len = fmt_alt(op, alt[k], p, i, e, val[k])) == 0) ++alt[k];
    }
    if (len > 0) {
      pos[k + 1] = i + len;
      ++k;
      alt[k] = 0;
      continue;
    }
    if (k == 0) break;  // no alternative left anywhere: no match
    --k;
    ++alt[k];
  }
  if (!matched || pos[n] != e) return false;
  int year = 1900, month = 1, day = 1, hour = 0, minute = 0, second = 0;
  for (int i = 0; i < n; ++i) {
    switch (m.fmt_op[i]) {
      case TM_FMT_Y: year = val[i]; break;
      case TM_FMT_y: year = val[i] <= 68 ? 2000 + val[i] : 1900 + val[i]; break;
      case TM_FMT_m: month = val[i]; break;
      case TM_FMT_d: day = val[i]; break;
      case TM_FMT_H: hour = val[i]; break;
      case TM_FMT_M: minute = val[i]; break;
      case TM_FMT_S: second = val[i]; break;
      default: break;
    }
  }
  if (year < 1 || second > 59) return false;  // "year 0 is out of range", "second must be in 0..59"
  const bool leap = (year % 4 == 0 && year % 100 != 0) || year % 400 == 0;
  const int mdays[12] = {31, leap ? 29 : 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  if (day > mdays[month - 1]) return false;  // "day is out of range for month"
  out = days_from_civil(year, month, day) * 86400 + hour * 3600 + minute * 60 + second;
  return true;
}

// ------------------------------------------------------------ row parse

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
__device__ __forceinline__ uint64_t hash_bytes(const unsigned char *p, int64_t s, int64_t e, uint64_t seed) {
  uint64_t h = 0xcbf29ce484222325ull ^ seed;
  for (int64_t i = s; i < e; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  return fmix64(h ^ (uint64_t)(e - s));
}

// key spans of one edge: [0] src bank, [1] src account, [2] dst bank,
// [3] dst account, [4] currency; begin = -1 marks "no bank column"
struct Spans {
  int64_t *beg;
  int32_t *len;
};

__global__ void k_parse(const __grid_constant__ tm_csv_mapping m, const char *__restrict__ bc, int64_t len,
                        const int64_t *__restrict__ rend, int64_t n_rows, const uint32_t *__restrict__ eidx,
                        const uint32_t *__restrict__ keep, int8_t *__restrict__ status,
                        unsigned long long *__restrict__ err_row, int64_t *__restrict__ ts_out,
                        double *__restrict__ amt_out, int8_t *__restrict__ lab_out,
                        uint64_t *__restrict__ node_key, uint64_t *__restrict__ cur_key, Spans sp) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  status[r] = kOk;
  if (!keep[r]) return;
  const unsigned char *p = reinterpret_cast<const unsigned char *>(bc);
  const Row w = row_at(bc, len, rend, r);
  const int64_t k = eidx[r];
  // split: field spans of the mapped columns (at most 8 distinct indices)
  constexpr int kCols = 8;
  const int cols[kCols] = {m.col_timestamp, m.col_src_bank, m.col_src_account, m.col_dst_bank,
                           m.col_dst_account, m.col_amount, m.col_currency, m.col_label};
  int64_t fs[kCols], fe[kCols];
#pragma unroll
  for (int c = 0; c < kCols; ++c) fs[c] = fe[c] = 0;
  int field = 0;
  int64_t start = w.s;
  const unsigned char delim = (unsigned char)m.delimiter;
  for (int64_t i = w.s;; ++i) {
    if (i == w.e || p[i] == delim) {
#pragma unroll
      for (int c = 0; c < kCols; ++c)
        if (cols[c] == field) fs[c] = start, fe[c] = i;
      ++field;
      start = i + 1;
      if (i == w.e) break;
    }
  }
  int st = kOk;
  if (field <= m.needed) st = TM_PARSE_COLUMNS;
  int64_t ts = 0;
  if (st == kOk) {
    int64_t s = fs[0], e = fe[0];
    strip(p, s, e);
    const int ri = parse_int(p, s, e, ts);
    if (ri == kUnsup) {
      st = kUnsup;
    } else if (ri != 0) {
      int64_t sec;
      if (m.n_fmt > 0 && strptime_epoch(m, p, s, e, sec)) {
        // int(dt.timestamp()) // max(tick_seconds, 1): floor division
        const int64_t t = m.tick_seconds;
        ts = sec / t - ((sec % t != 0) && ((sec < 0) != (t < 0)) ? 1 : 0);
      } else {
        st = TM_PARSE_TIMESTAMP;
      }
    }
    if (st == kOk && ts < 0) st = TM_PARSE_NEGATIVE;
  }
  double amt = 0.0;
  if (st == kOk && m.col_amount >= 0) st = parse_float(p, fs[5], fe[5], amt);
  int8_t lab = -1;
  if (st == kOk && m.col_label >= 0) {
    int64_t s = fs[7], e = fe[7];
    strip(p, s, e);
    const int64_t n = e - s;
    auto is = [&](const char *w, int wl) {
      if (n != wl) return false;
      for (int q = 0; q < wl; ++q) {
        unsigned char c = p[s + q];
        if (c >= 'A' && c <= 'Z') c |= 0x20;
        if (c != (unsigned char)w[q]) return false;
      }
      return true;
    };
    if (is("1", 1) || is("true", 4) || is("yes", 3)) lab = 1;
    else if (n == 0 || is("0", 1) || is("false", 5) || is("no", 2)) lab = 0;
    else st = TM_PARSE_LABEL;
  }
  if (st != kOk) {
    status[r] = (int8_t)st;
    atomicMin(err_row, (unsigned long long)r);
    return;
  }
  ts_out[k] = ts;
  amt_out[k] = amt;
  lab_out[k] = lab;
  // keys (node_of, txgraph.py:275-282; currency strip :299)
  uint64_t h[2];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int cb = side ? 3 : 1, ca = side ? 4 : 2;
    int64_t as = fs[ca], ae = fe[ca];
    strip(p, as, ae);
    uint64_t hk = hash_bytes(p, as, ae, 0x9e3779b97f4a7c15ull);
    int64_t bs = -1, be = -1;
    if (cols[cb] >= 0) {
      bs = fs[cb];
      be = fe[cb];
      strip(p, bs, be);
      hk = fmix64(hk ^ (hash_bytes(p, bs, be, 0x51ed270b27b2c3a5ull) * 0x9e3779b97f4a7c15ull) ^ 0x7f4a7c15ull);
    }
    h[side] = hk;
    sp.beg[5 * k + 2 * side] = bs;
    sp.len[5 * k + 2 * side] = (int32_t)(be - bs);
    sp.beg[5 * k + 2 * side + 1] = as;
    sp.len[5 * k + 2 * side + 1] = (int32_t)(ae - as);
  }
  node_key[2 * k] = h[0];
  node_key[2 * k + 1] = h[1];
  int64_t cs = 0, ce = 0;
  if (m.col_currency >= 0) {
    cs = fs[6];
    ce = fe[6];
    strip(p, cs, ce);
  }
  cur_key[k] = hash_bytes(p, cs, ce, 0x2545f4914f6cdd1dull);
  sp.beg[5 * k + 4] = cs;
  sp.len[5 * k + 4] = (int32_t)(ce - cs);
}

// ------------------------------------------------------------ first-seen ids

__device__ __forceinline__ bool bytes_eq(const unsigned char *p, int64_t a, int32_t la, int64_t b, int32_t lb) {
  if (la != lb) return false;
  for (int32_t i = 0; i < la; ++i)
    if (p[a + i] != p[b + i]) return false;
  return true;
}

// key of position q: node keys (q = 2 * edge + side) use spans 2*side,
// 2*side+1; currency keys (q = edge) use span 4
__device__ __forceinline__ bool keys_eq(const unsigned char *p, const Spans &sp, bool node, uint32_t x,
                                        uint32_t y) {
  if (!node) return bytes_eq(p, sp.beg[5 * (size_t)x + 4], sp.len[5 * (size_t)x + 4],
                             sp.beg[5 * (size_t)y + 4], sp.len[5 * (size_t)y + 4]);
  const size_t bx = 5 * (size_t)(x >> 1) + 2 * (x & 1), by = 5 * (size_t)(y >> 1) + 2 * (y & 1);
  const bool hx = sp.beg[bx] >= 0, hy = sp.beg[by] >= 0;
  if (hx != hy) return false;
  if (hx && !bytes_eq(p, sp.beg[bx], sp.len[bx], sp.beg[by], sp.len[by])) return false;
  return bytes_eq(p, sp.beg[bx + 1], sp.len[bx + 1], sp.beg[by + 1], sp.len[by + 1]);
}

// run heads of the sorted keys (+ byte comparison inside equal-hash runs)
__global__ void k_heads(const uint64_t *__restrict__ ks, const uint32_t *__restrict__ vs, int64_t n,
                        const char *__restrict__ bc, Spans sp, bool node,
                        unsigned long long *__restrict__ head, unsigned *collision) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool h = i == 0 || ks[i] != ks[i - 1];
  head[i] = h ? 1ull : 0ull;
  if (!h && !keys_eq(reinterpret_cast<const unsigned char *>(bc), sp, node, vs[i], vs[i - 1]))
    atomicOr(collision, 1u);
}

// first[pos of each run head] = 1
__global__ void k_first(const unsigned long long *__restrict__ head_scan, const uint64_t *__restrict__ ks,
                        const uint32_t *__restrict__ vs, int64_t n, uint32_t *__restrict__ run_first,
                        unsigned long long *__restrict__ first) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || ks[i] != ks[i - 1]) {
    run_first[head_scan[i]] = vs[i];
    first[vs[i]] = 1ull;
  }
}

// id of every position = rank of its run's first position among first positions
__global__ void k_assign(const unsigned long long *__restrict__ head_scan, const uint64_t *__restrict__ ks,
                         const uint32_t *__restrict__ vs, int64_t n, const uint32_t *__restrict__ run_first,
                         const unsigned long long *__restrict__ first_scan, bool node,
                         int64_t *__restrict__ src, int64_t *__restrict__ dst, int32_t *__restrict__ cur) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool h = i == 0 || ks[i] != ks[i - 1];
  const int64_t run = (int64_t)head_scan[i] - (h ? 0 : 1);
  const int64_t id = (int64_t)first_scan[run_first[run]];
  const uint32_t q = vs[i];
  if (node) (q & 1 ? dst : src)[q >> 1] = id;
  else cur[q] = (int32_t)id;
}

__global__ void k_iota(uint32_t *__restrict__ v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

// vocabulary spans in code order: code of run r = first_scan[run_first[r]]
__global__ void k_vocab(const uint32_t *__restrict__ run_first, int64_t runs,
                        const unsigned long long *__restrict__ first_scan, Spans sp,
                        int64_t *__restrict__ vspan) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= runs) return;
  const uint32_t e = run_first[r];
  const int64_t code = (int64_t)first_scan[e];
  vspan[2 * code] = sp.beg[5 * (size_t)e + 4];
  vspan[2 * code + 1] = sp.len[5 * (size_t)e + 4];
}

__global__ void k_gather_bytes(const char *__restrict__ bc, const int64_t *__restrict__ vspan,
                               const int64_t *__restrict__ off, int64_t n, char *__restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x;
  if (c >= n) return;
  for (int64_t i = threadIdx.x; i < vspan[2 * c + 1]; i += blockDim.x) out[off[c] + i] = bc[vspan[2 * c] + i];
}

// dense first-seen ids of n keys (hash, position) -> returns #distinct
int first_seen_ids(uint64_t *keys, int64_t n, bool node, const char *bc, Spans sp, int64_t *src,
                   int64_t *dst, int32_t *cur, DevBuf &scratch_v, DevBuf &scratch_k2, DevBuf &scratch_v2,
                   DevBuf &head, DevBuf &first, DevBuf &run_first, unsigned *flag, cudaStream_t s,
                   int64_t *n_distinct, DevBuf *vocab_span) {
  int rc;
  if ((rc = scratch_v.ensure(4 * (size_t)n)) || (rc = scratch_k2.ensure(8 * (size_t)n)) ||
      (rc = scratch_v2.ensure(4 * (size_t)n)) || (rc = head.ensure(8 * (size_t)(n + 1))) ||
      (rc = first.ensure(8 * (size_t)(n + 1))) || (rc = run_first.ensure(4 * (size_t)n)))
    return rc;
  k_iota<<<grid_for(n, 256), 256, 0, s>>>(scratch_v.as<uint32_t>(), n);
  TM_LAUNCHED("k_iota");
  uint64_t *ks;
  uint32_t *vs;
  if ((rc = radix_sort_pairs(keys, scratch_v.as<uint32_t>(), scratch_k2.as<uint64_t>(), scratch_v2.as<uint32_t>(),
                             n, 64, s, &ks, &vs)))
    return rc;
  unsigned long long *hd = head.as<unsigned long long>();
  TM_CUDA(cudaMemsetAsync(hd + n, 0, 8, s));
  k_heads<<<grid_for(n, 256), 256, 0, s>>>(ks, vs, n, bc, sp, node, hd, flag);
  TM_LAUNCHED("k_heads");
  if ((rc = scan_u64_exclusive(hd, n + 1, s))) return rc;
  unsigned long long runs = 0;
  TM_CUDA(cudaMemcpyAsync(&runs, hd + n, 8, cudaMemcpyDeviceToHost, s));
  unsigned long long *fs = first.as<unsigned long long>();
  TM_CUDA(cudaMemsetAsync(fs, 0, 8 * (size_t)(n + 1), s));
  k_first<<<grid_for(n, 256), 256, 0, s>>>(hd, ks, vs, n, run_first.as<uint32_t>(), fs);
  TM_LAUNCHED("k_first");
  if ((rc = scan_u64_exclusive(fs, n + 1, s))) return rc;
  k_assign<<<grid_for(n, 256), 256, 0, s>>>(hd, ks, vs, n, run_first.as<uint32_t>(), fs, node, src, dst, cur);
  TM_LAUNCHED("k_assign");
  TM_CUDA(cudaStreamSynchronize(s));
  *n_distinct = (int64_t)runs;
  if (vocab_span) {
    if ((rc = vocab_span->ensure(16 * (size_t)(runs > 0 ? runs : 1)))) return rc;
    k_vocab<<<grid_for((int64_t)runs, 256), 256, 0, s>>>(run_first.as<uint32_t>(), (int64_t)runs, fs, sp,
                                                        vocab_span->as<int64_t>());
    TM_LAUNCHED("k_vocab");
  }
  return TM_OK;
}

}  // namespace
}  // namespace tmb

using namespace tmb;

extern "C" int tm_ingest_csv(int device, const char *buf, int64_t len, int on_device, const tm_csv_mapping *m,
                             void *stream, tm_ingest **out, tm_ingest_info *info) {
  if (!out || !info || !m) return fail(TM_E_BAD_ARG, "NULL argument");
  *out = nullptr;
  *info = tm_ingest_info{};
  info->err_row = -1;
  if (len < 0 || (len > 0 && !buf)) return fail(TM_E_BAD_ARG, "bad buffer");
  if (m->n_fmt < 0 || m->n_fmt > TM_FMT_MAX) return fail(TM_E_BAD_ARG, "bad timestamp format program");
  if (m->tick_seconds < 1) return fail(TM_E_BAD_ARG, "tick_seconds must be >= 1");
  if (m->col_timestamp < 0 || m->col_src_account < 0 || m->col_dst_account < 0)
    return fail(TM_E_BAD_ARG, "timestamp and account columns are required");
  if (m->delimiter < 0 || m->delimiter > 127 || m->delimiter == '\n' || m->delimiter == '\r' ||
      m->delimiter == '"')
    return fail(TM_E_BAD_ARG, "delimiter must be one ASCII byte other than CR, LF and '\"'");
  int ndev = 0;
  TM_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(TM_E_BAD_ARG, "bad device ordinal");
  TM_CUDA(cudaSetDevice(device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  tm_ingest *h = new tm_ingest();
  h->device = device;
  h->stream = s;
  auto done = [&](int rc) {
    if (rc) delete h;
    else *out = h;
    return rc;
  };
  int rc;
  const char *bc = buf;
  DevBuf bytes;  // the input on the device (released when the call returns)
  if (!on_device && len > 0) {
    if ((rc = bytes.ensure((size_t)len + 16))) return done(rc);
    TM_CUDA(cudaMemcpyAsync(bytes.p, buf, (size_t)len, cudaMemcpyHostToDevice, s));
    bc = bytes.as<char>();
  }
  // 1. rows
  const int64_t tiles = (len + kTileBytes - 1) / kTileBytes;
  DevBuf counts, rend, flags;
  if ((rc = counts.ensure(8 * (size_t)(tiles + 1))) || (rc = flags.ensure(16))) return done(rc);
  TM_CUDA(cudaMemsetAsync(flags.p, 0, 16, s));
  unsigned *quote = flags.as<unsigned>(), *collision = flags.as<unsigned>() + 1;
  TM_CUDA(cudaMemsetAsync(counts.p, 0, 8 * (size_t)(tiles + 1), s));
  if (tiles > 0) {
    k_term_count<<<(unsigned)tiles, kTileThreads, 0, s>>>(bc, len, counts.as<unsigned long long>(), quote);
    TM_LAUNCHED("k_term_count");
  }
  if ((rc = scan_u64_exclusive(counts.as<unsigned long long>(), tiles + 1, s))) return done(rc);
  unsigned long long nterm = 0;
  unsigned hflags[2] = {0, 0};
  char last = 0;
  TM_CUDA(cudaMemcpyAsync(&nterm, counts.as<unsigned long long>() + tiles, 8, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaMemcpyAsync(hflags, flags.p, 8, cudaMemcpyDeviceToHost, s));
  if (len > 0) TM_CUDA(cudaMemcpyAsync(&last, bc + len - 1, 1, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  if (hflags[0]) {  // quoted fields: the csv quoting state machine is not implemented
    info->err_row = 0;
    info->err_status = TM_PARSE_UNSUPPORTED;
    info->err_begin = 0;
    info->err_end = 0;
    delete h;
    return TM_OK;
  }
  const bool tail = len > 0 && last != '\n' && last != '\r';
  const int64_t R = (int64_t)nterm + (tail ? 1 : 0);
  if (R >= (int64_t)UINT32_MAX / 2) return done(fail(TM_E_OVERFLOW, "too many rows"));
  if ((rc = rend.ensure(8 * (size_t)(R > 0 ? R : 1)))) return done(rc);
  if (tiles > 0) {
    k_term_write<<<(unsigned)tiles, kTileThreads, 0, s>>>(bc, len, counts.as<unsigned long long>(), rend.as<int64_t>());
    TM_LAUNCHED("k_term_write");
  }
  if (tail) TM_CUDA(cudaMemcpyAsync(rend.as<int64_t>() + nterm, &len, 8, cudaMemcpyHostToDevice, s));
  h->n_rows = R;
  info->n_rows = R;
  // 2. records: keep flags + scan
  DevBuf keep, eidx;
  if ((rc = keep.ensure(4 * (size_t)(R + 1))) || (rc = eidx.ensure(4 * (size_t)(R + 1)))) return done(rc);
  TM_CUDA(cudaMemsetAsync(keep.p, 0, 4 * (size_t)(R + 1), s));
  if (R > 0) {
    k_keep<<<grid_for(R, 256), 256, 0, s>>>(bc, len, rend.as<int64_t>(), R, (char)m->delimiter, keep.as<uint32_t>());
    TM_LAUNCHED("k_keep");
  }
  if ((rc = exclusive_scan_u32(keep.as<uint32_t>(), eidx.as<uint32_t>(), R + 1, s))) return done(rc);
  uint32_t E32 = 0;
  TM_CUDA(cudaMemcpyAsync(&E32, eidx.as<uint32_t>() + R, 4, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  const int64_t E = E32;
  h->n_edges = E;
  info->n_edges = E;
  // 3. fields
  const size_t Ea = (size_t)(E > 0 ? E : 1);
  DevBuf status, err, node_key, cur_key, sbeg, slen;
  if ((rc = status.ensure((size_t)(R > 0 ? R : 1))) || (rc = err.ensure(8)) || (rc = h->time.ensure(8 * Ea)) ||
      (rc = h->amount.ensure(8 * Ea)) || (rc = h->label.ensure(Ea)) || (rc = node_key.ensure(16 * Ea)) ||
      (rc = cur_key.ensure(8 * Ea)) || (rc = sbeg.ensure(8 * 5 * Ea)) || (rc = slen.ensure(4 * 5 * Ea)) ||
      (rc = h->src.ensure(8 * Ea)) || (rc = h->dst.ensure(8 * Ea)) || (rc = h->currency.ensure(4 * Ea)))
    return done(rc);
  TM_CUDA(cudaMemsetAsync(err.p, 0xff, 8, s));
  Spans sp{sbeg.as<int64_t>(), slen.as<int32_t>()};
  if (R > 0) {
    k_parse<<<grid_for(R, 128), 128, 0, s>>>(*m, bc, len, rend.as<int64_t>(), R, eidx.as<uint32_t>(),
                                             keep.as<uint32_t>(), status.as<int8_t>(),
                                             err.as<unsigned long long>(), h->time.as<int64_t>(),
                                             h->amount.as<double>(), h->label.as<int8_t>(),
                                             node_key.as<uint64_t>(), cur_key.as<uint64_t>(), sp);
    TM_LAUNCHED("k_parse");
  }
  unsigned long long erow = ~0ull;
  TM_CUDA(cudaMemcpyAsync(&erow, err.p, 8, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  if (erow != ~0ull) {
    int8_t st = 0;
    int64_t span[2] = {0, 0};
    TM_CUDA(cudaMemcpyAsync(&st, status.as<int8_t>() + erow, 1, cudaMemcpyDeviceToHost, s));
    if (erow > 0) TM_CUDA(cudaMemcpyAsync(&span[0], rend.as<int64_t>() + erow - 1, 8, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaMemcpyAsync(&span[1], rend.as<int64_t>() + erow, 8, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    info->err_row = (int64_t)erow;
    info->err_status = st;
    info->err_begin = erow > 0 ? span[0] + 1 : 0;
    info->err_end = span[1];
    delete h;
    return TM_OK;
  }
  // 4. first-seen ids: nodes over 2E keys, currencies over E keys
  DevBuf v1, k2, v2, head, first, run_first, vspan;
  if (E > 0) {
    if ((rc = first_seen_ids(node_key.as<uint64_t>(), 2 * E, true, bc, sp, h->src.as<int64_t>(),
                             h->dst.as<int64_t>(), nullptr, v1, k2, v2, head, first, run_first, collision, s,
                             &h->n_nodes, nullptr)))
      return done(rc);
    if ((rc = first_seen_ids(cur_key.as<uint64_t>(), E, false, bc, sp, nullptr, nullptr,
                             h->currency.as<int32_t>(), v1, k2, v2, head, first, run_first, collision, s,
                             &h->n_cur, &vspan)))
      return done(rc);
    // vocabulary strings, gathered while the input is still on the device
    const int64_t nc = h->n_cur;
    std::vector<int64_t> span(2 * (size_t)nc), off((size_t)nc + 1, 0);
    TM_CUDA(cudaMemcpyAsync(span.data(), vspan.p, 16 * (size_t)nc, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    for (int64_t c = 0; c < nc; ++c) off[c + 1] = off[c] + span[2 * c + 1];
    if ((rc = h->vocab_off.ensure(8 * (size_t)(nc + 1))) || (rc = h->vocab_bytes.ensure((size_t)off[nc] + 1)))
      return done(rc);
    TM_CUDA(cudaMemcpyAsync(h->vocab_off.p, off.data(), 8 * (size_t)(nc + 1), cudaMemcpyHostToDevice, s));
    if (off[nc] > 0) {
      k_gather_bytes<<<(unsigned)nc, 64, 0, s>>>(bc, vspan.as<int64_t>(), h->vocab_off.as<int64_t>(), nc,
                                                 h->vocab_bytes.as<char>());
      TM_LAUNCHED("k_gather_bytes");
    }
  }
  TM_CUDA(cudaMemcpyAsync(hflags, flags.p, 8, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  if (hflags[1]) {
    info->err_row = 0;
    info->err_status = TM_PARSE_COLLISION;
    delete h;
    return TM_OK;
  }
  info->n_nodes = h->n_nodes;
  info->n_currency = h->n_cur;
  *out = h;
  return TM_OK;
}

extern "C" int tm_ingest_fetch(tm_ingest *h, int64_t *src, int64_t *dst, int64_t *time, double *amount,
                               int32_t *currency, int8_t *label) {
  if (!h) return fail(TM_E_BAD_ARG, "NULL handle");
  TM_CUDA(cudaSetDevice(h->device));
  const size_t E = (size_t)h->n_edges;
  if (E == 0) return TM_OK;
  cudaStream_t s = h->stream;
  if (src) TM_CUDA(cudaMemcpyAsync(src, h->src.p, 8 * E, cudaMemcpyDeviceToHost, s));
  if (dst) TM_CUDA(cudaMemcpyAsync(dst, h->dst.p, 8 * E, cudaMemcpyDeviceToHost, s));
  if (time) TM_CUDA(cudaMemcpyAsync(time, h->time.p, 8 * E, cudaMemcpyDeviceToHost, s));
  if (amount) TM_CUDA(cudaMemcpyAsync(amount, h->amount.p, 8 * E, cudaMemcpyDeviceToHost, s));
  if (currency) TM_CUDA(cudaMemcpyAsync(currency, h->currency.p, 4 * E, cudaMemcpyDeviceToHost, s));
  if (label) TM_CUDA(cudaMemcpyAsync(label, h->label.p, E, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  return TM_OK;
}

extern "C" int tm_ingest_vocab(tm_ingest *h, int64_t *offsets, char *bytes, int64_t cap) {
  if (!h || !offsets) return fail(TM_E_BAD_ARG, "NULL argument");
  TM_CUDA(cudaSetDevice(h->device));
  const int64_t n = h->n_cur;
  cudaStream_t s = h->stream;
  offsets[0] = 0;
  if (n > 0) TM_CUDA(cudaMemcpyAsync(offsets, h->vocab_off.p, 8 * (size_t)(n + 1), cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  const int64_t total = offsets[n];
  if (!bytes || total == 0) return TM_OK;
  if (cap < total) return fail(TM_E_BAD_ARG, "vocab byte buffer too small");
  TM_CUDA(cudaMemcpyAsync(bytes, h->vocab_bytes.p, (size_t)total, cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  return TM_OK;
}

extern "C" int tm_ingest_graph(tm_ingest *h, tm_graph **out) {
  if (!h || !out) return fail(TM_E_BAD_ARG, "NULL argument");
  return tm_graph_build(h->device, h->n_nodes, h->n_edges, h->src.as<int64_t>(), h->dst.as<int64_t>(),
                        h->time.as<int64_t>(), 1, h->stream, out);
}

extern "C" void tm_ingest_free(tm_ingest *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  delete h;
}
