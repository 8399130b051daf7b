// DOT ingestion on the device: parse_dot (graphio.py:79-199) over the UTF-8
// bytes of the text, one thread per line.
//
//  1. line boundaries: str.splitlines' terminators (\n, \r, \r\n, \v, \f,
//     \x1c-\x1e, U+0085, U+2028, U+2029) flagged per byte and compacted;
//  2. per line: the '//' cut, str.strip (Unicode whitespace), '#' lines, the
//     digraph header (graphio.py:98-107) on the first content line, the
//     closing brace (graphio.py:109-114);
//  3. per line, twice (count, then write at scanned offsets): the statement
//     split (_split_statements, graphio.py:202-217), the edge / node statement
//     grammar (_EDGE_STMT / _NODE_STMT, graphio.py:67-70) and the attribute
//     list (_ATTR_RE, graphio.py:47-62), restated as deterministic scanners
//     (every regex there has a unique match);
//     the first failing line carries the reference's error;
//  4. names: canonical bytes (unquoted, \" -> ") hashed into an open-address
//     table, first occurrence by atomicMin, equality verified byte by byte;
//     appearance rank by a scan of the first-occurrence flags;
//  5. ids (graphio.py:145-158): n<digits> / <digits> names keep their number
//     (first appearance wins), the rest count up from max + 1;
//  6. attributes (graphio.py:160-183): last value per known key, Python
//     float() on the device (Eisel-Lemire with the published 128-bit powers of
//     five, exact for <= 19 significant digits; a longer literal whose two
//     bounds disagree is decided by a big-integer comparison with the
//     midpoint), int(float()) for size/bytes (values beyond int64 — Python
//     ints — are listed for the host).
//
// The caller gets counts and the first error from hs_dot_parse, then copies
// the per-name / per-edge / per-attribute arrays with hs_dot_fetch, or builds
// the device CSR of the parsed graph with hs_dot_csr.
#include "common.cuh"
#include "pow5_table.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <climits>
#include <cstring>
#include <vector>

namespace {

typedef uint8_t u8;

// ------------------------------------------------------------ characters ---
__host__ __device__ inline bool ascii_ws(u8 c) {
  return c == 0x20 || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

// bytes of the whitespace character (str.isspace) starting at p, 0 if none
__host__ __device__ inline int ws_at(const u8 *s, int p, int e) {
  const u8 c = s[p];
  if (c < 0x80) return ascii_ws(c) ? 1 : 0;
  if (c == 0xC2) return (p + 1 < e && (s[p + 1] == 0x85 || s[p + 1] == 0xA0)) ? 2 : 0;
  if (p + 2 >= e) return 0;
  const u8 c1 = s[p + 1], c2 = s[p + 2];
  if (c == 0xE1) return (c1 == 0x9A && c2 == 0x80) ? 3 : 0;                // U+1680
  if (c == 0xE2) {
    if (c1 == 0x80)  // U+2000-200A, U+2028, U+2029, U+202F
      return ((c2 >= 0x80 && c2 <= 0x8A) || c2 == 0xA8 || c2 == 0xA9 || c2 == 0xAF) ? 3 : 0;
    return (c1 == 0x81 && c2 == 0x9F) ? 3 : 0;                             // U+205F
  }
  if (c == 0xE3) return (c1 == 0x80 && c2 == 0x80) ? 3 : 0;                // U+3000
  return 0;
}

// bytes of the whitespace character ending at p - 1 (p > b), 0 if none
__host__ __device__ inline int ws_before(const u8 *s, int b, int p) {
  const u8 c = s[p - 1];
  if (c < 0x80) return ascii_ws(c) ? 1 : 0;
  if (p - 2 >= b && s[p - 2] == 0xC2) return (c == 0x85 || c == 0xA0) ? 2 : 0;
  if (p - 3 >= b && ws_at(s, p - 3, p) == 3) return 3;
  return 0;
}

__host__ __device__ inline int skip_ws(const u8 *s, int p, int e) {
  int k;
  while (p < e && (k = ws_at(s, p, e)) > 0) p += k;
  return p;
}

__host__ __device__ inline int rskip_ws(const u8 *s, int b, int e) {
  int k;
  while (e > b && (k = ws_before(s, b, e)) > 0) e -= k;
  return e;
}

__host__ __device__ inline bool is_digit(u8 c) { return c >= '0' && c <= '9'; }
__host__ __device__ inline bool id_start(u8 c) {
  return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_';
}
__host__ __device__ inline bool id_char(u8 c) { return id_start(c) || is_digit(c); }
__host__ __device__ inline bool name_char(u8 c) { return id_char(c) || c == '.'; }

// bytes of the last character of [b, e) (UTF-8 continuation bytes skipped)
__host__ __device__ inline int last_char_len(const u8 *s, int b, int e) {
  int p = e - 1;
  while (p > b && (s[p] & 0xC0) == 0x80) --p;
  return e - p;
}

// Canonical bytes of a token or attribute value: a leading '"' drops the
// first and the last character and turns \" into " (graphio.py:57-58, 73-76).
struct Canon {
  const u8 *s;
  int p, e;
  __host__ __device__ Canon(const u8 *s_, int b, int e_) : s(s_), p(b), e(e_) {
    if (e > b && s[b] == '"') {
      e = e - b == 1 ? b + 1 : e - last_char_len(s, b, e);
      p = b + 1;
      quoted = true;
    }
  }
  bool quoted = false;
  __host__ __device__ int next() {  // -1 at the end
    if (p >= e) return -1;
    if (quoted && s[p] == '\\' && p + 1 < e && s[p + 1] == '"') {
      p += 2;
      return '"';
    }
    return s[p++];
  }
};

__device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ uint64_t canon_hash(const u8 *s, int b, int e) {
  Canon c(s, b, e);
  uint64_t h = 0xcbf29ce484222325ull;
  int64_t n = 0;
  for (int x; (x = c.next()) >= 0; ++n) h = (h ^ (uint64_t)x) * 0x100000001b3ull;
  h = mix64(h ^ ((uint64_t)n << 56));
  return h ? h : 1;  // 0 marks an empty table slot
}

__device__ bool canon_eq(const u8 *s, int b1, int e1, int b2, int e2) {
  Canon a(s, b1, e1), b(s, b2, e2);
  for (;;) {
    const int x = a.next(), y = b.next();
    if (x != y) return false;
    if (x < 0) return true;
  }
}

__device__ bool canon_is(const u8 *s, int b, int e, const char *lit) {
  Canon c(s, b, e);
  for (int i = 0;; ++i) {
    const int x = c.next();
    if (lit[i] == 0) return x < 0;
    if (x != (u8)lit[i]) return false;
  }
}

__host__ __device__ inline bool span_is(const u8 *s, int b, int e, const char *lit) {
  int i = 0;
  for (; lit[i]; ++i)
    if (b + i >= e || s[b + i] != (u8)lit[i]) return false;
  return b + i == e;
}

// ---------------------------------------------------- Python float() ------
// Eisel-Lemire (fast_float's compute_float for binary64; exact whenever the
// decimal significand fits 19 digits, Mushtak & Lemire 2023).
#ifdef __CUDA_ARCH__
#define HS_POW5 kPow5Dev
#else
#define HS_POW5 kPow5Host
#endif
__device__ const uint64_t kPow5Dev[] = {HS_POW5_TABLE};
const uint64_t kPow5Host[] = {HS_POW5_TABLE};

__host__ __device__ inline void mul128(uint64_t a, uint64_t b, uint64_t &hi, uint64_t &lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 r = (unsigned __int128)a * b;
  lo = (uint64_t)r;
  hi = (uint64_t)(r >> 64);
#endif
}

__host__ __device__ inline int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

// (mantissa with the implicit bit cleared) | (biased exponent << 52)
__host__ __device__ uint64_t eisel_lemire(int64_t q, uint64_t w) {
  if (w == 0 || q < HS_POW5_MIN_Q) return 0;
  if (q > HS_POW5_MAX_Q) return 0x7FFull << 52;
  const int lz = clz64(w);
  w <<= lz;
  const int idx = 2 * (int)(q - HS_POW5_MIN_Q);
  uint64_t hi, lo;
  mul128(w, HS_POW5[idx], hi, lo);
  if ((hi & 0x1FFull) == 0x1FFull) {  // 55 bits of precision wanted
    uint64_t hi2, lo2;
    mul128(w, HS_POW5[idx + 1], hi2, lo2);
    lo += hi2;
    if (hi2 > lo) ++hi;
  }
  const int upper = (int)(hi >> 63);
  const int shift = upper + 64 - 52 - 3;
  uint64_t m = hi >> shift;
  int32_t p2 = (int32_t)((((152170 + 65536) * (int32_t)q) >> 16) + 63) + upper - lz + 1023;
  if (p2 <= 0) {  // subnormal
    if (-p2 + 1 >= 64) return 0;
    m >>= -p2 + 1;
    m += m & 1;
    m >>= 1;
    p2 = m < (1ull << 52) ? 0 : 1;
    return (m & ~(1ull << 52)) | ((uint64_t)p2 << 52);
  }
  if (lo <= 1 && q >= -4 && q <= 23 && (m & 3) == 1 && (m << shift) == hi) m &= ~1ull;
  m += m & 1;
  m >>= 1;
  if (m >= (2ull << 52)) {
    m = 1ull << 52;
    ++p2;
  }
  m &= ~(1ull << 52);
  if (p2 >= 0x7FF) return 0x7FFull << 52;
  return m | ((uint64_t)p2 << 52);
}

__host__ __device__ inline double bits_double(uint64_t b) {
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
}

__host__ __device__ inline u8 lower(u8 c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

__host__ __device__ inline bool ieq(const u8 *s, int b, int e, const char *lit) {
  int i = 0;
  for (; lit[i]; ++i)
    if (b + i >= e || lower(s[b + i]) != (u8)lit[i]) return false;
  return b + i == e;
}

// Exact decision for a literal whose 19-digit bounds round differently: the
// full significand (up to kMaxDigits digits, a nonzero tail kept as a sticky
// bit) against the halfway point between the two candidates, in big integers
// (the "digit comparison" fallback of the Eisel-Lemire literature).
constexpr int kLimbs = 100;       // 3200 bits
constexpr int kMaxDigits = 800;   // > 767, the most a binary64 midpoint needs

struct Big {
  uint32_t v[kLimbs];
  int n;  // used limbs
  __host__ __device__ void set(uint64_t x) {
    n = 0;
    while (x) {
      v[n++] = (uint32_t)x;
      x >>= 32;
    }
  }
  __host__ __device__ void mul_add(uint32_t m, uint32_t a) {
    uint64_t c = a;
    for (int i = 0; i < n; ++i) {
      const uint64_t t = (uint64_t)v[i] * m + c;
      v[i] = (uint32_t)t;
      c = t >> 32;
    }
    if (c && n < kLimbs) v[n++] = (uint32_t)c;
  }
  __host__ __device__ void mul_pow5(int k) {
    while (k >= 13) {
      mul_add(1220703125u, 0);  // 5^13
      k -= 13;
    }
    uint32_t m = 1;
    while (k-- > 0) m *= 5;
    if (m > 1) mul_add(m, 0);
  }
  __host__ __device__ void shl(int bits) {
    if (n == 0 || bits <= 0) return;
    const int w = bits / 32, b = bits % 32;
    int nn = n + w + 1;
    if (nn > kLimbs) nn = kLimbs;
    for (int i = nn - 1; i >= 0; --i) {
      const int s0 = i - w;
      uint32_t hi = s0 >= 0 && s0 < n ? v[s0] : 0;
      uint32_t lo = s0 - 1 >= 0 && s0 - 1 < n ? v[s0 - 1] : 0;
      v[i] = b ? (hi << b) | (lo >> (32 - b)) : hi;
    }
    n = nn;
    while (n > 0 && v[n - 1] == 0) --n;
  }
};

__host__ __device__ int big_cmp(const Big &a, const Big &b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.v[i] != b.v[i]) return a.v[i] < b.v[i] ? -1 : 1;
  return 0;
}

// bits of the correctly rounded binary64 of the decimal literal [b, e)
// (already validated: digits, '.', '_', exponent), given the lower candidate
__host__ __device__ uint64_t round_exact(const u8 *s, int b, int e, uint64_t lo_bits) {
  Big D, H;
  D.n = 0;
  int nd = 0;
  bool sticky = false;
  int64_t e10 = 0, ex = 0;
  bool frac = false, exp = false, eneg = false;
  for (int p = b; p < e; ++p) {
    const u8 c = s[p];
    if (c == '_') continue;
    if (exp) {
      if (c == '-') eneg = true;
      else if (c >= '0' && c <= '9' && ex < 100000000000ll) ex = ex * 10 + (c - '0');
      continue;
    }
    if (c == '.') {
      frac = true;
      continue;
    }
    if (c == 'e' || c == 'E') {
      exp = true;
      continue;
    }
    if (c < '0' || c > '9') continue;  // sign
    const int d = c - '0';
    if (nd == 0 && d == 0) {
      if (frac) --e10;
      continue;
    }
    if (nd < kMaxDigits) {
      D.mul_add(10, d);
      ++nd;
      if (frac) --e10;
    } else {
      sticky |= d != 0;
      if (!frac) ++e10;
    }
  }
  int64_t E = e10 + (eneg ? -ex : ex);
  // halfway point above the lower candidate: (2 m1 + 1) 2^(e1 - 1)
  const uint64_t f = lo_bits & ((1ull << 52) - 1);
  const int be = (int)(lo_bits >> 52);
  const uint64_t m1 = be ? (f | (1ull << 52)) : f;
  const int e1 = be ? be - 1075 : -1074;
  H.set(2 * m1 + 1);
  // D 10^E  vs  H 2^(e1 - 1)
  if (E >= 0) {
    D.mul_pow5((int)E);
    const int64_t k = E - (e1 - 1);
    if (k >= 0) D.shl((int)k);
    else H.shl((int)-k);
  } else {
    H.mul_pow5((int)-E);
    const int64_t t = (int64_t)e1 - 1 - E;
    if (t >= 0) H.shl((int)t);
    else D.shl((int)-t);
  }
  int c = big_cmp(D, H);
  if (c == 0 && sticky) c = 1;
  if (c > 0 || (c == 0 && (m1 & 1))) return lo_bits + 1;
  return lo_bits;
}

enum : int { kFloatOk = 0, kFloatBad = 1, kFloatSlow = 2 };

// Python float(str) on the canonical bytes of [b, e): surrounding Unicode
// whitespace, sign, inf/infinity/nan (any case), decimal digits with single
// underscores between digits, optional fraction and exponent.
__host__ __device__ int py_float(const u8 *raw, int rb, int re, double *out) {
  // canonicalise into a bounded window: a quoted value may hold \" pairs,
  // which never form a number anyway
  bool quoted = re > rb && raw[rb] == '"';
  int b = rb, e = re;
  if (quoted) {
    e = e - b == 1 ? b + 1 : e - last_char_len(raw, b, e);
    b = b + 1;
    for (int i = b; i < e; ++i)
      if (raw[i] == '\\' || raw[i] == '"') return kFloatBad;
  }
  const u8 *s = raw;
  b = skip_ws(s, b, e);
  e = rskip_ws(s, b, e);
  if (b >= e) return kFloatBad;
  bool neg = false;
  if (s[b] == '+' || s[b] == '-') neg = s[b++] == '-';
  double v;
  if (ieq(s, b, e, "inf") || ieq(s, b, e, "infinity")) {
    v = bits_double(0x7FF0000000000000ull);
  } else if (ieq(s, b, e, "nan")) {
    v = bits_double(0x7FF8000000000000ull);
  } else {
    uint64_t w = 0;
    int nd = 0;
    int64_t e10 = 0;
    bool trunc = false, any = false;
    int p = b;
    auto under_ok = [&](int i) { return i > b && is_digit(s[i - 1]) && i + 1 < e && is_digit(s[i + 1]); };
    for (; p < e; ++p) {  // integer part
      const u8 c = s[p];
      if (c == '_' && under_ok(p)) continue;
      if (!is_digit(c)) break;
      any = true;
      const int d = c - '0';
      if (nd == 0 && d == 0) continue;
      if (nd < 19) {
        w = w * 10 + d;
        ++nd;
      } else {
        ++e10;
        trunc |= d != 0;
      }
    }
    if (p < e && s[p] == '.') {
      ++p;
      for (; p < e; ++p) {
        const u8 c = s[p];
        if (c == '_' && under_ok(p)) continue;
        if (!is_digit(c)) break;
        any = true;
        const int d = c - '0';
        if (nd == 0 && d == 0) {
          --e10;
        } else if (nd < 19) {
          w = w * 10 + d;
          ++nd;
          --e10;
        } else {
          trunc |= d != 0;
        }
      }
    }
    if (!any) return kFloatBad;
    if (p < e && (s[p] == 'e' || s[p] == 'E')) {
      ++p;
      bool eneg = false;
      if (p < e && (s[p] == '+' || s[p] == '-')) eneg = s[p++] == '-';
      const int d0 = p;
      int64_t x = 0;
      for (; p < e; ++p) {
        const u8 c = s[p];
        if (c == '_' && p > d0 && under_ok(p)) continue;
        if (!is_digit(c)) break;
        if (x < 100000000000ll) x = x * 10 + (c - '0');
      }
      if (p == d0) return kFloatBad;
      e10 += eneg ? -x : x;
    }
    if (p != e) return kFloatBad;
    uint64_t bits = 0;
    if (w != 0) {
      const int64_t q = e10 < -100000 ? -100000 : (e10 > 100000 ? 100000 : e10);
      bits = eisel_lemire(q, w);
      if (trunc && eisel_lemire(q, w + 1) != bits) {
        if (e10 < -100000 || e10 > 100000) return kFloatSlow;  // absurd exponents
        bits = round_exact(s, b, e, bits);
      }
    }
    v = bits_double(bits);
  }
  *out = neg ? -v : v;
  return kFloatOk;
}


// ------------------------------------------------------------ grammar -----
// A token: "..." (first unescaped quote closes; \<char> pairs skipped) or a
// run of [A-Za-z0-9_.]; returns the end, or -1.
__device__ int token_end(const u8 *s, int p, int e) {
  if (p >= e) return -1;
  if (s[p] == '"') {
    for (int q = p + 1; q < e;) {
      if (s[q] == '\\') {
        if (q + 1 >= e) return -1;
        q += 2;
      } else if (s[q] == '"') {
        return q + 1;
      } else {
        ++q;
      }
    }
    return -1;
  }
  int q = p;
  while (q < e && name_char(s[q])) ++q;
  return q > p ? q : -1;
}

// Start of the shortest suffix matching \s*;?\s*$ (every later start matches too).
__device__ int tail_start(const u8 *s, int b, int e) {
  int r = rskip_ws(s, b, e);
  if (r > b && s[r - 1] == ';') r = rskip_ws(s, b, r - 1);
  return r;
}

// (?:\[(.*)\])?\s*;?\s*$ after a token ending at p: attribute text [ab, ae)
// (ab = ae = 0 when absent); false when the statement does not match.
__device__ bool attrs_span(const u8 *s, int p, int e, int T, int *ab, int *ae) {
  const int q = skip_ws(s, p, e);
  *ab = *ae = 0;
  if (q >= T) return true;
  if (s[q] != '[') return false;
  int j = e - 1;
  while (j > q && s[j] != ']') --j;
  if (j <= q || j + 1 < T) return false;
  *ab = q + 1;
  *ae = j;
  return true;
}

enum : int {
  kErrNone = 0,
  kErrHeader = 1,     // expected a digraph header, got {line!r}
  kErrUndirected = 2, // undirected graphs are not supported
  kErrStmt = 3,       // cannot parse statement {stmt!r}
  kErrAttr = 4,       // bad attribute syntax near {text[pos:pos+20]!r}
  kErrNoGraph = 5,    // no digraph found
  kErrBrace = 6,      // missing closing brace
};

// key classes (graphio.py:12-14)
enum : u8 { kKind = 0, kSize = 1, kWcpu = 2, kWgpu = 3, kBytes = 4, kWxfer = 5, kStyle = 6, kOther = 7 };

__device__ u8 key_class(const u8 *s, int b, int e) {
  if (span_is(s, b, e, "kind")) return kKind;
  if (span_is(s, b, e, "size")) return kSize;
  if (span_is(s, b, e, "weight_cpu")) return kWcpu;
  if (span_is(s, b, e, "weight_gpu")) return kWgpu;
  if (span_is(s, b, e, "bytes")) return kBytes;
  if (span_is(s, b, e, "weight_xfer")) return kWxfer;
  if (span_is(s, b, e, "part") || span_is(s, b, e, "color") || span_is(s, b, e, "style") ||
      span_is(s, b, e, "fillcolor") || span_is(s, b, e, "device") || span_is(s, b, e, "start") ||
      span_is(s, b, e, "end"))
    return kStyle;
  return kOther;
}

// Attribute list (_parse_attrs): calls f(k0, k1, v0, v1) per pair; returns the
// failing position (>= 0) or -1.
template <class F>
__device__ int parse_attrs(const u8 *s, int ab, int ae, F f) {
  int pos = ab;
  while (pos < ae) {
    int q = skip_ws(s, pos, ae);
    int end = -1, k0 = 0, k1 = 0, v0 = 0, v1 = 0;
    if (q < ae && id_start(s[q])) {
      k0 = q++;
      while (q < ae && id_char(s[q])) ++q;
      k1 = q;
      q = skip_ws(s, q, ae);
      if (q < ae && s[q] == '=') {
        q = skip_ws(s, q + 1, ae);
        v0 = q;
        auto close = [&](int r) -> int {  // \s*(?:,|$) after a value ending at r
          r = skip_ws(s, r, ae);
          if (r == ae) return r;
          return s[r] == ',' ? r + 1 : -1;
        };
        if (q < ae && s[q] == '"') {
          const int qe = token_end(s, q, ae);
          if (qe > 0 && (end = close(qe)) >= 0) v1 = qe;
        }
        if (end < 0) {  // [^,\]\s]+
          int r = q;
          while (r < ae && s[r] != ',' && s[r] != ']' && !ws_at(s, r, ae)) ++r;
          if (r > q && (end = close(r)) >= 0) v1 = r;
        }
      }
    }
    if (end < 0) return skip_ws(s, pos, ae) < ae ? pos : -1;
    f(k0, k1, v0, v1);
    pos = end;
  }
  return -1;
}

struct LineErr {
  int kind = kErrNone, a = 0, b = 0, c = 0;
};

// Statements of one body line [b, e): edge / node declarations handed to the
// sink; returns false (with err set) at the first failing statement.
template <class Sink>
__device__ bool line_statements(const u8 *s, int b, int e, Sink &sink, LineErr &err) {
  int depth = 0, a = b;
  bool quoted = false;
  for (int p = b; p <= e; ++p) {
    bool cut = p == e;
    if (!cut) {
      const u8 c = s[p];
      if (c == '"') quoted = !quoted;
      else if (!quoted && c == '[') ++depth;
      else if (!quoted && c == ']') --depth;
      cut = c == ';' && depth == 0 && !quoted;
    }
    if (!cut) continue;
    const int sb = skip_ws(s, a, p), se = rskip_ws(s, sb, p);
    a = p + 1;
    if (sb >= se) continue;
    const int T = tail_start(s, sb, se);
    const int t1 = token_end(s, sb, se);
    int ab, ae;
    bool done = false;
    if (t1 > 0) {
      const int q = skip_ws(s, t1, se);
      if (q + 1 < se && s[q] == '-' && s[q + 1] == '>') {
        const int d0 = skip_ws(s, q + 2, se), d1 = token_end(s, d0, se);
        if (d1 > 0 && attrs_span(s, d1, se, T, &ab, &ae)) {
          const int bad = sink.edge(sb, t1, d0, d1, ab, ae);
          if (bad >= 0) {
            err = {kErrAttr, ab, ae, bad};
            return false;
          }
          done = true;
        }
      }
      if (!done && attrs_span(s, t1, se, T, &ab, &ae)) {
        if (!canon_is(s, sb, t1, "node") && !canon_is(s, sb, t1, "edge") &&
            !canon_is(s, sb, t1, "graph")) {
          const int bad = sink.node(sb, t1, ab, ae);
          if (bad >= 0) {
            err = {kErrAttr, ab, ae, bad};
            return false;
          }
        }
        done = true;
      }
    }
    if (!done) {
      err = {kErrStmt, sb, se, 0};
      return false;
    }
  }
  return true;
}

struct CountSink {
  const u8 *s;
  int occ = 0, edges = 0, nodes = 0, attrs = 0;
  __device__ int edge(int, int, int, int, int ab, int ae) {
    occ += 2;
    ++edges;
    return parse_attrs(s, ab, ae, [&](int, int, int, int) { ++attrs; });
  }
  __device__ int node(int, int, int ab, int ae) {
    occ += 1;
    ++nodes;
    return parse_attrs(s, ab, ae, [&](int, int, int, int) { ++attrs; });
  }
};

struct Out {  // parse records, laid out by the count pass's scans
  int32_t *occ_b, *occ_e;                 // name occurrences, appearance order
  int32_t *edge_occ, *edge_ab, *edge_an;  // edge declarations (src occ; dst = +1)
  int32_t *node_occ, *node_ab, *node_an;  // node statements
  int32_t *attr_k0, *attr_k1, *attr_v0, *attr_v1;
  u8 *attr_cls;
};

struct FillSink {
  const u8 *s;
  Out o;
  int occ, edges, nodes, attrs;
  __device__ void put_attr(int k0, int k1, int v0, int v1) {
    o.attr_k0[attrs] = k0;
    o.attr_k1[attrs] = k1;
    o.attr_v0[attrs] = v0;
    o.attr_v1[attrs] = v1;
    o.attr_cls[attrs] = key_class(s, k0, k1);
    ++attrs;
  }
  __device__ int edge(int s0, int s1, int d0, int d1, int ab, int ae) {
    o.occ_b[occ] = s0;
    o.occ_e[occ] = s1;
    o.occ_b[occ + 1] = d0;
    o.occ_e[occ + 1] = d1;
    o.edge_occ[edges] = occ;
    o.edge_ab[edges] = attrs;
    parse_attrs(s, ab, ae, [&](int k0, int k1, int v0, int v1) { put_attr(k0, k1, v0, v1); });
    o.edge_an[edges] = attrs - o.edge_ab[edges];
    occ += 2;
    ++edges;
    return -1;
  }
  __device__ int node(int n0, int n1, int ab, int ae) {
    o.occ_b[occ] = n0;
    o.occ_e[occ] = n1;
    o.node_occ[nodes] = occ;
    o.node_ab[nodes] = attrs;
    parse_attrs(s, ab, ae, [&](int k0, int k1, int v0, int v1) { put_attr(k0, k1, v0, v1); });
    o.node_an[nodes] = attrs - o.node_ab[nodes];
    ++occ;
    ++nodes;
    return -1;
  }
};

// global scalars of one parse (device)
enum : int {
  G_H = 0,        // first content line (the header), INT_MAX if none
  G_C = 1,        // closing line, INT_MAX if none
  G_E = 2,        // first line with an error, INT_MAX if none
  G_NL = 3,       // '\n' count
  G_FATAL = 4,    // header error
  G_HNAME_B = 5,  // graph name group [b, e) (b < 0: none)
  G_HNAME_E = 6,
  G_ERRK = 7, G_ERRA = 8, G_ERRB = 9, G_ERRC = 10,  // header error record
  G_U = 11,        // unique names
  G_COLLIDE = 12,  // a hash collision was seen (the parse is refused)
  G_ROOT = 13,     // first name (rank) whose kind is SOURCE, INT_MAX if none
  G_BIGID = 14,    // a numeric name beyond 2^62
  G_NSLOW = 15,    // literals left to the host
  G_ZERO = 16,     // some name holds id 0
  G_COUNT = 17,
};

// ------------------------------------------------------------ kernels -----
// line terminators of str.splitlines: length of the terminator starting at
// byte i (0: none); \r\n is one terminator
__device__ __forceinline__ int term_at(const u8 *s, int L, int i, u8 c) {
  if (c == '\n') return (i > 0 && s[i - 1] == '\r') ? 0 : 1;
  if (c == '\r') return (i + 1 < L && s[i + 1] == '\n') ? 2 : 1;
  if (c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) return 1;
  if (c == 0xC2) return (i + 1 < L && s[i + 1] == 0x85) ? 2 : 0;
  if (c == 0xE2) return (i + 2 < L && s[i + 1] == 0x80 && (s[i + 2] == 0xA8 || s[i + 2] == 0xA9)) ? 3 : 0;
  return 0;
}

constexpr int kChunk = 16;  // bytes per thread (one 16-byte load)

// pass 1: terminators per 16-byte chunk (and the '\n' count); pass 2 writes
// their positions at the scanned offsets
template <bool kWrite>
__global__ void __launch_bounds__(256) terms(const u8 *s, int L, int32_t *cnt, const int32_t *off,
                                             int32_t *term, int32_t *g) {
  const int64_t nch = ((int64_t)L + kChunk - 1) / kChunk;
  int nl = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nch;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i0 = (int)(t * kChunk);
    uint32_t x[4];
    if (i0 + kChunk <= L) {
      const uint4 v = __ldg((const uint4 *)(s + i0));
      x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = 0;
#pragma unroll
      for (int q = 0; q < kChunk; ++q)
        if (i0 + q < L) x[q >> 2] |= (uint32_t)s[i0 + q] << (8 * (q & 3));
    }
    // candidate bytes (<= 0x1e, or a U+0085 / U+2028/9 lead byte) as a 16-bit
    // mask: the loop below runs once per candidate, not once per byte
    uint32_t mask = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t hit = __vcmpleu4(x[q], 0x1e1e1e1eu) | __vcmpeq4(x[q], 0xC2C2C2C2u) |
                           __vcmpeq4(x[q], 0xE2E2E2E2u);
      const uint32_t y = (hit >> 7) & 0x01010101u;
      mask |= (((y * 0x01020408u) >> 24) & 0xFu) << (4 * q);
    }
    if (L - i0 < kChunk) mask &= (1u << (L - i0)) - 1;
    int c = 0, w = kWrite ? off[t] : 0;
    while (mask) {
      const int q = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint32_t word = q < 4 ? x[0] : (q < 8 ? x[1] : (q < 12 ? x[2] : x[3]));
      const u8 ch = (u8)(word >> (8 * (q & 3)));
      nl += ch == '\n';
      if (term_at(s, L, i0 + q, ch)) {
        if (kWrite) term[w++] = i0 + q;
        ++c;
      }
    }
    if (!kWrite) cnt[t] = c;
  }
  if (!kWrite) {
    for (int o = 16; o; o >>= 1) nl += __shfl_down_sync(0xffffffffu, nl, o);
    if ((threadIdx.x & 31) == 0 && nl) atomicAdd(g + G_NL, nl);
  }
}

// terminator length at a recorded position
__device__ __forceinline__ int term_len(const u8 *s, int L, int i) { return term_at(s, L, i, s[i]); }

// per line: '//' cut + strip -> [lb, le); content lines (non-empty, not '#')
__global__ void line_spans(const u8 *s, int L, const int32_t *term, int nterm, int nlines,
                           int32_t *lb, int32_t *le, u8 *kind, int32_t *g) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nlines; k += gridDim.x * blockDim.x) {
    const int b = k == 0 ? 0 : term[k - 1] + term_len(s, L, term[k - 1]);
    int e = k < nterm ? term[k] : L;
    // first "//": 16-byte aligned windows, byte scan only where a '/' shows up
    // (the text is 16-byte aligned, so a window never crosses its end)
    for (int w0 = b & ~15; w0 < e - 1; w0 += 16) {
      const uint4 v = w0 + 16 <= L ? __ldg((const uint4 *)(s + w0)) : make_uint4(~0u, ~0u, ~0u, ~0u);
      const uint32_t hit = __vcmpeq4(v.x, 0x2f2f2f2fu) | __vcmpeq4(v.y, 0x2f2f2f2fu) |
                           __vcmpeq4(v.z, 0x2f2f2f2fu) | __vcmpeq4(v.w, 0x2f2f2f2fu);
      if (!hit && w0 + 16 <= L) continue;
      int p = w0 > b ? w0 : b;
      const int pe = w0 + 16 < e - 1 ? w0 + 16 : e - 1;
      for (; p < pe; ++p)
        if (s[p] == '/' && s[p + 1] == '/') break;
      if (p < pe) {
        e = p;
        break;
      }
    }
    const int x = skip_ws(s, b, e), y = rskip_ws(s, x, e);
    lb[k] = x;
    le[k] = y;
    const bool content = x < y && s[x] != '#';
    kind[k] = content ? 1 : 0;
    if (content) atomicMin(g + G_H, k);
  }
}

// the digraph header on line H (graphio.py:98-107); the rest of the line
// becomes its body
__global__ void header(const u8 *s, int32_t *lb, const int32_t *le, u8 *kind, int32_t *g) {
  const int H = g[G_H];
  if (H == INT_MAX) return;
  const int b = lb[H], e = le[H];
  int p = b;
  if (e - p >= 6 && span_is(s, p, p + 6, "strict") && p + 6 < e && ws_at(s, p + 6, e))
    p = skip_ws(s, p + 6, e);
  bool di = false, ok = true;
  if (e - p >= 7 && span_is(s, p, p + 7, "digraph")) {
    di = true;
    p += 7;
  } else if (e - p >= 5 && span_is(s, p, p + 5, "graph")) {
    p += 5;
  } else {
    ok = false;
  }
  bool brace = false;
  int n0 = 0, n1 = 0;
  if (ok) {
    p = skip_ws(s, p, e);
    n0 = p;
    while (p < e && (id_char(s[p]) || s[p] == '"')) ++p;
    n1 = p;
    p = skip_ws(s, p, e);
    if (p < e && s[p] == '{') {
      brace = true;
      p = skip_ws(s, p + 1, e);
    }
  }
  if (!ok || (!brace && p != e)) {
    g[G_FATAL] = 1;
    g[G_ERRK] = kErrHeader;
    g[G_ERRA] = b;
    g[G_ERRB] = e;
    return;
  }
  if (!di) {
    g[G_FATAL] = 1;
    g[G_ERRK] = kErrUndirected;
    return;
  }
  g[G_HNAME_B] = n1 > n0 ? n0 : -1;
  g[G_HNAME_E] = n1;
  lb[H] = p;  // already stripped on the right; p skipped the left
  kind[H] = p < e ? 1 : 0;
}

// body span of a line after its closing brace handling; close: 0 none,
// 1 "}" alone (no statements), 2 statements then close
__device__ inline int body(const u8 *s, int &b, int &e) {
  if (e - b == 1 && s[b] == '}') return 1;
  if (s[e - 1] == '}' && !(e - b >= 2 && s[e - 2] == '"')) {
    e = rskip_ws(s, b, e - 1);
    return 2;
  }
  return 0;
}

__global__ void find_close(const u8 *s, const int32_t *lb, const int32_t *le, const u8 *kind,
                           int nlines, int32_t *g) {
  const int H = g[G_H];
  if (H == INT_MAX || g[G_FATAL]) return;
  for (int k = H + blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += gridDim.x * blockDim.x) {
    if (!kind[k]) continue;
    int b = lb[k], e = le[k];
    if (body(s, b, e)) atomicMin(g + G_C, k);
  }
}

// The bytes of a block's lines (one line per thread, consecutive lines) staged
// in shared memory with coalesced 16-byte loads, so the per-thread scanners
// read shared memory instead of 32 scattered L1 lines per warp load. Returns
// the base to index with global byte offsets: the staged copy, or the text
// itself when the span does not fit.
constexpr int kStage = 32 * 1024;

__device__ const u8 *stage_lines(const u8 *s, int L, const int32_t *lb, const int32_t *le,
                                 int k0, int nlines, u8 *smem) {
  __shared__ int sb, se;
  if (threadIdx.x == 0) {
    const int k1 = min(k0 + (int)blockDim.x, nlines) - 1;
    sb = lb[k0] & ~15;
    se = max(le[k1], sb);
  }
  __syncthreads();
  const int b0 = sb, n = se - sb;
  if (n > kStage) return s;
  for (int i = threadIdx.x * 16; i < n; i += blockDim.x * 16) {
    if (b0 + i + 16 <= L) {
      *(uint4 *)(smem + i) = __ldg((const uint4 *)(s + b0 + i));
    } else {
      for (int q = 0; q < 16 && b0 + i + q < L; ++q) smem[i + q] = s[b0 + i + q];
    }
  }
  __syncthreads();
  return smem - b0;
}

__global__ void __launch_bounds__(256) count_lines(const u8 *text, int L, const int32_t *lb,
                                                   const int32_t *le, const u8 *kind, int nlines,
                                                   int32_t *g, int32_t *cnt, int32_t *err) {
  __shared__ __align__(16) u8 smem[kStage];
  const int H = g[G_H];
  const int last = g[G_C] == INT_MAX ? nlines - 1 : g[G_C];
  const bool run = H != INT_MAX && !g[G_FATAL];
  for (int k0 = blockIdx.x * blockDim.x; k0 < nlines; k0 += gridDim.x * blockDim.x) {
    const u8 *s = run ? stage_lines(text, L, lb, le, k0, nlines, smem) : text;
    const int k = k0 + threadIdx.x;
    if (k < nlines) {
      CountSink c{s};
      if (run && k >= H && k <= last && kind[k]) {
        int b = lb[k], e = le[k];
        if (body(s, b, e) != 1) {
          LineErr le_;
          if (!line_statements(s, b, e, c, le_)) {
            err[4 * k + 0] = le_.kind;
            err[4 * k + 1] = le_.a;
            err[4 * k + 2] = le_.b;
            err[4 * k + 3] = le_.c;
            atomicMin(g + G_E, k);
          }
        }
      }
      cnt[k] = c.occ;
      cnt[nlines + k] = c.edges;
      cnt[2 * nlines + k] = c.nodes;
      cnt[3 * nlines + k] = c.attrs;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) fill_lines(const u8 *text, int L, const int32_t *lb,
                                                  const int32_t *le, const u8 *kind, int nlines,
                                                  const int32_t *g, const int32_t *off, int base1,
                                                  int base2, int base3, Out o) {
  __shared__ __align__(16) u8 smem[kStage];
  const int H = g[G_H];
  const int last = g[G_C] == INT_MAX ? nlines - 1 : g[G_C];
  for (int k0 = blockIdx.x * blockDim.x; k0 < nlines; k0 += gridDim.x * blockDim.x) {
    const u8 *s = stage_lines(text, L, lb, le, k0, nlines, smem);
    const int k = k0 + threadIdx.x;
    if (k < nlines && k >= H && k <= last && kind[k]) {
      int b = lb[k], e = le[k];
      if (body(s, b, e) != 1) {
        FillSink f{s, o, off[k], off[nlines + k] - base1, off[2 * nlines + k] - base2,
                   off[3 * nlines + k] - base3};
        LineErr le_;
        line_statements(s, b, e, f, le_);
      }
    }
    __syncthreads();
  }
}

// names: open-address table of canonical hashes, first occurrence per slot
__global__ void name_insert(const u8 *s, int n, const int32_t *ob, const int32_t *oe,
                            uint64_t *key, uint32_t *first, uint32_t mask, uint32_t *slot_of) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t h = canon_hash(s, ob[i], oe[i]);
    uint32_t slot = (uint32_t)h & mask;
    for (;;) {
      const unsigned long long prev =
          atomicCAS((unsigned long long *)&key[slot], 0ull, (unsigned long long)h);
      if (prev == 0 || prev == h) break;
      slot = (slot + 1) & mask;
    }
    atomicMin(&first[slot], (uint32_t)i);
    slot_of[i] = slot;
  }
}

__global__ void name_heads(const u8 *s, int n, const int32_t *ob, const int32_t *oe,
                           const uint32_t *first, const uint32_t *slot_of, int32_t *head,
                           int32_t *g) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t f = first[slot_of[i]];
    head[i] = f == (uint32_t)i;
    if (f != (uint32_t)i && !canon_eq(s, ob[i], oe[i], ob[f], oe[f])) g[G_COLLIDE] = 1;
  }
}

// rank_of_occ = exclusive scan of head; per occurrence its name's rank
__global__ void name_ranks(int n, const uint32_t *first, const uint32_t *slot_of,
                           const int32_t *head, const int32_t *rank_scan, int32_t *name_of,
                           int32_t *uniq_occ) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = rank_scan[first[slot_of[i]]];
    name_of[i] = r;
    if (head[i]) uniq_occ[r] = i;
  }
}

// n?(\d+)$ on the canonical name: its number, -1 if none, -2 beyond 2^62
__device__ int64_t name_number(const u8 *s, int b, int e) {
  Canon c(s, b, e);
  int x = c.next();
  if (x == 'n') x = c.next();
  if (x < '0' || x > '9') return -1;
  int64_t v = 0;
  bool big = false;
  for (; x >= 0; x = c.next()) {
    if (x < '0' || x > '9') return -1;
    if (v > (1ll << 62) / 10) big = true;
    else v = v * 10 + (x - '0');
  }
  return big || v > (1ll << 62) ? -2 : v;
}

__global__ void number_insert(const u8 *s, int U, const int32_t *uniq_occ, const int32_t *ob,
                              const int32_t *oe, int64_t *num, uint64_t *key, uint32_t *first,
                              uint32_t mask, int32_t *g) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < U; r += gridDim.x * blockDim.x) {
    const int o = uniq_occ[r];
    const int64_t v = name_number(s, ob[o], oe[o]);
    num[r] = v;
    if (v == -2) g[G_BIGID] = 1;
    if (v < 0) continue;
    const uint64_t h = (uint64_t)v + 1;
    uint32_t slot = (uint32_t)mix64(h) & mask;
    for (;;) {
      const unsigned long long prev =
          atomicCAS((unsigned long long *)&key[slot], 0ull, (unsigned long long)h);
      if (prev == 0 || prev == h) break;
      slot = (slot + 1) & mask;
    }
    atomicMin(&first[slot], (uint32_t)r);
  }
}

// ids: numbered names that won their number keep it; flags the rest
// (warp-uniform trips: the max reduction runs on full warps)
__global__ void number_assign(int U, const int64_t *num, const uint64_t *key,
                              const uint32_t *first, uint32_t mask, int64_t *id, int32_t *rest,
                              unsigned long long *max_taken, int32_t *g) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < U; base += stride) {
    const int64_t r = base + threadIdx.x;
    bool won = false;
    int64_t v = -1;
    if (r < U) {
      v = num[r];
      if (v >= 0) {
        const uint64_t h = (uint64_t)v + 1;
        uint32_t slot = (uint32_t)mix64(h) & mask;
        while (key[slot] != h) slot = (slot + 1) & mask;
        won = first[slot] == (uint32_t)r;
      }
      id[r] = won ? v : -1;
      rest[r] = !won;
      if (won && v == 0) g[G_ZERO] = 1;
    }
    unsigned long long mx = won ? (unsigned long long)v : 0ull;
    for (int o = 16; o; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_taken, mx);
  }
}

__global__ void number_rest(int U, const int32_t *rest, const int32_t *rest_scan,
                            const unsigned long long *max_taken, int64_t *id) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < U; r += gridDim.x * blockDim.x)
    if (rest[r]) id[r] = (int64_t)*max_taken + 1 + rest_scan[r];
}

// last node attribute per (name, known key) and the owner of every attribute
__global__ void node_attrs(int nnodes, const int32_t *node_occ, const int32_t *node_ab,
                          const int32_t *node_an, const int32_t *name_of, const u8 *cls,
                          int32_t *last, int32_t *owner) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nnodes; t += gridDim.x * blockDim.x) {
    const int r = name_of[node_occ[t]];
    for (int i = node_ab[t], j = 0; j < node_an[t]; ++i, ++j) {
      owner[i] = r;
      if (cls[i] <= kWgpu) atomicMax(&last[4 * r + cls[i]], i);
    }
  }
}

// error order key: nodes in appearance order (size, weight_cpu, weight_gpu),
// then edges in declaration order (bytes, weight_xfer) — graphio.py:160-183
enum : int { kConvBad = 1, kConvInf = 2, kConvNan = 3 };

__device__ void conv_error(unsigned long long *err, int64_t order, int kind) {
  atomicMin(err, ((unsigned long long)order << 3) | (unsigned long long)kind);
}

// a literal the device could not round: listed for the host (order key, attr)
__device__ void slow_literal(int64_t order, int attr, int64_t *slow, int32_t *g) {
  const int k = atomicAdd(g + G_NSLOW, 1);
  slow[2 * k] = order;
  slow[2 * k + 1] = attr;
}

__device__ double conv_float(const u8 *s, const int32_t *v0, const int32_t *v1, int a,
                             int64_t order, unsigned long long *err, int64_t *slow, int32_t *g) {
  if (a < 0) return 0.0;
  double x = 0.0;
  const int st = py_float(s, v0[a], v1[a], &x);
  if (st == kFloatBad) conv_error(err, order, kConvBad);
  if (st == kFloatSlow) slow_literal(order, a, slow, g);
  return x;
}

__device__ int64_t conv_int(const u8 *s, const int32_t *v0, const int32_t *v1, int a,
                            int64_t order, unsigned long long *err, int64_t *slow, int32_t *g) {
  if (a < 0) return 0;
  double x = 0.0;
  const int st = py_float(s, v0[a], v1[a], &x);
  if (st == kFloatBad) {
    conv_error(err, order, kConvBad);
    return 0;
  }
  if (st == kFloatSlow) {
    slow_literal(order, a, slow, g);
    return 0;
  }
  if (x != x) {
    conv_error(err, order, kConvNan);
    return 0;
  }
  if (x == __longlong_as_double(0x7FF0000000000000ll) ||
      x == -__longlong_as_double(0x7FF0000000000000ll)) {
    conv_error(err, order, kConvInf);
    return 0;
  }
  if (!(x > -9223372036854775808.0 && x < 9223372036854775808.0)) {
    slow_literal(order, a, slow, g);  // a Python int beyond int64: the host converts
    return 0;
  }
  return (int64_t)x;  // truncation toward zero, as int()
}

__global__ void name_values(const u8 *s, int U, const int32_t *last, const int32_t *v0,
                            const int32_t *v1, int64_t *size, double *wc, double *wg,
                            int32_t *kind_attr, unsigned long long *err, int64_t *slow,
                            int32_t *g) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < U; r += gridDim.x * blockDim.x) {
    const int ka = last[4 * r + kKind];
    kind_attr[r] = ka;
    if (ka >= 0 && canon_is(s, v0[ka], v1[ka], "SOURCE")) atomicMin(g + G_ROOT, r);
    size[r] = conv_int(s, v0, v1, last[4 * r + kSize], 3ll * r, err, slow, g);
    wc[r] = conv_float(s, v0, v1, last[4 * r + kWcpu], 3ll * r + 1, err, slow, g);
    wg[r] = conv_float(s, v0, v1, last[4 * r + kWgpu], 3ll * r + 2, err, slow, g);
  }
}

__global__ void edge_values(const u8 *s, int U, int E, const int32_t *edge_occ,
                            const int32_t *edge_ab, const int32_t *edge_an, const int32_t *name_of,
                            const u8 *cls, const int32_t *v0, const int32_t *v1, int32_t *src,
                            int32_t *dst, int64_t *nbytes, double *wx, int32_t *owner,
                            u8 *has_pred, unsigned long long *err, int64_t *slow, int32_t *g) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < E; t += gridDim.x * blockDim.x) {
    const int o = edge_occ[t];
    src[t] = name_of[o];
    dst[t] = name_of[o + 1];
    has_pred[name_of[o + 1]] = 1;
    int lb = -1, lw = -1;
    for (int i = edge_ab[t], j = 0; j < edge_an[t]; ++i, ++j) {
      owner[i] = -1 - t;
      if (cls[i] == kBytes) lb = i;
      if (cls[i] == kWxfer) lw = i;
    }
    const int64_t base = 3ll * U + 2ll * t;
    nbytes[t] = conv_int(s, v0, v1, lb, base, err, slow, g);
    wx[t] = conv_float(s, v0, v1, lw, base + 1, err, slow, g);
  }
}

__global__ void canon_hashes(const u8 *s, int n, const int32_t *idx, const int32_t *b,
                             const int32_t *e, uint64_t *h) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = idx ? idx[i] : i;
    h[i] = a < 0 ? 0 : canon_hash(s, b[a], e[a]);
  }
}

}  // namespace

// ------------------------------------------------------------ CSR -------
// node keys: ids of the names, then the synthesized root (index U)
__global__ void csr_node_keys(int U, const int64_t *id, int64_t root_id, bool synth,
                              uint64_t *key, int32_t *val) {
  const int n = U + (synth ? 1 : 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    key[i] = (uint64_t)(i < U ? id[i] : root_id);
    val[i] = i;
  }
}

__global__ void csr_invert(int n, const int32_t *order, int32_t *pos) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    pos[order[i]] = i;
}

// edge keys (src index << 32 | dst index): declarations, then root -> every
// name without a predecessor (graphio.py:192-198)
__global__ void csr_edge_keys(int E, const int32_t *src, const int32_t *dst, const int32_t *pos,
                              int R, const int32_t *nopred, int root_pos, int shift, uint64_t *key,
                              int32_t *val) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E + R; i += gridDim.x * blockDim.x) {
    const uint32_t a = i < E ? pos[src[i]] : root_pos;
    const uint32_t b = i < E ? pos[dst[i]] : pos[nopred[i - E]];
    key[i] = ((uint64_t)a << shift) | b;
    val[i] = i;
  }
}

// a later duplicate edge replaces the earlier one (graph.py:66-69): keep the
// last of every run of equal keys (the sort is stable)
// 1 if key[] is not non-decreasing (then a stable radix sort is needed;
// emit_dot's output is already in order)
__global__ void not_sorted(int n, const uint64_t *key, int32_t *flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += gridDim.x * blockDim.x)
    if (key[i] > key[i + 1]) *flag = 1;
}

__global__ void csr_keep_last(int M, const uint64_t *key, u8 *keep) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x)
    keep[i] = i + 1 == M || key[i] != key[i + 1];
}

__global__ void csr_nodes(int n, int U, const uint64_t *skey, const int32_t *order,
                          const double *wc, const double *wg, int64_t *ids, double *w_cpu,
                          double *w_gpu, int64_t *out_ptr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
    out_ptr[i] = 0;
    if (i == n) continue;
    const int r = order[i];
    ids[i] = (int64_t)skey[i];
    w_cpu[i] = r < U ? wc[r] : 0.0;
    w_gpu[i] = r < U ? wg[r] : 0.0;
  }
}

__global__ void csr_edges(int m, int E, int shift, const uint64_t *key, const int32_t *val,
                          const int64_t *nbytes, const double *wx, int32_t *out_dst,
                          double *w_xfer, int64_t *bytes, unsigned long long *deg) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    const uint64_t k = key[j];
    const int t = val[j];
    out_dst[j] = (int32_t)(k & ((1ull << shift) - 1));
    w_xfer[j] = t < E ? wx[t] : 0.0;
    bytes[j] = t < E ? nbytes[t] : 0;
    atomicAdd(&deg[(k >> shift) + 1], 1ull);
  }
}

// ------------------------------------------------------------ host side ---
namespace {

template <typename T>
cudaError_t dmalloc(T **p, size_t n, cudaStream_t s) {
  return cudaMallocAsync((void **)p, (n ? n : 1) * sizeof(T), s);
}

struct DotParse {
  cudaStream_t s = nullptr;
  const u8 *text = nullptr;
  int L = 0, U = 0, E = 0, NA = 0, NO = 0, NN = 0, nslow = 0;
  int root_rank = -1;
  bool zero_taken = false;
  int64_t max_id = 0;
  std::vector<void *> bufs;
  // per name
  int64_t *id = nullptr, *size = nullptr;
  int32_t *kind_attr = nullptr;
  double *wc = nullptr, *wg = nullptr;
  u8 *has_pred = nullptr;
  // per edge
  int32_t *src = nullptr, *dst = nullptr;
  int64_t *nbytes = nullptr;
  double *wx = nullptr;
  // per attribute
  Out o{};
  int32_t *owner = nullptr;
  int64_t *slow = nullptr;
  // CSR (hs_dot_csr_size)
  int csr_n = -1, csr_m = 0, csr_root = -1, csr_shift = 32;
  uint64_t *node_key = nullptr, *edge_key = nullptr;
  int32_t *node_order = nullptr, *edge_val = nullptr;
  template <typename T>
  cudaError_t alloc(T **p, size_t n) {
    cudaError_t e = dmalloc(p, n, s);
    if (e == cudaSuccess) bufs.push_back(*p);
    return e;
  }
  ~DotParse() {
    for (void *p : bufs) cudaFreeAsync(p, s);
  }
};

template <typename T>
int exscan(const T *in, T *out, int64_t n, cudaStream_t s) {
  if (n <= 0) return HS_OK;
  size_t tb = 0;
  HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
  hs::Scratch<char> tmp;
  HS_CHECK_CUDA(tmp.alloc(tb, s));
  HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
  hs::count_launch(1);
  return HS_OK;
}

uint32_t table_size(int64_t n) {
  uint64_t t = 16;
  while (t < 2 * (uint64_t)n) t <<= 1;
  return (uint32_t)t;
}

}  // namespace

extern "C" int hs_dot_parse(const uint8_t *text, int64_t len, hs_dot_info_t *info, void **handle,
                            void *stream) {
  HS_REQUIRE(info && handle && (text || len == 0) && len >= 0, HS_EINVAL,
             "hs_dot_parse: null argument");
  HS_REQUIRE(len < (1ll << 31) - 16, HS_ELIMIT, "hs_dot_parse: DOT text beyond 2^31 bytes");
  HS_REQUIRE(((uintptr_t)text & 15) == 0, HS_EINVAL, "hs_dot_parse: text must be 16-byte aligned");
  *handle = nullptr;
  memset(info, 0, sizeof *info);
  cudaStream_t s = (cudaStream_t)stream;
  DotParse *P = new DotParse;
  P->s = s;
  P->text = text;
  P->L = (int)len;
  auto fail = [&](int rc) {
    delete P;
    return rc;
  };
  const int L = (int)len;
  const int B = 256;
  int32_t *g;
  if (P->alloc(&g, G_COUNT)) return fail(HS_ECUDA);
  int32_t g0[G_COUNT] = {};
  g0[G_H] = g0[G_C] = g0[G_E] = g0[G_ROOT] = INT_MAX;
  if (cudaMemcpyAsync(g, g0, sizeof g0, cudaMemcpyHostToDevice, s)) return fail(HS_ECUDA);

  // 1. line terminators
  const int64_t nch = ((int64_t)L + kChunk - 1) / kChunk;
  int32_t *tcnt, *toff, *term = nullptr;
  if (P->alloc(&tcnt, nch + 1) || P->alloc(&toff, nch + 1)) return fail(HS_ECUDA);
  int nterm = 0, nlines = 0;
  if (L > 0) {
    const int tg = hs::grid_for(nch, B);
    terms<false><<<tg, B, 0, s>>>(text, L, tcnt, nullptr, nullptr, g);
    hs::count_launch();
    if (cudaMemsetAsync(tcnt + nch, 0, 4, s)) return fail(HS_ECUDA);
    if (exscan(tcnt, toff, nch + 1, s)) return fail(HS_ECUDA);
    if (cudaMemcpyAsync(&nterm, toff + nch, 4, cudaMemcpyDeviceToHost, s) ||
        cudaStreamSynchronize(s))
      return fail(HS_ECUDA);
    if (P->alloc(&term, (size_t)nterm + 1)) return fail(HS_ECUDA);
    terms<true><<<tg, B, 0, s>>>(text, L, nullptr, toff, term, g);
    hs::count_launch();
    int last_end = 0;
    if (nterm > 0) {
      int32_t t = 0;
      u8 tail[3] = {0, 0, 0};
      if (cudaMemcpyAsync(&t, term + nterm - 1, 4, cudaMemcpyDeviceToHost, s) ||
          cudaStreamSynchronize(s) ||
          cudaMemcpyAsync(tail, text + t, L - t < 3 ? L - t : 3, cudaMemcpyDeviceToHost, s) ||
          cudaStreamSynchronize(s))
        return fail(HS_ECUDA);
      // the last terminator's length (\r\n, U+0085 and U+2028/9 are longer)
      int len = 1;
      if (tail[0] == '\r' && L - t > 1 && tail[1] == '\n') len = 2;
      if (tail[0] == 0xC2) len = 2;
      if (tail[0] == 0xE2) len = 3;
      last_end = t + len;
    }
    nlines = nterm + (last_end < L ? 1 : 0);
  }

  // 2-3. lines: spans, header, closing line, counts and the first error
  const int nl1 = nlines > 0 ? nlines : 1;
  int32_t *lb, *le, *cnt, *off, *err;
  u8 *kind;
  if (P->alloc(&lb, nl1) || P->alloc(&le, nl1) || P->alloc(&kind, nl1) ||
      P->alloc(&cnt, 4 * (size_t)nl1 + 1) || P->alloc(&off, 4 * (size_t)nl1 + 1) ||
      P->alloc(&err, 4 * (size_t)nl1))
    return fail(HS_ECUDA);
  if (nlines > 0) {
    const int lg = hs::grid_for(nlines, B);
    line_spans<<<lg, B, 0, s>>>(text, L, term, nterm, nlines, lb, le, kind, g);
    header<<<1, 1, 0, s>>>(text, lb, le, kind, g);
    find_close<<<lg, B, 0, s>>>(text, lb, le, kind, nlines, g);
    count_lines<<<lg, B, 0, s>>>(text, L, lb, le, kind, nlines, g, cnt, err);
    hs::count_launch(4);
    if (cudaMemsetAsync(cnt + 4 * (size_t)nlines, 0, 4, s)) return fail(HS_ECUDA);
    if (exscan(cnt, off, 4 * (int64_t)nlines + 1, s)) return fail(HS_ECUDA);
  }
  int32_t gh[G_COUNT];
  int32_t tot[5] = {0, 0, 0, 0, 0};  // offsets of the four count runs + total
  if (cudaMemcpyAsync(gh, g, sizeof gh, cudaMemcpyDeviceToHost, s)) return fail(HS_ECUDA);
  if (nlines > 0)
    for (int q = 1; q <= 4; ++q)
      if (cudaMemcpyAsync(&tot[q], off + (size_t)q * nlines, 4, cudaMemcpyDeviceToHost, s))
        return fail(HS_ECUDA);
  if (cudaStreamSynchronize(s)) return fail(HS_ECUDA);
  info->name_b = -1;
  info->root_rank = -1;
  info->conv_err = -1;
  const int nl_count = gh[G_NL];
  if (gh[G_H] == INT_MAX) {
    info->status = kErrNoGraph;
    info->err_line = nl_count + 1 > 1 ? nl_count + 1 : 1;
    return fail(HS_OK);
  }
  if (gh[G_FATAL]) {
    info->status = gh[G_ERRK];
    info->err_line = gh[G_H] + 1;
    info->err_a = gh[G_ERRA];
    info->err_b = gh[G_ERRB];
    return fail(HS_OK);
  }
  info->name_b = gh[G_HNAME_B];
  info->name_e = gh[G_HNAME_E];
  if (gh[G_E] != INT_MAX) {
    int32_t er[4];
    if (cudaMemcpyAsync(er, err + 4 * (size_t)gh[G_E], sizeof er, cudaMemcpyDeviceToHost, s) ||
        cudaStreamSynchronize(s))
      return fail(HS_ECUDA);
    info->status = er[0];
    info->err_line = gh[G_E] + 1;
    info->err_a = er[1];
    info->err_b = er[2];
    info->err_c = er[3];
    return fail(HS_OK);
  }
  if (gh[G_C] == INT_MAX) {
    info->status = kErrBrace;
    info->err_line = nl_count + 1;
    return fail(HS_OK);
  }
  // run totals: occ | edges | nodes | attrs
  const int NO = tot[1], E = tot[2] - tot[1], NN = tot[3] - tot[2], NA = tot[4] - tot[3];
  P->NO = NO;
  P->E = E;
  P->NN = NN;
  P->NA = NA;

  // 4. records
  Out &o = P->o;
  if (P->alloc(&o.occ_b, NO) || P->alloc(&o.occ_e, NO) || P->alloc(&o.edge_occ, E) ||
      P->alloc(&o.edge_ab, E) || P->alloc(&o.edge_an, E) || P->alloc(&o.node_occ, NN) ||
      P->alloc(&o.node_ab, NN) || P->alloc(&o.node_an, NN) || P->alloc(&o.attr_k0, NA) ||
      P->alloc(&o.attr_k1, NA) || P->alloc(&o.attr_v0, NA) || P->alloc(&o.attr_v1, NA) ||
      P->alloc(&o.attr_cls, NA))
    return fail(HS_ECUDA);
  if (NO > 0 || NA > 0) {
    fill_lines<<<hs::grid_for(nlines, B), B, 0, s>>>(text, L, lb, le, kind, nlines, g, off, tot[1],
                                                     tot[2], tot[3], o);
    hs::count_launch();
  }

  // 5. names: dedup, appearance ranks
  uint32_t *slot_of, *first;
  uint64_t *key;
  int32_t *head, *rank, *name_of, *uniq_occ;
  const uint32_t T1 = table_size(NO);
  if (P->alloc(&slot_of, NO) || P->alloc(&first, T1) || P->alloc(&key, T1) ||
      P->alloc(&head, NO + 1) || P->alloc(&rank, NO + 1) || P->alloc(&name_of, NO))
    return fail(HS_ECUDA);
  if (cudaMemsetAsync(first, 0xff, T1 * 4ull, s) || cudaMemsetAsync(key, 0, T1 * 8ull, s) ||
      cudaMemsetAsync(head + NO, 0, 4, s))
    return fail(HS_ECUDA);
  const int og = hs::grid_for(NO, B);
  if (NO > 0) {
    name_insert<<<og, B, 0, s>>>(text, NO, o.occ_b, o.occ_e, key, first, T1 - 1, slot_of);
    name_heads<<<og, B, 0, s>>>(text, NO, o.occ_b, o.occ_e, first, slot_of, head, g);
    hs::count_launch(2);
  }
  if (exscan(head, rank, (int64_t)NO + 1, s)) return fail(HS_ECUDA);
  int U = 0;
  if (cudaMemcpyAsync(&U, rank + NO, 4, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
    return fail(HS_ECUDA);
  P->U = U;
  if (P->alloc(&uniq_occ, U)) return fail(HS_ECUDA);
  if (NO > 0) {
    name_ranks<<<og, B, 0, s>>>(NO, first, slot_of, head, rank, name_of, uniq_occ);
    hs::count_launch();
  }

  // 6. ids
  int64_t *num;
  uint64_t *key2;
  uint32_t *first2;
  int32_t *rest, *rest_scan;
  unsigned long long *max_taken;
  const uint32_t T2 = table_size(U);
  if (P->alloc(&num, U) || P->alloc(&key2, T2) || P->alloc(&first2, T2) ||
      P->alloc(&rest, U + 1) || P->alloc(&rest_scan, U + 1) || P->alloc(&max_taken, 1) ||
      P->alloc(&P->id, U))
    return fail(HS_ECUDA);
  if (cudaMemsetAsync(first2, 0xff, T2 * 4ull, s) || cudaMemsetAsync(key2, 0, T2 * 8ull, s) ||
      cudaMemsetAsync(max_taken, 0, 8, s) || cudaMemsetAsync(rest + U, 0, 4, s))
    return fail(HS_ECUDA);
  const int ug = hs::grid_for(U, B);
  if (U > 0) {
    number_insert<<<ug, B, 0, s>>>(text, U, uniq_occ, o.occ_b, o.occ_e, num, key2, first2, T2 - 1,
                                   g);
    number_assign<<<ug, B, 0, s>>>(U, num, key2, first2, T2 - 1, P->id, rest, max_taken, g);
    hs::count_launch(2);
  }
  if (exscan(rest, rest_scan, (int64_t)U + 1, s)) return fail(HS_ECUDA);
  if (U > 0) {
    number_rest<<<ug, B, 0, s>>>(U, rest, rest_scan, max_taken, P->id);
    hs::count_launch();
  }

  // 7. attributes and values
  int32_t *last;
  unsigned long long *cerr;
  if (P->alloc(&last, 4 * (size_t)U) || P->alloc(&P->owner, NA) || P->alloc(&P->size, U) ||
      P->alloc(&P->wc, U) || P->alloc(&P->wg, U) || P->alloc(&P->kind_attr, U) ||
      P->alloc(&P->has_pred, U) || P->alloc(&P->src, E) || P->alloc(&P->dst, E) ||
      P->alloc(&P->nbytes, E) || P->alloc(&P->wx, E) || P->alloc(&cerr, 1) ||
      P->alloc(&P->slow, 2 * ((size_t)NA + 1)))
    return fail(HS_ECUDA);
  if (cudaMemsetAsync(last, 0xff, 16ull * U, s) || cudaMemsetAsync(cerr, 0xff, 8, s) ||
      cudaMemsetAsync(P->has_pred, 0, U, s))
    return fail(HS_ECUDA);
  if (NN > 0) {
    node_attrs<<<hs::grid_for(NN, B), B, 0, s>>>(NN, o.node_occ, o.node_ab, o.node_an, name_of,
                                                o.attr_cls, last, P->owner);
    hs::count_launch();
  }
  if (U > 0) {
    name_values<<<ug, B, 0, s>>>(text, U, last, o.attr_v0, o.attr_v1, P->size, P->wc, P->wg,
                                 P->kind_attr, cerr, P->slow, g);
    hs::count_launch();
  }
  if (E > 0) {
    edge_values<<<hs::grid_for(E, B), B, 0, s>>>(text, U, E, o.edge_occ, o.edge_ab, o.edge_an,
                                                 name_of, o.attr_cls, o.attr_v0, o.attr_v1,
                                                 P->src, P->dst, P->nbytes, P->wx, P->owner,
                                                 P->has_pred, cerr, P->slow, g);
    hs::count_launch();
  }
  unsigned long long ce = 0, mt = 0;
  if (cudaMemcpyAsync(gh, g, sizeof gh, cudaMemcpyDeviceToHost, s) ||
      cudaMemcpyAsync(&ce, cerr, 8, cudaMemcpyDeviceToHost, s) ||
      cudaMemcpyAsync(&mt, max_taken, 8, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
    return fail(HS_ECUDA);
  if (gh[G_COLLIDE]) {
    hs::set_error("hs_dot_parse: 64-bit name hash collision (two distinct names)");
    return fail(HS_ELIMIT);
  }
  if (gh[G_BIGID]) {
    hs::set_error("hs_dot_parse: numbered node name beyond 2^62");
    return fail(HS_ELIMIT);
  }
  P->nslow = gh[G_NSLOW];
  P->root_rank = gh[G_ROOT] == INT_MAX ? -1 : gh[G_ROOT];
  P->zero_taken = gh[G_ZERO] != 0;
  // the largest id: max numbered id, or the last sequential one
  int64_t max_id = (int64_t)mt;
  {
    int32_t nrest = 0;
    if (U > 0 && (cudaMemcpyAsync(&nrest, rest_scan + U, 4, cudaMemcpyDeviceToHost, s) ||
                  cudaStreamSynchronize(s)))
      return fail(HS_ECUDA);
    if (nrest > 0) max_id = (int64_t)mt + nrest;
  }
  P->max_id = max_id;
  info->n_names = U;
  info->n_edges = E;
  info->n_attrs = NA;
  info->n_slow = P->nslow;
  info->root_rank = P->root_rank;
  info->conv_err = ce == ~0ull ? -1 : (int64_t)ce;
  info->max_id = max_id;
  *handle = P;
  return HS_OK;
}

namespace {
struct NoPred {
  const u8 *hp;
  __host__ __device__ bool operator()(int r) const { return !hp[r]; }
};

// stable sort of (key, value) pairs over key bits [0, bits); keys already in
// order are copied instead
int sort_pairs(const uint64_t *kin, uint64_t *kout, const int32_t *vin, int32_t *vout, int n,
               int bits, cudaStream_t s) {
  if (n <= 0) return HS_OK;
  hs::Scratch<int32_t> flag;
  HS_CHECK_CUDA(flag.alloc(1, s));
  HS_CHECK_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
  not_sorted<<<hs::grid_for(n, 256), 256, 0, s>>>(n, kin, flag.p);
  HS_CHECK_LAUNCH();
  int32_t unsorted = 0;
  HS_CHECK_CUDA(cudaMemcpyAsync(&unsorted, flag.p, 4, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  if (!unsorted) {
    HS_CHECK_CUDA(cudaMemcpyAsync(kout, kin, 8ull * n, cudaMemcpyDeviceToDevice, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(vout, vin, 4ull * n, cudaMemcpyDeviceToDevice, s));
    return HS_OK;
  }
  bits = bits < 1 ? 1 : (bits > 64 ? 64 : bits);
  size_t tb = 0;
  HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, bits, s));
  hs::Scratch<char> tmp;
  HS_CHECK_CUDA(tmp.alloc(tb, s));
  HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kin, kout, vin, vout, n, 0, bits, s));
  hs::count_launch(4);
  return HS_OK;
}

int bit_width(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}
}  // namespace

extern "C" int hs_dot_fetch(void *handle, const hs_dot_host_t *h, void *stream) {
  HS_REQUIRE(handle && h, HS_EINVAL, "hs_dot_fetch: null argument");
  DotParse *P = (DotParse *)handle;
  cudaStream_t s = (cudaStream_t)stream;
  const int U = P->U, E = P->E, NA = P->NA;
  auto cp = [&](void *dst, const void *src, size_t bytes) -> cudaError_t {
    if (!dst || !bytes) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  };
  hs::Scratch<uint64_t> kh;
  HS_CHECK_CUDA(kh.alloc(U, s));
  if (U > 0 && h->kind_hash) {
    canon_hashes<<<hs::grid_for(U, 256), 256, 0, s>>>(P->text, U, P->kind_attr, P->o.attr_v0,
                                                      P->o.attr_v1, kh.p);
    HS_CHECK_LAUNCH();
  }
  HS_CHECK_CUDA(cp(h->id, P->id, 8ull * U));
  HS_CHECK_CUDA(cp(h->kind_attr, P->kind_attr, 4ull * U));
  HS_CHECK_CUDA(cp(h->kind_hash, kh.p, 8ull * U));
  HS_CHECK_CUDA(cp(h->size, P->size, 8ull * U));
  HS_CHECK_CUDA(cp(h->w_cpu, P->wc, 8ull * U));
  HS_CHECK_CUDA(cp(h->w_gpu, P->wg, 8ull * U));
  HS_CHECK_CUDA(cp(h->has_pred, P->has_pred, 1ull * U));
  HS_CHECK_CUDA(cp(h->src, P->src, 4ull * E));
  HS_CHECK_CUDA(cp(h->dst, P->dst, 4ull * E));
  HS_CHECK_CUDA(cp(h->bytes, P->nbytes, 8ull * E));
  HS_CHECK_CUDA(cp(h->w_xfer, P->wx, 8ull * E));
  HS_CHECK_CUDA(cp(h->k0, P->o.attr_k0, 4ull * NA));
  HS_CHECK_CUDA(cp(h->k1, P->o.attr_k1, 4ull * NA));
  HS_CHECK_CUDA(cp(h->v0, P->o.attr_v0, 4ull * NA));
  HS_CHECK_CUDA(cp(h->v1, P->o.attr_v1, 4ull * NA));
  HS_CHECK_CUDA(cp(h->owner, P->owner, 4ull * NA));
  HS_CHECK_CUDA(cp(h->cls, P->o.attr_cls, 1ull * NA));
  HS_CHECK_CUDA(cp(h->slow, P->slow, 16ull * P->nslow));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  return HS_OK;
}

extern "C" int hs_dot_csr_size(void *handle, int64_t *n_out, int64_t *m_out, void *stream) {
  HS_REQUIRE(handle && n_out && m_out, HS_EINVAL, "hs_dot_csr_size: null argument");
  DotParse *P = (DotParse *)handle;
  cudaStream_t s = (cudaStream_t)stream;
  const int U = P->U, E = P->E, B = 256;
  const bool synth = P->root_rank < 0;
  const int n = U + (synth ? 1 : 0);
  const int64_t root_id = !synth ? -1 : (P->zero_taken ? P->max_id + 1 : 0);
  HS_REQUIRE(n < INT_MAX, HS_ELIMIT, "hs_dot_csr_size: too many nodes");
  // nodes ascending by id
  hs::Scratch<uint64_t> nk;
  hs::Scratch<int32_t> nv, pos;
  HS_CHECK_CUDA(nk.alloc(n, s));
  HS_CHECK_CUDA(nv.alloc(n, s));
  HS_CHECK_CUDA(pos.alloc(n, s));
  if (!P->node_key) {
    HS_CHECK_CUDA(P->alloc(&P->node_key, n));
    HS_CHECK_CUDA(P->alloc(&P->node_order, n));
  }
  if (n > 0) {
    csr_node_keys<<<hs::grid_for(n, B), B, 0, s>>>(U, P->id, root_id, synth, nk.p, nv.p);
    HS_CHECK_LAUNCH();
  }
  const int64_t top_id = root_id > P->max_id ? root_id : P->max_id;
  int rc = sort_pairs(nk.p, P->node_key, nv.p, P->node_order, n, bit_width((uint64_t)top_id), s);
  if (rc) return rc;
  if (n > 0) {
    csr_invert<<<hs::grid_for(n, B), B, 0, s>>>(n, P->node_order, pos.p);
    HS_CHECK_LAUNCH();
  }
  // names without a predecessor feed from the synthesized root
  hs::Scratch<int32_t> nopred, nR;
  HS_CHECK_CUDA(nopred.alloc(U, s));
  HS_CHECK_CUDA(nR.alloc(1, s));
  int R = 0;
  if (synth && U > 0) {
    size_t tb = 0;
    thrust::counting_iterator<int32_t> it(0);
    HS_CHECK_CUDA(cub::DeviceSelect::If(nullptr, tb, it, nopred.p, nR.p, U, NoPred{P->has_pred}, s));
    hs::Scratch<char> tmp;
    HS_CHECK_CUDA(tmp.alloc(tb, s));
    HS_CHECK_CUDA(cub::DeviceSelect::If(tmp.p, tb, it, nopred.p, nR.p, U, NoPred{P->has_pred}, s));
    hs::count_launch();
    HS_CHECK_CUDA(cudaMemcpyAsync(&R, nR.p, 4, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  int root_pos = 0;
  if (n > 0) {
    const int rr = synth ? U : P->root_rank;
    HS_CHECK_CUDA(cudaMemcpyAsync(&root_pos, pos.p + rr, 4, cudaMemcpyDeviceToHost, s));
  }
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  const int M = E + R;
  P->csr_shift = bit_width((uint64_t)(n > 1 ? n - 1 : 1));
  hs::Scratch<uint64_t> ek, eks;
  hs::Scratch<int32_t> ev, evs;
  hs::Scratch<u8> keep;
  HS_CHECK_CUDA(ek.alloc(M, s));
  HS_CHECK_CUDA(ev.alloc(M, s));
  HS_CHECK_CUDA(eks.alloc(M, s));
  HS_CHECK_CUDA(evs.alloc(M, s));
  HS_CHECK_CUDA(keep.alloc(M, s));
  if (M > 0) {
    csr_edge_keys<<<hs::grid_for(M, B), B, 0, s>>>(E, P->src, P->dst, pos.p, R, nopred.p,
                                                   root_pos, P->csr_shift, ek.p, ev.p);
    HS_CHECK_LAUNCH();
  }
  rc = sort_pairs(ek.p, eks.p, ev.p, evs.p, M, 2 * P->csr_shift, s);
  if (rc) return rc;
  int m = 0;
  if (M > 0) {
    csr_keep_last<<<hs::grid_for(M, B), B, 0, s>>>(M, eks.p, keep.p);
    HS_CHECK_LAUNCH();
    if (P->edge_key) {
      cudaFreeAsync(P->edge_key, s);
      cudaFreeAsync(P->edge_val, s);
    }
    HS_CHECK_CUDA(dmalloc(&P->edge_key, M, s));
    HS_CHECK_CUDA(dmalloc(&P->edge_val, M, s));
    P->bufs.push_back(P->edge_key);
    P->bufs.push_back(P->edge_val);
    hs::Scratch<int32_t> nm;
    HS_CHECK_CUDA(nm.alloc(1, s));
    size_t tb = 0;
    HS_CHECK_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, eks.p, keep.p, P->edge_key, nm.p, M, s));
    hs::Scratch<char> tmp;
    HS_CHECK_CUDA(tmp.alloc(tb, s));
    HS_CHECK_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, eks.p, keep.p, P->edge_key, nm.p, M, s));
    HS_CHECK_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, evs.p, keep.p, P->edge_val, nm.p, M, s));
    hs::count_launch(2);
    HS_CHECK_CUDA(cudaMemcpyAsync(&m, nm.p, 4, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  P->csr_n = n;
  P->csr_m = m;
  P->csr_root = n > 0 ? root_pos : -1;
  *n_out = n;
  *m_out = m;
  return HS_OK;
}

extern "C" int hs_dot_csr(void *handle, int64_t *out_ptr, int32_t *out_dst, int64_t *ids,
                          double *w_cpu, double *w_gpu, double *w_xfer, int64_t *bytes,
                          int32_t *root_host, void *stream) {
  HS_REQUIRE(handle && root_host, HS_EINVAL, "hs_dot_csr: null argument");
  DotParse *P = (DotParse *)handle;
  HS_REQUIRE(P->csr_n >= 0, HS_EINVAL, "hs_dot_csr: call hs_dot_csr_size first");
  cudaStream_t s = (cudaStream_t)stream;
  const int n = P->csr_n, m = P->csr_m, B = 256;
  HS_REQUIRE(out_ptr && (n == 0 || (ids && w_cpu && w_gpu)) &&
                 (m == 0 || (out_dst && w_xfer && bytes)),
             HS_EINVAL, "hs_dot_csr: null output");
  csr_nodes<<<hs::grid_for(n + 1, B), B, 0, s>>>(n, P->U, P->node_key, P->node_order, P->wc,
                                                 P->wg, ids, w_cpu, w_gpu, out_ptr);
  HS_CHECK_LAUNCH();
  if (m > 0) {
    csr_edges<<<hs::grid_for(m, B), B, 0, s>>>(m, P->E, P->csr_shift, P->edge_key, P->edge_val,
                                               P->nbytes,
                                               P->wx, out_dst, w_xfer, bytes,
                                               (unsigned long long *)out_ptr);
    HS_CHECK_LAUNCH();
    // degrees at out_ptr[1..n] -> inclusive prefix in place
    size_t tb = 0;
    HS_CHECK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, out_ptr + 1, out_ptr + 1, n, s));
    hs::Scratch<char> tmp;
    HS_CHECK_CUDA(tmp.alloc(tb, s));
    HS_CHECK_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, out_ptr + 1, out_ptr + 1, n, s));
    hs::count_launch();
  }
  *root_host = P->csr_root;
  return HS_OK;
}

extern "C" int hs_dot_release(void *handle) {
  delete (DotParse *)handle;
  return HS_OK;
}

// Python float() of bytes on the host with the device's code (tests)
extern "C" int hs_dot_py_float(const uint8_t *bytes, int64_t len, double *out) {
  HS_REQUIRE(out && (bytes || len == 0) && len >= 0 && len < INT_MAX, HS_EINVAL,
             "hs_dot_py_float: bad argument");
  return py_float(bytes, 0, (int)len, out);
}
