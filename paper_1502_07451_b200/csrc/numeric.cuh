// Bit-exact restatements of the reference's floating-point reductions.
//
//  * PySum — CPython >= 3.12 builtin sum() over floats (bltinmodule.c,
//    builtin_sum_impl): the int start 0 absorbs the first float (0 + x),
//    then Neumaier-compensated accumulation, compensation added once at the
//    end if it is nonzero and finite. Every `sum(...)` in
//    partition.py (lines 65, 67, 69, 103, 149, 163, 166, 178, 225, 241, 242,
//    268) is this reduction, in the reference's iteration order.
//  * SuperAcc — exact fixed-point accumulator over the full double range,
//    rounded once to nearest-even: the value math.fsum returns
//    (costs.py:248-249, graph.py:329-331), computable in any order.
#pragma once
#include <stdint.h>
#include <math.h>
#include <string.h>

namespace hs {

__host__ __device__ inline double bits_to_double(uint64_t b) {
  double r;
  memcpy(&r, &b, sizeof r);
  return r;
}

struct PySum {
  double f = 0.0, c = 0.0;
  bool started = false;
  __host__ __device__ void add(double x) {
    if (!started) {
      f = 0.0 + x;
      started = true;
      return;
    }
    double t = f + x;
    if (fabs(f) >= fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  __host__ __device__ double result() const {
    double r = f;
    if (c != 0.0 && isfinite(c)) r += c;
    return r;
  }
};

// Fixed point: bit 0 of the accumulator weighs 2^-1074 (smallest subnormal).
// 67 limbs of 32 significant bits cover every finite double plus carry room.
constexpr int kAccLimbs = 67;

// Adds x into signed 64-bit limbs (deferred carries; each limb receives at
// most 2^32 per add, so 2^31 adds per limb are safe).
template <typename AddFn>
__device__ __forceinline__ void superacc_split(double x, AddFn add) {
  uint64_t bits = (uint64_t)__double_as_longlong(x);
  uint64_t ex = (bits >> 52) & 0x7ff;
  uint64_t mant = bits & ((1ull << 52) - 1);
  if (ex == 0 && mant == 0) return;
  int p;
  if (ex == 0) {
    p = 0;
  } else {
    mant |= 1ull << 52;
    p = (int)ex - 1;
  }
  int li = p >> 5, sh = p & 31;
  unsigned __int128 v = ((unsigned __int128)mant) << sh;
  int64_t c0 = (int64_t)(uint32_t)v;
  int64_t c1 = (int64_t)(uint32_t)(v >> 32);
  int64_t c2 = (int64_t)(uint32_t)(v >> 64);
  if (bits >> 63) { c0 = -c0; c1 = -c1; c2 = -c2; }
  if (c0) add(li, c0);
  if (c1) add(li + 1, c1);
  if (c2) add(li + 2, c2);
}

// Normalises the limbs and rounds to the nearest double (ties to even).
__host__ __device__ inline double superacc_round(const int64_t *limbs) {
  uint32_t d[kAccLimbs + 1];
  int64_t carry = 0;
  for (int i = 0; i < kAccLimbs; ++i) {
    int64_t v = limbs[i] + carry;
    d[i] = (uint32_t)((uint64_t)v & 0xffffffffull);
    carry = v >> 32;  // arithmetic shift
  }
  bool neg = carry < 0;
  if (neg) {  // two's complement negate the magnitude
    uint64_t c = 1;
    for (int i = 0; i < kAccLimbs; ++i) {
      uint64_t v = (uint64_t)(uint32_t)~d[i] + c;
      d[i] = (uint32_t)v;
      c = v >> 32;
    }
  }
  int top = -1;
  for (int i = kAccLimbs - 1; i >= 0 && top < 0; --i)
    if (d[i]) {
      int b = 31;
      while (!((d[i] >> b) & 1u)) --b;
      top = i * 32 + b;
    }
  if (top < 0) return 0.0;
  auto bit = [&](int pos) -> uint64_t {
    if (pos < 0) return 0;
    return (d[pos >> 5] >> (pos & 31)) & 1u;
  };
  double r;
  if (top < 53) {
    uint64_t m = 0;
    for (int pos = top; pos >= 0; --pos) m = (m << 1) | bit(pos);
    // m * 2^-1074 is exactly representable (subnormal or lowest binade)
    uint64_t b = m;  // subnormal encoding when m < 2^52
    if (m >> 52) {   // normal in the lowest binade: exponent field 1
      b = (1ull << 52) | (m & ((1ull << 52) - 1));
    }
    r = bits_to_double(b);
  } else {
    uint64_t m = 0;
    for (int pos = top; pos > top - 53; --pos) m = (m << 1) | bit(pos);
    uint64_t rnd = bit(top - 53);
    bool sticky = false;
    for (int pos = top - 54; pos >= 0 && !sticky; --pos) sticky = bit(pos) != 0;
    if (rnd && (sticky || (m & 1))) {
      ++m;
      if (m >> 53) { m >>= 1; ++top; }
    }
    int64_t bexp = (int64_t)top - 51;  // biased exponent
    if (bexp >= 2047) {
      r = bits_to_double(0x7ff0000000000000ull);
    } else {
      uint64_t b = ((uint64_t)bexp << 52) | (m & ((1ull << 52) - 1));
      r = bits_to_double(b);
    }
  }
  return neg ? -r : r;
}

}  // namespace hs
