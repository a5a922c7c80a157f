// ddmath.cuh — device error-free transformations, double-double arithmetic and exact int128 <-> fp64
// conversions for the ozr kernels. Every EFT uses the _rn intrinsics, which the compiler never
// contracts into FMAs, so TwoSum (§2.2) and the pair arithmetic
// (lines 155-161) are evaluated exactly as written regardless of -fmad.
#pragma once
#include <cstdint>

namespace ozr {

typedef __int128 i128;
typedef unsigned __int128 u128;

struct dd {
  double hi, lo;
};

__device__ __forceinline__ void two_sum(double a, double b, double& x, double& y) {
  x = __dadd_rn(a, b);
  double z = __dsub_rn(x, a);
  y = __dadd_rn(__dsub_rn(a, __dsub_rn(x, z)), __dsub_rn(b, z));
}
__device__ __forceinline__ void fast_two_sum(double a, double b, double& x, double& y) {
  x = __dadd_rn(a, b);
  y = __dsub_rn(b, __dsub_rn(x, a));
}
__device__ __forceinline__ void two_prod(double a, double b, double& x, double& y) {
  x = __dmul_rn(a, b);
  y = __fma_rn(a, b, -x);
}
// accurate double-double addition
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  double s, e, t, f;
  two_sum(a.hi, b.hi, s, e);
  two_sum(a.lo, b.lo, t, f);
  e = __dadd_rn(e, t);
  fast_two_sum(s, e, s, e);
  e = __dadd_rn(e, f);
  dd r;
  fast_two_sum(s, e, r.hi, r.lo);
  return r;
}
// (a.hi + a.lo) * b
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  double p, e;
  two_prod(a.hi, b, p, e);
  e = __fma_rn(a.lo, b, e);
  dd r;
  fast_two_sum(p, e, r.hi, r.lo);
  return r;
}
// a / b in double-double (one Newton correction)
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  double q1 = __ddiv_rn(a.hi, b.hi);
  dd p = dd_mul_d(b, q1);
  dd r = dd_add(a, dd{-p.hi, -p.lo});
  double q2 = __ddiv_rn(r.hi, b.hi);
  dd o;
  fast_two_sum(q1, q2, o.hi, o.lo);
  return o;
}

// Correctly rounded (RNE) conversion of a signed 128-bit integer to fp64.
__device__ __forceinline__ double i128_to_f64(i128 x) {
  if (x == 0) return 0.0;
  const bool neg = x < 0;
  u128 a = neg ? static_cast<u128>(-x) : static_cast<u128>(x);
  const uint64_t hi = static_cast<uint64_t>(a >> 64);
  double r;
  if (hi == 0) {
    r = __ull2double_rn(static_cast<uint64_t>(a));
  } else {
    const int lz = __clzll(static_cast<long long>(hi));
    const u128 b = a << lz;  // leading one at bit 127
    uint64_t top = static_cast<uint64_t>(b >> 64);
    top |= (static_cast<uint64_t>(b) != 0) ? 1ull : 0ull;  // sticky bit below the 11 guard bits
    r = scalbn(__ull2double_rn(top), 64 - lz);
  }
  return neg ? -r : r;
}
// Exact conversion of an integer-valued fp64 to int128.
__device__ __forceinline__ i128 f64int_to_i128(double h) {
  if (fabs(h) < 9007199254740992.0) return static_cast<i128>(static_cast<long long>(h));
  int e;
  const double m = frexp(h, &e);  // h = m 2^e, 0.5 <= |m| < 1, e > 53
  const long long mi = static_cast<long long>(scalbn(m, 53));
  return static_cast<i128>(mi) << (e - 53);
}
// Correctly rounded double-double of an exact int128: hi = RN(x), lo = RN(x - hi).
__device__ __forceinline__ dd i128_to_dd(i128 x) {
  dd r;
  r.hi = i128_to_f64(x);
  r.lo = i128_to_f64(x - f64int_to_i128(r.hi));
  return r;
}
// Integer nearest to an fp64 (RNE), exactly, as int128 (|x| < 2^126).
__device__ __forceinline__ i128 rint_to_i128(double x) { return f64int_to_i128(rint(x)); }

// ⌈log2 v⌉ for v > 0 from the exponent field (R2); 0 for v == 0.
__device__ __forceinline__ int ceil_log2_d(double v) {
  if (v == 0.0) return 0;
  int e;
  const double m = frexp(v, &e);
  return (m == 0.5) ? e - 1 : e;
}

// R5: k excess-128 base-256 digits of p, most significant first: p = Σ d_s 256^{k-s}, d_s ∈ [-128,127].
// w = p + Σ_{s=2..k} 128·256^{k-s}; d_s = byte(w) - 128 for s >= 2 (from the least significant),
// d_1 = w >> 8(k-1) (arithmetic shift = floor). Writes d[0..k-1].
__device__ __forceinline__ void excess_digits(i128 p, int k, int* d) {
  i128 off = 0;
  for (int s = 1; s < k; ++s) off = (off << 8) | 128;
  i128 w = p + off;
  for (int s = k - 1; s >= 1; --s) {
    d[s] = static_cast<int>(static_cast<uint32_t>(w) & 0xFFu) - 128;
    w >>= 8;
  }
  d[0] = static_cast<int>(static_cast<long long>(w));
}

}  // namespace ozr
