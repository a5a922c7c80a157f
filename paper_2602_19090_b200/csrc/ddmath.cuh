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

// 2^k as an fp64 built from its bit pattern (exact; valid for -1022 <= k <= 1023).
__device__ __forceinline__ double pow2i(int k) {
  return __longlong_as_double(static_cast<long long>(1023 + k) << 52);
}
// x · 2^k, exact for normal results: one multiply in the common range, scalbn otherwise.
__device__ __forceinline__ double ldexp_fast(double x, int k) {
  if (k >= -1022 && k <= 1023) return x * pow2i(k);
  return scalbn(x, k);
}

// Correctly rounded (RNE) conversion of a signed 128-bit integer to fp64.
__device__ __forceinline__ double i128_to_f64(i128 x) {
  const bool neg = x < 0;
  const u128 a = neg ? static_cast<u128>(-x) : static_cast<u128>(x);
  const uint64_t hi = static_cast<uint64_t>(a >> 64);
  double r;
  if (hi == 0) {
    r = __ull2double_rn(static_cast<uint64_t>(a));
  } else {
    const int lz = __clzll(static_cast<long long>(hi));
    const u128 b = a << lz;  // leading one at bit 127
    uint64_t top = static_cast<uint64_t>(b >> 64);
    top |= (static_cast<uint64_t>(b) != 0) ? 1ull : 0ull;  // sticky bit below the 11 guard bits
    r = __ull2double_rn(top) * pow2i(64 - lz);
  }
  return neg ? -r : r;
}
// RN(L0·2^32 + L1) for |L0|, |L1| < 2^55 (two recombination limbs) without 128-bit arithmetic: with
// s = L0 + ⌊L1/2^32⌋ and b = L1 mod 2^32 the value is s·2^32 + b. For |s| < 2^47 both are exact doubles and
// one fma rounds once; otherwise the value has ≥ 80 bits, so its bits below 2^25 only act as a sticky bit:
// RN((s·2^7 + ⌊b/2^25⌋) | sticky)·2^25.
__device__ __forceinline__ double limbs2_rn(long long L0, long long L1) {
  const long long s = L0 + (L1 >> 32);
  const unsigned long long b = static_cast<unsigned long long>(L1) & 0xFFFFFFFFull;
  if (s > -(1LL << 47) && s < (1LL << 47)) return fma(static_cast<double>(s), 4294967296.0, static_cast<double>(b));
  long long t = s * 128 + static_cast<long long>(b >> 25);
  if (b & 0x1FFFFFFull) t |= 1;
  return __ll2double_rn(t) * 33554432.0;
}
// Exact conversion of an integer-valued fp64 to int128 (bit-level: mantissa << exponent).
__device__ __forceinline__ i128 f64int_to_i128(double h) {
  if (fabs(h) < 9007199254740992.0) return static_cast<i128>(__double2ll_rz(h));
  const long long bits = __double_as_longlong(h);
  const int ex = static_cast<int>((bits >> 52) & 0x7FF) - 1075;  // h = ±m 2^ex, m in [2^52, 2^53)
  const long long m = (bits & 0xFFFFFFFFFFFFFLL) | 0x10000000000000LL;
  const i128 v = static_cast<i128>(static_cast<u128>(m) << ex);
  return (bits < 0) ? -v : v;
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

// ⌈log2 v⌉ for v > 0 from the exponent field (R2); 0 for v == 0 (v normal).
__device__ __forceinline__ int ceil_log2_d(double v) {
  if (v == 0.0) return 0;
  const long long bits = __double_as_longlong(v);
  const int be = static_cast<int>((bits >> 52) & 0x7FF);
  if (be == 0) {  // subnormal: fall back
    int e;
    const double m = frexp(v, &e);
    return (m == 0.5) ? e - 1 : e;
  }
  const bool pow2 = (bits & 0xFFFFFFFFFFFFFLL) == 0;
  return be - 1023 + (pow2 ? 0 : 1);
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
