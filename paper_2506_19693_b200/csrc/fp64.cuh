// Exact modular arithmetic on the FP64 pipe for primes < 2^46 (used by the
// NTT and the basis conversion).  Residues are exact integers in doubles;
// t = Y*W - q*p with q = rint(Y*(W/p)), h = Y*W (rounded), l = fma(Y, W, -h)
// (the exact product error), t = fma(-q, p, h) + l: an exact integer with
// |t| <= 1.5p whenever |Y| < 2^51 and 0 <= W < p < 2^46.
#pragma once
#include <stdint.h>

namespace ckb_f64 {

constexpr double kRint = 6755399441055744.0;  // 1.5 * 2^52

__device__ __forceinline__ double u64_to_f64(uint64_t v) {  // exact for v < 2^52
  return __longlong_as_double((long long)(v | 0x4330000000000000ull)) - 4503599627370496.0;
}

__device__ __forceinline__ uint64_t f64_to_u64(double d) {  // exact for 0 <= d < 2^52
  return (uint64_t)__double_as_longlong(d + 4503599627370496.0) - 0x4330000000000000ull;
}

__device__ __forceinline__ double mulmod_f64(double Y, double W, double Wp, double p) {
  const double q = (Y * Wp + kRint) - kRint;
  const double h = Y * W;
  const double l = fma(Y, W, -h);
  return fma(-q, p, h) + l;
}

// v mod p into [-p/2, p/2] (exact)
__device__ __forceinline__ double center_f64(double v, double p, double pinv) {
  const double q = (v * pinv + kRint) - kRint;
  return fma(-q, p, v);
}

// v mod p into [0, p)
__device__ __forceinline__ double canon_f64(double v, double p, double pinv) {
  const double r = center_f64(v, p, pinv);
  return r < 0.0 ? r + p : r;
}

// v mod p into [0, p) as an integer (|v| < 2^51).  The remainder is formed on
// the 1.5 * 2^52 offset, kRint + (v - q p) — exact, the sum lies in
// (2^52, 2^53) — so it falls out of the bit pattern as a signed integer and
// the sign fix-up is integer work: 4 FP64-pipe instructions instead of the 7
// of f64_to_u64(canon_f64(v)) (the FP64 pipe is the binding one in the NTT).
__device__ __forceinline__ uint64_t canon_u64(double v, double p, double pinv) {
  const double q = (v * pinv + kRint) - kRint;
  const double rk = fma(-q, p, v + kRint);
  long long r = __double_as_longlong(rk) - __double_as_longlong(kRint);
  r += (r >> 63) & (long long)p;
  return (uint64_t)r;
}

}  // namespace ckb_f64
