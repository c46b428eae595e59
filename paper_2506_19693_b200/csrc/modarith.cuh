// Word-size modular arithmetic for RNS-CKKS limbs (primes p < 2^62).
//
// Shared by the device kernels and by the host-side table builders so the
// same code can be unit-tested on the CPU against unsigned __int128.
//
//  * Shoup multiplication by a constant w (twiddles, CRT constants):
//      w' = floor(w * 2^64 / p);  q = hi(x * w');  r = x*w - q*p in [0, 2p)
//    valid for any 64-bit x, which is what the lazy Harvey butterflies need.
//  * Barrett multiplication of two canonical residues (Hadamard products,
//    key inner products): mu = floor(2^(2k) / p) with k = bitlen(p);
//    q3 = ((x >> (k-1)) * mu) >> (k+1) underestimates floor(x/p) by <= 2,
//    so r = x - q3*p lies in [0, 3p) and two conditional subtractions finish.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define CKB_HD __host__ __device__ __forceinline__
#else
#define CKB_HD inline
#endif

namespace ckb {

// Per-prime constants; laid out as 4 x u64 in the device modulus table.
struct Mod {
  uint64_t p;      // the prime
  uint64_t mu;     // floor(2^(2k) / p)
  uint64_t k;      // bit length of p
  uint64_t two_p;  // 2p (lazy-reduction bound)
};

CKB_HD uint64_t mulhi(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

CKB_HD uint64_t add_mod(uint64_t a, uint64_t b, uint64_t p) {
  uint64_t s = a + b;
  return s >= p ? s - p : s;
}

CKB_HD uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t p) {
  return a >= b ? a - b : a + p - b;
}

CKB_HD uint64_t neg_mod(uint64_t a, uint64_t p) { return a == 0 ? 0 : p - a; }

// Shoup: x * w mod p with precomputed ws = floor(w * 2^64 / p); result in [0, 2p).
CKB_HD uint64_t mul_shoup_lazy(uint64_t x, uint64_t w, uint64_t ws, uint64_t p) {
  uint64_t q = mulhi(x, ws);
  return x * w - q * p;
}

CKB_HD uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t ws, uint64_t p) {
  uint64_t r = mul_shoup_lazy(x, w, ws, p);
  return r >= p ? r - p : r;
}

// Barrett reduction of a 128-bit value (hi, lo) < 2^(2k) to [0, p).
CKB_HD uint64_t barrett_reduce128(uint64_t hi, uint64_t lo, const Mod& m) {
  const uint32_t k = (uint32_t)m.k;
  // q1 = x >> (k-1)  (< 2^(k+1) <= 2^63)
  uint64_t q1 = (lo >> (k - 1)) | (hi << (65 - k));
  // q3 = (q1 * mu) >> (k+1)
  uint64_t plo = q1 * m.mu;
  uint64_t phi = mulhi(q1, m.mu);
  uint64_t q3 = (plo >> (k + 1)) | (phi << (63 - k));
  uint64_t r = lo - q3 * m.p;
  if (r >= m.two_p) r -= m.two_p;
  if (r >= m.p) r -= m.p;
  return r;
}

// a * b mod p for canonical a, b.
CKB_HD uint64_t mul_mod(uint64_t a, uint64_t b, const Mod& m) {
  return barrett_reduce128(mulhi(a, b), a * b, m);
}

// x mod p for x < 16p (p < 2^60): four conditional subtractions.
CKB_HD uint64_t reduce_16p(uint64_t x, uint64_t p) {
  x = x >= 8 * p ? x - 8 * p : x;
  x = x >= 4 * p ? x - 4 * p : x;
  x = x >= 2 * p ? x - 2 * p : x;
  return x >= p ? x - p : x;
}

// (hi, lo) += a * b, 128-bit multiply-accumulate.
CKB_HD void mac128(uint64_t& hi, uint64_t& lo, uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\tmadc.hi.u64 %1, %2, %3, %1;"
      : "+l"(lo), "+l"(hi)
      : "l"(a), "l"(b));
#else
  unsigned __int128 acc = ((unsigned __int128)hi << 64) | lo;
  acc += (unsigned __int128)a * b;
  hi = (uint64_t)(acc >> 64);
  lo = (uint64_t)acc;
#endif
}

// x mod p for an arbitrary 64-bit x.
CKB_HD uint64_t reduce64(uint64_t x, const Mod& m) {
  if (x < m.p) return x;
  if (m.k >= 32) return barrett_reduce128(0, x, m);
  return x % m.p;
}

// (hi * 2^64 + lo) mod p for any 128-bit value, given r64 = 2^64 mod p and
// its Shoup companion.
CKB_HD uint64_t reduce128_any(uint64_t hi, uint64_t lo, uint64_t r64, uint64_t r64s,
                              const Mod& m);

// Centered residue of x (canonical mod q) reduced into prime m:
// value v = x if x <= q/2 else x - q  (reference: ring.py:341-342, keys.py:85-86),
// returned as v mod p in [0, p).
CKB_HD uint64_t centered_into(uint64_t x, uint64_t q, const Mod& m) {
  if (x > (q >> 1)) {
    uint64_t mag = reduce64(q - x, m);
    return mag == 0 ? 0 : m.p - mag;
  }
  return reduce64(x, m);
}

CKB_HD uint64_t reduce128_any(uint64_t hi, uint64_t lo, uint64_t r64, uint64_t r64s,
                              const Mod& m) {
  const uint64_t h = mul_shoup(hi, r64, r64s, m.p);
  return add_mod(h, reduce64(lo, m), m.p);
}

// Carry-free dot products.  An operand x < 2^61 is split as x = hi*2^30 + lo
// (lo < 2^30, hi < 2^31); the four partial sums of 32x32-bit products then
// grow by < 2^61 per term, so up to 8 terms accumulate in plain 64-bit words
// with one IMAD.WIDE.U32 each (the 128-bit mad.lo.cc/madc.hi pair costs ~16
// instructions per term).  fold() turns the partials into the exact 128-bit
// sum.  Packed form of a split constant: (hi << 32) | lo.
struct Split30 {
  uint32_t lo, hi;
};

CKB_HD Split30 split30(uint64_t x) {
  return Split30{(uint32_t)(x & 0x3FFFFFFFull), (uint32_t)(x >> 30)};
}

CKB_HD uint64_t pack30(uint64_t x) { return ((x >> 30) << 32) | (x & 0x3FFFFFFFull); }

CKB_HD Split30 unpack30(uint64_t w) { return Split30{(uint32_t)w, (uint32_t)(w >> 32)}; }

struct Acc4 {
  uint64_t s00 = 0, s01 = 0, s10 = 0, s11 = 0;
  CKB_HD void mac(Split30 a, Split30 b) {
#if defined(__CUDA_ARCH__)
    // one IMAD.WIDE.U32 each (plain C++ lets the compiler widen a factor)
    asm("mad.wide.u32 %0, %4, %6, %0;\n\t"
        "mad.wide.u32 %1, %4, %7, %1;\n\t"
        "mad.wide.u32 %2, %5, %6, %2;\n\t"
        "mad.wide.u32 %3, %5, %7, %3;"
        : "+l"(s00), "+l"(s01), "+l"(s10), "+l"(s11)
        : "r"(a.lo), "r"(a.hi), "r"(b.lo), "r"(b.hi));
#else
    s00 += (uint64_t)a.lo * b.lo;
    s01 += (uint64_t)a.lo * b.hi;
    s10 += (uint64_t)a.hi * b.lo;
    s11 += (uint64_t)a.hi * b.hi;
#endif
  }
  // (hi:lo) += s00 + (s01 + s10) * 2^30 + s11 * 2^60
  CKB_HD void fold_into(uint64_t& hi, uint64_t& lo) const {
    const uint64_t mid = s01 + s10;
    const uint64_t mid_c = mid < s01 ? 1ull : 0ull;  // carry of the 65-bit mid
    // mid * 2^30 = (mid_c:mid) << 30
    const uint64_t m_lo = mid << 30;
    const uint64_t m_hi = (mid >> 34) | (mid_c << 30);
    const uint64_t t_lo = s11 << 60;
    const uint64_t t_hi = s11 >> 4;
    uint64_t l = lo + s00;
    uint64_t h = hi + (l < s00 ? 1ull : 0ull);
    l += m_lo;
    h += m_hi + (l < m_lo ? 1ull : 0ull);
    l += t_lo;
    h += t_hi + (l < t_lo ? 1ull : 0ull);
    lo = l;
    hi = h;
  }
};

// Same for primes of at least 32 bits, branch-free: hi*2^64 via Shoup, lo via
// Barrett (lo < 2^64 <= 2^(2k)).
CKB_HD uint64_t reduce128_big(uint64_t hi, uint64_t lo, uint64_t r64, uint64_t r64s,
                              const Mod& m) {
  const uint64_t h = mul_shoup_lazy(hi, r64, r64s, m.p);     // [0, 2p)
  const uint64_t l = barrett_reduce128(0, lo, m);            // [0, p)
  uint64_t s = h + l;                                        // [0, 3p)
  s = s >= m.two_p ? s - m.two_p : s;
  return s >= m.p ? s - m.p : s;
}

// ---- host-only helpers for table construction -----------------------------
inline uint64_t shoup_of(uint64_t w, uint64_t p) {
  return (uint64_t)(((unsigned __int128)w << 64) / p);
}
inline uint64_t mul_mod_host(uint64_t a, uint64_t b, uint64_t p) {
  return (uint64_t)(((unsigned __int128)a * b) % p);
}
inline uint64_t pow_mod_host(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  b %= p;
  while (e) {
    if (e & 1) r = mul_mod_host(r, b, p);
    b = mul_mod_host(b, b, p);
    e >>= 1;
  }
  return r;
}
inline uint64_t inv_mod_host(uint64_t a, uint64_t p) {  // p prime
  return pow_mod_host(a % p, p - 2, p);
}
inline uint32_t bitlen(uint64_t x) {
  uint32_t k = 0;
  while (x) { ++k; x >>= 1; }
  return k;
}
inline Mod make_mod(uint64_t p) {
  Mod m;
  m.p = p;
  m.k = bitlen(p);
  m.mu = (uint64_t)(((unsigned __int128)1 << (2 * m.k)) / p);
  m.two_p = 2 * p;
  return m;
}

}  // namespace ckb
