// Host-side check of the device modular arithmetic (paper_2506_19693_b200/csrc/modarith.cuh)
// against unsigned __int128 on random operands; compiled and run by tests/test_native_host.py.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "../../paper_2506_19693_b200/csrc/modarith.cuh"

using namespace ckb;

static bool is_prime(uint64_t n) {
  if (n < 2) return false;
  for (uint64_t p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    if (n % p == 0) return n == p;
  }
  uint64_t d = n - 1; int s = 0;
  while (!(d & 1)) { d >>= 1; ++s; }
  for (uint64_t a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    uint64_t x = pow_mod_host(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; ++r) { x = mul_mod_host(x, x, n); if (x == n - 1) { comp = false; break; } }
    if (comp) return false;
  }
  return true;
}

int main() {
  std::mt19937_64 rng(12345);
  int fails = 0;
  for (int bits : {20, 28, 30, 31, 32, 33, 40, 41, 50, 59, 60, 61}) {
    // a few primes = 1 mod 2^17 just below 2^bits (or any prime for small bits)
    uint64_t step = bits > 20 ? (1ull << 17) : 2;
    uint64_t p = ((1ull << bits) - 1) / step * step + 1;
    int found = 0;
    while (found < 3 && p > step) {
      if (p < (1ull << bits) && is_prime(p)) {
        ++found;
        Mod m = make_mod(p);
        for (int t = 0; t < 200000; ++t) {
          uint64_t a = rng() % p, b = rng() % p, x = rng();
          if (t < 4) { a = p - 1 - t; b = p - 1; }
          uint64_t want = mul_mod_host(a, b, p);
          if (mul_mod(a, b, m) != want) { ++fails; printf("mul_mod p=%llu a=%llu b=%llu\n", (unsigned long long)p, (unsigned long long)a, (unsigned long long)b); }
          uint64_t ws = shoup_of(b, p);
          if (mul_shoup(x, b, ws, p) != (uint64_t)(((unsigned __int128)x * b) % p)) ++fails;
          if (mul_shoup_lazy(x, b, ws, p) >= 2 * p) ++fails;
          if (reduce64(x, m) != x % p) ++fails;
          uint64_t q = 1000003ull + 2 * (rng() % (1ull << 58));
          uint64_t xr = rng() % q;
          __int128 c = (xr > q / 2) ? (__int128)xr - (__int128)q : (__int128)xr;
          __int128 cm = c % (__int128)p; if (cm < 0) cm += p;
          if (centered_into(xr, q, m) != (uint64_t)cm) ++fails;
          if (bits <= 60) {
            uint64_t y = rng() % (16 * p);
            if (reduce_16p(y, p) != y % p) ++fails;
          }
          {
            uint64_t hi = 0, lo = 0;
            unsigned __int128 want128 = 0;
            for (int k = 0; k < 5; ++k) {
              uint64_t u = rng() % p, v = rng() % p;
              mac128(hi, lo, u, v);
              want128 += (unsigned __int128)u * v;
            }
            uint64_t r64 = (uint64_t)(((unsigned __int128)1 << 64) % p);
            if (reduce128_any(hi, lo, r64, shoup_of(r64, p), m) != (uint64_t)(want128 % p)) ++fails;
          }
        }
      }
      p -= step;
    }
  }
  printf("fails=%d\n", fails);
  return fails ? 1 : 0;
}
