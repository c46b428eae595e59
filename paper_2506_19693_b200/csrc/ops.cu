// Limb arithmetic, key switching, rescale, automorphism and conversion kernels
// (sm_100a) replacing ciphermlp/ckks/{ring,keys,backend}.py numpy routines.
#include "common.cuh"
#include "fp64.cuh"
#include <cstring>

using namespace ckb_internal;
using ckb::Mod;

namespace {

// ===========================================================================
// Element-wise limb arithmetic
// ===========================================================================

// Limb-wise arithmetic, two coefficients per thread (16-byte accesses); b
// (and c) broadcast with a period of brows rows when brows > 0.  The row
// index is a 32-bit quantity, so the limb and broadcast-row lookups are
// 32-bit modulos once per coefficient pair.
template <int OP>
__device__ __forceinline__ uint64_t ew_op(uint64_t x, uint64_t y, uint64_t z, const Mod& m) {
  if constexpr (OP == 0) return ckb::add_mod(x, y, m.p);
  if constexpr (OP == 1) return ckb::sub_mod(x, y, m.p);
  if constexpr (OP == 2) return ckb::mul_mod(x, y, m);
  if constexpr (OP == 3) return ckb::neg_mod(x, m.p);
  return ckb::add_mod(ckb::mul_mod(x, y, m), z, m.p);
}

template <int OP>
__global__ void __launch_bounds__(256) k_elementwise(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
    const uint64_t* __restrict__ c, size_t pairs, unsigned brows, int log_n, unsigned limbs,
    RingDev R, LimbMap lm) {
  const int lh = log_n - 1;
  const size_t hmask = ((size_t)1 << lh) - 1;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < pairs;
       t += (size_t)gridDim.x * blockDim.x) {
    const unsigned row = (unsigned)(t >> lh);
    const size_t n = (t & hmask) * 2;
    const Mod m = load_mod(R, lm.p[row % limbs]);
    const size_t i = ((size_t)row << log_n) + n;
    const size_t ib = brows ? ((size_t)(row % brows) << log_n) + n : i;
    const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(a + i);
    ulonglong2 y = make_ulonglong2(0, 0), z = make_ulonglong2(0, 0);
    if constexpr (OP != 3) y = *reinterpret_cast<const ulonglong2*>(b + ib);
    if constexpr (OP == 4) z = *reinterpret_cast<const ulonglong2*>(c + ib);
    *reinterpret_cast<ulonglong2*>(out + i) =
        make_ulonglong2(ew_op<OP>(x.x, y.x, z.x, m), ew_op<OP>(x.y, y.y, z.y, m));
  }
}

// out = sum_t x_t (.) pt_t over the coefficient-wise products, one reduction:
// the ciphertext operand of term t is x0 (idx -1) or stack + idx[t]*xstride,
// each [items][comps*limbs][N]; its plaintext is pts + t*ptstride, [limbs][N]
// broadcast over items and components.  128-bit lazy sums (T <= 64 terms of
// products < 2^124).  Replaces the mul_pt + add_ct chain of a BSGS row.
struct TermIdx {
  int16_t p[64];
};

__global__ void __launch_bounds__(256) k_pt_mac(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ x0,
    const uint64_t* __restrict__ stack, size_t xstride, TermIdx ti,
    const uint64_t* __restrict__ pts, size_t ptstride, int T, size_t pairs, int log_n,
    unsigned limbs, RingDev R, LimbMap lm) {
  const int lh = log_n - 1;
  const size_t hmask = ((size_t)1 << lh) - 1;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < pairs;
       t += (size_t)gridDim.x * blockDim.x) {
    const unsigned row = (unsigned)(t >> lh);
    const size_t n = (t & hmask) * 2;
    const unsigned l = row % limbs;
    const size_t i = ((size_t)row << log_n) + n;
    const size_t ip = ((size_t)l << log_n) + n;
    uint64_t h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll 4
    for (int k = 0; k < T; ++k) {
      const uint64_t* xs = ti.p[k] < 0 ? x0 : stack + (size_t)ti.p[k] * xstride;
      const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(xs + i);
      const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(pts + k * ptstride + ip));
      ckb::mac128(h0, l0, x.x, w.x);
      ckb::mac128(h1, l1, x.y, w.y);
    }
    const uint64_t* mm = R.mods + (size_t)lm.p[l] * kModStride;
    const Mod m{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
    const uint64_t r64 = __ldg(mm + 8), r64s = __ldg(mm + 9);
    *reinterpret_cast<ulonglong2*>(out + i) =
        make_ulonglong2(ckb::reduce128_any(h0, l0, r64, r64s, m),
                        ckb::reduce128_any(h1, l1, r64, r64s, m));
  }
}

struct ScalarTab {
  uint64_t v[kMaxLimbs];
  uint64_t s[kMaxLimbs];
};

__global__ void k_scalar_mul(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                             size_t total, int log_n, int limbs, RingDev R, LimbMap lm,
                             ScalarTab sc) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i >> log_n) % limbs;
    const uint64_t p = __ldg(R.mods + (size_t)lm.p[l] * kModStride);
    out[i] = ckb::mul_shoup(a[i], sc.v[l], sc.s[l], p);
  }
}

// a * b mod p on the FP64 pipe for p < 2^46 (canonical a, b): q = rint(a (b/p))
// is within 1 of a b / p (relative error < 2^-51), so t = (a b - q p) is
// formed exactly from h = fl(a b), l = a b - h and lies in (-1.5p, 1.5p).
__device__ __forceinline__ double mulmod2_f64(double a, double b, double p, double pinv) {
  return ckb_f64::mulmod_f64(a, b, b * pinv, p);
}

// Two coefficients per thread with 16-byte loads and stores (N >= 2).  Rows
// whose prime is < 2^46 (warp-uniform: a warp covers 64 coefficients of one
// row) multiply on the FP64 pipe, the others with Barrett products.
__global__ void k_tensor2(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                          const uint64_t* __restrict__ b, size_t total, int log_n, int limbs,
                          RingDev R, LimbMap lm) {
  const size_t N = (size_t)1 << log_n;
  const size_t poly = (size_t)limbs * N;
  for (size_t i = 2 * (blockIdx.x * (size_t)blockDim.x + threadIdx.x); i < total;
       i += 2 * (size_t)gridDim.x * blockDim.x) {
    const unsigned row = (unsigned)(i >> log_n);
    const unsigned bi = row / (unsigned)limbs;
    const int l = (int)(row - bi * (unsigned)limbs);
    const size_t off = i - (size_t)bi * poly;
    const Mod m = load_mod(R, lm.p[l]);
    const uint64_t* pa = a + (size_t)bi * 2 * poly + off;
    const uint64_t* pb = b + (size_t)bi * 2 * poly + off;
    const ulonglong2 a0 = __ldcs(reinterpret_cast<const ulonglong2*>(pa));
    const ulonglong2 a1 = __ldcs(reinterpret_cast<const ulonglong2*>(pa + poly));
    const ulonglong2 b0 = __ldcs(reinterpret_cast<const ulonglong2*>(pb));
    const ulonglong2 b1 = __ldcs(reinterpret_cast<const ulonglong2*>(pb + poly));
    uint64_t* po = out + (size_t)bi * 3 * poly + off;
    ulonglong2 d0, d1, d2;
#ifndef CKB_TENSOR_NO_F64
    if ((m.p >> 46) == 0) {
      using namespace ckb_f64;
      const double p = (double)m.p, pinv = 1.0 / p;
      const double x0[2] = {u64_to_f64(a0.x), u64_to_f64(a0.y)};
      const double x1[2] = {u64_to_f64(a1.x), u64_to_f64(a1.y)};
      const double y0[2] = {u64_to_f64(b0.x), u64_to_f64(b0.y)};
      const double y1[2] = {u64_to_f64(b1.x), u64_to_f64(b1.y)};
      uint64_t r0[2], r1[2], r2[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        r0[c] = canon_u64(mulmod2_f64(x0[c], y0[c], p, pinv), p, pinv);
        r1[c] = canon_u64(mulmod2_f64(x0[c], y1[c], p, pinv) +
                                         mulmod2_f64(x1[c], y0[c], p, pinv), p, pinv);
        r2[c] = canon_u64(mulmod2_f64(x1[c], y1[c], p, pinv), p, pinv);
      }
      d0 = make_ulonglong2(r0[0], r0[1]);
      d1 = make_ulonglong2(r1[0], r1[1]);
      d2 = make_ulonglong2(r2[0], r2[1]);
    } else
#endif
    {
      d0.x = ckb::mul_mod(a0.x, b0.x, m);
      d0.y = ckb::mul_mod(a0.y, b0.y, m);
      d1.x = ckb::add_mod(ckb::mul_mod(a0.x, b1.x, m), ckb::mul_mod(a1.x, b0.x, m), m.p);
      d1.y = ckb::add_mod(ckb::mul_mod(a0.y, b1.y, m), ckb::mul_mod(a1.y, b0.y, m), m.p);
      d2.x = ckb::mul_mod(a1.x, b1.x, m);
      d2.y = ckb::mul_mod(a1.y, b1.y, m);
    }
    *reinterpret_cast<ulonglong2*>(po) = d0;
    *reinterpret_cast<ulonglong2*>(po + poly) = d1;
    *reinterpret_cast<ulonglong2*>(po + 2 * poly) = d2;
  }
}

__global__ void k_tensor(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                         const uint64_t* __restrict__ b, size_t total, int log_n, int limbs,
                         RingDev R, LimbMap lm) {
  const size_t N = (size_t)1 << log_n;
  const size_t poly = (size_t)limbs * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t bi = i / poly, off = i - bi * poly;
    const int l = (int)(off >> log_n);
    const Mod m = load_mod(R, lm.p[l]);
    const uint64_t* pa = a + bi * 2 * poly + off;
    const uint64_t* pb = b + bi * 2 * poly + off;
    const uint64_t a0 = pa[0], a1 = pa[poly], b0 = pb[0], b1 = pb[poly];
    uint64_t* po = out + bi * 3 * poly + off;
    po[0] = ckb::mul_mod(a0, b0, m);
    po[poly] = ckb::add_mod(ckb::mul_mod(a0, b1, m), ckb::mul_mod(a1, b0, m), m.p);
    po[2 * poly] = ckb::mul_mod(a1, b1, m);
  }
}

// ===========================================================================
// Key switching: ModUp and the key inner product
// ===========================================================================

// One thread per (batch, digit, coefficient); writes the digit's value in
// every extended limb (coalesced across coefficients).
// Digit j of item b covers limbs [j*alpha, j*alpha + cnt).  With skip_own the
// digit's own limbs are not written (their NTT is already the input's NTT, read
// directly by k_ks_inner) and each digit has ext - alpha output rows, ordered
// as the ext basis without the own limbs.
__device__ __forceinline__ int digit_row(int e, int first, int cnt, int skip_own) {
  return skip_own ? (e < first ? e : e - cnt) : e;
}

// One CTA = one digit (blockIdx.y) over a range of (item, coefficient pair);
// the digit's conversion constants and every ext limb's modulus constants are
// staged in shared memory.  alpha > 1: y_i = [x_i qhat_i^-1]_{q_i}, then per
// ext limb a 128-bit lazy sum of y_i [qhat_i]_{p_e} and one reduction.  Two
// coefficients per thread (16-byte loads and stores).
struct ModSm {
  uint64_t p, mu, k, two_p, r64, r64s;
};

template <int AMAX>
__global__ void __launch_bounds__(256) k_modup(uint64_t* __restrict__ out,
                                                const uint64_t* __restrict__ in, size_t in_bstride,
                                                int batch, int limbs, int ext, int alpha,
                                                int item_rows, int out_rows, int skip_own,
                                                int log_n, RingDev R, LimbMap lm, LimbMap em,
                                                const uint64_t* __restrict__ bconv) {
  extern __shared__ uint64_t sm[];
  ModSm* mods = reinterpret_cast<ModSm*>(sm);
  uint64_t* ctab = sm + 6 * ext;
  const size_t N = (size_t)1 << log_n;
  const int j = blockIdx.y;
  const int first = j * alpha;
  const int cnt = min(alpha, limbs - first);
  const size_t stride_i = 2 + 2 * (size_t)ext;
  for (int e = threadIdx.x; e < ext; e += blockDim.x) {
    const uint64_t* mm = R.mods + (size_t)em.p[e] * kModStride;
    mods[e] = ModSm{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3), __ldg(mm + 8),
                    __ldg(mm + 9)};
  }
  if (AMAX > 1) {  // [qhat_i]_{p_e} staged in split form (pack30) for the carry-free sum
    const uint64_t* tab = bconv + (size_t)j * alpha * stride_i;
    for (int q = threadIdx.x; q < cnt * (int)stride_i; q += blockDim.x) {
      const int c = q % (int)stride_i;
      const uint64_t v = __ldg(tab + q);
      ctab[q] = (c >= 2 && !(c & 1)) ? ckb::pack30(v) : v;
    }
  }
  __syncthreads();
  const size_t half = N >> 1;
  const size_t total = (size_t)batch * half;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = (t & (half - 1)) * 2;
    const size_t bi = t / half;
    const uint64_t* src = in + bi * in_bstride + n;
    uint64_t* dst = out + (bi * (size_t)item_rows + (size_t)j * out_rows) * N + n;
    if (AMAX == 1) {
      const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(src + (size_t)first * N);
      const uint64_t q = __ldg(R.mods + (size_t)lm.p[first] * kModStride);
      for (int e = 0; e < ext; ++e) {
        if (e == first) {
          if (!skip_own) *reinterpret_cast<ulonglong2*>(dst + (size_t)e * N) = x;
          continue;
        }
        const ModSm ms = mods[e];
        const Mod m{ms.p, ms.mu, ms.k, ms.two_p};
        ulonglong2 o;
        o.x = ckb::centered_into(x.x, q, m);
        o.y = ckb::centered_into(x.y, q, m);
        *reinterpret_cast<ulonglong2*>(dst + (size_t)digit_row(e, first, 1, skip_own) * N) = o;
      }
    } else {
      ckb::Split30 y0[AMAX], y1[AMAX];
#pragma unroll
      for (int i = 0; i < AMAX; ++i) {
        if (i < cnt) {
          const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(src + (size_t)(first + i) * N);
          const uint64_t q = __ldg(R.mods + (size_t)lm.p[first + i] * kModStride);
          y0[i] = ckb::split30(ckb::mul_shoup(x.x, ctab[i * stride_i], ctab[i * stride_i + 1], q));
          y1[i] = ckb::split30(ckb::mul_shoup(x.y, ctab[i * stride_i], ctab[i * stride_i + 1], q));
        } else {
          y0[i] = y1[i] = ckb::Split30{0, 0};  // short last digit: zero terms
        }
      }
      for (int e = 0; e < ext; ++e) {
        if (e >= first && e < first + cnt) {
          if (!skip_own)
            *reinterpret_cast<ulonglong2*>(dst + (size_t)e * N) =
                *reinterpret_cast<const ulonglong2*>(src + (size_t)e * N);
          continue;
        }
        uint64_t h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll
        for (int i0 = 0; i0 < AMAX; i0 += 8) {  // <= 8 terms per 64-bit partial
          ckb::Acc4 a0, a1;
#pragma unroll
          for (int i = i0; i < (i0 + 8 < AMAX ? i0 + 8 : AMAX); ++i) {
            const ckb::Split30 c = ckb::unpack30((i < cnt) ? ctab[i * stride_i + 2 + 2 * e] : 0);
            a0.mac(y0[i], c);
            a1.mac(y1[i], c);
          }
          a0.fold_into(h0, l0);
          a1.fold_into(h1, l1);
        }
        const ModSm ms = mods[e];
        const Mod m{ms.p, ms.mu, ms.k, ms.two_p};
        ulonglong2 o;
        if (ms.k >= 32) {  // warp-uniform
          o.x = ckb::reduce128_big(h0, l0, ms.r64, ms.r64s, m);
          o.y = ckb::reduce128_big(h1, l1, ms.r64, ms.r64s, m);
        } else {
          o.x = ckb::reduce128_any(h0, l0, ms.r64, ms.r64s, m);
          o.y = ckb::reduce128_any(h1, l1, ms.r64, ms.r64s, m);
        }
        *reinterpret_cast<ulonglong2*>(dst + (size_t)digit_row(e, first, cnt, skip_own) * N) = o;
      }
    }
  }
}

// ModUp on both arithmetic pipes.  For a digit whose input primes are all
// < 2^46 (y_i exact in a double) the outputs on primes < 2^46 are summed on the
// FP64 pipe, sum_i mulmod_f64(y_i, c_ie) (|sum| < 1.5 * AMAX * p < 2^51, exact),
// and the other outputs (60-bit special primes) on the integer pipe as in
// k_modup; warps at different outputs keep both pipes busy.  One coefficient
// per thread (register budget).  Smem: ModSm per ext limb, the integer table in
// pack30 form, then per (i, e) {double(c), double(c)/p_e} and per e 1/p_e.
template <int AMAX, bool COMPACT>
__global__ void __launch_bounds__(256) k_modup_mixed(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ in, size_t in_bstride, int batch,
    int limbs, int ext, int alpha, int n_digits, int out_rows, int skip_own, int log_n,
    int item_rows,
    RingDev R, LimbMap lm, LimbMap em, const uint64_t* __restrict__ bconv) {
  extern __shared__ uint64_t sm[];
  ModSm* mods = reinterpret_cast<ModSm*>(sm);
  uint64_t* ctab = sm + 6 * ext;
  const size_t stride_i = 2 + 2 * (size_t)ext;
  double2* cd = reinterpret_cast<double2*>(ctab + (size_t)alpha * stride_i);
  double* pinv = reinterpret_cast<double*>(cd + (size_t)alpha * ext);
  __shared__ int f64in;
  const size_t N = (size_t)1 << log_n;
  const int j = blockIdx.y;
  const int first = j * alpha;
  const int cnt = min(alpha, limbs - first);
  for (int e = threadIdx.x; e < ext; e += blockDim.x) {
    const uint64_t* mm = R.mods + (size_t)em.p[e] * kModStride;
    const uint64_t pe = __ldg(mm);
    mods[e] = ModSm{pe, __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3), __ldg(mm + 8),
                    __ldg(mm + 9)};
    pinv[e] = 1.0 / (double)pe;
  }
  const uint64_t* tab = bconv + (size_t)j * alpha * stride_i;
  for (int q = threadIdx.x; q < cnt * (int)stride_i; q += blockDim.x) {
    const int c = q % (int)stride_i;
    const uint64_t v = __ldg(tab + q);
    ctab[q] = (c >= 2 && !(c & 1)) ? ckb::pack30(v) : v;
  }
  for (int q = threadIdx.x; q < cnt * ext; q += blockDim.x) {
    const int i = q / ext, e = q % ext;
    const uint64_t c = __ldg(tab + (size_t)i * stride_i + 2 + 2 * e);
    const double pe = (double)__ldg(R.mods + (size_t)em.p[e] * kModStride);
    cd[q] = make_double2((double)c, (double)c / pe);
  }
  if (threadIdx.x == 0) {
    int ok = 1;
    for (int i = 0; i < cnt; ++i)
      ok &= (__ldg(R.mods + (size_t)lm.p[first + i] * kModStride) >> 46) == 0;
    f64in = ok;
  }
  __syncthreads();
  const bool fin = f64in;
  const size_t total = (size_t)batch * N;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = t & (N - 1);
    const size_t bi = t >> log_n;
    const uint64_t* src = in + bi * in_bstride + n;
    // uniform digits (every digit item_rows / n_digits rows): the index form the
    // kernel was tuned with; compact layout of a short last digit otherwise
    uint64_t* dst = COMPACT ? out + (bi * (size_t)item_rows + (size_t)j * out_rows) * N + n
                            : out + (bi * n_digits + j) * (size_t)out_rows * N + n;
    uint64_t y[AMAX];
    double yd[AMAX];
#pragma unroll
    for (int i = 0; i < AMAX; ++i) {
      if (i < cnt) {
        const uint64_t q = __ldg(R.mods + (size_t)lm.p[first + i] * kModStride);
        y[i] = ckb::mul_shoup(src[(size_t)(first + i) * N], ctab[i * stride_i],
                              ctab[i * stride_i + 1], q);
      } else {
        y[i] = 0;
      }
      yd[i] = ckb_f64::u64_to_f64(y[i]);  // only used when fin (then y < 2^46)
    }
    for (int e = 0; e < ext; ++e) {
      if (e >= first && e < first + cnt) {
        if (!skip_own) dst[(size_t)e * N] = src[(size_t)e * N];
        continue;
      }
      const ModSm ms = mods[e];
      uint64_t o;
      if (fin && (ms.p >> 46) == 0) {  // warp-uniform: FP64 pipe
        const double pd = (double)ms.p;
        double acc[2] = {0.0, 0.0};  // two independent add chains
#pragma unroll
        for (int i = 0; i < AMAX; ++i)
          if (i < cnt) {
            const double2 c = cd[i * ext + e];
            acc[i & 1] += ckb_f64::mulmod_f64(yd[i], c.x, c.y, pd);
          }
        o = ckb_f64::canon_u64(acc[0] + acc[1], pd, pinv[e]);
      } else {  // integer pipe (Acc4 carry-free sums, one reduction)
        uint64_t h = 0, l = 0;
#pragma unroll
        for (int i0 = 0; i0 < AMAX; i0 += 8) {
          ckb::Acc4 a;
#pragma unroll
          for (int i = i0; i < (i0 + 8 < AMAX ? i0 + 8 : AMAX); ++i)
            if (i < cnt) a.mac(ckb::split30(y[i]), ckb::unpack30(ctab[i * stride_i + 2 + 2 * e]));
          a.fold_into(h, l);
        }
        const Mod m{ms.p, ms.mu, ms.k, ms.two_p};
        o = ms.k >= 32 ? ckb::reduce128_big(h, l, ms.r64, ms.r64s, m)
                       : ckb::reduce128_any(h, l, ms.r64, ms.r64s, m);
      }
      dst[(size_t)digit_row(e, first, cnt, skip_own) * N] = o;
    }
  }
}

// ModUp v2 (alpha > 1): the digit's outputs are split once per CTA into an
// FP64 list (output prime < 2^46 and every digit prime < 2^46: y_i exact in a
// double, sum_i mulmod_f64 on the FP64 pipe) and an integer list (Acc4
// carry-free sums + one reduction on the integer pipes), so the per-output loops
// carry no class branches, and each thread converts TWO coefficients (16-byte
// loads and stores; the constants loaded from shared memory serve both).
// y_i is kept in doubles: the exact value when the digit is FP64-class, else
// the bit pattern of the u64 (the integer loop reads it back either way).
// Smem: [nf][AMAX] double2 {c, c/p} | [nf] double2 {p, 1/p} | [ni][AMAX] pack30(c)
//       | [ni] ModSm | [nf + ni] int row index | [AMAX] {qinv, shoup, q}.
#ifndef CKB_MODUP_MINB
#define CKB_MODUP_MINB 2
#endif
template <int AMAX>
__global__ void __launch_bounds__(256, CKB_MODUP_MINB) k_modup_v2(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ in, size_t in_bstride, int batch,
    int limbs, int ext, int alpha, int out_rows, int item_rows, int skip_own, int log_n,
    RingDev R, LimbMap lm, LimbMap em, const uint64_t* __restrict__ bconv) {
  extern __shared__ __align__(16) uint64_t sm[];
  __shared__ int s_nf, s_ni, s_fin;
  const size_t N = (size_t)1 << log_n;
  const int j = blockIdx.y;
  const int first = j * alpha;
  const int cnt = min(alpha, limbs - first);
  const size_t stride_i = 2 + 2 * (size_t)ext;
  const uint64_t* tab = bconv + (size_t)j * alpha * stride_i;
  double2* fc = reinterpret_cast<double2*>(sm);
  double2* fpp = fc + (size_t)ext * AMAX;
  uint64_t* ic = reinterpret_cast<uint64_t*>(fpp + ext);
  ModSm* ims = reinterpret_cast<ModSm*>(ic + (size_t)ext * AMAX);
  int* rowi = reinterpret_cast<int*>(ims + ext);       // [ext]: f rows then i rows
  uint64_t* qc = reinterpret_cast<uint64_t*>(rowi + 2 * ext + 2);
  if (threadIdx.x == 0) {
    int fin = 1;
    for (int i = 0; i < cnt; ++i)
      fin &= (__ldg(R.mods + (size_t)lm.p[first + i] * kModStride) >> 46) == 0;
    int nf = 0, ni = 0;
    for (int e = 0; e < ext; ++e) {
      if (e >= first && e < first + cnt) continue;
      const bool f = fin && (__ldg(R.mods + (size_t)em.p[e] * kModStride) >> 46) == 0;
      const int row = digit_row(e, first, cnt, skip_own);
      if (f) rowi[nf++] = (e << 16) | row;
      else rowi[ext + ni++] = (e << 16) | row;
    }
    s_nf = nf;
    s_ni = ni;
    s_fin = fin;
  }
  __syncthreads();
  const int nf = s_nf, ni = s_ni;
  const bool fin = s_fin;
  for (int q = threadIdx.x; q < nf * AMAX; q += blockDim.x) {
    const int a = q / AMAX, i = q % AMAX;
    const int e = rowi[a] >> 16;
    const double pe = (double)__ldg(R.mods + (size_t)em.p[e] * kModStride);
    const double c = i < cnt ? (double)__ldg(tab + (size_t)i * stride_i + 2 + 2 * e) : 0.0;
    fc[q] = make_double2(c, c / pe);
  }
  for (int a = threadIdx.x; a < nf; a += blockDim.x) {
    const double pe = (double)__ldg(R.mods + (size_t)em.p[rowi[a] >> 16] * kModStride);
    fpp[a] = make_double2(pe, 1.0 / pe);
  }
  for (int q = threadIdx.x; q < ni * AMAX; q += blockDim.x) {
    const int b = q / AMAX, i = q % AMAX;
    const int e = rowi[ext + b] >> 16;
    ic[q] = i < cnt ? ckb::pack30(__ldg(tab + (size_t)i * stride_i + 2 + 2 * e)) : 0;
  }
  for (int b = threadIdx.x; b < ni; b += blockDim.x) {
    const uint64_t* mm = R.mods + (size_t)em.p[rowi[ext + b] >> 16] * kModStride;
    ims[b] = ModSm{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3), __ldg(mm + 8),
                   __ldg(mm + 9)};
  }
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    qc[3 * i] = __ldg(tab + (size_t)i * stride_i);
    qc[3 * i + 1] = __ldg(tab + (size_t)i * stride_i + 1);
    qc[3 * i + 2] = __ldg(R.mods + (size_t)lm.p[first + i] * kModStride);
  }
  __syncthreads();
  const size_t half = N >> 1;
  const size_t total = (size_t)batch * half;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = (t & (half - 1)) * 2;
    const size_t bi = t / half;
    const uint64_t* src = in + bi * in_bstride + n;
    uint64_t* dst = out + (bi * (size_t)item_rows + (size_t)j * out_rows) * N + n;
    double y0[AMAX], y1[AMAX];
#pragma unroll
    for (int i = 0; i < AMAX; ++i) {
      if (i < cnt) {
        const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(src + (size_t)(first + i) * N));
        const uint64_t w = qc[3 * i], ws = qc[3 * i + 1], q = qc[3 * i + 2];
        const uint64_t a = ckb::mul_shoup(x.x, w, ws, q), b = ckb::mul_shoup(x.y, w, ws, q);
        y0[i] = fin ? ckb_f64::u64_to_f64(a) : __longlong_as_double((long long)a);
        y1[i] = fin ? ckb_f64::u64_to_f64(b) : __longlong_as_double((long long)b);
        if (!skip_own)
          *reinterpret_cast<ulonglong2*>(dst + (size_t)(first + i) * N) = x;
      } else {
        y0[i] = y1[i] = 0.0;  // short last digit: zero terms (0.0 has bit pattern 0)
      }
    }
    for (int a = 0; a < nf; ++a) {  // FP64 pipe
      const double2 pp = fpp[a];
      const double2* cr = fc + (size_t)a * AMAX;
      double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
#pragma unroll
      for (int i = 0; i < AMAX; i += 2) {
        const double2 c = cr[i];
        s00 += ckb_f64::mulmod_f64(y0[i], c.x, c.y, pp.x);
        s10 += ckb_f64::mulmod_f64(y1[i], c.x, c.y, pp.x);
        if (i + 1 < AMAX) {
          const double2 d = cr[i + 1];
          s01 += ckb_f64::mulmod_f64(y0[i + 1], d.x, d.y, pp.x);
          s11 += ckb_f64::mulmod_f64(y1[i + 1], d.x, d.y, pp.x);
        }
      }
      ulonglong2 o;
      o.x = ckb_f64::canon_u64(s00 + s01, pp.x, pp.y);
      o.y = ckb_f64::canon_u64(s10 + s11, pp.x, pp.y);
      *reinterpret_cast<ulonglong2*>(dst + (size_t)(rowi[a] & 0xFFFF) * N) = o;
    }
    for (int b = 0; b < ni; ++b) {  // integer pipes
      const uint64_t* cr = ic + (size_t)b * AMAX;
      uint64_t h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll
      for (int i0 = 0; i0 < AMAX; i0 += 8) {  // <= 8 terms per 64-bit partial
        ckb::Acc4 a0, a1;
#pragma unroll
        for (int i = i0; i < (i0 + 8 < AMAX ? i0 + 8 : AMAX); ++i) {
          const ckb::Split30 c = ckb::unpack30(cr[i]);
          const uint64_t u0 = fin ? ckb_f64::f64_to_u64(y0[i]) : (uint64_t)__double_as_longlong(y0[i]);
          const uint64_t u1 = fin ? ckb_f64::f64_to_u64(y1[i]) : (uint64_t)__double_as_longlong(y1[i]);
          a0.mac(ckb::split30(u0), c);
          a1.mac(ckb::split30(u1), c);
        }
        a0.fold_into(h0, l0);
        a1.fold_into(h1, l1);
      }
      const ModSm ms = ims[b];
      const Mod m{ms.p, ms.mu, ms.k, ms.two_p};
      ulonglong2 o;
      if (ms.k >= 32) {  // CTA-uniform
        o.x = ckb::reduce128_big(h0, l0, ms.r64, ms.r64s, m);
        o.y = ckb::reduce128_big(h1, l1, ms.r64, ms.r64s, m);
      } else {
        o.x = ckb::reduce128_any(h0, l0, ms.r64, ms.r64s, m);
        o.y = ckb::reduce128_any(h1, l1, ms.r64, ms.r64s, m);
      }
      *reinterpret_cast<ulonglong2*>(dst + (size_t)(rowi[ext + b] & 0xFFFF) * N) = o;
    }
  }
}

inline size_t modup_v2_smem(int ext, int amax) {
  return (size_t)ext * amax * 16 + (size_t)ext * 16 + (size_t)ext * amax * 8 +
         (size_t)ext * sizeof(ModSm) + (2 * (size_t)ext + 2) * 4 + 3 * (size_t)amax * 8 + 16;
}

// Optional addend folded into the inner product for the first `limbs` ext
// limbs (the Q limbs): acc_b[e] += b[e] * P_e and acc_a[e] += a[e] * P_e
// (P_e = the special modulus mod q_e, with its Shoup word), so the ModDown
// that follows yields x P^-1 + addend without reading the addend again.
struct KsFold {
  const uint64_t* b;  // item i, limb e at b + i*bs + e*N (NULL: no fold)
  const uint64_t* a;  // likewise for the a output (NULL: none)
  size_t bs, as;
  const uint64_t* mul;  // [limbs][2] {P mod q_e, shoup}
  int limbs;
};

// acc[b][c][e] = sum_j digit_j[e] * key_b[j][c][key_limb(e)] with 128-bit lazy
// accumulation and one reduction per output.  With own != NULL the digits'
// own limbs come from `own` (the NTT-domain input the digits were cut from);
// od.p[e] is the digit that owns ext limb e (-1 for none), and digit j holds
// limb e at row e - (e >= (j+1)*alpha ? alpha : 0).  ND > 0: fully unrolled.
template <int ND>
__global__ void __launch_bounds__(256) k_ks_inner(
    uint64_t* __restrict__ acc, const uint64_t* __restrict__ dig, int batch, int nd, int ext,
    int out_rows, int item_rows, int alpha, int limbs, const uint64_t* __restrict__ own,
    size_t own_bstride, int log_n,
    const uint64_t* __restrict__ key, const uint64_t* const* __restrict__ key_ptrs, int key_limbs,
    RingDev R, LimbMap em, LimbMap km, LimbMap od, KsFold fold) {
  const size_t N = (size_t)1 << log_n;
  const int lh = log_n - 1;
  const size_t total = (size_t)batch * ext << lh;
  const size_t krow = 2 * (size_t)key_limbs * N;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = (t & ((N >> 1) - 1)) * 2;
    const unsigned be = (unsigned)(t >> lh);
    const int e = (int)(be % (unsigned)ext);
    const size_t bi = be / (unsigned)ext;
    const uint64_t* K = key_ptrs ? key_ptrs[bi] : key;
    const uint64_t* kb = K + (size_t)km.p[e] * N + n;
    const uint64_t* ka = kb + (size_t)key_limbs * N;
    const int owner = own ? od.p[e] : -1;
    const uint64_t* dbase = dig + bi * (size_t)item_rows * N + n;
    ulonglong2 x[ND], b[ND], a[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j) {  // issue every load first
      const int cj = min(alpha, limbs - j * alpha);  // digit j's width (last may be short)
      const int row = own ? e - (e >= j * alpha + cj ? cj : 0) : e;
      const uint64_t* xp = (j == owner) ? own + bi * own_bstride + (size_t)e * N + n
                                        : dbase + ((size_t)j * out_rows + row) * N;
      x[j] = *reinterpret_cast<const ulonglong2*>(xp);
      b[j] = __ldg(reinterpret_cast<const ulonglong2*>(kb + j * krow));
      a[j] = __ldg(reinterpret_cast<const ulonglong2*>(ka + j * krow));
    }
    const uint64_t* mm = R.mods + (size_t)em.p[e] * kModStride;
    const Mod m{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
    const uint64_t r64 = __ldg(mm + 8), r64s = __ldg(mm + 9);
    const bool fold_e = fold.b != nullptr && e < fold.limbs;
    ulonglong2 fb = make_ulonglong2(0, 0), fa = make_ulonglong2(0, 0);
    uint64_t fP = 0;
    if (fold_e) {
      fP = __ldg(fold.mul + 2 * e);
      fb = *reinterpret_cast<const ulonglong2*>(fold.b + bi * fold.bs + (size_t)e * N + n);
      if (fold.a) fa = *reinterpret_cast<const ulonglong2*>(fold.a + bi * fold.as + (size_t)e * N + n);
    }
    ulonglong2 ob, oa;
#ifndef CKB_KSS_INT
    if ((m.p >> 46) == 0) {  // warp-uniform: the FP64 pipe, exact products
      using namespace ckb_f64;
      const double pd = (double)m.p, pinv = 1.0 / pd;
      double sb0 = 0, sb1 = 0, sa0 = 0, sa1 = 0;
#pragma unroll
      for (int j = 0; j < ND; ++j) {
        const double x0 = u64_to_f64(x[j].x), x1 = u64_to_f64(x[j].y);
        const double b0 = u64_to_f64(b[j].x), b1 = u64_to_f64(b[j].y);
        const double a0 = u64_to_f64(a[j].x), a1 = u64_to_f64(a[j].y);
        sb0 += mulmod_f64(x0, b0, b0 * pinv, pd);
        sb1 += mulmod_f64(x1, b1, b1 * pinv, pd);
        sa0 += mulmod_f64(x0, a0, a0 * pinv, pd);
        sa1 += mulmod_f64(x1, a1, a1 * pinv, pd);
      }
      if (fold_e) {
        const double P = u64_to_f64(fP), Pp = P * pinv;
        sb0 += mulmod_f64(u64_to_f64(fb.x), P, Pp, pd);
        sb1 += mulmod_f64(u64_to_f64(fb.y), P, Pp, pd);
        sa0 += mulmod_f64(u64_to_f64(fa.x), P, Pp, pd);
        sa1 += mulmod_f64(u64_to_f64(fa.y), P, Pp, pd);
      }
      ob = make_ulonglong2(canon_u64(sb0, pd, pinv), canon_u64(sb1, pd, pinv));
      oa = make_ulonglong2(canon_u64(sa0, pd, pinv), canon_u64(sa1, pd, pinv));
    } else
#endif
    {
    uint64_t hb0 = 0, lb0 = 0, ha0 = 0, la0 = 0, hb1 = 0, lb1 = 0, ha1 = 0, la1 = 0;
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      ckb::mac128(hb0, lb0, x[j].x, b[j].x);
      ckb::mac128(ha0, la0, x[j].x, a[j].x);
      ckb::mac128(hb1, lb1, x[j].y, b[j].y);
      ckb::mac128(ha1, la1, x[j].y, a[j].y);
    }
    if (fold_e) {
      ckb::mac128(hb0, lb0, fb.x, fP);
      ckb::mac128(hb1, lb1, fb.y, fP);
      ckb::mac128(ha0, la0, fa.x, fP);
      ckb::mac128(ha1, la1, fa.y, fP);
    }
    if (m.k >= 32) {
      ob = make_ulonglong2(ckb::reduce128_big(hb0, lb0, r64, r64s, m),
                           ckb::reduce128_big(hb1, lb1, r64, r64s, m));
      oa = make_ulonglong2(ckb::reduce128_big(ha0, la0, r64, r64s, m),
                           ckb::reduce128_big(ha1, la1, r64, r64s, m));
    } else {
      ob = make_ulonglong2(ckb::reduce128_any(hb0, lb0, r64, r64s, m),
                           ckb::reduce128_any(hb1, lb1, r64, r64s, m));
      oa = make_ulonglong2(ckb::reduce128_any(ha0, la0, r64, r64s, m),
                           ckb::reduce128_any(ha1, la1, r64, r64s, m));
    }
    }
    uint64_t* o = acc + (bi * 2 * ext + e) * N + n;
    *reinterpret_cast<ulonglong2*>(o) = ob;
    *reinterpret_cast<ulonglong2*>(o + (size_t)ext * N) = oa;
  }
}

// Runtime digit count (alpha = 1 chains with many digits).
// One key for the whole batch (relinearisation, a single rotation step): each
// thread owns one (ext limb, coefficient pair), loads that pair of every key
// row ONCE into registers and walks the batch, so the key is read from memory
// once per batch instead of once per item (the per-item form re-read the
// 90 MB relinearisation key from L2 for each of the 64 items of config 2).
template <int ND>
__global__ void __launch_bounds__(256, 2) k_ks_inner_shared(
    uint64_t* __restrict__ acc, const uint64_t* __restrict__ dig, int batch, int ext,
    int out_rows, int item_rows, int alpha, int limbs, const uint64_t* __restrict__ own,
    size_t own_bstride, int log_n, const uint64_t* __restrict__ key, int key_limbs, RingDev R,
    LimbMap em, LimbMap km, LimbMap od, KsFold fold) {
  const size_t N = (size_t)1 << log_n;
  const int lh = log_n - 1;
  const size_t total = (size_t)ext << lh;
  const size_t krow = 2 * (size_t)key_limbs * N;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = (t & ((N >> 1) - 1)) * 2;
    const int e = (int)(t >> lh);
    const uint64_t* kb = key + (size_t)km.p[e] * N + n;
    const uint64_t* ka = kb + (size_t)key_limbs * N;
    ulonglong2 b[ND], a[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      b[j] = __ldg(reinterpret_cast<const ulonglong2*>(kb + j * krow));
      a[j] = __ldg(reinterpret_cast<const ulonglong2*>(ka + j * krow));
    }
    const int owner = own ? od.p[e] : -1;
    size_t rowoff[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const int cj = min(alpha, limbs - j * alpha);
      const int row = own ? e - (e >= j * alpha + cj ? cj : 0) : e;
      rowoff[j] = ((size_t)j * out_rows + row) * N + n;
    }
    const uint64_t* mm = R.mods + (size_t)em.p[e] * kModStride;
    const Mod m{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
    const uint64_t r64 = __ldg(mm + 8), r64s = __ldg(mm + 9);
    const bool fold_e = fold.b != nullptr && e < fold.limbs;
    const uint64_t fP = fold_e ? __ldg(fold.mul + 2 * e) : 0;
    // x[0..ND) the digits; with a fold, x[ND] / x[ND+1] the b / a addends
    auto load_item = [&](int bi, ulonglong2* x) {
      const uint64_t* dbase = dig + (size_t)bi * item_rows * N;
#pragma unroll
      for (int j = 0; j < ND; ++j) {
        const uint64_t* xp = (j == owner) ? own + bi * own_bstride + (size_t)e * N + n
                                          : dbase + rowoff[j];
        x[j] = __ldcs(reinterpret_cast<const ulonglong2*>(xp));
      }
      if (fold_e) {
        x[ND] = *reinterpret_cast<const ulonglong2*>(fold.b + bi * fold.bs + (size_t)e * N + n);
        x[ND + 1] = fold.a ? *reinterpret_cast<const ulonglong2*>(fold.a + bi * fold.as +
                                                                  (size_t)e * N + n)
                           : make_ulonglong2(0, 0);
      }
    };
    ulonglong2 xn[ND + 2];
    load_item(0, xn);
    for (int bi = 0; bi < batch; ++bi) {
      ulonglong2 x[ND + 2];
#pragma unroll
      for (int j = 0; j < ND + 2; ++j) x[j] = xn[j];
#ifndef CKB_KSS_NO_PREFETCH
      if (bi + 1 < batch) load_item(bi + 1, xn);  // next item's loads in flight during this MAC
#endif
      ulonglong2 ob, oa;
#ifndef CKB_KSS_INT
      if ((m.p >> 46) == 0) {  // warp-uniform: the FP64 pipe, exact products
        using namespace ckb_f64;
        const double pd = (double)m.p, pinv = 1.0 / pd;
        double sb0 = 0, sb1 = 0, sa0 = 0, sa1 = 0;
#pragma unroll
        for (int j = 0; j < ND; ++j) {
          const double x0 = u64_to_f64(x[j].x), x1 = u64_to_f64(x[j].y);
          const double b0 = u64_to_f64(b[j].x), b1 = u64_to_f64(b[j].y);
          const double a0 = u64_to_f64(a[j].x), a1 = u64_to_f64(a[j].y);
          sb0 += mulmod_f64(x0, b0, b0 * pinv, pd);
          sb1 += mulmod_f64(x1, b1, b1 * pinv, pd);
          sa0 += mulmod_f64(x0, a0, a0 * pinv, pd);
          sa1 += mulmod_f64(x1, a1, a1 * pinv, pd);
        }
        if (fold_e) {
          const double P = u64_to_f64(fP), Pp = P * pinv;
          sb0 += mulmod_f64(u64_to_f64(x[ND].x), P, Pp, pd);
          sb1 += mulmod_f64(u64_to_f64(x[ND].y), P, Pp, pd);
          sa0 += mulmod_f64(u64_to_f64(x[ND + 1].x), P, Pp, pd);
          sa1 += mulmod_f64(u64_to_f64(x[ND + 1].y), P, Pp, pd);
        }
        ob = make_ulonglong2(canon_u64(sb0, pd, pinv), canon_u64(sb1, pd, pinv));
        oa = make_ulonglong2(canon_u64(sa0, pd, pinv), canon_u64(sa1, pd, pinv));
      } else
#endif
      {
      uint64_t hb0 = 0, lb0 = 0, ha0 = 0, la0 = 0, hb1 = 0, lb1 = 0, ha1 = 0, la1 = 0;
#pragma unroll
      for (int j = 0; j < ND; ++j) {
        ckb::mac128(hb0, lb0, x[j].x, b[j].x);
        ckb::mac128(ha0, la0, x[j].x, a[j].x);
        ckb::mac128(hb1, lb1, x[j].y, b[j].y);
        ckb::mac128(ha1, la1, x[j].y, a[j].y);
      }
      if (fold_e) {
        ckb::mac128(hb0, lb0, x[ND].x, fP);
        ckb::mac128(hb1, lb1, x[ND].y, fP);
        ckb::mac128(ha0, la0, x[ND + 1].x, fP);
        ckb::mac128(ha1, la1, x[ND + 1].y, fP);
      }
      if (m.k >= 32) {
        ob = make_ulonglong2(ckb::reduce128_big(hb0, lb0, r64, r64s, m),
                             ckb::reduce128_big(hb1, lb1, r64, r64s, m));
        oa = make_ulonglong2(ckb::reduce128_big(ha0, la0, r64, r64s, m),
                             ckb::reduce128_big(ha1, la1, r64, r64s, m));
      } else {
        ob = make_ulonglong2(ckb::reduce128_any(hb0, lb0, r64, r64s, m),
                             ckb::reduce128_any(hb1, lb1, r64, r64s, m));
        oa = make_ulonglong2(ckb::reduce128_any(ha0, la0, r64, r64s, m),
                             ckb::reduce128_any(ha1, la1, r64, r64s, m));
      }
      }
      uint64_t* o = acc + ((size_t)bi * 2 * ext + e) * N + n;
      __stcs(reinterpret_cast<ulonglong2*>(o), ob);
      __stcs(reinterpret_cast<ulonglong2*>(o + (size_t)ext * N), oa);
#ifdef CKB_KSS_NO_PREFETCH
      if (bi + 1 < batch) load_item(bi + 1, xn);
#endif
    }
  }
}

__global__ void __launch_bounds__(256) k_ks_inner_any(
    uint64_t* __restrict__ acc, const uint64_t* __restrict__ dig, int batch, int nd, int ext,
    int out_rows, int item_rows, int alpha, int limbs, const uint64_t* __restrict__ own,
    size_t own_bstride, int log_n,
    const uint64_t* __restrict__ key, const uint64_t* const* __restrict__ key_ptrs, int key_limbs,
    RingDev R, LimbMap em, LimbMap km, LimbMap od) {
  const size_t N = (size_t)1 << log_n;
  const size_t total = (size_t)batch * ext * N;
  const size_t krow = 2 * (size_t)key_limbs * N;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = t & (N - 1);
    const size_t be = t >> log_n;
    const int e = (int)(be % ext);
    const size_t bi = be / ext;
    const uint64_t* K = key_ptrs ? key_ptrs[bi] : key;
    const uint64_t* kb = K + (size_t)km.p[e] * N + n;
    const uint64_t* ka = kb + (size_t)key_limbs * N;
    const int owner = own ? od.p[e] : -1;
    const uint64_t* dbase = dig + bi * (size_t)item_rows * N + n;
    uint64_t hb = 0, lb = 0, ha = 0, la = 0;
    for (int j = 0; j < nd; ++j) {
      const int cj = min(alpha, limbs - j * alpha);  // digit j's width (last may be short)
      const int row = own ? e - (e >= j * alpha + cj ? cj : 0) : e;
      const uint64_t x = (j == owner) ? own[bi * own_bstride + (size_t)e * N + n]
                                      : dbase[((size_t)j * out_rows + row) * N];
      ckb::mac128(hb, lb, x, __ldg(kb + j * krow));
      ckb::mac128(ha, la, x, __ldg(ka + j * krow));
    }
    const uint64_t* mm = R.mods + (size_t)em.p[e] * kModStride;
    const Mod m{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
    const uint64_t r64 = __ldg(mm + 8), r64s = __ldg(mm + 9);
    uint64_t* o = acc + (bi * 2 * ext + e) * N + n;
    o[0] = ckb::reduce128_any(hb, lb, r64, r64s, m);
    o[(size_t)ext * N] = ckb::reduce128_any(ha, la, r64, r64s, m);
  }
}

// ===========================================================================
// Exact divide-and-round (rescale / ModDown / level adjust)
// ===========================================================================

constexpr int kMaxDrop = 16;
// first-drop width from which the correction takes the fast basis-conversion
// form (k_divround_corr_hps) when the caller passes its table
constexpr int kHpsMinDrop = 6;
// |frac - 1/2| below which rho is settled by exact_rho (ckb_ring.flags
// CKB_RING_HPS_EXACT lowers it to 0: every coefficient takes the exact path)
constexpr double kHpsMargin = 0.5 - 0x1p-30;

// acc - r * M  (mod p) for a signed centered remainder r and a Shoup constant M.
__device__ __forceinline__ uint64_t sub_rm(uint64_t acc, int64_t r, uint64_t M, uint64_t Ms,
                                           uint64_t p) {
  const uint64_t mag = (uint64_t)(r < 0 ? -r : r);
  uint64_t prod = ckb::mul_shoup_lazy(mag, M, Ms, p);
  prod = prod >= p ? prod - p : prod;
  return r < 0 ? ckb::add_mod(acc, prod, p) : ckb::sub_mod(acc, prod, p);
}

__device__ __forceinline__ int64_t centered(uint64_t x, uint64_t p) {
  return x > (p >> 1) ? (int64_t)x - (int64_t)p : (int64_t)x;
}

// Exact sequential divide-and-round by the last n1 (then n2) limbs, evaluated
// in mixed radix: dropping p_0, p_1, ... one at a time (ring.py:171-183) gives
//   result_j = (x_j - sum_u r_u M_u) * (prod_u p_u)^-1  (mod q_j),
// with M_u = p_0 ... p_{u-1} and r_u the centered residue of the partially
// divided value at p_u — the same integers, so the output is bit-identical.
// tab1: [limbs][n1+1][2] {M_u mod p_j, shoup} and {(M_t)^-1 mod p_j or P^-1}
// tab2: [m1][n2+1][2] likewise for the second chain.
template <int D1, int D2>
__global__ void __launch_bounds__(256, 2) k_divround(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ in, size_t in_stride,
    const uint64_t* __restrict__ addend, int add_polys, int add_period, int add_stride,
    int polys, int limbs, int n1, int n2, int log_n, RingDev R, LimbMap lm, ScalarTab pre,
    int has_pre, const uint64_t* __restrict__ tab1, const uint64_t* __restrict__ tab2) {
  const size_t N = (size_t)1 << log_n;
  const size_t total = (size_t)polys * N;
  const int m1 = limbs - n1;
  const int m2 = m1 - n2;
  const int s1 = 2 * (n1 + 1), s2 = 2 * (n2 + 1);
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = t & (N - 1);
    const size_t pidx = t >> log_n;
    const uint64_t* src = in + pidx * in_stride + n;
    const uint64_t* add = nullptr;
    if (addend) {
      const size_t ph = pidx % add_period;
      if ((int)ph < add_polys) add = addend + ((pidx / add_period) * add_stride + ph) * m1 * N + n;
    }
    uint64_t* dst = out + pidx * m2 * N + n;

    auto load = [&](int l, uint64_t p) -> uint64_t {
      uint64_t v = src[(size_t)l * N];
      if (has_pre) v = ckb::mul_shoup(v, pre.v[l], pre.s[l], p);
      return v;
    };
    int64_t r1[D1 > 0 ? D1 : 1], r2[D2 > 0 ? D2 : 1];
#pragma unroll
    for (int d = 0; d < D1; ++d) {
      if (d < n1) {
        const int li = limbs - 1 - d;
        const uint64_t p = __ldg(R.mods + (size_t)lm.p[li] * kModStride);
        const uint64_t* T = tab1 + (size_t)li * s1;
        uint64_t acc = load(li, p);
#pragma unroll
        for (int u = 0; u < D1; ++u)
          if (u < d) acc = sub_rm(acc, r1[u], __ldg(T + 2 * u), __ldg(T + 2 * u + 1), p);
        acc = ckb::mul_shoup(acc, __ldg(T + 2 * n1), __ldg(T + 2 * n1 + 1), p);
        r1[d] = centered(acc, p);
      }
    }
    auto stage1 = [&](int l) -> uint64_t {
      const uint64_t p = __ldg(R.mods + (size_t)lm.p[l] * kModStride);
      uint64_t v = load(l, p);
      if (n1) {
        const uint64_t* T = tab1 + (size_t)l * s1;
#pragma unroll
        for (int u = 0; u < D1; ++u)
          if (u < n1) v = sub_rm(v, r1[u], __ldg(T + 2 * u), __ldg(T + 2 * u + 1), p);
        v = ckb::mul_shoup(v, __ldg(T + 2 * n1), __ldg(T + 2 * n1 + 1), p);
      }
      if (add) v = ckb::add_mod(v, add[(size_t)l * N], p);
      return v;
    };
#pragma unroll
    for (int d = 0; d < D2; ++d) {
      if (d < n2) {
        const int li = m1 - 1 - d;
        const uint64_t p = __ldg(R.mods + (size_t)lm.p[li] * kModStride);
        const uint64_t* T = tab2 + (size_t)li * s2;
        uint64_t acc = stage1(li);
#pragma unroll
        for (int u = 0; u < D2; ++u)
          if (u < d) acc = sub_rm(acc, r2[u], __ldg(T + 2 * u), __ldg(T + 2 * u + 1), p);
        acc = ckb::mul_shoup(acc, __ldg(T + 2 * n2), __ldg(T + 2 * n2 + 1), p);
        r2[d] = centered(acc, p);
      }
    }
    for (int l = 0; l < m2; ++l) {
      uint64_t v = stage1(l);
      if (n2) {
        const uint64_t p = __ldg(R.mods + (size_t)lm.p[l] * kModStride);
        const uint64_t* T = tab2 + (size_t)l * s2;
#pragma unroll
        for (int u = 0; u < D2; ++u)
          if (u < n2) v = sub_rm(v, r2[u], __ldg(T + 2 * u), __ldg(T + 2 * u + 1), p);
        v = ckb::mul_shoup(v, __ldg(T + 2 * n2), __ldg(T + 2 * n2 + 1), p);
      }
      dst[(size_t)l * N] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// NTT-domain divide-and-round.  With x (and the addend) in the NTT domain, the
// exact result (x_j * P1^-1 + add_j - E_j) * P2^-1 needs only the
// coefficient-domain values of the dropped limbs: the correction polynomial
//   E_j = (sum_u r1_u M1_u) * P1^-1 + sum_u r2_u M2_u   (mod q_j)
// is built here from those limbs (T, coefficient domain) and is then
// transformed with one forward NTT per output limb.
// T per poly: rows [0, n1+n2) = x limbs [m2, limbs) (coefficient domain),
//             rows [n1+n2, n1+2*n2) = addend limbs [m2, m1) (coefficient domain).
// tabE: [m2][n1+n2][2] {M1_u * P1^-1 mod q_j, shoup} then {M2_u mod q_j, shoup}.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t add_rm(uint64_t acc, int64_t r, uint64_t M, uint64_t Ms,
                                           uint64_t p) {
  return sub_rm(acc, -r, M, Ms, p);
}

// V coefficients per thread (2: 16-byte accesses; 1 for wide drops, whose
// remainder arrays would otherwise cap occupancy); the E loop's per-limb
// constants (modulus, r64, and the tabE row) are staged in shared memory.
template <int V>
__device__ __forceinline__ void ld_v(uint64_t* x, const uint64_t* p) {
  if constexpr (V == 2) {
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
    x[0] = v.x;
    x[1] = v.y;
  } else {
    x[0] = *p;
  }
}

template <int V>
__device__ __forceinline__ void st_v(uint64_t* p, const uint64_t* x) {
  if constexpr (V == 2) {
    *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(x[0], x[1]);
  } else {
    *p = x[0];
  }
}

// acc_c - sum_{u<cnt} r_u[c] * M_u  (mod p) for V lanes at once, with one
// reduction instead of cnt sequential modular steps: each term is made
// non-negative as (C - r_u) M_u with C = p << (clz(p) - 4) in [2^59, 2^60) a
// multiple of p (|r_u| < 2^59), so the 128-bit lazy sum stays below
// 2^125 for up to 16 terms.  Bit-identical to the sub_rm chain.
template <int D, int V>
__device__ __forceinline__ void sub_rm_lazy(uint64_t* acc, const int64_t (*r)[V], int cnt,
                                            const uint64_t* __restrict__ Tb, const uint64_t* mm) {
  const uint64_t p = __ldg(mm);
  const int64_t C = (int64_t)(p << (__clzll((long long)p) - 4));
  uint64_t h[V], l[V];
#pragma unroll
  for (int c = 0; c < V; ++c) {
    h[c] = 0;
    l[c] = acc[c];
  }
#pragma unroll
  for (int u = 0; u < D; ++u)
    if (u < cnt) {
      const uint64_t M = __ldg(Tb + 2 * u);
#pragma unroll
      for (int c = 0; c < V; ++c) ckb::mac128(h[c], l[c], (uint64_t)(C - r[u][c]), M);
    }
  const Mod m{p, __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
  const uint64_t r64 = __ldg(mm + 8), r64s = __ldg(mm + 9);
  if (m.k >= 32) {  // warp-uniform
#pragma unroll
    for (int c = 0; c < V; ++c) acc[c] = ckb::reduce128_big(h[c], l[c], r64, r64s, m);
  } else {
#pragma unroll
    for (int c = 0; c < V; ++c) acc[c] = ckb::reduce128_any(h[c], l[c], r64, r64s, m);
  }
}

template <int D1, int D2, int V>
__global__ void __launch_bounds__(256, V == 2 ? 2 : 3) k_divround_corr(
    uint64_t* __restrict__ E, const uint64_t* __restrict__ T, int has_add, int polys, int limbs,
    int n1, int n2, int log_n, RingDev R, LimbMap lm, const uint64_t* __restrict__ tab1,
    const uint64_t* __restrict__ tab2, const uint64_t* __restrict__ tabE) {
  extern __shared__ uint64_t sm[];
  const size_t N = (size_t)1 << log_n;
  const int m1 = limbs - n1;
  const int m2 = m1 - n2;
  const int s1 = 2 * (n1 + 1), s2 = 2 * (n2 + 1), sE = 2 * (n1 + n2 + 1);
  const int row_w = 6 + sE;  // {p, mu, k, 2p, r64, r64s} then the tabE row
  for (int q = threadIdx.x; q < m2 * row_w; q += blockDim.x) {
    const int j = q / row_w, c = q % row_w;
    const uint64_t* mm = R.mods + (size_t)lm.p[j] * kModStride;
    uint64_t v;
    if (c < 6) {
      v = c < 4 ? __ldg(mm + c) : __ldg(mm + 4 + c);
    } else {  // tabE row
      v = __ldg(tabE + (size_t)j * sE + c - 6);
    }
    sm[q] = v;
  }
  __syncthreads();
  const size_t per = N / V;
  const size_t total = (size_t)polys * per;
  const int trows = n1 + n2 + (has_add ? n2 : 0);
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = (t % per) * V;
    const size_t pidx = t / per;
    const uint64_t* src = T + pidx * trows * N + n;
    int64_t r1[D1 > 0 ? D1 : 1][V], r2[D2 > 0 ? D2 : 1][V];
#pragma unroll
    for (int d = 0; d < D1; ++d) {
      if (d < n1) {
        const int li = limbs - 1 - d;
        const uint64_t p = __ldg(R.mods + (size_t)lm.p[li] * kModStride);
        const uint64_t* Tb = tab1 + (size_t)li * s1;
        uint64_t a[V];
        ld_v<V>(a, src + (size_t)(li - m2) * N);
        if (d >= 2) {  // compile-time after unrolling
          sub_rm_lazy<D1, V>(a, r1, d, Tb, R.mods + (size_t)lm.p[li] * kModStride);
        } else {
#pragma unroll
          for (int u = 0; u < D1; ++u)
            if (u < d) {
              const uint64_t M = __ldg(Tb + 2 * u), Ms = __ldg(Tb + 2 * u + 1);
#pragma unroll
              for (int c = 0; c < V; ++c) a[c] = sub_rm(a[c], r1[u][c], M, Ms, p);
            }
        }
        const uint64_t W = __ldg(Tb + 2 * n1), Ws = __ldg(Tb + 2 * n1 + 1);
#pragma unroll
        for (int c = 0; c < V; ++c) r1[d][c] = centered(ckb::mul_shoup(a[c], W, Ws, p), p);
      }
    }
#pragma unroll
    for (int d = 0; d < D2; ++d) {
      if (d < n2) {
        const int li = m1 - 1 - d;
        const uint64_t p = __ldg(R.mods + (size_t)lm.p[li] * kModStride);
        uint64_t v[V];
        ld_v<V>(v, src + (size_t)(li - m2) * N);
        if (n1) {
          const uint64_t* Ta = tab1 + (size_t)li * s1;
          if (n1 >= 2) {
            sub_rm_lazy<D1, V>(v, r1, n1, Ta, R.mods + (size_t)lm.p[li] * kModStride);
          } else {
#pragma unroll
            for (int u = 0; u < D1; ++u)
              if (u < n1) {
                const uint64_t M = __ldg(Ta + 2 * u), Ms = __ldg(Ta + 2 * u + 1);
#pragma unroll
                for (int c = 0; c < V; ++c) v[c] = sub_rm(v[c], r1[u][c], M, Ms, p);
              }
          }
          const uint64_t W = __ldg(Ta + 2 * n1), Ws = __ldg(Ta + 2 * n1 + 1);
#pragma unroll
          for (int c = 0; c < V; ++c) v[c] = ckb::mul_shoup(v[c], W, Ws, p);
        }
        if (has_add) {
          uint64_t a[V];
          ld_v<V>(a, src + (size_t)(n1 + n2 + li - m2) * N);
#pragma unroll
          for (int c = 0; c < V; ++c) v[c] = ckb::add_mod(v[c], a[c], p);
        }
        const uint64_t* Tb = tab2 + (size_t)li * s2;
#pragma unroll
        for (int u = 0; u < D2; ++u)
          if (u < d) {
            const uint64_t M = __ldg(Tb + 2 * u), Ms = __ldg(Tb + 2 * u + 1);
#pragma unroll
            for (int c = 0; c < V; ++c) v[c] = sub_rm(v[c], r2[u][c], M, Ms, p);
          }
        const uint64_t W = __ldg(Tb + 2 * n2), Ws = __ldg(Tb + 2 * n2 + 1);
#pragma unroll
        for (int c = 0; c < V; ++c) r2[d][c] = centered(ckb::mul_shoup(v[c], W, Ws, p), p);
      }
    }
    // E_j = sum_u r_u c_uj: each signed r is shifted by C_j (a multiple of q_j)
    // so every term is a non-negative word; 128-bit lazy sum and one
    // reduction per output.
    uint64_t* dst = E + pidx * m2 * N + n;
    for (int j = 0; j < m2; ++j) {
      const uint64_t* S = sm + (size_t)j * row_w;
      const uint64_t* Te = S + 6;
      const int64_t off = (int64_t)Te[2 * (n1 + n2)];
      uint64_t h[V], l[V];
#pragma unroll
      for (int c = 0; c < V; ++c) h[c] = l[c] = 0;
#pragma unroll
      for (int u = 0; u < D1; ++u)
        if (u < n1) {
          const uint64_t cc = Te[2 * u];
#pragma unroll
          for (int c = 0; c < V; ++c) ckb::mac128(h[c], l[c], (uint64_t)(r1[u][c] + off), cc);
        }
#pragma unroll
      for (int u = 0; u < D2; ++u)
        if (u < n2) {
          const uint64_t cc = Te[2 * (n1 + u)];
#pragma unroll
          for (int c = 0; c < V; ++c) ckb::mac128(h[c], l[c], (uint64_t)(r2[u][c] + off), cc);
        }
      const Mod m{S[0], S[1], S[2], S[3]};
      uint64_t o[V];
      if (m.k >= 32) {  // warp-uniform
#pragma unroll
        for (int c = 0; c < V; ++c) o[c] = ckb::reduce128_big(h[c], l[c], S[4], S[5], m);
      } else {
#pragma unroll
        for (int c = 0; c < V; ++c) o[c] = ckb::reduce128_any(h[c], l[c], S[4], S[5], m);
      }
      st_v<V>(dst + (size_t)j * N, o);
    }
  }
}

// Wide first drops (n1 >= 6 special primes): the centred residue of x mod P1
// from one fast basis conversion instead of the O(n1^2) mixed-radix chain.
//   y_u = [x_u (P1/p_u)^-1]_{p_u},  S = sum_u y_u (P1/p_u),  rho = round(S/P1)
//   c1 = S - rho P1 (the centred residue: |c1| < P1/2 since P1 is odd)
//   E1_j = c1 P1^-1 = sum_u y_u [p_u^-1]_{q_j} - rho  (mod q_j)
// rho = rint(sum_u y_u / p_u) in FP64 (error < 2^-47 for n1 <= 16).  When the
// fractional part lies within 2^-30 of 1/2 (probability ~2^-29 per
// coefficient) rho is settled exactly by exact_rho below, so the integers are
// always the sequential chain's and the output is bit-identical.
// tabH: [m1][n1] {p_u^-1 mod q_j} for every kept limb, then [n1][2]
// {(P1/p_u)^-1 mod p_u, shoup}.  Smem per output row: {p, mu, k, 2p, r64,
// r64s}, the tabE row (C_j and the r2 constants), then the tabH row.

// Rare path: S/P1 = floor(f) + 1/2 +- 2^-30, so rho is floor(f) when the
// centred residue c1 is positive and floor(f) + 1 when it is negative.  The
// sign of c1 is that of its top nonzero centred mixed-radix digit (the digits
// of the sequential chain, ring.py:171-183); local arrays are fine here.
__device__ __noinline__ uint64_t exact_rho(const uint64_t* __restrict__ src, size_t N, int limbs,
                                           int m2, int n1, double f,
                                           const uint64_t* __restrict__ tab1, RingDev R,
                                           const LimbMap& lm) {
  int64_t r[kMaxDrop];
  const int s1 = 2 * (n1 + 1);
  int64_t top = 0;
  for (int d = 0; d < n1; ++d) {
    const int li = limbs - 1 - d;
    const uint64_t p = __ldg(R.mods + (size_t)lm.p[li] * kModStride);
    const uint64_t* Tb = tab1 + (size_t)li * s1;
    uint64_t a = src[(size_t)(li - m2) * N];
    for (int u = 0; u < d; ++u) a = sub_rm(a, r[u], __ldg(Tb + 2 * u), __ldg(Tb + 2 * u + 1), p);
    r[d] = centered(ckb::mul_shoup(a, __ldg(Tb + 2 * n1), __ldg(Tb + 2 * n1 + 1), p), p);
    if (r[d] != 0) top = r[d];
  }
  // c1 == 0 (every digit zero; reached only when the margin is forced to 0):
  // S = rho * P1 exactly, so f is rho up to rounding
  if (top == 0) return (uint64_t)rint(f);
  const uint64_t fl = (uint64_t)floor(f);
  return top > 0 ? fl : fl + 1;
}

#ifndef CKB_CORR_MINB
#define CKB_CORR_MINB 3
#endif
// widest first drop handled two coefficients per thread (A/B: round 1 measured
// config 5's steady step 5.89 -> 5.77 s with 11, despite the spills of the
// <11, *, 2> instantiations under the 80-register bound)
#ifndef CKB_CORR_VV2_MAX
#define CKB_CORR_VV2_MAX 11
#endif
template <int D1, int D2, int V>
__global__ void __launch_bounds__(256, CKB_CORR_MINB) k_divround_corr_hps(
    uint64_t* __restrict__ E, const uint64_t* __restrict__ T, int has_add, int polys, int limbs,
    int n1, int n2, int log_n, RingDev R, LimbMap lm, const uint64_t* __restrict__ tab1,
    const uint64_t* __restrict__ tab2, const uint64_t* __restrict__ tabE,
    const uint64_t* __restrict__ tabH, double margin) {
  extern __shared__ uint64_t sm[];
  const size_t N = (size_t)1 << log_n;
  const int m1 = limbs - n1;
  const int m2 = m1 - n2;
  const int s1 = 2 * (n1 + 1), s2 = 2 * (n2 + 1), sE = 2 * (n1 + n2 + 1);
  const int row_w = 6 + sE + n1;
  for (int q = threadIdx.x; q < m2 * row_w; q += blockDim.x) {
    const int j = q / row_w, c = q % row_w;
    const uint64_t* mm = R.mods + (size_t)lm.p[j] * kModStride;
    uint64_t v;
    if (c < 6) {
      v = c < 4 ? __ldg(mm + c) : __ldg(mm + 4 + c);
    } else if (c < 6 + sE) {
      v = __ldg(tabE + (size_t)j * sE + c - 6);
    } else {
      v = __ldg(tabH + (size_t)j * n1 + c - 6 - sE);
    }
    sm[q] = v;
  }
  // per drop: (P1/p_u)^-1 pair, p_u and 1/p_u, after the rows
  uint64_t* dsm = sm + (size_t)m2 * row_w;
  double* dinv = reinterpret_cast<double*>(dsm + 3 * kMaxDrop);
  for (int u = threadIdx.x; u < n1; u += blockDim.x) {
    const uint64_t p = __ldg(R.mods + (size_t)lm.p[limbs - 1 - u] * kModStride);
    dsm[3 * u] = __ldg(tabH + (size_t)m1 * n1 + 2 * u);
    dsm[3 * u + 1] = __ldg(tabH + (size_t)m1 * n1 + 2 * u + 1);
    dsm[3 * u + 2] = p;
    dinv[u] = 1.0 / (double)p;
  }
  __syncthreads();
  const size_t per = N / V;
  const size_t total = (size_t)polys * per;
  const int trows = n1 + n2 + (has_add ? n2 : 0);
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = (t % per) * V;
    const size_t pidx = t / per;
    const uint64_t* src = T + pidx * trows * N + n;
    uint64_t y[D1][V];
    double f[V];
#pragma unroll
    for (int c = 0; c < V; ++c) f[c] = 0.0;
#pragma unroll
    for (int u = 0; u < D1; ++u) {
      if (u < n1) {
        uint64_t x[V];
        ld_v<V>(x, src + (size_t)(limbs - 1 - u - m2) * N);
#pragma unroll
        for (int c = 0; c < V; ++c) {
          y[u][c] = ckb::mul_shoup(x[c], dsm[3 * u], dsm[3 * u + 1], dsm[3 * u + 2]);
          f[c] = fma((double)y[u][c], dinv[u], f[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < V; ++c) y[u][c] = 0;
      }
    }
    uint64_t rho[V];
#pragma unroll
    for (int c = 0; c < V; ++c) {
      const double rho_d = rint(f[c]);
      rho[c] = fabs(f[c] - rho_d) < margin  // 0.5 - 2^-30 (0: CKB_RING_HPS_EXACT)
                   ? (uint64_t)rho_d
                   : exact_rho(src + c, N, limbs, m2, n1, f[c], tab1, R, lm);
    }
    int64_t r2[D2 > 0 ? D2 : 1][V];
#pragma unroll
    for (int d = 0; d < D2; ++d) {
      if (d < n2) {
        const int li = m1 - 1 - d;
        const uint64_t* mm = R.mods + (size_t)lm.p[li] * kModStride;
        const Mod m{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
        const uint64_t* Ta = tab1 + (size_t)li * s1;
        const uint64_t* H = tabH + (size_t)li * n1;
        const uint64_t* Tb = tab2 + (size_t)li * s2;
        uint64_t xv[V], av[V];
        ld_v<V>(xv, src + (size_t)(li - m2) * N);
        if (has_add) ld_v<V>(av, src + (size_t)(n1 + n2 + li - m2) * N);
#pragma unroll
        for (int c = 0; c < V; ++c) {
          // (x - c1) P1^-1 = x P1^-1 - E1 at this limb
          uint64_t v = ckb::mul_shoup(xv[c], __ldg(Ta + 2 * n1), __ldg(Ta + 2 * n1 + 1), m.p);
          uint64_t h = 0, l = (m.p << (__clzll((long long)m.p) - 4)) - rho[c];  // + k p
#pragma unroll
          for (int u = 0; u < D1; ++u)
            if (u < n1) ckb::mac128(h, l, y[u][c], __ldg(H + u));
          v = ckb::sub_mod(v, ckb::reduce128_any(h, l, __ldg(mm + 8), __ldg(mm + 9), m), m.p);
          if (has_add) v = ckb::add_mod(v, av[c], m.p);
#pragma unroll
          for (int u = 0; u < D2; ++u)
            if (u < d) v = sub_rm(v, r2[u][c], __ldg(Tb + 2 * u), __ldg(Tb + 2 * u + 1), m.p);
          r2[d][c] =
              centered(ckb::mul_shoup(v, __ldg(Tb + 2 * n2), __ldg(Tb + 2 * n2 + 1), m.p), m.p);
        }
      }
    }
    uint64_t* dst = E + pidx * m2 * N + n;
    for (int j = 0; j < m2; ++j) {
      const uint64_t* S = sm + (size_t)j * row_w;
      const uint64_t* Te = S + 6;
      const uint64_t* H = Te + sE;
      const int64_t off = (int64_t)Te[2 * (n1 + n2)];  // C_j: multiple of q_j in [2^59, 2^61)
      uint64_t h[V], l[V];
#pragma unroll
      for (int c = 0; c < V; ++c) {
        h[c] = 0;
        l[c] = (uint64_t)off - rho[c];
      }
#pragma unroll
      for (int u = 0; u < D1; ++u)
        if (u < n1) {
          const uint64_t hu = H[u];
#pragma unroll
          for (int c = 0; c < V; ++c) ckb::mac128(h[c], l[c], y[u][c], hu);
        }
#pragma unroll
      for (int u = 0; u < D2; ++u)
        if (u < n2) {
          const uint64_t tu = Te[2 * (n1 + u)];
#pragma unroll
          for (int c = 0; c < V; ++c) ckb::mac128(h[c], l[c], (uint64_t)(r2[u][c] + off), tu);
        }
      const Mod m{S[0], S[1], S[2], S[3]};
      uint64_t o[V];
      if (m.k >= 32) {  // warp-uniform
#pragma unroll
        for (int c = 0; c < V; ++c) o[c] = ckb::reduce128_big(h[c], l[c], S[4], S[5], m);
      } else {
#pragma unroll
        for (int c = 0; c < V; ++c) o[c] = ckb::reduce128_any(h[c], l[c], S[4], S[5], m);
      }
      st_v<V>(dst + (size_t)j * N, o);
    }
  }
}

// out_j = (x_j * P1^-1 + add_j - E_j) * P2^-1, all in the NTT domain.
__global__ void __launch_bounds__(256) k_divround_combine(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ x, size_t x_stride,
    const uint64_t* __restrict__ addend, int add_polys, int add_period, int add_stride,
    const uint64_t* __restrict__ E, int polys, int limbs, int n1, int n2, int log_n, RingDev R,
    LimbMap lm, const uint64_t* __restrict__ tab1, const uint64_t* __restrict__ tab2,
    const uint64_t* __restrict__ post, size_t post_stride) {
  // grid: x over coefficient pairs of one row, y over rows (poly, limb): the
  // row's constants are loaded once, every access is a 16-byte vector
  const size_t N = (size_t)1 << log_n;
  const int m1 = limbs - n1;
  const int m2 = m1 - n2;
  const size_t rows = (size_t)polys * m2;
  const int s1 = 2 * (n1 + 1), s2 = 2 * (n2 + 1);
  const size_t half = N >> 1;
  for (size_t pj = blockIdx.y; pj < rows; pj += gridDim.y) {
    const int j = (int)(pj % m2);
    const size_t pidx = pj / m2;
    const uint64_t p = __ldg(R.mods + (size_t)lm.p[j] * kModStride);
    uint64_t a1 = 0, a1s = 0, b2 = 0, b2s = 0;
    if (n1) {
      a1 = __ldg(tab1 + (size_t)j * s1 + 2 * n1);
      a1s = __ldg(tab1 + (size_t)j * s1 + 2 * n1 + 1);
    }
    if (n2) {
      b2 = __ldg(tab2 + (size_t)j * s2 + 2 * n2);
      b2s = __ldg(tab2 + (size_t)j * s2 + 2 * n2 + 1);
    }
    const uint64_t* xr = x + pidx * x_stride + (size_t)j * N;
    const uint64_t* ar = nullptr;
    if (addend) {
      const size_t ph = pidx % add_period;
      if ((int)ph < add_polys)
        ar = addend + ((pidx / add_period) * add_stride + ph) * m1 * N + (size_t)j * N;
    }
    const uint64_t* er = E + pj * N;
    const uint64_t* pr = post ? post + pidx * post_stride + (size_t)j * N : nullptr;
    uint64_t* orow = out + pj * N;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < half;
         q += (size_t)gridDim.x * blockDim.x) {
      const size_t n = 2 * q;
      ulonglong2 v = *reinterpret_cast<const ulonglong2*>(xr + n);
      const ulonglong2 e = *reinterpret_cast<const ulonglong2*>(er + n);
      ulonglong2 a = make_ulonglong2(0, 0);
      if (ar) a = *reinterpret_cast<const ulonglong2*>(ar + n);
      if (n1) {
        v.x = ckb::mul_shoup(v.x, a1, a1s, p);
        v.y = ckb::mul_shoup(v.y, a1, a1s, p);
      }
      if (ar) {
        v.x = ckb::add_mod(v.x, a.x, p);
        v.y = ckb::add_mod(v.y, a.y, p);
      }
      v.x = ckb::sub_mod(v.x, e.x, p);
      v.y = ckb::sub_mod(v.y, e.y, p);
      if (n2) {
        v.x = ckb::mul_shoup(v.x, b2, b2s, p);
        v.y = ckb::mul_shoup(v.y, b2, b2s, p);
      }
      if (pr) {  // fused accumulate: s + rot(s) (packing.py:193-208)
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(pr + n);
        v.x = ckb::add_mod(v.x, w.x, p);
        v.y = ckb::add_mod(v.y, w.y, p);
      }
      *reinterpret_cast<ulonglong2*>(orow + n) = v;
    }
  }
}

// NTT-domain automorphism: slot i of the bit-reversed NTT holds the value at
// psi^(2 brv(i) + 1), and (X -> X^g) maps it to psi^((2 brv(i) + 1) g), so
// out[i] = in[brv(((2 brv(i) + 1) g mod 2N - 1) / 2)] — a pure permutation.
__global__ void k_automorphism_ntt(uint64_t* __restrict__ out, const uint64_t* __restrict__ in,
                                   size_t total, int log_n, uint64_t g0,
                                   const uint64_t* __restrict__ g_items, int rows_per_item) {
  const uint64_t N = 1ull << log_n;
  const uint64_t mask2 = 2 * N - 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = i >> log_n;
    const uint32_t t = (uint32_t)(i & (N - 1));
    const uint64_t g = g_items ? __ldg(g_items + row / rows_per_item) : g0;
    const uint32_t bt = __brev(t) >> (32 - log_n);
    const uint64_t e = ((2ull * bt + 1) * g) & mask2;
    const uint32_t src = __brev((uint32_t)((e - 1) >> 1)) >> (32 - log_n);
    out[i] = in[row * N + src];
  }
}

// Blocked form.  In the bit-reversed evaluation order the automorphism maps
// the slots of an output block (fixed top bits of the index) onto ONE input
// block: bits 1..t of e*g mod 2N depend only on bits 1..t of e, and those are
// the top t index bits after the bit reversal.  So a CTA loads its source block
// contiguously (16-byte vectors), permutes inside shared memory and writes its
// output block contiguously: both global streams are coalesced, where the
// gather form read 8 bytes per 32-byte sector.
constexpr int kAutLogBlock = 11;  // 2048 slots = 16 KiB per CTA
__global__ void __launch_bounds__(256) k_automorphism_ntt_blk(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ in, int log_n, uint64_t g0,
    const uint64_t* __restrict__ g_items, int rows_per_item) {
  __shared__ __align__(16) uint64_t tile[1 << kAutLogBlock];
  const int lb = min(kAutLogBlock, log_n);
  const uint32_t B = 1u << lb;
  const int nblk = 1 << (log_n - lb);
  const size_t row = blockIdx.x / nblk;
  const uint32_t b = blockIdx.x % nblk;
  const uint64_t N = 1ull << log_n;
  const uint64_t mask2 = 2 * N - 1;
  const uint64_t g = g_items ? __ldg(g_items + row / rows_per_item) : g0;
  auto src_of = [&](uint32_t t) -> uint32_t {
    const uint32_t bt = __brev(t) >> (32 - log_n);
    const uint64_t e = ((2ull * bt + 1) * g) & mask2;
    return __brev((uint32_t)((e - 1) >> 1)) >> (32 - log_n);
  };
  const uint32_t t0 = b << lb;
  const uint32_t sb = src_of(t0) >> lb;
  const uint64_t* ib = in + row * N + (size_t)sb * B;
  for (uint32_t k = 2 * threadIdx.x; k < B; k += 2 * blockDim.x) {
    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(ib + k));
    tile[k] = v.x;
    tile[k + 1] = v.y;
  }
  __syncthreads();
  uint64_t* ob = out + row * N + (size_t)t0;
  for (uint32_t k = 2 * threadIdx.x; k < B; k += 2 * blockDim.x) {
    ulonglong2 v;
    v.x = tile[src_of(t0 + k) & (B - 1)];
    v.y = tile[src_of(t0 + k + 1) & (B - 1)];
    __stcs(reinterpret_cast<ulonglong2*>(ob + k), v);
  }
}

// x mod p for arbitrary 64-bit words (after an integer all-reduce of residues).
__global__ void k_reduce(uint64_t* __restrict__ out, const uint64_t* __restrict__ in, size_t total,
                         int log_n, int limbs, RingDev R, LimbMap lm) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)((i >> log_n) % limbs);
    out[i] = ckb::reduce64(in[i], load_mod(R, lm.p[l]));
  }
}

// ---------------------------------------------------------------------------
// Counter-based sampling: Philox4x32-10 keyed by a per-item 64-bit
// seed, counter = (coefficient, limb, stream, 0).  Uniform residues take 128
// random bits reduced mod p (bias < 2^-60); the error is rint(sigma * z) with z
// from Box-Muller (ring.py:148-158 distributions).
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__global__ void k_sample(uint64_t* __restrict__ a, int64_t* __restrict__ e,
                         const uint64_t* __restrict__ seeds, int items, int limbs, int log_n,
                         double sigma, RingDev R, LimbMap lm) {
  const size_t N = (size_t)1 << log_n;
  const size_t total = (size_t)items * (limbs + 1) * N;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const uint32_t n = (uint32_t)(t & (N - 1));
    const size_t rj = t >> log_n;
    const int j = (int)(rj % (limbs + 1));
    const size_t it = rj / (limbs + 1);
    const uint64_t sd = __ldg(seeds + it);
    const uint2 key = make_uint2((uint32_t)sd, (uint32_t)(sd >> 32));
    if (j < limbs) {
      if (!a) continue;
      const uint4 r = philox(make_uint4(n, (uint32_t)j, 0u, 0u), key);
      const uint64_t hi = ((uint64_t)r.x << 32) | r.y, lo = ((uint64_t)r.z << 32) | r.w;
      const uint64_t* mm = R.mods + (size_t)lm.p[j] * kModStride;
      Mod m;
      m.p = __ldg(mm);
      m.mu = __ldg(mm + 1);
      m.k = __ldg(mm + 2);
      m.two_p = __ldg(mm + 3);
      a[(it * limbs + j) * N + n] = ckb::reduce128_any(hi & 0x3FFFFFFFFFFFFFFFull, lo, __ldg(mm + 8),
                                                       __ldg(mm + 9), m);
    } else {
      if (!e) continue;
      const uint4 r = philox(make_uint4(n, 0xFFFFFFFFu, 1u, 0u), key);
      const double u1 = ((double)((((uint64_t)r.x << 32) | r.y) >> 11) + 1.0) * 0x1.0p-53;
      const double u2 = (double)((((uint64_t)r.z << 32) | r.w) >> 11) * 0x1.0p-53;
      const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
      e[it * N + n] = (int64_t)rint(sigma * z);
    }
  }
}

// ===========================================================================
// Automorphism and conversions
// ===========================================================================

// out[t] = sign * in[src(t)] with src from galois^-1 mod 2N (gather form of
// ring.py:226-231's scatter).
__global__ void k_automorphism(uint64_t* __restrict__ out, const uint64_t* __restrict__ in,
                               size_t total, int log_n, int limbs, uint64_t ginv0,
                               const uint64_t* __restrict__ ginv_items, int rows_per_item,
                               RingDev R, LimbMap lm) {
  const uint64_t N = 1ull << log_n;
  const uint64_t mask2 = 2 * N - 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = i >> log_n;
    const uint64_t t = i & (N - 1);
    const uint64_t ginv = ginv_items ? __ldg(ginv_items + row / rows_per_item) : ginv0;
    const uint64_t sidx2 = (t * ginv) & mask2;
    const uint64_t p = __ldg(R.mods + (size_t)lm.p[row % limbs] * kModStride);
    const uint64_t* src = in + row * N;
    if (sidx2 < N) {
      out[i] = src[sidx2];
    } else {
      out[i] = ckb::neg_mod(src[sidx2 - N], p);
    }
  }
}

__global__ void k_from_i64(uint64_t* __restrict__ out, const int64_t* __restrict__ in,
                           size_t total, int log_n, int limbs, RingDev R, LimbMap lm) {
  const size_t N = (size_t)1 << log_n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = i >> log_n;
    const size_t poly = row / limbs;
    const int l = (int)(row % limbs);
    const int64_t v = in[poly * N + (i & (N - 1))];
    const Mod m = load_mod(R, lm.p[l]);
    if (v >= 0) {
      out[i] = ckb::reduce64((uint64_t)v, m);
    } else {
      const uint64_t mag = ckb::reduce64((uint64_t)(-(v + 1)) + 1, m);
      out[i] = mag == 0 ? 0 : m.p - mag;
    }
  }
}

// Encoder (encoding.py:34-49): slot scatter into the conjugate-symmetric
// spectrum, then — after the forward FFT (cuFFT) — the twist, rounding and the
// residues of every limb in one pass.  bins / conj_bins cover all N indices
// exactly once (the odd residues mod 2N are +-5^i), so the scatter writes every
// spectrum entry: no zero fill.
__global__ void k_embed_scatter(double2* __restrict__ spec, const double* __restrict__ values,
                                int batch, int width, size_t vstride, double scale,
                                const int32_t* __restrict__ bins, int log_n) {
  const size_t N = (size_t)1 << log_n;
  const size_t half = N >> 1;
  const size_t total = (size_t)batch * half;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t b = t / half, i = t % half;
    const double v = (int)i < width ? values[b * vstride + i] * scale : 0.0;
    double2* row = spec + b * N;
    row[__ldg(bins + i)] = make_double2(v, 0.0);
    row[__ldg(bins + half + i)] = make_double2(v, 0.0);
  }
}

__device__ __forceinline__ uint64_t i64_residue(int64_t v, const Mod& m) {
  if (v >= 0) return ckb::reduce64((uint64_t)v, m);
  const uint64_t mag = ckb::reduce64((uint64_t)(-(v + 1)) + 1, m);
  return mag == 0 ? 0 : m.p - mag;
}

__global__ void k_embed_finish(uint64_t* __restrict__ out, const double2* __restrict__ spec,
                               int batch, int limbs, int log_n, const double2* __restrict__ twist,
                               unsigned long long* __restrict__ maxabs, RingDev R, LimbMap lm) {
  const size_t N = (size_t)1 << log_n;
  const double inv_n = 1.0 / (double)N;
  const size_t total = (size_t)batch * N;
  double local = 0.0;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t b = t >> log_n, j = t & (N - 1);
    const double2 w = spec[t];
    const double2 tw = __ldg(twist + j);  // {cos(pi j / N), sin(pi j / N)}
    // Re((w / N) * conj(psi^j))
    const double c = rint(w.x * inv_n * tw.x + w.y * inv_n * tw.y);
    local = fmax(local, fabs(c));
    const int64_t v = (int64_t)c;  // |c| < 2^62 whenever the caller's bound check passes
    uint64_t* o = out + (b * limbs) * N + j;
    for (int l = 0; l < limbs; ++l) o[(size_t)l * N] = i64_residue(v, load_mod(R, lm.p[l]));
  }
  if (maxabs) {  // non-negative doubles order like their bit patterns
    for (int off = 16; off; off >>= 1) local = fmax(local, __shfl_xor_sync(0xffffffffu, local, off));
    if ((threadIdx.x & 31) == 0)
      atomicMax(maxabs, (unsigned long long)__double_as_longlong(local));
  }
}

// Garner mixed-radix digits, centered by comparing x/Q with 1/2, then the
// value is rebuilt exactly modulo 2^64 when it fits in 63 bits (the case for
// every decryptable phase) and approximately otherwise.
__global__ void k_to_f64(double* __restrict__ out, const uint64_t* __restrict__ in, int polys,
                         int limbs, int log_n, RingDev R, LimbMap lm) {
  const size_t N = (size_t)1 << log_n;
  const size_t total = (size_t)polys * N;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t n = t & (N - 1);
    const size_t poly = t >> log_n;
    const uint64_t* src = in + poly * limbs * N + n;
    uint64_t v[kMaxLimbs];
    for (int i = 0; i < limbs; ++i) {
      const int pi = lm.p[i];
      const Mod mi = load_mod(R, pi);
      uint64_t x = src[(size_t)i * N];
      for (int s = 0; s < i; ++s) {
        const int ps = lm.p[s];
        const uint64_t* pr = R.pair + ((size_t)ps * R.np + pi) * 4;
        x = ckb::sub_mod(x, ckb::reduce64(v[s], mi), mi.p);
        x = ckb::mul_shoup(x, __ldg(pr), __ldg(pr + 1), mi.p);
      }
      v[i] = x;
    }
    // fraction x / Q = sum_i v_i / (q_i * ... * q_{limbs-1}), Horner from digit 0
    double f = 0.0;
    for (int i = 0; i < limbs; ++i) {
      const double q = (double)__ldg(R.mods + (size_t)lm.p[i] * kModStride);
      f = ((double)v[i] + f) / q;
    }
    const bool negative = f > 0.5;
    double approx = 0.0;
    uint64_t exact = 0, prod = 1;
    for (int i = 0; i < limbs; ++i) {
      const uint64_t q = __ldg(R.mods + (size_t)lm.p[i] * kModStride);
      const uint64_t u = negative ? (q - 1 - v[i]) : v[i];
      exact += u * prod;
      prod *= q;
    }
    for (int i = limbs - 1; i >= 0; --i) {
      const uint64_t q = __ldg(R.mods + (size_t)lm.p[i] * kModStride);
      const uint64_t u = negative ? (q - 1 - v[i]) : v[i];
      approx = approx * (double)q + (double)u;
    }
    if (negative) {
      exact += 1;
      approx += 1.0;
    }
    double mag = (approx < 4.0e18) ? (double)exact : approx;
    out[t] = negative ? -mag : mag;
  }
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================

static uint64_t f64_bits(double d) {
  uint64_t u;
  memcpy(&u, &d, sizeof u);
  return u;
}


// ---------------------------------------------------------------------------
// Packed residue transfer format (host <-> device copies): limb l of an item
// stores each residue in w_l bytes (5 below 2^40, 6 below 2^48, else 8: the
// ckb_ring size classes), little-endian, the item's limbs back to back:
// item i, limb l at byte i*item_bytes + off_l*N.  A thread moves 8 residues
// (64 B unpacked, 8*w_l B = w_l words packed; all offsets 8-byte aligned).
// ---------------------------------------------------------------------------
struct PackMap {
  int16_t w[kMaxLimbs];    // bytes per residue
  int32_t off[kMaxLimbs];  // prefix sum of w (bytes per coefficient before limb l)
};

__global__ void k_pack(uint64_t* __restrict__ out, const uint64_t* __restrict__ in,
                       size_t groups, int log_n, int limbs, int item_w, PackMap pm) {
  const size_t N = (size_t)1 << log_n;
  const int gpr = (int)(N >> 3);  // 8-residue groups per row
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < groups;
       g += (size_t)gridDim.x * blockDim.x) {
    const size_t row = g / gpr;
    const int c = (int)(g - row * gpr);
    const size_t item = row / limbs;
    const int l = (int)(row - item * limbs);
    const int w = pm.w[l];
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(in + row * N + 8 * (size_t)c);
    uint64_t v[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const ulonglong2 t = __ldcs(src + k);
      v[2 * k] = t.x;
      v[2 * k + 1] = t.y;
    }
    uint64_t* dst = out + (item * (size_t)item_w * N + (size_t)pm.off[l] * N) / 8 + (size_t)c * w;
    if (w == 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dst[k] = v[k];
      continue;
    }
    // concatenate 8 values of 8w bits into w words
    unsigned __int128 acc = 0;
    int bits = 0, o = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc |= (unsigned __int128)v[k] << bits;
      bits += 8 * w;
      if (bits >= 64) {
        dst[o++] = (uint64_t)acc;
        acc >>= 64;
        bits -= 64;
      }
    }
  }
}

__global__ void k_unpack(uint64_t* __restrict__ out, const uint64_t* __restrict__ in,
                         size_t groups, int log_n, int limbs, int item_w, PackMap pm) {
  const size_t N = (size_t)1 << log_n;
  const int gpr = (int)(N >> 3);
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < groups;
       g += (size_t)gridDim.x * blockDim.x) {
    const size_t row = g / gpr;
    const int c = (int)(g - row * gpr);
    const size_t item = row / limbs;
    const int l = (int)(row - item * limbs);
    const int w = pm.w[l];
    const uint64_t* src = in + (item * (size_t)item_w * N + (size_t)pm.off[l] * N) / 8 + (size_t)c * w;
    uint64_t v[8];
    if (w == 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcs(src + k);
    } else {
      const uint64_t mask = (1ull << (8 * w)) - 1;
      unsigned __int128 acc = 0;
      int bits = 0, i = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (bits < 8 * w) {
          acc |= (unsigned __int128)__ldcs(src + i++) << bits;
          bits += 64;
        }
        v[k] = (uint64_t)acc & mask;
        acc >>= 8 * w;
        bits -= 8 * w;
      }
    }
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(out + row * N + 8 * (size_t)c);
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[k] = make_ulonglong2(v[2 * k], v[2 * k + 1]);
  }
}

static int make_packmap(PackMap& pm, const RingDev& R, const LimbMap& lm, int limbs) {
  int off = 0;
  for (int l = 0; l < limbs; ++l) {
    const int pi = lm.p[l];
    const bool wide = (R.wide_mask[pi >> 6] >> (pi & 63)) & 1;
    const bool mid = (R.mid_mask[pi >> 6] >> (pi & 63)) & 1;
    pm.w[l] = (int16_t)(wide ? 8 : mid ? 6 : 5);
    pm.off[l] = off;
    off += pm.w[l];
  }
  return off;
}

extern "C" {

int ckb_version(void) { return 1; }

int ckb_build_tables(uint32_t log_n, const uint64_t* primes, uint32_t np, uint64_t* mods_out,
                     uint64_t* ntt_out, uint64_t* pair_out) {
  if (log_n < 1 || log_n > 20 || np == 0 || !primes) return CKB_E_ARG;
  const uint64_t N = 1ull << log_n;
  for (uint32_t i = 0; i < np; ++i) {
    const uint64_t p = primes[i];
    if (p < 3 || (p >> 60) != 0 || (p - 1) % (2 * N) != 0) return CKB_E_ARG;  // < 2^60
    // psi: smallest g >= 2 with psi = g^((p-1)/2N) != 1 and psi^N == -1
    const uint64_t cof = (p - 1) / (2 * N);
    uint64_t psi = 0;
    for (uint64_t g = 2; g < 10000; ++g) {
      const uint64_t c = ckb::pow_mod_host(g, cof, p);
      if (c != 1 && ckb::pow_mod_host(c, N, p) == p - 1) {
        psi = c;
        break;
      }
    }
    if (!psi) return CKB_E_ARG;
    const uint64_t psi_inv = ckb::inv_mod_host(psi, p);
    // [N] forward then [N] inverse {w, shoup(w)} pairs, bit-reversed powers
    uint64_t* t = ntt_out + (size_t)i * 4 * N;
    uint64_t acc = 1, acc_inv = 1;
    for (uint64_t j = 0; j < N; ++j) {
      // bit-reverse j over log_n bits
      uint64_t r = 0;
      for (uint32_t b = 0; b < log_n; ++b) r |= ((j >> b) & 1ull) << (log_n - 1 - b);
      if ((p >> 46) == 0) {  // FP64 NTT path (csrc/ntt.cu): [N] double(w) per direction
        t[r] = f64_bits((double)acc);
        t[2 * N + r] = f64_bits((double)acc_inv);
      } else {
        t[2 * r] = acc;
        t[2 * r + 1] = ckb::shoup_of(acc, p);
        t[2 * N + 2 * r] = acc_inv;
        t[2 * N + 2 * r + 1] = ckb::shoup_of(acc_inv, p);
      }
      acc = ckb::mul_mod_host(acc, psi, p);
      acc_inv = ckb::mul_mod_host(acc_inv, psi_inv, p);
    }
    if ((p >> 46) == 0) {
      // second half of each direction: the same twiddles, with the entries of
      // the two bottom stages ([N/2, N): 8 per thread, [N/4, N/2): 4 per
      // thread) interleaved by 16-byte chunk inside every warp's block of
      // 256 / 128 so the row phase's vector loads are contiguous per warp
      // (ntt.cu load_tw_f64_perm): chunk c of lane l at block + 64 c + 2 l.
      for (int dir = 0; dir < 2; ++dir) {
        const uint64_t* w = t + (size_t)dir * 2 * N;
        uint64_t* q = t + (size_t)dir * 2 * N + N;
        for (uint64_t j = 0; j < N; ++j) q[j] = w[j];
        for (int nt = 8; nt >= 4 && N >= 512; nt >>= 1) {
          const uint64_t lo = nt == 8 ? N / 2 : N / 4, blk = 32 * (uint64_t)nt;
          for (uint64_t b0 = lo; b0 < 2 * lo; b0 += blk)
            for (uint64_t l = 0; l < 32; ++l)
              for (uint64_t e = 0; e < (uint64_t)nt; ++e)
                q[b0 + (e / 2) * 64 + 2 * l + (e & 1)] = w[b0 + nt * l + e];
        }
      }
    }
    const ckb::Mod m = ckb::make_mod(p);
    const uint64_t ninv = ckb::inv_mod_host(N % p, p);
    // inv_psi_brv[1] = psi^-(N/2) (bit-reversed index 1), times N^-1
    const uint64_t fold = ckb::mul_mod_host(ckb::pow_mod_host(psi_inv, N / 2, p), ninv, p);
    uint64_t* mo = mods_out + (size_t)i * kModStride;
    mo[0] = m.p;
    mo[1] = m.mu;
    mo[2] = m.k;
    mo[3] = m.two_p;
    mo[4] = ninv;
    mo[5] = ckb::shoup_of(ninv, p);
    mo[6] = fold;
    mo[7] = ckb::shoup_of(fold, p);
    const uint64_t r64 = (uint64_t)(((unsigned __int128)1 << 64) % p);
    mo[8] = r64;
    mo[9] = ckb::shoup_of(r64, p);
    const double pinv = 1.0 / (double)p;  // the FP64 kernels' 1/p (IEEE division, as on the device)
    memcpy(&mo[10], &pinv, sizeof(double));
    for (int z = 11; z < kModStride; ++z) mo[z] = 0;
  }
  for (uint32_t i = 0; i < np; ++i) {
    for (uint32_t j = 0; j < np; ++j) {
      uint64_t* pr = pair_out + ((size_t)i * np + j) * 4;
      const uint64_t pj = primes[j];
      const uint64_t pim = primes[i] % pj;
      const uint64_t inv = (i == j || pim == 0) ? 0 : ckb::inv_mod_host(pim, pj);
      pr[0] = inv;
      pr[1] = ckb::shoup_of(inv, pj);
      pr[2] = pim;
      pr[3] = 0;
    }
  }
  return 0;
}

int ckb_elementwise(const ckb_ring* ring, int op, uint64_t* out, const uint64_t* a,
                    const uint64_t* b, const uint64_t* c, int rows, int limbs,
                    const int32_t* limb_prime, int b_rows, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || rows < 0 || op < 0 || op > 4) return CKB_E_ARG;
  if ((op != 3 && !b) || (op == 4 && !c) || b_rows < 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = (size_t)rows << R.log_n;
  if (!total) return 0;
  const unsigned brows = (b_rows && b_rows < rows) ? (unsigned)b_rows : 0u;
  const size_t pairs = total / 2;
  const int grid = grid_for(pairs, 256);
  cudaStream_t st = (cudaStream_t)stream;
  switch (op) {
#define CKB_EW(OP)                                                                            \
  case OP:                                                                                    \
    k_elementwise<OP><<<grid, 256, 0, st>>>(out, a, b, c, pairs, brows, (int)R.log_n,       \
                                           (unsigned)limbs, R, lm);                         \
    break;
    CKB_EW(0) CKB_EW(1) CKB_EW(2) CKB_EW(3) CKB_EW(4)
#undef CKB_EW
  }
  return finish();
}

// out[poly][j] = sum_k a[k][j] * X_k[poly][j]  (mod q_j), j < limbs: a linear
// combination of ciphertexts with per-limb integer scalars (the leaves of the
// Chebyshev evaluation in bootstrapping: constant plaintexts are scalars).
// X_k: polys of pstride[k] >= limbs limbs (a ciphertext at a higher level is
// read restricted to its first limbs).  128-bit lazy sum, one reduction.
struct TermPtrs {
  const uint64_t* p[16];
  int pstride[16];
};

__global__ void __launch_bounds__(256) k_scalar_mac(uint64_t* __restrict__ out, TermPtrs tp,
                                                    const uint64_t* __restrict__ sc, int K,
                                                    size_t pairs, int log_n, int limbs,
                                                    RingDev R, LimbMap lm) {
  const int lh = log_n - 1;
  const size_t hmask = ((size_t)1 << lh) - 1;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < pairs;
       t += (size_t)gridDim.x * blockDim.x) {
    const unsigned row = (unsigned)(t >> lh);
    const size_t n = (t & hmask) * 2;
    const unsigned poly = row / (unsigned)limbs, j = row % (unsigned)limbs;
    uint64_t h0 = 0, l0 = 0, h1 = 0, l1 = 0;
    for (int k = 0; k < K; ++k) {
      const uint64_t a = __ldg(sc + (size_t)k * limbs + j);
      const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(
          tp.p[k] + (((size_t)poly * tp.pstride[k] + j) << log_n) + n);
      ckb::mac128(h0, l0, x.x, a);
      ckb::mac128(h1, l1, x.y, a);
    }
    const uint64_t* mm = R.mods + (size_t)lm.p[j] * kModStride;
    const Mod m{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
    const uint64_t r64 = __ldg(mm + 8), r64s = __ldg(mm + 9);
    *reinterpret_cast<ulonglong2*>(out + ((size_t)row << log_n) + n) =
        make_ulonglong2(ckb::reduce128_any(h0, l0, r64, r64s, m),
                        ckb::reduce128_any(h1, l1, r64, r64s, m));
  }
}

int ckb_scalar_mac(const ckb_ring* ring, uint64_t* out, const uint64_t* const* terms_host,
                   const int32_t* term_limbs, const uint64_t* scalars, int n_terms, int polys,
                   int limbs, const int32_t* limb_prime, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || polys < 0 || n_terms < 1 || n_terms > 16 || !scalars ||
      !terms_host || !term_limbs)
    return CKB_E_ARG;
  TermPtrs tp;
  for (int k = 0; k < n_terms; ++k) {
    if (!terms_host[k] || term_limbs[k] < limbs) return CKB_E_ARG;
    tp.p[k] = terms_host[k];
    tp.pstride[k] = term_limbs[k];
  }
  const RingDev R = make_ring(ring);
  const size_t pairs = (((size_t)polys * limbs) << R.log_n) / 2;
  if (!pairs) return 0;
  k_scalar_mac<<<grid_for(pairs, 256), 256, 0, (cudaStream_t)stream>>>(
      out, tp, scalars, n_terms, pairs, (int)R.log_n, limbs, R, lm);
  return finish();
}

int ckb_pt_mac(const ckb_ring* ring, uint64_t* out, const uint64_t* x0, const uint64_t* stack,
               int64_t stack_stride, const int32_t* term_idx, const uint64_t* pts,
               int64_t pt_stride, int n_terms, int rows, int limbs, const int32_t* limb_prime,
               void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || rows < 0 || n_terms < 1 || n_terms > 64 || !pts ||
      !term_idx || pt_stride < 0 || stack_stride < 0)
    return CKB_E_ARG;
  TermIdx ti;
  for (int k = 0; k < n_terms; ++k) {
    if (term_idx[k] < -1 || term_idx[k] > 32767) return CKB_E_ARG;
    if ((term_idx[k] < 0 && !x0) || (term_idx[k] >= 0 && !stack)) return CKB_E_ARG;
    ti.p[k] = (int16_t)term_idx[k];
  }
  const RingDev R = make_ring(ring);
  const size_t pairs = ((size_t)rows << R.log_n) / 2;
  if (!pairs) return 0;
  k_pt_mac<<<grid_for(pairs, 256), 256, 0, (cudaStream_t)stream>>>(
      out, x0, stack, (size_t)stack_stride, ti, pts, (size_t)pt_stride, n_terms, pairs,
      (int)R.log_n, (unsigned)limbs, R, lm);
  return finish();
}

int ckb_scalar_mul(const ckb_ring* ring, uint64_t* out, const uint64_t* a, int rows, int limbs,
                   const int32_t* limb_prime, const uint64_t* scalars_host, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || rows < 0 || !scalars_host) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  ScalarTab sc;  // host pairs {value, shoup(value)} per limb
  for (int l = 0; l < limbs; ++l) {
    sc.v[l] = scalars_host[2 * l];
    sc.s[l] = scalars_host[2 * l + 1];
  }
  const size_t total = (size_t)rows << R.log_n;
  if (!total) return 0;
  k_scalar_mul<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      out, a, total, (int)R.log_n, limbs, R, lm, sc);
  return finish();
}

int ckb_tensor(const ckb_ring* ring, uint64_t* out, const uint64_t* a, const uint64_t* b,
               int batch, int limbs, const int32_t* limb_prime, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || batch < 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = ((size_t)batch * limbs) << R.log_n;
  if (!total) return 0;
  if (R.log_n >= 1) {  // pairs never straddle a limb
    k_tensor2<<<grid_for(total / 2, 256), 256, 0, (cudaStream_t)stream>>>(out, a, b, total,
                                                                          (int)R.log_n, limbs, R,
                                                                          lm);
    return finish();
  }
  k_tensor<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(out, a, b, total,
                                                                    (int)R.log_n, limbs, R, lm);
  return finish();
}

int ckb_modup(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int64_t in_batch_stride,
              int batch, int limbs, const int32_t* limb_prime, int ext_limbs, const int32_t* ext_prime,
              int alpha, const uint64_t* bconv, int skip_own, void* stream) {
  LimbMap lm, em;
  if (!make_map(lm, limb_prime, limbs) || !make_map(em, ext_prime, ext_limbs)) return CKB_E_LIMBS;
  if (alpha < 1 || alpha > 16 || ext_limbs < limbs || batch < 0) return CKB_E_ARG;
  if (alpha > 1 && !bconv) return CKB_E_ARG;
  for (int i = 0; i < limbs; ++i)
    if (lm.p[i] != em.p[i]) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const int nd = (limbs + alpha - 1) / alpha;
  const size_t total = (size_t)batch << R.log_n;
  if (!total || !nd) return 0;
  const size_t bstride = in_batch_stride > 0 ? (size_t)in_batch_stride : ((size_t)limbs << R.log_n);
  // per-digit row stride; a short last digit (skip_own) keeps ext - width rows
  const int out_rows = skip_own ? ext_limbs - alpha : ext_limbs;
  const int item_rows = skip_own ? (nd - 1) * out_rows + ext_limbs - (limbs - (nd - 1) * alpha)
                                 : nd * ext_limbs;
  // exact digit width (a rounded-up template would multiply by zero constants)
  using KernT = decltype(&k_modup<1>);
  static const KernT kerns[17] = {nullptr,       k_modup<1>,  k_modup<2>,  k_modup<3>,
                                  k_modup<4>,    k_modup<5>,  k_modup<6>,  k_modup<7>,
                                  k_modup<8>,    k_modup<9>,  k_modup<10>, k_modup<11>,
                                  k_modup<12>,   k_modup<13>, k_modup<14>, k_modup<15>,
                                  k_modup<16>};
  const int amax = alpha;
  auto kern = kerns[alpha];
  // both pipes when some digit is all FP64-class primes and some output is too
  auto is_f64 = [&](int pi) { return (R.f64_mask[pi >> 6] >> (pi & 63)) & 1; };
  bool digit_f64 = false, out_f64 = false;
  for (int d = 0; d < nd && !digit_f64; ++d) {
    bool ok = true;
    for (int i = d * alpha; i < std::min(limbs, (d + 1) * alpha); ++i) ok &= is_f64(lm.p[i]);
    digit_f64 = ok;
  }
  for (int e = 0; e < ext_limbs; ++e) out_f64 |= is_f64(em.p[e]);
  {
    const int rc = tc_modup(R, out, in, bstride, batch, limbs, lm, ext_limbs, em, alpha, bconv,
                            skip_own, out_rows, item_rows, (cudaStream_t)stream);
    if (rc != 1) return rc;
  }
#ifndef CKB_MODUP_V1
  if (alpha > 1) {  // per-class output lists, two coefficients per thread
    using KernV = decltype(&k_modup_v2<2>);
    static const KernV vk[17] = {nullptr, nullptr, k_modup_v2<2>, k_modup_v2<3>, k_modup_v2<4>,
                                 k_modup_v2<5>, k_modup_v2<6>, k_modup_v2<7>, k_modup_v2<8>,
                                 k_modup_v2<9>, k_modup_v2<10>, k_modup_v2<11>, k_modup_v2<12>,
                                 k_modup_v2<13>, k_modup_v2<14>, k_modup_v2<15>, k_modup_v2<16>};
    const size_t vsmem = modup_v2_smem(ext_limbs, alpha);
    if (vsmem > 200 * 1024) return CKB_E_ARG;
    if (vsmem > 48 * 1024)
      cudaFuncSetAttribute(vk[alpha], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsmem);
    const size_t work = (size_t)batch << (R.log_n - 1);
    dim3 vgrid((unsigned)std::max<size_t>(1, std::min<size_t>((work + 255) / 256, 4096 / nd + 1)),
               (unsigned)nd);
    vk[alpha]<<<vgrid, 256, vsmem, (cudaStream_t)stream>>>(
        out, in, bstride, batch, limbs, ext_limbs, alpha, out_rows, item_rows, skip_own,
        (int)R.log_n, R, lm, em, bconv);
    return finish();
  }
#endif
  if (alpha > 1 && alpha <= 16 && digit_f64 && out_f64) {
    using KernM = decltype(&k_modup_mixed<2, false>);
#define CKB_MM(C)                                                                            \
  {nullptr, nullptr, k_modup_mixed<2, C>, k_modup_mixed<3, C>, k_modup_mixed<4, C>,          \
   k_modup_mixed<5, C>, k_modup_mixed<6, C>, k_modup_mixed<7, C>, k_modup_mixed<8, C>,       \
   k_modup_mixed<9, C>, k_modup_mixed<10, C>, k_modup_mixed<11, C>, k_modup_mixed<12, C>,    \
   k_modup_mixed<13, C>, k_modup_mixed<14, C>, k_modup_mixed<15, C>, k_modup_mixed<16, C>}
    static const KernM mk_u[17] = CKB_MM(false);
    static const KernM mk_c[17] = CKB_MM(true);
#undef CKB_MM
    const bool compact = item_rows != nd * out_rows;
    const KernM* mkerns = compact ? mk_c : mk_u;
    const size_t msmem = (6 * (size_t)ext_limbs + (size_t)alpha * (2 + 2 * (size_t)ext_limbs)) * 8 +
                         (size_t)alpha * ext_limbs * 16 + (size_t)ext_limbs * 8;
    if (msmem > 48 * 1024)
      cudaFuncSetAttribute(mkerns[alpha], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem);
    const size_t work = (size_t)batch << R.log_n;
    dim3 mgrid((unsigned)std::max<size_t>(1, std::min<size_t>((work + 255) / 256, 4096 / nd + 1)),
               (unsigned)nd);
    mkerns[alpha]<<<mgrid, 256, msmem, (cudaStream_t)stream>>>(
        out, in, bstride, batch, limbs, ext_limbs, alpha, nd, out_rows, skip_own, (int)R.log_n,
        item_rows, R, lm, em, bconv);
    return finish();
  }
  const size_t smem = (6 * (size_t)ext_limbs +
                       (amax == 1 ? 0 : (size_t)alpha * (2 + 2 * (size_t)ext_limbs))) * 8;
  const size_t work = (size_t)batch << (R.log_n - 1);
  dim3 grid((unsigned)std::max<size_t>(1, std::min<size_t>((work + 255) / 256, 4096 / nd + 1)),
            (unsigned)nd);
  kern<<<grid, 256, smem, (cudaStream_t)stream>>>(out, in, bstride, batch, limbs, ext_limbs,
                                                   alpha, item_rows, out_rows, skip_own,
                                                   (int)R.log_n,
                                                   R, lm, em, bconv);
  return finish();
}

int ckb_ks_inner_fold(const ckb_ring* ring, uint64_t* acc, const uint64_t* digits, int batch,
                      int n_digits, int ext_limbs, const int32_t* ext_prime, int alpha, int limbs,
                      const uint64_t* own, int64_t own_batch_stride, const uint64_t* key,
                      const uint64_t* const* key_ptrs, int key_limbs, const int32_t* key_limb,
                      const uint64_t* fold_b, int64_t fold_b_stride, const uint64_t* fold_a,
                      int64_t fold_a_stride, const uint64_t* fold_mul, int fold_limbs,
                      void* stream) {
  KsFold fold{fold_b, fold_a, (size_t)fold_b_stride, (size_t)fold_a_stride, fold_mul,
              fold_limbs};
  if (fold_b && (!fold_mul || fold_limbs < 1 || fold_limbs > ext_limbs || fold_b_stride < 0 ||
                 fold_a_stride < 0))
    return CKB_E_ARG;
  if (fold_b && n_digits > 8) return CKB_E_ARG;  // the generic kernel has no fold
  LimbMap em, km, od;
  if (!make_map(em, ext_prime, ext_limbs) || !make_map(km, key_limb, ext_limbs))
    return CKB_E_LIMBS;
  if (batch < 0 || n_digits < 1 || (!key && !key_ptrs) || alpha < 1) return CKB_E_ARG;
  if (own && (limbs > n_digits * alpha || limbs <= (n_digits - 1) * alpha)) return CKB_E_ARG;
  for (int e = 0; e < ext_limbs; ++e) od.p[e] = (int16_t)(e < limbs ? e / alpha : -1);
  const RingDev R = make_ring(ring);
  const size_t total = ((size_t)batch * ext_limbs) << R.log_n;
  if (!total) return 0;
  const int out_rows = own ? ext_limbs - alpha : ext_limbs;  // as written by ckb_modup
  const int item_rows = own ? (n_digits - 1) * out_rows + ext_limbs - (limbs - (n_digits - 1) * alpha)
                            : n_digits * ext_limbs;
  const size_t ob = own_batch_stride > 0 ? (size_t)own_batch_stride : ((size_t)limbs << R.log_n);
  const int grid = grid_for(total / 2, 256);
  cudaStream_t st = (cudaStream_t)stream;
#ifndef CKB_KS_PER_ITEM
  if (key && !key_ptrs && batch > 1 && n_digits <= 4) {  // one key: read it once per batch
    const size_t pairs = (size_t)ext_limbs << (R.log_n - 1);
    const int g = (int)std::min<size_t>((pairs + 255) / 256, 148 * 8);
#define CKB_KSS(ND)                                                                         \
  k_ks_inner_shared<ND><<<g, 256, 0, st>>>(acc, digits, batch, ext_limbs, out_rows,         \
                                           item_rows, alpha, limbs, own, ob, (int)R.log_n,  \
                                           key, key_limbs, R, em, km, od, fold)
    switch (n_digits) {
      case 1: CKB_KSS(1); break;
      case 2: CKB_KSS(2); break;
      case 3: CKB_KSS(3); break;
      default: CKB_KSS(4); break;
    }
#undef CKB_KSS
    return finish();
  }
#endif
#define CKB_KS(ND)                                                                           \
  k_ks_inner<ND><<<grid, 256, 0, st>>>(acc, digits, batch, n_digits, ext_limbs, out_rows,   \
                                       item_rows, alpha, limbs, own, ob, (int)R.log_n, key, \
                                       key_ptrs,                                            \
                                       key_limbs, R, em, km, od, fold)
  switch (n_digits) {
    case 1: CKB_KS(1); break;
    case 2: CKB_KS(2); break;
    case 3: CKB_KS(3); break;
    case 4: CKB_KS(4); break;
    case 6: CKB_KS(6); break;
    case 5: CKB_KS(5); break;
    case 8: CKB_KS(8); break;
    default:
      k_ks_inner_any<<<grid_for(total, 256), 256, 0, st>>>(
          acc, digits, batch, n_digits, ext_limbs, out_rows, item_rows, alpha, limbs, own, ob,
          (int)R.log_n, key,
          key_ptrs, key_limbs, R, em, km, od);
      break;
  }
#undef CKB_KS
  return finish();
}

int ckb_ks_inner(const ckb_ring* ring, uint64_t* acc, const uint64_t* digits, int batch,
                 int n_digits, int ext_limbs, const int32_t* ext_prime, int alpha, int limbs,
                 const uint64_t* own, int64_t own_batch_stride, const uint64_t* key,
                 const uint64_t* const* key_ptrs, int key_limbs, const int32_t* key_limb,
                 void* stream) {
  return ckb_ks_inner_fold(ring, acc, digits, batch, n_digits, ext_limbs, ext_prime, alpha,
                           limbs, own, own_batch_stride, key, key_ptrs, key_limbs, key_limb,
                           nullptr, 0, nullptr, 0, nullptr, 0, stream);
}

int ckb_divround(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int64_t in_poly_stride,
                 const uint64_t* addend, int addend_polys, int addend_period, int addend_stride,
                 int polys, int limbs, const int32_t* limb_prime, int n_drop1, int n_drop2,
                 const uint64_t* prescale_host, const uint64_t* tab1, const uint64_t* tab2,
                 void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs)) return CKB_E_LIMBS;
  if (n_drop1 < 0 || n_drop2 < 0 || n_drop1 > kMaxDrop || n_drop2 > kMaxDrop ||
      n_drop1 + n_drop2 >= limbs || polys < 0)
    return CKB_E_ARG;
  if ((n_drop1 && !tab1) || (n_drop2 && !tab2)) return CKB_E_ARG;
  if (addend && (addend_period < 1 || addend_polys < 0 || addend_polys > addend_period ||
                 addend_stride < addend_polys))
    return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  ScalarTab pre;
  int has_pre = 0;
  if (prescale_host) {
    has_pre = 1;
    for (int l = 0; l < limbs; ++l) {
      pre.v[l] = prescale_host[2 * l];
      pre.s[l] = prescale_host[2 * l + 1];
    }
  }
  const size_t total = (size_t)polys << R.log_n;
  if (!total) return 0;
  const size_t stride = in_poly_stride > 0 ? (size_t)in_poly_stride : ((size_t)limbs << R.log_n);
  const int d1 = n_drop1 == 0 ? 0 : n_drop1 <= 1 ? 1 : n_drop1 <= 2 ? 2 : n_drop1 <= 4 ? 4
               : n_drop1 <= 8 ? 8 : 16;
  const int d2 = n_drop2 == 0 ? 0 : n_drop2 <= 1 ? 1 : n_drop2 <= 2 ? 2 : 8;
  const int grid = grid_for(total, 256);
  cudaStream_t st = (cudaStream_t)stream;
#define CKB_DR(A, B)                                                                          \
  if (d1 == A && d2 == B) {                                                                   \
    k_divround<A, B><<<grid, 256, 0, st>>>(out, in, stride, addend, addend ? addend_polys : 0, \
                                           addend ? addend_period : 1,                        \
                                           addend ? addend_stride : 0, polys, limbs, n_drop1,  \
                                           n_drop2, (int)R.log_n, R, lm, pre, has_pre, tab1,   \
                                           tab2);                                              \
    return finish();                                                                           \
  }
  CKB_DR(0, 1) CKB_DR(0, 2) CKB_DR(0, 8)
  CKB_DR(1, 0) CKB_DR(1, 1) CKB_DR(1, 2) CKB_DR(1, 8)
  CKB_DR(2, 0) CKB_DR(2, 1) CKB_DR(2, 2) CKB_DR(2, 8)
  CKB_DR(4, 0) CKB_DR(4, 1) CKB_DR(4, 2) CKB_DR(4, 8)
  CKB_DR(8, 0) CKB_DR(8, 1) CKB_DR(8, 2) CKB_DR(8, 8)
  CKB_DR(16, 0) CKB_DR(16, 1) CKB_DR(16, 2)
#undef CKB_DR
  return CKB_E_ARG;
}

int ckb_automorphism(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int rows, int limbs,
                     const int32_t* limb_prime, uint64_t galois, const uint64_t* galois_inv_items,
                     int rows_per_item, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || rows < 0) return CKB_E_ARG;
  if (galois_inv_items ? rows_per_item < 1 : (galois & 1) == 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const uint64_t two_n = 2ull << R.log_n;
  // inverse of an odd galois element modulo a power of two (Newton iteration)
  uint64_t g = galois & (two_n - 1), inv = g;
  for (int it = 0; it < 6; ++it) inv *= 2 - g * inv;
  inv &= two_n - 1;
  const size_t total = (size_t)rows << R.log_n;
  if (!total) return 0;
  k_automorphism<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      out, in, total, (int)R.log_n, limbs, inv, galois_inv_items, rows_per_item, R, lm);
  return finish();
}

int64_t ckb_packed_bytes(const ckb_ring* ring, int items, int limbs, const int32_t* limb_prime) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || items < 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  PackMap pm;
  return (int64_t)items * make_packmap(pm, R, lm, limbs) * ((int64_t)1 << R.log_n);
}

int ckb_pack(const ckb_ring* ring, uint8_t* out, const uint64_t* in, int items, int limbs,
             const int32_t* limb_prime, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || items < 0 || !out || !in) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  if (R.log_n < 3) return CKB_E_LOGN;
  PackMap pm;
  const int item_w = make_packmap(pm, R, lm, limbs);
  const size_t groups = ((size_t)items * limbs) << (R.log_n - 3);
  if (!groups) return 0;
  k_pack<<<grid_for(groups, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<uint64_t*>(out), in, groups, (int)R.log_n, limbs, item_w, pm);
  return finish();
}

int ckb_unpack(const ckb_ring* ring, uint64_t* out, const uint8_t* in, int items, int limbs,
               const int32_t* limb_prime, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || items < 0 || !out || !in) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  if (R.log_n < 3) return CKB_E_LOGN;
  PackMap pm;
  const int item_w = make_packmap(pm, R, lm, limbs);
  const size_t groups = ((size_t)items * limbs) << (R.log_n - 3);
  if (!groups) return 0;
  k_unpack<<<grid_for(groups, 256), 256, 0, (cudaStream_t)stream>>>(
      out, reinterpret_cast<const uint64_t*>(in), groups, (int)R.log_n, limbs, item_w, pm);
  return finish();
}

int ckb_from_i64(const ckb_ring* ring, uint64_t* out, const int64_t* in, int polys, int limbs,
                 const int32_t* limb_prime, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || polys < 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = ((size_t)polys * limbs) << R.log_n;
  if (!total) return 0;
  k_from_i64<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(out, in, total, (int)R.log_n,
                                                                      limbs, R, lm);
  return finish();
}

int ckb_embed_scatter(double* spec, const double* values, int batch, int width,
                      int64_t values_stride, double scale, const int32_t* bins, int log_n,
                      void* stream) {
  if (batch < 0 || width < 0 || width > (1 << (log_n - 1)) || log_n < 1 || log_n > 20 ||
      !spec || !bins || (width && !values))
    return CKB_E_ARG;
  const size_t total = (size_t)batch << (log_n - 1);
  if (!total) return 0;
  k_embed_scatter<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<double2*>(spec), values, batch, width,
      values_stride > 0 ? (size_t)values_stride : (size_t)width, scale, bins, log_n);
  return finish();
}

int ckb_embed_finish(const ckb_ring* ring, uint64_t* out, const double* spec, int batch,
                     int limbs, const int32_t* limb_prime, const double* twist, uint64_t* maxabs,
                     void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || batch < 0 || !out || !spec || !twist) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = (size_t)batch << R.log_n;
  if (!total) return 0;
  k_embed_finish<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      out, reinterpret_cast<const double2*>(spec), batch, limbs, (int)R.log_n,
      reinterpret_cast<const double2*>(twist), reinterpret_cast<unsigned long long*>(maxabs), R,
      lm);
  return finish();
}

int ckb_to_f64(const ckb_ring* ring, double* out, const uint64_t* in, int polys, int limbs,
               const int32_t* limb_prime, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || polys < 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = (size_t)polys << R.log_n;
  if (!total) return 0;
  k_to_f64<<<grid_for(total, 128), 128, 0, (cudaStream_t)stream>>>(out, in, polys, limbs,
                                                                    (int)R.log_n, R, lm);
  return finish();
}


int ckb_divround_ntt_corr(const ckb_ring* ring, uint64_t* E, const uint64_t* T, int has_addend,
                          int polys, int limbs, const int32_t* limb_prime, int n_drop1,
                          int n_drop2, const uint64_t* tab1, const uint64_t* tab2,
                          const uint64_t* tabE, const uint64_t* tabH, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs)) return CKB_E_LIMBS;
  if (n_drop1 < 0 || n_drop2 < 0 || n_drop1 > kMaxDrop || n_drop2 > kMaxDrop ||
      n_drop1 + n_drop2 >= limbs || n_drop1 + n_drop2 == 0 || polys < 0 || !tabE)
    return CKB_E_ARG;
  if ((n_drop1 && !tab1) || (n_drop2 && !tab2)) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = (size_t)polys << R.log_n;
  if (!total) return 0;
  // register arrays are sized by D1: exact widths for the special-prime
  // counts of the configs (6: config 2, 11: configs 3/4, 13: config 5)
  const int d1 = n_drop1 == 0 ? 0 : n_drop1 <= 1 ? 1 : n_drop1 <= 2 ? 2 : n_drop1 <= 4 ? 4
               : n_drop1 <= 6 ? 6 : n_drop1 <= 8 ? 8 : n_drop1 <= 11 ? 11 : n_drop1 <= 13 ? 13
               : 16;
  const int d2 = n_drop2 == 0 ? 0 : n_drop2 <= 1 ? 1 : n_drop2 <= 2 ? 2 : 8;
  cudaStream_t st0 = (cudaStream_t)stream;
  if (tabH && n_drop1 >= kHpsMinDrop && n_drop2 <= 2) {  // fast basis-conversion form
    const int rc = tc_corr(R, E, T, has_addend, polys, limbs, lm, n_drop1, n_drop2, tab1, tab2,
                           tabE, tabH, (R.flags & CKB_RING_HPS_EXACT) ? 0.0 : kHpsMargin, st0);
    if (rc != 1) return rc;
    const int m2h = limbs - n_drop1 - n_drop2;
    const size_t smh = (size_t)m2h * (6 + 2 * (n_drop1 + n_drop2 + 1) + n_drop1) * 8 +
                       4 * kMaxDrop * 8;
    if (smh > 200 * 1024) return CKB_E_ARG;
#define CKB_DH(A, B)                                                                        \
  if (d1 == A && d2 == B) {                                                                 \
    constexpr int VV = A <= CKB_CORR_VV2_MAX ? 2 : 1; /* two coefficients per thread */    \
    if (smh > 48 * 1024)                                                                    \
      cudaFuncSetAttribute(k_divround_corr_hps<A, B, VV>,                                   \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smh);          \
    k_divround_corr_hps<A, B, VV><<<grid_for(total / VV, 256), 256, smh, st0>>>(            \
        E, T, has_addend, polys, limbs, n_drop1, n_drop2, (int)R.log_n, R, lm, tab1, tab2,  \
        tabE, tabH, (R.flags & CKB_RING_HPS_EXACT) ? 0.0 : kHpsMargin);                                                          \
    return finish();                                                                        \
  }
    CKB_DH(6, 0) CKB_DH(6, 1) CKB_DH(6, 2) CKB_DH(8, 0) CKB_DH(8, 1) CKB_DH(8, 2)
    CKB_DH(11, 0) CKB_DH(11, 1) CKB_DH(11, 2) CKB_DH(13, 0) CKB_DH(13, 1) CKB_DH(13, 2)
    CKB_DH(16, 0) CKB_DH(16, 1) CKB_DH(16, 2)
#undef CKB_DH
  }
  const bool one = n_drop1 >= 11;  // wide drops: one coefficient per thread
  const int grid = grid_for(one ? total : total / 2, 256);
  cudaStream_t st = (cudaStream_t)stream;
  const int m2 = limbs - n_drop1 - n_drop2;
  const size_t smem = (size_t)m2 * (6 + 2 * (n_drop1 + n_drop2 + 1)) * 8;
  if (smem > 200 * 1024) return CKB_E_ARG;
#define CKB_DC_V(A, B, V)                                                                   \
  {                                                                                         \
    if (smem > 48 * 1024)                                                                   \
      cudaFuncSetAttribute(k_divround_corr<A, B, V>,                                        \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
    k_divround_corr<A, B, V><<<grid, 256, smem, st>>>(E, T, has_addend, polys, limbs,       \
                                                     n_drop1, n_drop2, (int)R.log_n, R, lm, \
                                                     tab1, tab2, tabE);                     \
    return finish();                                                                        \
  }
#define CKB_DC(A, B)                                                                        \
  if (d1 == A && d2 == B) {                                                                 \
    if constexpr (A >= 11) {                                                                \
      if (one) CKB_DC_V(A, B, 1)                                                            \
    }                                                                                       \
    CKB_DC_V(A, B, 2)                                                                       \
  }
  CKB_DC(0, 1) CKB_DC(0, 2) CKB_DC(0, 8)
  CKB_DC(1, 0) CKB_DC(1, 1) CKB_DC(1, 2) CKB_DC(1, 8)
  CKB_DC(2, 0) CKB_DC(2, 1) CKB_DC(2, 2) CKB_DC(2, 8)
  CKB_DC(4, 0) CKB_DC(4, 1) CKB_DC(4, 2) CKB_DC(4, 8)
  CKB_DC(6, 0) CKB_DC(6, 1) CKB_DC(6, 2)
  CKB_DC(8, 0) CKB_DC(8, 1) CKB_DC(8, 2) CKB_DC(8, 8)
  CKB_DC(11, 0) CKB_DC(11, 1) CKB_DC(11, 2)
  CKB_DC(13, 0) CKB_DC(13, 1) CKB_DC(13, 2)
  CKB_DC(16, 0) CKB_DC(16, 1) CKB_DC(16, 2)
#undef CKB_DC
#undef CKB_DC_V
  return CKB_E_ARG;
}

int ckb_divround_ntt_combine(const ckb_ring* ring, uint64_t* out, const uint64_t* x,
                             int64_t x_poly_stride, const uint64_t* addend, int addend_polys,
                             int addend_period, int addend_stride, const uint64_t* E, int polys,
                             int limbs, const int32_t* limb_prime, int n_drop1, int n_drop2,
                             const uint64_t* tab1, const uint64_t* tab2, void* stream) {
  return ckb_divround_ntt_combine_acc(ring, out, x, x_poly_stride, addend, addend_polys,
                                      addend_period, addend_stride, E, polys, limbs, limb_prime,
                                      n_drop1, n_drop2, tab1, tab2, nullptr, 0, stream);
}

int ckb_divround_ntt_combine_acc(const ckb_ring* ring, uint64_t* out, const uint64_t* x,
                                 int64_t x_poly_stride, const uint64_t* addend, int addend_polys,
                                 int addend_period, int addend_stride, const uint64_t* E,
                                 int polys, int limbs, const int32_t* limb_prime, int n_drop1,
                                 int n_drop2, const uint64_t* tab1, const uint64_t* tab2,
                                 const uint64_t* post, int64_t post_poly_stride, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs)) return CKB_E_LIMBS;
  if (n_drop1 < 0 || n_drop2 < 0 || n_drop1 + n_drop2 >= limbs || polys < 0 || !E)
    return CKB_E_ARG;
  if ((n_drop1 && !tab1) || (n_drop2 && !tab2)) return CKB_E_ARG;
  if (addend && (addend_period < 1 || addend_polys < 0 || addend_polys > addend_period ||
                 addend_stride < addend_polys))
    return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const int m2 = limbs - n_drop1 - n_drop2;
  const size_t total = ((size_t)polys * m2) << R.log_n;
  if (!total) return 0;
  const size_t xs = x_poly_stride > 0 ? (size_t)x_poly_stride : ((size_t)limbs << R.log_n);
  const size_t rows = (size_t)polys * (limbs - n_drop1 - n_drop2);
  const size_t pairs = (size_t)1 << (R.log_n - 1);
  dim3 grid((unsigned)std::max<size_t>(1, std::min<size_t>((pairs + 255) / 256, 64)),
            (unsigned)std::min<size_t>(rows, 65535));
  k_divround_combine<<<grid, 256, 0, (cudaStream_t)stream>>>(
      out, x, xs, addend, addend ? addend_polys : 0, addend ? addend_period : 1,
      addend ? addend_stride : 0, E, polys, limbs, n_drop1, n_drop2, (int)R.log_n, R, lm, tab1,
      tab2, post,
      post_poly_stride > 0 ? (size_t)post_poly_stride : ((size_t)m2 << R.log_n));
  return finish();
}

int ckb_automorphism_ntt(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int rows,
                         uint64_t galois, const uint64_t* galois_items, int rows_per_item,
                         void* stream) {
  if (rows < 0) return CKB_E_ARG;
  if (galois_items ? rows_per_item < 1 : (galois & 1) == 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = (size_t)rows << R.log_n;
  if (!total) return 0;
#ifndef CKB_AUT_GATHER
  if (R.log_n >= 1) {
    const int lb = std::min(kAutLogBlock, (int)R.log_n);
    const size_t blocks = (size_t)rows << (R.log_n - lb);
    k_automorphism_ntt_blk<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        out, in, (int)R.log_n, galois, galois_items, rows_per_item);
    return finish();
  }
#endif
  k_automorphism_ntt<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      out, in, total, (int)R.log_n, galois, galois_items, rows_per_item);
  return finish();
}

int ckb_reduce(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int rows, int limbs,
               const int32_t* limb_prime, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || rows < 0) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = (size_t)rows << R.log_n;
  if (!total) return 0;
  k_reduce<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(out, in, total, (int)R.log_n,
                                                                    limbs, R, lm);
  return finish();
}

int ckb_sample(const ckb_ring* ring, uint64_t* a, int64_t* e, const uint64_t* seeds, int items,
               int limbs, const int32_t* limb_prime, double sigma, void* stream) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || items < 0 || !seeds) return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const size_t total = ((size_t)items * (limbs + 1)) << R.log_n;
  if (!total) return 0;
  k_sample<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(a, e, seeds, items, limbs,
                                                                    (int)R.log_n, sigma, R, lm);
  return finish();
}

}  // extern "C"
