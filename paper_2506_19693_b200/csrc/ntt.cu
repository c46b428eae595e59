// Negacyclic NTT kernels (sm_100a): replaces NttPlan.forward/inverse
// (/root/reference/pkg/src/ciphermlp/ckks/ntt.py:121-154).
#include <cstdlib>

#include "common.cuh"
#include "fp64.cuh"

using namespace ckb_internal;
using namespace ckb_f64;

// Two register-round shapes (measured on B200, tools/ntt_micro.py):
//  * single phase (N <= 4096): radix-16 rounds, one 4096-element limb per CTA,
//    256 threads at an 80-register budget (3 CTAs/SM);
//  * two phases (N > 4096): radix-8 rounds, 2048-element tiles, 256 threads at
//    a 64-register budget (4 CTAs/SM) — 12% faster than radix-16 at N=2^16.
constexpr int kNttThreads = 256;
constexpr int kTwoPhaseTile = 2048;
using ckb::Mod;

namespace {

// ===========================================================================
// NTT
//
// A length-N negacyclic transform is run as one or two "phases".  A phase
// applies S = log2(G) consecutive radix-2 stages to independent groups of G
// elements, element (g, r) living at g*gstride + r*rstride of its limb:
//   * single phase (N <= 4096): one group = the whole limb;
//   * two phases (N > 4096): phase A = strided columns (the high stages of the
//     forward transform), phase B = contiguous rows (the low stages).
// Inside a CTA the tile (C groups x G) is staged in shared memory; each thread
// keeps 16 elements in registers and applies up to 4 stages per round
// (radix-16), with one smem exchange between rounds.  Butterflies are the
// Harvey lazy forms with Shoup twiddles and a 3-multiply quotient estimate:
// forward values live in [0, 8p), inverse values in [0, 4p) (see
// ntt_mul_lazy), and the last phase canonicalises.
// Twiddle of stage bit b for element r in group gidx (derivation in DESIGN.md):
//   idx = ((M0 + gt*gidx) << (S-1-b)) + (r >> (b+1))
// ===========================================================================

struct NttPhase {
  int limbs;
  int tiles_per_row;
  int C;        // groups per CTA
  int gstride;  // element stride between groups
  int rstride;  // element stride inside a group
  int M0;
  int gt;
  int last;     // forward: canonicalise; inverse: fold N^-1 into the top stage
  int row0;     // first row handled by this launch (for L2-resident chunking)
  int logC;     // log2(C)
  int items;    // > 0: rows enumerated limb-major (rows = items * limbs)
  int first;    // first phase of the transform: input is canonical uint64
                // (the FP64 path keeps doubles between the two phases)
  const uint64_t* src;  // out-of-place first phase: row (item i, limb l) is read
  size_t src_istride;   // from src + i*src_istride + l*N (NULL: in place)
  // block decode without integer divisions (set by prep_phase): tiles_per_row
  // is a power of two, rows split into (item, limb) by a multiply-high
  int log_tpr;
  uint32_t items_magic, limbs_magic;  // 0: divide
  int pf_dist;  // first phases: L2-prefetch the tile of block + pf_dist (0: off)
};

// floor(x / d) for 0 <= x <= max_x as __umulhi(x, magic): magic = floor(2^32/d)+1
// is exact while x * d < 2^32; 0 when that cannot be guaranteed.
inline uint32_t div_magic(int d, long long max_x) {
  if (d <= 1 || max_x * (long long)d >= (1ll << 32)) return 0;
  return (uint32_t)((1ull << 32) / (uint32_t)d) + 1;
}

__device__ __forceinline__ int fast_div(int x, int d, uint32_t magic) {
  return magic ? (int)__umulhi((uint32_t)x, magic) : x / d;
}

// Optional epilogue of a forward transform's last phase: the ModDown /
// rescale combine (ckb_divround_ntt_combine) applied to the transformed
// correction polynomial E as it is stored, so E never goes back to HBM:
//   out_j = ((x_j * P1^-1 + add_j - E_j) * P2^-1) + post_j   (mod q_j)
// The transformed rows are E's: row = poly * m2 + j.
struct CombineEp {
  uint64_t* out;  // NULL: no epilogue
  const uint64_t* x;
  size_t xs;      // x poly stride (elements)
  const uint64_t* add;
  int add_polys, add_period, add_stride, m1;
  const uint64_t* tab1;
  const uint64_t* tab2;
  int n1, n2;
  const uint64_t* post;
  size_t post_stride;
};

// Shared-memory slot of element r of group g: one pad word per 16 elements
// keeps the register rounds (r = w + 16k, r = 16w + k, ...) conflict-free, and
// the G/128 extra words of group stride spread the column phase's tile I/O
// (lanes = 4 rows x 4 column pairs) over distinct banks.  Chosen by
// enumerating every shared access pattern of the two-phase kernels (an XOR
// swizzle that is fully conflict-free costs more ALU issue than it saves).
template <int S>
__device__ __forceinline__ int sidx(int g, int r) {
  constexpr int G = 1 << S;
  return g * (G + G / 16 + G / 128) + r + (r >> 4);
}

// Slot offset of element k of a thread's register set: rbase has zero bits in
// [WLO, WLO+RB), so r = rbase + (k << WLO) adds without carries and
// sidx(g, r) = sidx(g, rbase) + koff(k), a compile-time constant per k.
template <int WLO>
__device__ __forceinline__ constexpr int koff(int k) {
  return (k << WLO) + ((k << WLO) >> 4);
}

// Barrier between register rounds: when a group's G/E threads fit in one warp
// (G/E <= 32), a warp only exchanges data with itself through shared memory.
template <int S, int RB>
__device__ __forceinline__ void round_sync() {
  if constexpr ((1 << (S - RB)) <= 32) {
    __syncwarp();
  } else {
    __syncthreads();
  }
}

// Integer butterflies.  The Shoup quotient q = hi64(x * ws) costs four 32-bit
// multiplies; the butterfly is bound by the multiplier pipe (ten per product),
// so the NTT estimates it with three, dropping the low x low partial product
// and the carries of the two cross products' low halves:
//   q' = xh wsh + hi32(xh wsl) + hi32(xl wsh)  in [q - 2, q],
// so x w - q' p lies in [0, 4p) instead of [0, 2p) (any x < 2^64).  The lazy
// ranges widen by one bit to absorb it at no extra instruction: forward values
// live in [0, 8p), inverse values in [0, 4p) (p < 2^60, ckb_build_tables).
// kLz = 2: the bound of a reduced value is 4p (CKB_NTT_SHOUP4: the exact
// quotient and the [0, 4p) / [0, 2p) ranges, kLz = 1).
#ifdef CKB_NTT_SHOUP4
constexpr int kLz = 1;
__device__ __forceinline__ uint64_t ntt_mul_lazy(uint64_t x, uint64_t w, uint64_t ws, uint64_t p) {
  return ckb::mul_shoup_lazy(x, w, ws, p);
}
#else
constexpr int kLz = 2;
__device__ __forceinline__ uint64_t ntt_mul_lazy(uint64_t x, uint64_t w, uint64_t ws, uint64_t p) {
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
  const uint32_t sl = (uint32_t)ws, sh = (uint32_t)(ws >> 32);
  const uint64_t q = (uint64_t)xh * sh + __umulhi(xh, sl) + __umulhi(xl, sh);
#ifdef CKB_NTT_MUL_PLAIN
  return x * w - q * p;
#else
  // x w + q (-p) mod 2^64 as two wide multiply-adds for the low words and four
  // 32-bit multiply-adds into the high word (no negation, no 64-bit add chain)
  const uint64_t np = 0 - p;  // loop-invariant
  const uint32_t wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
  const uint32_t ql = (uint32_t)q, qh = (uint32_t)(q >> 32);
  const uint32_t nl = (uint32_t)np, nh = (uint32_t)(np >> 32);
  const uint64_t t = (uint64_t)xl * wl + (uint64_t)ql * nl;
  const uint32_t hi = (uint32_t)(t >> 32) + xh * wl + xl * wh + qh * nl + ql * nh;
  return ((uint64_t)hi << 32) | (uint32_t)t;
#endif
}
#endif

// Harvey forward (CT) butterfly, values in [0, 2 lz): lz = kLz * 2p.
// RED = false (kLz == 2 only): the conditional subtraction of X is skipped.
// Both outputs carry X's bound plus lz (the product side absorbs any Y), and
// p < 2^60 leaves room for 16p: alternating stages reduce X from [0, 16p) to
// [0, 8p) (outputs < 12p) and skip the reduction (inputs < 12p, outputs
// < 16p), which halves the compare/select work of the forward transform.
template <bool RED = true>
__device__ __forceinline__ void ct_bfly(uint64_t& X, uint64_t& Y, uint64_t W, uint64_t Ws,
                                        uint64_t p, uint64_t lz) {
  uint64_t a = X;
  if constexpr (RED) a = X >= lz ? X - lz : X;
  const uint64_t t = ntt_mul_lazy(Y, W, Ws, p);
  X = a + t;
  Y = a - t + lz;
}

// Harvey inverse (GS) butterfly, values in [0, lz).
__device__ __forceinline__ void gs_bfly(uint64_t& X, uint64_t& Y, uint64_t W, uint64_t Ws,
                                        uint64_t p, uint64_t lz) {
  uint64_t sum = X + Y;
  sum = sum >= lz ? sum - lz : sum;
  const uint64_t d = X - Y + lz;
  X = sum;
  Y = ntt_mul_lazy(d, W, Ws, p);
}

// The same butterfly with bound tracking (kLz == 2; b = 4p is the bound of a
// product).  Values live in [0, 2b); FRESH: both inputs are products of the
// previous stage (< b), so the sum (< 2b) needs no reduction and the difference
// is offset by b instead of 2b.  Inside a register round the inputs of a
// butterfly share their history, so FRESH is a compile-time property of the
// element index: 3/8 of the butterflies skip the compare/select.
template <bool FRESH>
__device__ __forceinline__ void gs_bfly_t(uint64_t& X, uint64_t& Y, uint64_t W, uint64_t Ws,
                                          uint64_t p, uint64_t b) {
  uint64_t sum = X + Y;
  if constexpr (!FRESH) sum = sum >= 2 * b ? sum - 2 * b : sum;
  const uint64_t d = X - Y + (FRESH ? b : 2 * b);
  X = sum;
  Y = ntt_mul_lazy(d, W, Ws, p);
}

// One radix-16 round: the thread's 16 elements differ in bits [WLO, WLO+4) of
// r; stages b in (HI-1 .. LO) for the forward, (LO .. HI-1) for the inverse.
// The twiddle of the butterfly at k is tw[t0(b) + (k >> (bb+1))]: only
// 1, 2, 4, 8 distinct values per stage, loaded once each.
template <int S, int RB, int HI>
__device__ __forceinline__ void fwd_rounds(uint64_t* s, const ulonglong2* __restrict__ tw,
                                           uint64_t p,
                                           uint64_t two_p, int gq, int tbase, int w, int last) {
  if constexpr (HI > 0) {
    constexpr int E = 1 << RB;  // elements per thread
    constexpr int Q = HI < RB ? HI : RB;
    constexpr int LO = HI - Q;
    constexpr int WLO = HI - RB > 0 ? HI - RB : 0;
    const int rbase = (w & ((1 << WLO) - 1)) | ((w >> WLO) << (WLO + RB));
    uint64_t x[E];
    uint64_t* sb = s + sidx<S>(gq, rbase);
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = sb[koff<WLO>(k)];
#pragma unroll
    for (int b = HI - 1; b >= LO; --b) {
      const int bb = b - WLO;
      const int t0 = (tbase << (S - 1 - b)) + (rbase >> (b + 1));
      uint64_t Wv[E / 2], Wsv[E / 2];
#pragma unroll
      for (int i = 0; i < E / 2; ++i) {
        if (i < ((E / 2) >> bb)) {
          const ulonglong2 wp = __ldg(tw + t0 + i);  // {w, shoup(w)}
          Wv[i] = wp.x;
          Wsv[i] = wp.y;
        }
      }
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << bb)) continue;
        const int i = k >> (bb + 1);
#if defined(CKB_NTT_SHOUP4) || defined(CKB_NTT_CT_REDUCE_ALL)
        ct_bfly(x[k], x[k | (1 << bb)], Wv[i], Wsv[i], p, kLz * two_p);
#else
        // stage i = S-1-b of the phase: even stages reduce X by 8p (inputs
        // < 16p: a phase may end on a skipping stage), odd stages skip
        if (((S - 1 - b) & 1) == 0) {
          uint64_t& X = x[k];
          X = X >= 4 * two_p ? X - 4 * two_p : X;
        }
        ct_bfly<false>(x[k], x[k | (1 << bb)], Wv[i], Wsv[i], p, 2 * two_p);
#endif
      }
    }
    if (LO == 0 && last) {
#pragma unroll
      for (int k = 0; k < E; ++k) {
        uint64_t X = x[k];
#if !defined(CKB_NTT_SHOUP4) && !defined(CKB_NTT_CT_REDUCE_ALL)
        X = X >= 4 * two_p ? X - 4 * two_p : X;
#endif
        if (kLz == 2) X = X >= 2 * two_p ? X - 2 * two_p : X;
        X = X >= two_p ? X - two_p : X;
        x[k] = X >= p ? X - p : X;
      }
    }
#pragma unroll
    for (int k = 0; k < E; ++k) sb[koff<WLO>(k)] = x[k];
    round_sync<S, RB>();
    fwd_rounds<S, RB, LO>(s, tw, p, two_p, gq, tbase, w, last);
  }
}

template <int S, int RB, int LO>
__device__ __forceinline__ void inv_rounds(uint64_t* s, const ulonglong2* __restrict__ tw,
                                           uint64_t p,
                                           uint64_t two_p, uint64_t ninv, uint64_t ninvs,
                                           uint64_t fw, uint64_t fws, int gq, int tbase, int w,
                                           int last) {
  if constexpr (LO < S) {
    constexpr int E = 1 << RB;
    constexpr int Q = (S - LO) < RB ? (S - LO) : RB;
    constexpr int HI = LO + Q;
    constexpr int WLO = LO < S - RB ? LO : S - RB;
    const int rbase = (w & ((1 << WLO) - 1)) | ((w >> WLO) << (WLO + RB));
    uint64_t x[E];
    uint64_t* sb = s + sidx<S>(gq, rbase);
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = sb[koff<WLO>(k)];
#pragma unroll
    for (int b = LO; b < HI; ++b) {
      const int bb = b - WLO;
      if (b == S - 1 && last) {
        // top stage of the whole transform with N^-1 folded in
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (k & (1 << bb)) continue;
          const uint64_t X = x[k], Y = x[k | (1 << bb)];
#if defined(CKB_NTT_SHOUP4) || defined(CKB_NTT_GS_REDUCE_ALL)
          uint64_t sum = X + Y;
          sum = sum >= kLz * two_p ? sum - kLz * two_p : sum;
          x[k] = ckb::mul_shoup(sum, ninv, ninvs, p);
          x[k | (1 << bb)] = ckb::mul_shoup(X - Y + kLz * two_p, fw, fws, p);
#else
          // inputs < 8p: the exact Shoup products take any 64-bit operand
          x[k] = ckb::mul_shoup(X + Y, ninv, ninvs, p);
          x[k | (1 << bb)] = ckb::mul_shoup(X - Y + 4 * two_p, fw, fws, p);
#endif
        }
      } else {
        const int t0 = (tbase << (S - 1 - b)) + (rbase >> (b + 1));
        uint64_t Wv[E / 2], Wsv[E / 2];
#pragma unroll
        for (int i = 0; i < E / 2; ++i) {
          if (i < ((E / 2) >> bb)) {
            const ulonglong2 wp = __ldg(tw + t0 + i);
            Wv[i] = wp.x;
            Wsv[i] = wp.y;
          }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (k & (1 << bb)) continue;
          const int i = k >> (bb + 1);
#if defined(CKB_NTT_SHOUP4) || defined(CKB_NTT_GS_REDUCE_ALL)
          gs_bfly(x[k], x[k | (1 << bb)], Wv[i], Wsv[i], p, kLz * two_p);
#else
          // fresh: not the round's first stage, and the element was on the
          // product side of the previous stage (bit bb-1 of k)
          if (b > LO && ((k >> (bb > 0 ? bb - 1 : 0)) & 1))
            gs_bfly_t<true>(x[k], x[k | (1 << bb)], Wv[i], Wsv[i], p, 2 * two_p);
          else
            gs_bfly_t<false>(x[k], x[k | (1 << bb)], Wv[i], Wsv[i], p, 2 * two_p);
#endif
        }
      }
    }
#pragma unroll
    for (int k = 0; k < E; ++k) sb[koff<WLO>(k)] = x[k];
    round_sync<S, RB>();
    inv_rounds<S, RB, HI>(s, tw, p, two_p, ninv, ninvs, fw, fws, gq, tbase, w, last);
  }
}

// ---------------------------------------------------------------------------
// FP64 NTT path (primes < 2^46).  The integer butterfly is bound by the
// 32-bit multiplier pipe (ten multiplies per Shoup product) while the FP64
// pipe idles; B200 runs DFMA at full rate (ckb_alu_probe_f64: 2.27 T
// butterflies/s vs 0.80 T for the integer form).  Residues are held as exact
// integers in doubles and a product t = Y*W - q*p is formed exactly:
//   q = rint(Y * (W/p)),  h = Y*W (rounded),  l = fma(Y, W, -h) (exact),
//   t = fma(-q, p, h) + l  (exact integer, |t| <= 1.5p).
// Bounds (p < 2^46): forward values grow by <= 1.5p per stage (|v| < 27p over
// 17 stages, < 2^51, so Y*(W/p) stays below the 2^51 rint range); inverse
// sums double per stage: after every register round (<= 4 stages) the sum-side
// outputs are reduced to [-p/2, p/2] and the product-side outputs (<= 1.5p)
// are kept, so a round's inputs are <= 1.5p and its differences <= 24p.
// All arithmetic is exact integer arithmetic, so results equal the integer
// path's bit for bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ct_bfly_f64(double& X, double& Y, double W, double Wp, double p) {
  const double t = mulmod_f64(Y, W, Wp, p);
  const double a = X;
  X = a + t;
  Y = a - t;
}

__device__ __forceinline__ void gs_bfly_f64(double& X, double& Y, double W, double Wp, double p) {
  const double a = X, b = Y;
  X = a + b;
  Y = mulmod_f64(a - b, W, Wp, p);
}

// A thread's twiddles for one stage are NT consecutive entries starting at a
// multiple of NT (t0 = (tbase << (S-1-b)) + (rbase >> (b+1)) with rbase's
// low bits zero), so they load as 16-byte vectors.
template <int NT>
__device__ __forceinline__ void load_tw_f64(const double* __restrict__ tw, int t0, double* Wv,
                                            double* Wpv, double pinv) {
  if constexpr (NT >= 2) {
#pragma unroll
    for (int i = 0; i < NT; i += 2) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(tw + t0 + i));
      Wv[i] = v.x;
      Wv[i + 1] = v.y;
    }
  } else {
    Wv[0] = __ldg(tw + t0);
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) Wpv[i] = Wv[i] * pinv;
}

// Bottom round of a row phase (register bits = the low bits of r): thread T of
// the launch needs NT consecutive twiddles starting at NT*T, so a warp's vector
// load strides 8*NT bytes between lanes and touches 4x (NT = 8) / 2x (NT = 4)
// the cache lines it uses.  The table's second half (ckb_build_tables) holds
// the same entries with each warp's block of 32*NT interleaved by 16-byte
// chunk: chunk c of lane l at block + 64 c + 2 l, so every load is one
// contiguous 512 bytes per warp.
template <int NT>
__device__ __forceinline__ void load_tw_f64_perm(const double* __restrict__ ptab, int t0, double* Wv,
                                                 double* Wpv, double pinv) {
  static_assert(NT >= 2, "");
  const int lane = threadIdx.x & 31;
  const double* b = ptab + t0 - (NT - 2) * lane;
#pragma unroll
  for (int c = 0; c < NT / 2; ++c) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(b + 64 * c));
    Wv[2 * c] = v.x;
    Wv[2 * c + 1] = v.y;
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) Wpv[i] = Wv[i] * pinv;
}

__device__ __forceinline__ void load_tw_f64_pn(int nt, const double* __restrict__ ptab, int t0,
                                               double* Wv, double* Wpv, double pinv) {
  switch (nt) {  // constant after unrolling
    case 8: load_tw_f64_perm<8>(ptab, t0, Wv, Wpv, pinv); break;
    case 4: load_tw_f64_perm<4>(ptab, t0, Wv, Wpv, pinv); break;
    case 2: load_tw_f64_perm<2>(ptab, t0, Wv, Wpv, pinv); break;
    default: load_tw_f64<1>(ptab, t0, Wv, Wpv, pinv); break;
  }
}

__device__ __forceinline__ void load_tw_f64_n(int nt, const double* __restrict__ tw, int t0,
                                              double* Wv, double* Wpv, double pinv) {
  switch (nt) {  // constant after unrolling
    case 8: load_tw_f64<8>(tw, t0, Wv, Wpv, pinv); break;
    case 4: load_tw_f64<4>(tw, t0, Wv, Wpv, pinv); break;
    case 2: load_tw_f64<2>(tw, t0, Wv, Wpv, pinv); break;
    default: load_tw_f64<1>(tw, t0, Wv, Wpv, pinv); break;
  }
}

// Stores of a two-phase transform.  The first phase's outputs are read back by
// the second phase of the same row chunk and should stay in L2 (MID); the last
// phase's outputs stream out (st.cs).  CKB_NTT_MID_STORE: 0 = streaming store
// (st.cs), 1 = plain store, 2 = L2 evict_last cache hint (default).  Measured
// (tools/ab_mid.sh, 96 MiB chunks, one-pass ncu DRAM counters): DRAM bytes per
// forward transform 1.95x -> 1.43x the algorithmic bytes, inverse 1.50x ->
// 1.39x; HMult / HRot batch -1%.
#ifndef CKB_NTT_MID_STORE
#define CKB_NTT_MID_STORE 2
#endif
__device__ __forceinline__ void st_mid(uint64_t* g, uint64_t v) {
#if CKB_NTT_MID_STORE == 2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(g), "l"(v), "l"(pol) : "memory");
#elif CKB_NTT_MID_STORE == 1
  *g = v;
#else
  __stcs(g, v);
#endif
}
__device__ __forceinline__ void st_mid2(uint64_t* g, ulonglong2 v) {
#if CKB_NTT_MID_STORE == 2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(g), "l"(v.x), "l"(v.y),
               "l"(pol)
               : "memory");
#else
  *reinterpret_cast<ulonglong2*>(g) = v;
#endif
}

// Global I/O of the FP64 register rounds.  CM = false: the first round may
// read contiguous rows straight from global memory (gsrc), rounds exchange
// through shared memory with warp-local syncs where a group fits in a warp,
// and the last round stores to shared memory (tile store).  CM = true (column
// mapping, second phases): the first round reads and the last round writes
// global memory with element stride gs; one CTA barrier between rounds.
template <int E, int WLO, bool CM>
__device__ __forceinline__ void load_round_f64(double* x, const uint64_t* sb,
                                               const uint64_t* __restrict__ gsrc, int gs,
                                               int rbase, bool u64in) {
  if (CM && gsrc) {
    const uint64_t* g = gsrc + (size_t)rbase * gs;
    const size_t step = (size_t)gs << WLO;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const uint64_t v = __ldcs(g + k * step);
      x[k] = u64in ? u64_to_f64(v) : __longlong_as_double((long long)v);
    }
  } else if (!CM && gsrc) {
    const uint64_t* g = gsrc + rbase;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const uint64_t v = __ldcs(g + (k << WLO));
      x[k] = u64in ? u64_to_f64(v) : __longlong_as_double((long long)v);
    }
  } else if (u64in) {  // canonical residues staged raw in shared memory
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = u64_to_f64(sb[koff<WLO>(k)]);
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = __longlong_as_double((long long)sb[koff<WLO>(k)]);
  }
}

template <int S, int RB, bool CM>
__device__ __forceinline__ void rsync() {
  if constexpr (CM) {
    __syncthreads();
  } else {
    round_sync<S, RB>();
  }
}

// PT: the bottom round (WLO == 0) reads the interleaved copy of the table
// (tw + N), see load_tw_f64_perm.
template <int S, int RB, int HI, bool CM, bool PT = false>
__device__ __forceinline__ void fwd_rounds_f64(uint64_t* s, const double* __restrict__ tw,
                                               double p, double pinv, int gq, int tbase, int w,
                                               int last, const uint64_t* gsrc, uint64_t* gdst,
                                               int gs, bool u64in) {
  if constexpr (HI > 0) {
    constexpr int E = 1 << RB;
    constexpr int Q = HI < RB ? HI : RB;
    constexpr int LO = HI - Q;
    constexpr int WLO = HI - RB > 0 ? HI - RB : 0;
    const int rbase = (w & ((1 << WLO) - 1)) | ((w >> WLO) << (WLO + RB));
    double x[E];
    uint64_t* sb = s + sidx<S>(gq, rbase);
    load_round_f64<E, WLO, CM>(x, sb, HI == S ? gsrc : nullptr, gs, rbase, HI == S && u64in);
#pragma unroll
    for (int b = HI - 1; b >= LO; --b) {
      const int bb = b - WLO;
      const int t0 = (tbase << (S - 1 - b)) + (rbase >> (b + 1));
      double Wv[E / 2], Wpv[E / 2];
      if constexpr (PT && WLO == 0)
        load_tw_f64_pn((E / 2) >> bb, tw + ((size_t)1 << (2 * S)), t0, Wv, Wpv, pinv);
      else
        load_tw_f64_n((E / 2) >> bb, tw, t0, Wv, Wpv, pinv);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << bb)) continue;
        const int i = k >> (bb + 1);
        ct_bfly_f64(x[k], x[k | (1 << bb)], Wv[i], Wpv[i], p);
      }
    }
    if constexpr (CM && LO == 0) {  // column mapping: straight to global memory
      const size_t step = (size_t)gs << WLO;
      uint64_t* g = gdst + (size_t)rbase * gs;
      if (last) {
#pragma unroll
        for (int k = 0; k < E; ++k) __stcs(g + k * step, canon_u64(x[k], p, pinv));
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k) st_mid(g + k * step, (uint64_t)__double_as_longlong(x[k]));
      }
      return;
    }
    if (LO == 0 && last) {
#pragma unroll
      for (int k = 0; k < E; ++k)
        sb[koff<WLO>(k)] = canon_u64(x[k], p, pinv);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) sb[koff<WLO>(k)] = (uint64_t)__double_as_longlong(x[k]);
    }
    rsync<S, RB, CM>();
    fwd_rounds_f64<S, RB, LO, CM, PT>(s, tw, p, pinv, gq, tbase, w, last, gsrc, gdst, gs, u64in);
  }
}

template <int S, int RB, int LO, bool CM, bool PT = false>
__device__ __forceinline__ void inv_rounds_f64(uint64_t* s, const double* __restrict__ tw,
                                               double p, double pinv, double ninv, double ninvp,
                                               double fw, double fwp, int gq, int tbase, int w,
                                               int last, const uint64_t* gsrc, uint64_t* gdst,
                                               int gs, bool u64in) {
  if constexpr (LO < S) {
    constexpr int E = 1 << RB;
    constexpr int Q = (S - LO) < RB ? (S - LO) : RB;
    constexpr int HI = LO + Q;
    constexpr int WLO = LO < S - RB ? LO : S - RB;
    const int rbase = (w & ((1 << WLO) - 1)) | ((w >> WLO) << (WLO + RB));
    double x[E];
    uint64_t* sb = s + sidx<S>(gq, rbase);
    load_round_f64<E, WLO, CM>(x, sb, LO == 0 ? gsrc : nullptr, gs, rbase, LO == 0 && u64in);
#pragma unroll
    for (int b = LO; b < HI; ++b) {
      const int bb = b - WLO;
      if (b == S - 1 && last) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (k & (1 << bb)) continue;
          const double X = x[k], Y = x[k | (1 << bb)];
          x[k] = mulmod_f64(X + Y, ninv, ninvp, p);
          x[k | (1 << bb)] = mulmod_f64(X - Y, fw, fwp, p);
        }
      } else {
        const int t0 = (tbase << (S - 1 - b)) + (rbase >> (b + 1));
        double Wv[E / 2], Wpv[E / 2];
        if constexpr (PT && WLO == 0)
          load_tw_f64_pn((E / 2) >> bb, tw + ((size_t)1 << (2 * S)), t0, Wv, Wpv, pinv);
        else
          load_tw_f64_n((E / 2) >> bb, tw, t0, Wv, Wpv, pinv);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (k & (1 << bb)) continue;
          const int i = k >> (bb + 1);
          gs_bfly_f64(x[k], x[k | (1 << bb)], Wv[i], Wpv[i], p);
        }
      }
    }
    // Re-centring between rounds: an element whose last stage of this round
    // made it the product side of its butterfly (bit HI-1-WLO of k set) is a
    // mulmod_f64 output, |v| <= 1.5p, and goes on as it is; the sum sides (up
    // to 16x the round's input bound) are reduced to [-p/2, p/2].  A round's
    // inputs are then <= 1.5p, its differences <= 24p < 2^51 / 2^46 p.
    auto recentre = [&](int k) {
      return ((k >> (HI - 1 - WLO)) & 1) ? x[k] : center_f64(x[k], p, pinv);
    };
    if constexpr (CM && HI == S) {
      const size_t step = (size_t)gs << WLO;
      uint64_t* g = gdst + (size_t)rbase * gs;
      if (last) {
#pragma unroll
        for (int k = 0; k < E; ++k) __stcs(g + k * step, canon_u64(x[k], p, pinv));
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          st_mid(g + k * step, (uint64_t)__double_as_longlong(recentre(k)));
      }
      return;
    }
    if (HI == S && last) {
#pragma unroll
      for (int k = 0; k < E; ++k)
        sb[koff<WLO>(k)] = canon_u64(x[k], p, pinv);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) sb[koff<WLO>(k)] = (uint64_t)__double_as_longlong(recentre(k));
    }
    rsync<S, RB, CM>();
    inv_rounds_f64<S, RB, HI, CM, PT>(s, tw, p, pinv, ninv, ninvp, fw, fwp, gq, tbase, w, last,
                                      gsrc, gdst, gs, u64in);
  }
}

#ifndef CKB_NTT_MODE0_MINB
#define CKB_NTT_MODE0_MINB 3
#endif
// MODE 0: per-CTA dispatch on the row's prime class; 1: FP64 rows only; 2:
// integer rows only; 3: FP64 rows, column-mapped direct global I/O.
// ST = 1 / 2: the column / row phase of a two-phase transform with
// log2 N = 2S, whose geometry is then a compile-time fact (strides 1 and G,
// 2048/G groups per CTA, which phase is first and last, the twiddle base):
// global addresses become immediate offsets of one base pointer (a runtime
// stride costs six integer instructions per load and store), the first/last
// variants of the I/O disappear, and the radix-16 row phase's bottom round
// reads the interleaved twiddle copy (load_tw_f64_perm).  In a MODE 0 launch
// with ST the FP64 rows' CTAs also take the column-mapped / direct I/O paths
// of MODE 3 / MODE 1 (the choice is CTA-uniform).
// resident CTAs per SM (register caps) of the compile-time-geometry kernels,
// A/B on tools/ntt_micro.py: inverse row phase 8 / 7 / 6 CTAs: 1.491 / 1.442 /
// 1.397 ms per 3072-row inverse transform
#ifndef CKB_NTT_M5_INV_MINB
#define CKB_NTT_M5_INV_MINB 6
#endif
#ifndef CKB_NTT_M4_INV_MINB
#define CKB_NTT_M4_INV_MINB 8
#endif
#ifndef CKB_NTT_PF_DIST
#define CKB_NTT_PF_DIST 296  // 2 CTAs per SM ahead (A/B 148..888: 1.376 / 1.370 / 1.370 / 1.374 / 1.375 / 1.379 ms)
#endif
#ifndef CKB_NTT_ST_FWD_MINB
#define CKB_NTT_ST_FWD_MINB 6
#endif
template <int S, bool FWD, int RBT, int MODE = 0, int ST = 0>
__global__ void __launch_bounds__(MODE == 1 || MODE == 3 ? 128 : kNttThreads,
                                  MODE == 1 || MODE == 3
                                      ? (FWD ? (ST ? CKB_NTT_ST_FWD_MINB : 6)
                                             : (ST == 2   ? CKB_NTT_M5_INV_MINB
                                                : ST == 1 ? CKB_NTT_M4_INV_MINB
                                                          : 8))
                                                         : (RBT == 3 ? 4 : CKB_NTT_MODE0_MINB))
    k_ntt_phase(uint64_t* __restrict__ data, NttPhase ph, RingDev R, LimbMap lm, CombineEp ep) {
  constexpr int G = 1 << S;
  constexpr bool kStCol = ST == 1, kStRow = ST == 2, kSt = ST != 0;
  constexpr bool kF64Only = MODE == 1 || MODE == 3;
  // forward: columns then rows; inverse: rows then columns
  const int p_first = kSt ? (FWD == kStCol ? 1 : 0) : ph.first;
  const int p_last = kSt ? (FWD == kStCol ? 0 : 1) : ph.last;
  const int p_rstride = kStCol ? G : kStRow ? 1 : ph.rstride;
  const int p_gstride = kStCol ? 1 : kStRow ? G : ph.gstride;
  const int p_logC = kSt ? (S < 11 ? 11 - S : 0) : ph.logC;
  constexpr int RB = S < RBT ? S : RBT;  // log2 elements per thread
  constexpr int E = 1 << RB;
  extern __shared__ uint64_t smem[];
  const int N = 1 << R.log_n;
  const int rl = ph.row0 + (int)(blockIdx.x >> ph.log_tpr);
  // limb-major enumeration keeps one prime's twiddle table hot in L2 per chunk
  int limb, item;  // row = item * limbs + limb
  if (ph.items) {
    limb = fast_div(rl, ph.items, ph.items_magic);
    item = rl - limb * ph.items;
  } else {
    item = fast_div(rl, ph.limbs, ph.limbs_magic);
    limb = rl - item * ph.limbs;
  }
  const int row = item * ph.limbs + limb;
  const int tile = blockIdx.x & (ph.tiles_per_row - 1);
  const int pi = lm.p[limb];
  const uint64_t* mm = R.mods + (size_t)pi * kModStride;
  const uint64_t p = __ldg(mm), two_p = __ldg(mm + 3);
  const bool f64 = kF64Only || (MODE == 0 && (p >> 46) == 0);  // CTA-uniform
  if ((kF64Only && (p >> 46) != 0) || (MODE == 2 && (p >> 46) == 0)) return;
  uint64_t* base = data + (size_t)row * N;
  // tile loads of an out-of-place first phase come from the source row
  const uint64_t* ibase = ph.src ? ph.src + (size_t)item * ph.src_istride + (size_t)limb * N
                                 : base;
  const int C = kSt ? (1 << (S < 11 ? 11 - S : 0)) : ph.C;
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int g0 = tile * C;
#ifndef CKB_NTT_NO_L2_PREFETCH
  // The forward transform's first (column) phase streams its tiles from DRAM
  // at ~33% occupancy: each CTA asks L2 for the tile of a CTA that will start
  // soon (block index + pf_dist), so that CTA's strided loads are L2 hits.
  // (A/B: the inverse's first, row phase and the forward's second phase are slower with it)
  if (kStCol && FWD && ph.pf_dist) {
    const unsigned b2 = blockIdx.x + (unsigned)ph.pf_dist;
    if (b2 < gridDim.x) {
      const int rl2 = ph.row0 + (int)(b2 >> ph.log_tpr);
      int limb2, item2;
      if (ph.items) {
        limb2 = fast_div(rl2, ph.items, ph.items_magic);
        item2 = rl2 - limb2 * ph.items;
      } else {
        item2 = fast_div(rl2, ph.limbs, ph.limbs_magic);
        limb2 = rl2 - item2 * ph.limbs;
      }
      const uint64_t* b2p = ph.src ? ph.src + (size_t)item2 * ph.src_istride + (size_t)limb2 * N
                                   : data + (size_t)(item2 * ph.limbs + limb2) * N;
      const int t2 = (int)(b2 & (unsigned)(ph.tiles_per_row - 1));
      for (int r = tid; r < G; r += T)  // G rows of C words: one line per row
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b2p + (size_t)r * G + (size_t)t2 * C));
    }
  }
#endif
  const bool rows_contig = p_rstride == 1;

  // tile -> smem, 16-byte vectors (pairs adjacent in global memory).  Every
  // thread moves exactly E/2 pairs (C*G/2 pairs over C*G/E threads); all
  // loads are issued before the first shared store.
  // Contiguous rows with a group per (part of a) warp: thread t moves pairs
  // lt + (G/E) i of its own group (still 16-byte coalesced), so the whole
  // phase only exchanges data inside a warp (__syncwarp, no CTA barrier).
  constexpr bool kWarpGroups = (G / E) <= 32;
  const bool warp_local = kWarpGroups && rows_contig;
  auto pair_of = [&](int i, int& g, int& r) -> size_t {  // i-th pair of this thread
    const int e = 2 * (tid + i * T);
    if (rows_contig) {
      if (kWarpGroups) {  // group tid/(G/E), pair (tid % (G/E)) + (G/E) i
        g = tid / (G / E);
        r = 2 * (tid % (G / E) + (G / E) * i);
      } else {
        g = e >> S;
        r = e & (G - 1);
      }
      return (size_t)(g0 + g) * p_gstride + r;
    }
    r = e >> p_logC;
    g = e & (C - 1);
    return (size_t)r * p_rstride + g0 + g;
  };
  // FP64 path on contiguous rows of a second phase (input = the first phase's
  // L2-resident doubles): the first register round reads global memory
  // directly, no tile staging through shared memory.  Measured (A/B,
  // tools/ab_ntt.sh): forward -3%; a first phase streaming from DRAM is 9%
  // faster with the 16-byte tile loads, so it keeps them.
  const bool direct = f64 && warp_local && !p_first;
#ifndef CKB_NO_COMBINE_PREFETCH
  // Fused ModDown combine: the x and addend tiles this thread combines in the
  // epilogue are copied into shared memory asynchronously (cp.async, no
  // registers held) while the rounds run, so the epilogue reads them without
  // exposing DRAM latency.  Each thread fetches exactly its own pairs: a
  // cp.async.wait_all before the epilogue is the only synchronisation.
  uint64_t* pf = smem + (size_t)C * (G + G / 16 + G / 128);
  const bool prefetch = FWD && ep.out && p_last && rows_contig;
  const uint64_t* pf_add = nullptr;
  if (prefetch) {
    const int j = limb;
    const unsigned pidx = (unsigned)item;
    const uint64_t* xr = ep.x + (size_t)pidx * ep.xs + (size_t)j * N;
    if (ep.add) {
      const unsigned phs = pidx % (unsigned)ep.add_period;
      if ((int)phs < ep.add_polys)
        pf_add = ep.add +
                 ((size_t)(pidx / (unsigned)ep.add_period) * ep.add_stride + phs) * ep.m1 * N +
                 (size_t)j * N;
    }
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      int g, r;
      const size_t off = pair_of(i, g, r);
      const unsigned sx = (unsigned)__cvta_generic_to_shared(pf + 2 * ((size_t)i * T + tid));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sx), "l"(xr + off));
      if (pf_add) {
        const unsigned sa =
            (unsigned)__cvta_generic_to_shared(pf + 2 * ((size_t)(E / 2 + i) * T + tid));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(pf_add + off));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
#endif
  // FP64-only kernel, column phase: lanes span the tile's C columns
  // (gq = tid % C, w = tid / C) so both the first round's loads and the last
  // round's stores go straight to global memory (each warp instruction
  // touches 32/C rows x C contiguous words); one shared exchange between the
  // two radix-16 rounds, behind a CTA barrier.
  // (second phases only, chosen by the host: a first phase streaming from
  // DRAM keeps the 16-byte tile loads — A/B: forward column phase +5% with
  // the column mapping, inverse column phase -4%)
  // (MODE 0 + ST: the FP64 rows of a mixed column phase take it too)
  constexpr bool kColF64 = MODE == 3 || (MODE == 0 && kStCol);  // FP64 rows column-mapped
  const bool colmap = MODE == 3 || (kColF64 && f64);
  if (!direct && !colmap) {
    ulonglong2 v[E / 2];
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      int g, r;
      v[i] = __ldcs(reinterpret_cast<const ulonglong2*>(ibase + pair_of(i, g, r)));
    }
    if (f64 && p_first) {  // canonical residues -> exact doubles
#pragma unroll
      for (int i = 0; i < E / 2; ++i) {
        v[i].x = (uint64_t)__double_as_longlong(u64_to_f64(v[i].x));
        v[i].y = (uint64_t)__double_as_longlong(u64_to_f64(v[i].y));
      }
    }
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      int g, r;
      pair_of(i, g, r);
      smem[sidx<S>(g, r)] = v[i].x;
      if (rows_contig)
        smem[sidx<S>(g, r + 1)] = v[i].y;
      else
        smem[sidx<S>(g + 1, r)] = v[i].y;
    }
  }
  if (warp_local)
    __syncwarp();
  else if (!colmap)
    __syncthreads();

  // (log2 N <= 16 keeps |x P^-1 + add - E| below 2^51 for the epilogue's products)
  const bool raw_e = FWD && p_last && f64 && R.log_n <= 16;
  const int gq = colmap ? (tid & (C - 1)) : tid / (G / E);
  const int w = colmap ? (tid >> p_logC) : tid % (G / E);
  const int tbase = kStCol ? 1 : kStRow ? G + g0 + gq : ph.M0 + ph.gt * (g0 + gq);
  // per prime: N forward then N inverse {w, shoup(w)} pairs
  const ulonglong2* tables = reinterpret_cast<const ulonglong2*>(R.ntt + (size_t)pi * 4 * N);
  if (MODE != 2 && f64) {
    const double pd = (double)p, pinv = __longlong_as_double((long long)__ldg(mm + 10));  // 1/p
    // FP64-path table: [N] double(w) forward, [N] w/p, then the inverse pair
    const double* dtab = reinterpret_cast<const double*>(R.ntt + (size_t)pi * 4 * N);
    // (a column-mapped first phase reads the out-of-place source directly)
    const uint64_t* gsrc = colmap ? ibase + g0 + gq
                                  : (direct ? base + (size_t)(g0 + gq) * p_gstride : nullptr);
    uint64_t* gdst = colmap ? base + g0 + gq : nullptr;
    const int gs = colmap ? p_rstride : 1;
    if constexpr (FWD) {
      // fused combine: E stays a (non-canonical, |E| < 27p) double for the epilogue
      const int f_last = (ep.out && raw_e) ? 0 : p_last;
      fwd_rounds_f64<S, RB, S, kColF64, kStRow && RB == 4>(smem, dtab, pd, pinv, gq, tbase, w,
                                                           f_last, gsrc, gdst, gs,
                                                           gsrc != nullptr && p_first);
    } else {
      const double ninv = u64_to_f64(__ldg(mm + 4)), fw = u64_to_f64(__ldg(mm + 6));
      inv_rounds_f64<S, RB, 0, kColF64, kStRow && RB == 4>(
          smem, dtab + 2 * N, pd, pinv, ninv, ninv * pinv, fw, fw * pinv, gq, tbase, w, p_last,
          gsrc, gdst, gs, gsrc != nullptr && p_first);
    }
    if constexpr (kColF64) return;  // stored straight to global memory
  } else if constexpr (!kF64Only) {
    if constexpr (FWD) {
      fwd_rounds<S, RB, S>(smem, tables, p, two_p, gq, tbase, w, p_last);
    } else {
      inv_rounds<S, RB, 0>(smem, tables + N, p, two_p, __ldg(mm + 4), __ldg(mm + 5),
                           __ldg(mm + 6), __ldg(mm + 7), gq, tbase, w, p_last);
    }
  }
  if (warp_local)
    __syncwarp();
  else
    __syncthreads();  // the tile store reads across groups

  if (FWD && ep.out && p_last) {  // fused combine (rows are contiguous here)
    const int j = limb;
    const unsigned pidx = (unsigned)item;
    const int s1 = 2 * (ep.n1 + 1), s2 = 2 * (ep.n2 + 1);
    uint64_t a1 = 0, a1s = 0, b2 = 0, b2s = 0;
    if (ep.n1) {
      a1 = __ldg(ep.tab1 + (size_t)j * s1 + 2 * ep.n1);
      a1s = __ldg(ep.tab1 + (size_t)j * s1 + 2 * ep.n1 + 1);
    }
    if (ep.n2) {
      b2 = __ldg(ep.tab2 + (size_t)j * s2 + 2 * ep.n2);
      b2s = __ldg(ep.tab2 + (size_t)j * s2 + 2 * ep.n2 + 1);
    }
    const uint64_t* xr = ep.x + (size_t)pidx * ep.xs + (size_t)j * N;
    const uint64_t* ar = nullptr;
    if (ep.add) {
      const unsigned phs = pidx % (unsigned)ep.add_period;
      if ((int)phs < ep.add_polys)
        ar = ep.add +
             ((size_t)(pidx / (unsigned)ep.add_period) * ep.add_stride + phs) * ep.m1 * N +
             (size_t)j * N;
    }
    const uint64_t* pr =
        ep.post ? ep.post + (size_t)pidx * ep.post_stride + (size_t)j * N : nullptr;
    uint64_t* orow = ep.out + (size_t)row * N;
#ifndef CKB_NO_COMBINE_PREFETCH
    if (prefetch) asm volatile("cp.async.wait_all;\n" ::: "memory");
#endif
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      int g, r;
      const size_t off = pair_of(i, g, r);
      const uint64_t e0 = smem[sidx<S>(g, r)], e1 = smem[sidx<S>(g, r + 1)];
#ifndef CKB_NO_COMBINE_PREFETCH
      ulonglong2 v = prefetch ? *reinterpret_cast<const ulonglong2*>(pf + 2 * ((size_t)i * T + tid))
                              : *reinterpret_cast<const ulonglong2*>(xr + off);
#else
      ulonglong2 v = *reinterpret_cast<const ulonglong2*>(xr + off);
#endif
#ifndef CKB_COMBINE_INT
      if (f64) {  // the combine on the FP64 pipe (exact; same integers)
        const double pd = (double)p, pinv = __longlong_as_double((long long)__ldg(mm + 10));
        double c[2] = {u64_to_f64(v.x), u64_to_f64(v.y)};
        const double ev[2] = {raw_e ? __longlong_as_double((long long)e0) : u64_to_f64(e0),
                              raw_e ? __longlong_as_double((long long)e1) : u64_to_f64(e1)};
        const double a1d = u64_to_f64(a1), b2d = u64_to_f64(b2);
        ulonglong2 a = make_ulonglong2(0, 0), w2 = make_ulonglong2(0, 0);
        if (ar) {
#ifndef CKB_NO_COMBINE_PREFETCH
          a = prefetch ? *reinterpret_cast<const ulonglong2*>(pf + 2 * ((size_t)(E / 2 + i) * T + tid))
                       : *reinterpret_cast<const ulonglong2*>(ar + off);
#else
          a = *reinterpret_cast<const ulonglong2*>(ar + off);
#endif
        }
        if (pr) w2 = *reinterpret_cast<const ulonglong2*>(pr + off);
        const double av[2] = {u64_to_f64(a.x), u64_to_f64(a.y)};
        const double wv[2] = {u64_to_f64(w2.x), u64_to_f64(w2.y)};
        uint64_t o[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double t = ep.n1 ? mulmod_f64(c[h], a1d, a1d * pinv, pd) : c[h];  // |t| < 1.5p
          t = t + av[h] - ev[h];                                            // |t| < 3.5p
          if (ep.n2) t = mulmod_f64(t, b2d, b2d * pinv, pd);                // |t| < 1.5p
          t += wv[h];
          o[h] = canon_u64(t, pd, pinv);
        }
        *reinterpret_cast<ulonglong2*>(orow + off) = make_ulonglong2(o[0], o[1]);
        continue;
      }
#endif
      if (ep.n1) {
        v.x = ckb::mul_shoup(v.x, a1, a1s, p);
        v.y = ckb::mul_shoup(v.y, a1, a1s, p);
      }
      if (ar) {
#ifndef CKB_NO_COMBINE_PREFETCH
        const ulonglong2 a =
            prefetch ? *reinterpret_cast<const ulonglong2*>(pf + 2 * ((size_t)(E / 2 + i) * T + tid))
                     : *reinterpret_cast<const ulonglong2*>(ar + off);
#else
        const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(ar + off);
#endif
        v.x = ckb::add_mod(v.x, a.x, p);
        v.y = ckb::add_mod(v.y, a.y, p);
      }
      v.x = ckb::sub_mod(v.x, e0, p);
      v.y = ckb::sub_mod(v.y, e1, p);
      if (ep.n2) {
        v.x = ckb::mul_shoup(v.x, b2, b2s, p);
        v.y = ckb::mul_shoup(v.y, b2, b2s, p);
      }
      if (pr) {
        const ulonglong2 w2 = *reinterpret_cast<const ulonglong2*>(pr + off);
        v.x = ckb::add_mod(v.x, w2.x, p);
        v.y = ckb::add_mod(v.y, w2.y, p);
      }
      *reinterpret_cast<ulonglong2*>(orow + off) = v;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < E / 2; ++i) {
    int g, r;
    const size_t off = pair_of(i, g, r);
    ulonglong2 v;
    v.x = smem[sidx<S>(g, r)];
    v.y = rows_contig ? smem[sidx<S>(g, r + 1)] : smem[sidx<S>(g + 1, r)];
#if CKB_NTT_MID_STORE == 2 || !defined(CKB_NTT_NO_LAST_CS)
    if (p_last) {
#ifndef CKB_NTT_NO_LAST_CS
      __stcs(reinterpret_cast<ulonglong2*>(base + off), v);
#else
      *reinterpret_cast<ulonglong2*>(base + off) = v;
#endif
    } else {
      st_mid2(base + off, v);
    }
#else
    *reinterpret_cast<ulonglong2*>(base + off) = v;
#endif
  }
}

template <bool FWD, int RBT, int MODE = 0, int ST = 0>
int launch_phase(int S, uint64_t* data, const NttPhase& ph, int nrows, const RingDev& R,
                 const LimbMap& lm, cudaStream_t st, const CombineEp& ep = CombineEp{}) {
  const int G = 1 << S;
  const int RB = S < RBT ? S : RBT;
  const int threads = ph.C * G >> RB;
  size_t smem = (size_t)ph.C * (G + G / 16 + G / 128) * sizeof(uint64_t);
#ifndef CKB_NO_COMBINE_PREFETCH
  if (FWD && ep.out && ph.last && ph.rstride == 1)  // prefetched x (and addend) tiles
    smem += (ep.add ? 2 : 1) * (size_t)ph.C * G * sizeof(uint64_t);
#endif
  const int blocks = nrows * ph.tiles_per_row;
  if (blocks <= 0) return 0;
  if (threads > kNttThreads) return CKB_E_LOGN;
  NttPhase q = ph;  // block decode constants
  q.log_tpr = 0;
  while ((1 << q.log_tpr) < ph.tiles_per_row) ++q.log_tpr;
  if ((1 << q.log_tpr) != ph.tiles_per_row) return CKB_E_LOGN;
  q.items_magic = ph.items ? div_magic(ph.items, (long long)ph.row0 + nrows) : 0;
  q.limbs_magic = div_magic(ph.limbs, (long long)ph.row0 + nrows);
  q.pf_dist = CKB_NTT_PF_DIST;
#define CKB_NTT_CASE(SS)                                                           \
  case SS:                                                                         \
    if (smem > 48 * 1024)                                                          \
      cudaFuncSetAttribute(k_ntt_phase<SS, FWD, RBT, MODE, ST>,                    \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_ntt_phase<SS, FWD, RBT, MODE, ST><<<blocks, threads, smem, st>>>(data, q, R, lm, ep); \
    break;
  if constexpr (ST != 0) {  // log2 N = 2S in 14..20
    constexpr bool col = ST == 1;
    if (S < 7 || S > 10 || ph.C != (1 << (11 - S)) || ph.rstride != (col ? G : 1) ||
        ph.gstride != (col ? 1 : G) || ph.M0 != (col ? 1 : G) || ph.gt != (col ? 0 : 1) ||
        ph.first != (FWD == col ? 1 : 0) || ph.last != (FWD == col ? 0 : 1))
      return CKB_E_ARG;
    switch (S) {
      CKB_NTT_CASE(7)
      CKB_NTT_CASE(8)
      CKB_NTT_CASE(9)
      CKB_NTT_CASE(10)
      default:
        return CKB_E_LOGN;
    }
  } else {
    switch (S) {
      CKB_NTT_CASE(4)
      CKB_NTT_CASE(5)
      CKB_NTT_CASE(6)
      CKB_NTT_CASE(7)
      CKB_NTT_CASE(8)
      CKB_NTT_CASE(9)
      CKB_NTT_CASE(10)
      CKB_NTT_CASE(11)
      CKB_NTT_CASE(12)
      default:
        return CKB_E_LOGN;
    }
  }
#undef CKB_NTT_CASE
  return 0;
}

// Register rounds of the per-CTA-dispatch and integer kernels: radix-16 in
// forward transforms (mixed launches then run their FP64 rows radix-16; the
// integer rows are equal either way), radix-8 in inverse ones (integer
// inverse rows 6% faster at radix-8) — A/B on tools/ntt_micro.py and bench.
// Launches holding rows of both prime classes run as ONE launch of the
// per-CTA-dispatch kernel (MODE 0: radix-8 for both paths): FP64-row CTAs and
// integer-row CTAs then share the SMs, the FP64/L1-latency-bound and the
// multiplier-bound work overlapping (measured: c2 479 -> 485 GB/s, config-4
// steady step forward NTT -5%, against the class-split MODE 1 + MODE 2 pair
// whose FP64 kernel alone is faster).  ckb_ring.flags CKB_RING_NTT_SPLIT
// restores the split.

// Rows of a two-phase transform are processed in chunks whose intermediate
// stays in L2 between the phases.  96 MB measured best for one stream
// (config-4 step -2%, config-2 sequential NTT -7% against 48 MB); callers
// running transforms on several streams at once give each a share
// (ckb_ring.ntt_chunk_bytes; bench.py's concurrent HMult/HRot pair uses 48 MB).
constexpr size_t kDefaultNttChunkBytes = (size_t)96 << 20;

template <bool FWD>
int ntt_run(const ckb_ring* ring, uint64_t* data, int rows, int limbs, const int32_t* limb_prime,
            void* stream, const uint64_t* src = nullptr, size_t src_istride = 0,
            const CombineEp& ep = CombineEp{}) {
  LimbMap lm;
  if (!make_map(lm, limb_prime, limbs) || rows < 0) return CKB_E_LIMBS;
  if (rows == 0) return 0;
  const RingDev R = make_ring(ring);
  const int logn = (int)R.log_n;
  if (logn < 4 || logn > 20) return CKB_E_LOGN;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = 1 << logn;
  if (logn <= 12) {
    NttPhase ph{limbs, 1, 1, 0, 1, 1, 0, 1, 0, 0, 0, 1, src, src_istride};
    int rc = launch_phase<FWD, 4>(logn, data, ph, rows, R, lm, st, ep);
    return rc ? rc : finish();
  }
  const int s2 = logn / 2;        // low stages (contiguous rows, phase B)
  const int s1 = logn - s2;       // high stages (strided columns, phase A)
  if (s1 > 12) return CKB_E_LOGN;
  const int GA = 1 << s1, GB = 1 << s2;
  const int CA = std::max(1, kTwoPhaseTile / GA), CB = std::max(1, kTwoPhaseTile / GB);
  // prime classes of this launch (host copy in the ring): FP64 rows go to the
  // radix-16 FP64 kernel, integer rows to the radix-8 integer kernel
  bool any_f64 = false, any_int = false;
  for (int i = 0; i < limbs; ++i) {
    const int pi = lm.p[i];
    ((R.f64_mask[pi >> 6] >> (pi & 63)) & 1 ? any_f64 : any_int) = true;
  }
  // phase A: groups are the GB columns, elements strided by GB
  auto lg = [](int v) { int l = 0; while ((1 << l) < v) ++l; return l; };
  const int items = (rows % limbs == 0 && rows / limbs > 1) ? rows / limbs : 0;
  NttPhase pa{limbs, GB / CA, CA, 1, GB, 1, 0, FWD ? 0 : 1, 0, lg(CA), items, FWD ? 1 : 0,
              FWD ? src : nullptr, src_istride};
  // phase B: groups are the GA rows of GB contiguous elements
  NttPhase pb{limbs, GA / CB, CB, GB, 1, N / GB, 1, FWD ? 1 : 0, 0, lg(CB), items, FWD ? 0 : 1,
              FWD ? nullptr : src, src_istride};
  // Chunk rows so one chunk's intermediate stays in the 126 MB L2 between phases.
  const size_t budget = R.ntt_chunk_bytes ? (size_t)R.ntt_chunk_bytes : kDefaultNttChunkBytes;
  const int chunk = std::max(1, (int)(budget / ((size_t)N * 8)));
  const bool mixed_one_kernel = !(R.flags & CKB_RING_NTT_SPLIT);
  for (int r0 = 0; r0 < rows; r0 += chunk) {
    const int nr = std::min(chunk, rows - r0);
    pa.row0 = r0;
    pb.row0 = r0;
    int rc = 0;
    auto run = [&](int S, const NttPhase& ph) {
      const bool cm = ph.rstride != 1;  // column phase
#ifndef CKB_NTT_NO_STATIC
      const bool st2 = logn == 2 * S && S >= 7 && S <= 10;  // compile-time geometry (ST)
#else
      const bool st2 = false;
#endif
      if (!any_f64 || (any_int && mixed_one_kernel)) {
#ifndef CKB_NTT_NO_STATIC_MIXED
        if (st2)
          return cm ? launch_phase<FWD, FWD ? 4 : 3, 0, 1>(S, data, ph, nr, R, lm, st, ep)
                    : launch_phase<FWD, FWD ? 4 : 3, 0, 2>(S, data, ph, nr, R, lm, st, ep);
#endif
        return launch_phase<FWD, FWD ? 4 : 3, 0>(S, data, ph, nr, R, lm, st, ep);
      }
      // column phases (first or second) of pure-FP64 launches: column-mapped
      // direct global I/O (MODE 3) — first passes too since round 2
      // (ModDown combine -4%, batch NTT -1%, tools/ks_micro.py A/B)
      int r = cm ? (st2 ? launch_phase<FWD, 4, 3, 1>(S, data, ph, nr, R, lm, st, ep)
                        : launch_phase<FWD, 4, 3>(S, data, ph, nr, R, lm, st, ep))
                 : (st2 ? launch_phase<FWD, 4, 1, 2>(S, data, ph, nr, R, lm, st, ep)
                        : launch_phase<FWD, 4, 1>(S, data, ph, nr, R, lm, st, ep));
      if (!r && any_int) r = launch_phase<FWD, FWD ? 4 : 3, 2>(S, data, ph, nr, R, lm, st, ep);
      return r;
    };
    if (FWD) {
      rc = run(s1, pa);
      if (!rc) rc = run(s2, pb);
    } else {
      rc = run(s2, pb);
      if (!rc) rc = run(s1, pa);
    }
    if (rc) return rc;
  }
  return finish();
}

// ---------------------------------------------------------------------------
// Key switching: the digits' forward NTT row phase fused with the key inner
// product (keys.py:91-97).  ModUp's digits, after the column phase, are
// finished row tile by row tile; one CTA owns (item, extended limb e, tile)
// and, for every digit j, transforms digit j's row of limb e (or, for the limb
// the digit owns, reads the NTT-domain input it was cut from), multiplies it
// by key_j's (b, a) rows and accumulates — so the transformed digits never go
// to HBM and the separate inner-product pass (k_ks_inner) disappears.
// Accumulators live in shared memory (each thread owns its pairs: no barrier
// between digits beyond the tile's own); FP64-class rows accumulate exact
// mulmod_f64 terms (|acc| <= 1.5 p nd), integer rows Barrett products.
// ---------------------------------------------------------------------------
struct KsMac {
  uint64_t* acc;                 // [batch][2][ext][N]
  const uint64_t* dig;           // [batch][item_rows][N] after the column phase
  const uint64_t* own;           // NTT-domain input limbs, item stride own_bs
  size_t own_bs;
  const uint64_t* key;           // one key, or
  const uint64_t* const* key_ptrs;  // one key per item
  int key_limbs, nd, ext, out_rows, item_rows, alpha, m, item0, tiles;
};

template <int S, int RBT>
__global__ void __launch_bounds__(128, 4)
    k_ntt_rows_mac(KsMac km, RingDev R, LimbMap em, LimbMap kmap) {
  constexpr int G = 1 << S;
  constexpr int RB = S < RBT ? S : RBT;
  constexpr int E = 1 << RB;
  constexpr int C = kTwoPhaseTile / G;  // rows (groups) per tile
  constexpr int T = C * G / E;          // threads
  static_assert((G / E) <= 32, "row groups must be warp-local");
  extern __shared__ uint64_t smem[];
  double2* accb = reinterpret_cast<double2*>(smem + C * (G + G / 16 + G / 128));
  double2* acca = accb + (E / 2) * T;
  const int N = 1 << R.log_n;
  const int tid = threadIdx.x;
  const int tile = blockIdx.x % km.tiles;
  const int e = (blockIdx.x / km.tiles) % km.ext;
  const int item = km.item0 + blockIdx.x / (km.tiles * km.ext);
  const int pi = em.p[e];
  const uint64_t* mm = R.mods + (size_t)pi * kModStride;
  const uint64_t p = __ldg(mm), two_p = __ldg(mm + 3);
  const bool f64 = (p >> 46) == 0;  // CTA-uniform
  const Mod mod{p, __ldg(mm + 1), __ldg(mm + 2), two_p};
  const double pd = (double)p, pinv = 1.0 / pd;
  const int g0 = tile * C;
  const int gq = tid / (G / E), w = tid % (G / E);
  const int tbase = N / G + g0 + gq;  // row phase: M0 = N/G, gt = 1
  const uint64_t* K = km.key_ptrs ? km.key_ptrs[item] : km.key;
  const size_t krow = 2 * (size_t)km.key_limbs * N;
  const uint64_t* kb0 = K + (size_t)kmap.p[e] * N;
  const int owner = e < km.m ? e / km.alpha : -1;
  auto pair_off = [&](int i, int& g, int& r) -> size_t {  // warp-local pairs of my row
    g = tid / (G / E);
    r = 2 * (tid % (G / E) + (G / E) * i);
    return (size_t)(g0 + g) * G + r;
  };
  for (int j = 0; j < km.nd; ++j) {
    const bool is_own = j == owner;
    if (!is_own) {
      const int cj = min(km.alpha, km.m - j * km.alpha);
      const int drow = j * km.out_rows + (e >= j * km.alpha + cj ? e - cj : e);
      const uint64_t* base = km.dig + ((size_t)item * km.item_rows + drow) * N;
      if (f64) {
        const double* dtab = reinterpret_cast<const double*>(R.ntt + (size_t)pi * 4 * N);
        fwd_rounds_f64<S, RB, S, false>(smem, dtab, pd, pinv, gq, tbase, w, 1,
                                        base + (size_t)(g0 + gq) * G, nullptr, 1, false);
      } else {
        ulonglong2 v[E / 2];
#pragma unroll
        for (int i = 0; i < E / 2; ++i) {
          int g, r;
          v[i] = __ldcs(reinterpret_cast<const ulonglong2*>(base + pair_off(i, g, r)));
        }
#pragma unroll
        for (int i = 0; i < E / 2; ++i) {
          int g, r;
          pair_off(i, g, r);
          smem[sidx<S>(g, r)] = v[i].x;
          smem[sidx<S>(g, r + 1)] = v[i].y;
        }
        __syncwarp();
        const ulonglong2* tables = reinterpret_cast<const ulonglong2*>(R.ntt + (size_t)pi * 4 * N);
        fwd_rounds<S, RB, S>(smem, tables, p, two_p, gq, tbase, w, 1);
      }
      __syncwarp();
    }
    const uint64_t* kb = kb0 + j * krow;
    const uint64_t* ka = kb + (size_t)km.key_limbs * N;
    const uint64_t* orow = is_own ? km.own + (size_t)item * km.own_bs + (size_t)e * N : nullptr;
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      int g, r;
      const size_t off = pair_off(i, g, r);
      ulonglong2 x;
      if (is_own) {
        x = *reinterpret_cast<const ulonglong2*>(orow + off);
      } else {
        x.x = smem[sidx<S>(g, r)];
        x.y = smem[sidx<S>(g, r + 1)];
      }
      const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(kb + off));
      const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(ka + off));
      const int slot = i * T + tid;
      if (f64) {
        const double x0 = u64_to_f64(x.x), x1 = u64_to_f64(x.y);
        const double b0 = u64_to_f64(b.x), b1 = u64_to_f64(b.y);
        const double a0 = u64_to_f64(a.x), a1 = u64_to_f64(a.y);
        double2 tb = make_double2(mulmod_f64(x0, b0, b0 * pinv, pd), mulmod_f64(x1, b1, b1 * pinv, pd));
        double2 ta = make_double2(mulmod_f64(x0, a0, a0 * pinv, pd), mulmod_f64(x1, a1, a1 * pinv, pd));
        if (j) {
          const double2 pb = accb[slot], pa = acca[slot];
          tb.x += pb.x;
          tb.y += pb.y;
          ta.x += pa.x;
          ta.y += pa.y;
        }
        accb[slot] = tb;
        acca[slot] = ta;
      } else {
        uint64_t tb0 = ckb::mul_mod(x.x, b.x, mod), tb1 = ckb::mul_mod(x.y, b.y, mod);
        uint64_t ta0 = ckb::mul_mod(x.x, a.x, mod), ta1 = ckb::mul_mod(x.y, a.y, mod);
        if (j) {
          const double2 pb = accb[slot], pa = acca[slot];
          tb0 = ckb::add_mod(tb0, (uint64_t)__double_as_longlong(pb.x), p);
          tb1 = ckb::add_mod(tb1, (uint64_t)__double_as_longlong(pb.y), p);
          ta0 = ckb::add_mod(ta0, (uint64_t)__double_as_longlong(pa.x), p);
          ta1 = ckb::add_mod(ta1, (uint64_t)__double_as_longlong(pa.y), p);
        }
        accb[slot] = make_double2(__longlong_as_double((long long)tb0),
                                  __longlong_as_double((long long)tb1));
        acca[slot] = make_double2(__longlong_as_double((long long)ta0),
                                  __longlong_as_double((long long)ta1));
      }
    }
    __syncwarp();  // the next digit's rounds reuse the tile
  }
  uint64_t* ob = km.acc + ((size_t)item * 2 * km.ext + e) * N;
  uint64_t* oa = ob + (size_t)km.ext * N;
#pragma unroll
  for (int i = 0; i < E / 2; ++i) {
    int g, r;
    const size_t off = pair_off(i, g, r);
    const int slot = i * T + tid;
    const double2 vb = accb[slot], va = acca[slot];
    ulonglong2 b, a;
    if (f64) {
      b = make_ulonglong2(canon_u64(vb.x, pd, pinv), canon_u64(vb.y, pd, pinv));
      a = make_ulonglong2(canon_u64(va.x, pd, pinv), canon_u64(va.y, pd, pinv));
    } else {
      b = make_ulonglong2((uint64_t)__double_as_longlong(vb.x), (uint64_t)__double_as_longlong(vb.y));
      a = make_ulonglong2((uint64_t)__double_as_longlong(va.x), (uint64_t)__double_as_longlong(va.y));
    }
    *reinterpret_cast<ulonglong2*>(ob + off) = b;
    *reinterpret_cast<ulonglong2*>(oa + off) = a;
  }
}

// ALU ceiling probe (the IMAD pipe is the NTT's binding
// roofline, so its peak is measured, not assumed).  Each thread keeps 8
// residues in registers and runs radix-8 rounds of the same lazy CT butterfly
// the NTT uses, twiddles in registers: no memory traffic at all.
__global__ void __launch_bounds__(256) k_alu_probe(uint64_t p, uint64_t w0, int iters,
                                                   uint64_t* __restrict__ sink) {
  const uint64_t two_p = 2 * p;
  uint64_t x[8], W[3], Ws[3];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (threadIdx.x * 8 + k + blockIdx.x) % p;
  W[0] = w0;
  W[1] = (w0 * 3 + threadIdx.x) % p;
  W[2] = (w0 * 7 + blockIdx.x) % p;
#pragma unroll
  for (int i = 0; i < 3; ++i) Ws[i] = (uint64_t)(((unsigned __int128)W[i] << 64) / p);
#if defined(CKB_NTT_SHOUP4) || defined(CKB_NTT_CT_REDUCE_ALL)
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 2; b >= 0; --b) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (!(k & (1 << b))) ct_bfly(x[k], x[k | (1 << b)], W[b], Ws[b], p, kLz * two_p);
    }
  }
#else
  // the NTT's stage schedule: reducing and skipping stages alternate (fwd_rounds)
  for (int it = 0; it < iters; it += 2) {
#pragma unroll
    for (int st = 0; st < 6; ++st) {
      const int b = 2 - st % 3;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k & (1 << b)) continue;
        if ((st & 1) == 0) x[k] = x[k] >= 4 * two_p ? x[k] - 4 * two_p : x[k];
        ct_bfly<false>(x[k], x[k | (1 << b)], W[b], Ws[b], p, 2 * two_p);
      }
    }
  }
#endif
  uint64_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= x[k];
  if (acc == 0x5A5A5A5A5A5A5A5Aull) sink[0] = acc;  // keeps the loop live
}

// FP64 variant of the probe: the same radix-8 rounds on the FP64 pipe.
__global__ void __launch_bounds__(256) k_alu_probe_f64(double p, double w0, int iters,
                                                       uint64_t* __restrict__ sink) {
  double x[8], W[3], Wp[3];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (double)((threadIdx.x * 8 + k + blockIdx.x) % 1000003);
  W[0] = w0;
  W[1] = fmod(w0 * 3.0 + threadIdx.x, p);
  W[2] = fmod(w0 * 7.0 + blockIdx.x, p);
#pragma unroll
  for (int i = 0; i < 3; ++i) Wp[i] = W[i] / p;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 2; b >= 0; --b) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (!(k & (1 << b))) ct_bfly_f64(x[k], x[k | (1 << b)], W[b], Wp[b], p);
    }
  }
  double acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += x[k];
  if (acc == 1234.5) sink[0] = 1;
}

}  // namespace

extern "C" {

int ckb_ntt_forward(const ckb_ring* ring, uint64_t* data, int rows, int limbs,
                    const int32_t* limb_prime, void* stream) {
  return ntt_run<true>(ring, data, rows, limbs, limb_prime, stream);
}

int ckb_ntt_inverse(const ckb_ring* ring, uint64_t* data, int rows, int limbs,
                    const int32_t* limb_prime, void* stream) {
  return ntt_run<false>(ring, data, rows, limbs, limb_prime, stream);
}

int ckb_ntt_forward_combine(const ckb_ring* ring, uint64_t* out, uint64_t* E, const uint64_t* x,
                            int64_t x_poly_stride, const uint64_t* addend, int addend_polys,
                            int addend_period, int addend_stride, int polys, int limbs,
                            const int32_t* limb_prime, int n_drop1, int n_drop2,
                            const uint64_t* tab1, const uint64_t* tab2, const uint64_t* post,
                            int64_t post_poly_stride, void* stream) {
  if (n_drop1 < 0 || n_drop2 < 0 || n_drop1 + n_drop2 >= limbs || polys < 0 || !E || !out || !x)
    return CKB_E_ARG;
  if ((n_drop1 && !tab1) || (n_drop2 && !tab2)) return CKB_E_ARG;
  if (addend && (addend_period < 1 || addend_polys < 0 || addend_polys > addend_period ||
                 addend_stride < addend_polys))
    return CKB_E_ARG;
  const int m2 = limbs - n_drop1 - n_drop2;
  if (!polys) return 0;
  CombineEp ep;
  ep.out = out;
  ep.x = x;
  ep.xs = x_poly_stride > 0 ? (size_t)x_poly_stride : ((size_t)limbs << ring->log_n);
  ep.add = addend;
  ep.add_polys = addend ? addend_polys : 0;
  ep.add_period = addend ? addend_period : 1;
  ep.add_stride = addend ? addend_stride : 0;
  ep.m1 = limbs - n_drop1;
  ep.tab1 = tab1;
  ep.tab2 = tab2;
  ep.n1 = n_drop1;
  ep.n2 = n_drop2;
  ep.post = post;
  ep.post_stride = post_poly_stride > 0 ? (size_t)post_poly_stride : ((size_t)m2 << ring->log_n);
  // the transform's rows are E's: m2 limbs per poly, primes = the first m2 of the basis
  return ntt_run<true>(ring, E, polys * m2, m2, limb_prime, stream, nullptr, 0, ep);
}

int ckb_ntt_forward_from(const ckb_ring* ring, uint64_t* dst, const uint64_t* src,
                         int64_t src_item_stride, int rows, int limbs, const int32_t* limb_prime,
                         void* stream) {
  if (!src || src_item_stride < 0) return CKB_E_ARG;
  return ntt_run<true>(ring, dst, rows, limbs, limb_prime, stream, src,
                       src_item_stride ? (size_t)src_item_stride : ((size_t)limbs << ring->log_n));
}

int ckb_ntt_inverse_from(const ckb_ring* ring, uint64_t* dst, const uint64_t* src,
                         int64_t src_item_stride, int rows, int limbs, const int32_t* limb_prime,
                         void* stream) {
  if (!src || src_item_stride < 0) return CKB_E_ARG;
  return ntt_run<false>(ring, dst, rows, limbs, limb_prime, stream, src,
                        src_item_stride ? (size_t)src_item_stride : ((size_t)limbs << ring->log_n));
}


int ckb_ks_ntt_mac(const ckb_ring* ring, uint64_t* acc, uint64_t* digits, int batch, int limbs,
                   int alpha, int ext_limbs, const int32_t* ext_prime, const int32_t* digit_prime,
                   const uint64_t* own, int64_t own_batch_stride, const uint64_t* key,
                   const uint64_t* const* key_ptrs, int key_limbs, const int32_t* key_limb,
                   void* stream) {
  LimbMap em, kmap;
  if (!make_map(em, ext_prime, ext_limbs) || !make_map(kmap, key_limb, ext_limbs))
    return CKB_E_LIMBS;
  if (batch < 0 || alpha < 1 || limbs < 1 || ext_limbs <= limbs || !own || !digits || !acc ||
      (!key && !key_ptrs))
    return CKB_E_ARG;
  const RingDev R = make_ring(ring);
  const int logn = (int)R.log_n;
  if (logn <= 12 || logn > 20) return CKB_E_LOGN;  // two-phase transforms only
  const int nd = (limbs + alpha - 1) / alpha;
  const int out_rows = ext_limbs - alpha;
  const int item_rows = (nd - 1) * out_rows + ext_limbs - (limbs - (nd - 1) * alpha);
  if (item_rows > kMaxLimbs) return CKB_E_LIMBS;
  LimbMap dm;
  if (!make_map(dm, digit_prime, item_rows)) return CKB_E_LIMBS;
  if (!batch) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = 1 << logn;
  const int s2 = logn / 2, s1 = logn - s2;
  if (s1 > 12 || s2 != 8) return CKB_E_LOGN;  // the fused row kernel is built for 256-row groups
  const int GA = 1 << s1, GB = 1 << s2;
  const int CA = std::max(1, kTwoPhaseTile / GA), CB = std::max(1, kTwoPhaseTile / GB);
  auto lg = [](int v) { int l = 0; while ((1 << l) < v) ++l; return l; };
  bool any_f64 = false, any_int = false;
  for (int i = 0; i < item_rows; ++i) {
    const int pi = dm.p[i];
    ((R.f64_mask[pi >> 6] >> (pi & 63)) & 1 ? any_f64 : any_int) = true;
  }
  const size_t budget = R.ntt_chunk_bytes ? (size_t)R.ntt_chunk_bytes : kDefaultNttChunkBytes;
  const int chunk = std::max(1, (int)(budget / ((size_t)item_rows * N * 8)));
  const bool mixed_one_kernel = !(R.flags & CKB_RING_NTT_SPLIT);
  KsMac km{acc, digits, own, own_batch_stride > 0 ? (size_t)own_batch_stride : ((size_t)limbs << logn),
           key, key_ptrs, key_limbs, nd, ext_limbs, out_rows, item_rows, alpha, limbs, 0, GA / CB};
  constexpr int S = 8, RBT = 4;
  constexpr int G = 1 << S, E = 1 << RBT, C = kTwoPhaseTile / G, T = C * G / E;
  const size_t smem = (size_t)C * (G + G / 16 + G / 128) * 8 + 2 * (size_t)(E / 2) * T * 16;
  static bool attr = false;  // idempotent, set before the first launch of this process
  if (!attr) {
    cudaFuncSetAttribute(k_ntt_rows_mac<S, RBT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  for (int i0 = 0; i0 < batch; i0 += chunk) {
    const int ni = std::min(chunk, batch - i0);
    uint64_t* data = digits + (size_t)i0 * item_rows * N;
    // column phase of the chunk's digit rows (limb-major within the chunk)
    NttPhase pa{item_rows, GB / CA, CA, 1, GB, 1, 0, 0, 0, lg(CA), ni > 1 ? ni : 0, 1, nullptr, 0};
    int rc;
    const int rows = ni * item_rows;
    if (!any_f64 || (any_int && mixed_one_kernel)) {
      rc = launch_phase<true, 4, 0>(s1, data, pa, rows, R, dm, st);
    } else {
      rc = launch_phase<true, 4, 1>(s1, data, pa, rows, R, dm, st);
      if (!rc && any_int) rc = launch_phase<true, 4, 2>(s1, data, pa, rows, R, dm, st);
    }
    if (rc) return rc;
    km.item0 = i0;
    const int blocks = ni * ext_limbs * km.tiles;
    k_ntt_rows_mac<S, RBT><<<blocks, T, smem, st>>>(km, R, em, kmap);
  }
  return finish();
}

int ckb_alu_probe(uint64_t p, uint64_t w, int iters, int blocks, uint64_t* sink, void* stream) {
  if (p < 3 || (p >> 60) != 0 || w >= p || iters < 1 || (iters & 1) || blocks < 1 || !sink)
    return CKB_E_ARG;
  k_alu_probe<<<blocks, 256, 0, (cudaStream_t)stream>>>(p, w, iters, sink);
  return finish();
}

int ckb_alu_probe_f64(uint64_t p, uint64_t w, int iters, int blocks, uint64_t* sink,
                      void* stream) {
  if (p < 3 || (p >> 47) != 0 || w >= p || iters < 1 || blocks < 1 || !sink) return CKB_E_ARG;
  k_alu_probe_f64<<<blocks, 256, 0, (cudaStream_t)stream>>>((double)p, (double)w, iters, sink);
  return finish();
}
}  // extern "C"
