// Basis conversions on the 5th-generation tensor cores (tcgen05.mma kind::i8,
// sm_100a): ModUp (keys.py:84-90, the digit lift) and the fast-conversion
// ModDown correction (keys.py:98-99 with ring.py:165-189's rescale drops).
//
// Both are the same contraction.  Per coefficient (a GEMM row) a handful of
// 64-bit values v_u (the digit's y_i = [x_i qhat_i^-1]_{q_i}; for ModDown the
// y_u of the dropped special primes, rho and the rescale remainders) meet a
// per-output constant C_uj:  out_j = sum_u v_u C_uj  mod p_j.
//
// Byte slicing with pre-shifted constants: write v_u = sum_a 2^(8a) v_u[a]
// (bytes) and d_uaj = 2^(8a) C_uj mod p_j = sum_b 2^(8b) d_uaj[b].  Then
//   out_j = sum_b 2^(8b) P_jb  (mod p_j),   P_jb = sum_{u,a} v_u[a] d_uaj[b]
// and P is one u8 x u8 -> s32 GEMM: A = [rows x 8U] (each row's values as raw
// little-endian bytes), B = [(j, b) x 8U] (the constant bytes).  Each P_jb is
// < 8U * 255^2 < 2^24, so the recombination sum_b 2^(8b) P_jb stays below 2^56
// for the <= 5 byte columns of a prime < 2^40 (one Barrett reduction of a
// 64-bit word) and below 2^80 for the 8 columns of a wider prime (a 128-bit
// Barrett).  Everything is exact integer arithmetic, so the outputs equal the
// CUDA-core kernels' bit for bit (tests/test_gpu_parity.py::test_tc_*).
//
// The tensor cores take the whole multiply-accumulate (round 2's CUDA-core
// ModUp spent ~1,000 instructions per coefficient-digit on it); what is left on
// the CUDA cores is the per-value premultiply, 16-byte shared stores of the A
// rows, and per output 1-2 TMEM loads, a shift-add and one reduction.
//
// CTA = 4 warps, persistent over 128-coefficient tiles.  Per tile: every
// thread computes its row's values and stores them into the A tile (K-major,
// no swizzle: 8-row x 16-byte core matrices); one thread issues the MMAs
// (M=128, N<=256 per instruction, K=32 per step) into a TMEM accumulator and
// commits to an mbarrier; the next tile's inputs are loaded while the MMAs run;
// then warp w reads TMEM lanes 32w..32w+31 (its 32 rows) and stores the
// outputs (a warp stores 32 consecutive coefficients of one limb: 256 B).
// The constant matrix B is built once per CTA in shared memory.
#include "common.cuh"

using namespace ckb_internal;

namespace {

constexpr int kTcRows = 128;      // GEMM M (one TMEM lane per coefficient)
constexpr int kTcThreads = 128;   // per TMEM lane set; CTAs run 128 * h threads (h = 1, 2, 4)
constexpr int kTcMaxThreads = 512;
constexpr int kNarrowBits = 40;   // primes < 2^40: 5 byte columns, else 8

// ---------------------------------------------------------------------------
// PTX wrappers (tcgen05, mbarrier)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  const uint32_t a = su32(b);
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// warp-wide (all 32 lanes of one warp)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// D[tmem] (+)= A[smem] . B[smem]^T, u8 x u8 -> s32
__device__ __forceinline__ void mma_u8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(bar))
      : "memory");
}

// 8 consecutive accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
// wait for this thread's tcgen05.ld; the empty asm ties every register read
// after the wait (plain code could otherwise be scheduled above it)
template <int NV>
__device__ __forceinline__ void tmem_wait(uint32_t* v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < NV; ++i) asm volatile("" : "+r"(v[i]));
}

// Instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A/B u8 (format 0),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_u8(int m, int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// Shared-memory matrix descriptor, no swizzle: start >> 4, leading byte offset
// (between the two 16-byte core matrices of one K=32 step) >> 4, stride byte
// offset (between 8-row groups) >> 4, version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Byte offset of (row r, 16-byte K chunk c) in a K-major no-swizzle operand
// with kp bytes per row: core matrix (r/8, c) is 128 contiguous bytes.
__device__ __forceinline__ uint32_t kmaj_off(int r, int c, int kp) {
  return (uint32_t)((r >> 3) * (kp * 8) + c * 128 + (r & 7) * 16);
}

// ---------------------------------------------------------------------------
// The shared GEMM / epilogue machinery
// ---------------------------------------------------------------------------
// One output limb.  The narrow epilogue reads only the first 32 bytes.
struct __align__(16) TcSlot {
  uint64_t p;      // output modulus
  uint64_t addc;   // additive constant (mod p)
  uint32_t mu32;   // floor(2^(31+k) / p): 32-bit quotient estimate (0: generic path)
  uint32_t sh;     // k - 1
  uint32_t roff;   // row * N (elements from the tile's output base)
  int key;         // constant lookup index (ext limb / kept limb)
  uint64_t mu, k, two_p, r64, r64s;  // Barrett (wide outputs) and the generic reduction
  uint64_t w256s;                    // floor(256 * 2^64 / p): B-matrix byte shifts
  int row, pad;
};

// Column layout of the accumulator, by output prime size: narrow (<= 40
// bits, 5 byte columns, read in groups of 8 outputs = 40 columns), mid (41..48
// bits, 6 columns, groups of 4 = 24 columns), wide (>= 49 bits, 8 columns,
// pairs).  Each class starts 8-aligned.  Work units (one group or pair each)
// are spread over the warps that share a TMEM lane quarter.
struct TcCols {
  int n_narrow, n_mid, n_wide, col_mid, col_wide, n_mma, n_alloc;
  int u_narrow, u_mid, u_wide;  // work units per class
};

__host__ __device__ inline int tc_class_of_bits(int k) { return k <= 40 ? 0 : k <= 48 ? 1 : 2; }

__host__ __device__ inline TcCols tc_cols(int n_narrow, int n_mid, int n_wide) {
  TcCols c;
  c.n_narrow = n_narrow;
  c.n_mid = n_mid;
  c.n_wide = n_wide;
  c.col_mid = (5 * n_narrow + 7) & ~7;
  c.col_wide = (c.col_mid + 6 * n_mid + 7) & ~7;
  const int used = c.col_wide + 8 * n_wide;
  c.n_mma = (used + 15) & ~15;
  c.u_narrow = (n_narrow + 7) / 8;
  c.u_mid = (n_mid + 3) / 4;
  c.u_wide = (n_wide + 1) / 2;
  int read = c.n_mma;
  read = read > 40 * c.u_narrow ? read : 40 * c.u_narrow;
  read = read > c.col_mid + 24 * c.u_mid ? read : c.col_mid + 24 * c.u_mid;
  read = read > c.col_wide + 16 * c.u_wide ? read : c.col_wide + 16 * c.u_wide;
  int a = 32;
  while (a < read) a <<= 1;
  c.n_alloc = a;
  return c;
}

__host__ __device__ inline int tc_col0(const TcCols& c, int s) {
  if (s < c.n_narrow) return 5 * s;
  if (s < c.n_narrow + c.n_mid) return c.col_mid + 6 * (s - c.n_narrow);
  return c.col_wide + 8 * (s - c.n_narrow - c.n_mid);
}

// floor(2^e / p) for 63 <= e <= 95 and p >= 2^(e-63) (setup only: bitwise long division)
__device__ inline uint64_t div_pow2(int e, uint64_t p) {
  uint64_t q = (1ull << 63) / p, r = (1ull << 63) - q * p;
  for (int i = 63; i < e; ++i) {
    q <<= 1;
    r <<= 1;  // r < p < 2^63
    if (r >= p) {
      r -= p;
      q |= 1;
    }
  }
  return q;
}

// B[col][8u + a] = byte b of 2^(8a) C_uj mod p_j for the column (j, b).
// cfun(u, slot) returns C_uj (canonical).  B is zeroed first (padding rows and
// the K padding).  All threads participate; ends with a CTA barrier.
template <typename CF>
__device__ void tc_build_b(uint8_t* B, int kp, int n_rows, const TcSlot* slots, TcCols cols,
                           int nvals, CF cfun) {
  for (int i = threadIdx.x; i < n_rows * kp / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(B)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const int nslots = cols.n_narrow + cols.n_mid + cols.n_wide;
  // one (slot, value) per thread: d_0 = C, d_{a+1} = 256 d_a mod p (Shoup)
  for (int q = threadIdx.x; q < nslots * nvals; q += blockDim.x) {
    const int s = q / nvals;
    const int u = q % nvals;
    const TcSlot& S = slots[s];
    const uint64_t w = 256;  // NTT primes exceed 2^9
    const uint64_t w256s = S.w256s;
    uint64_t d = cfun(u, s);
    const int col0 = tc_col0(cols, s);
    const int nb = s < cols.n_narrow ? 5 : s < cols.n_narrow + cols.n_mid ? 6 : 8;
    for (int a = 0; a < 8; ++a) {
      const int kk = 8 * u + a;
      for (int b = 0; b < nb; ++b)
        B[kmaj_off(col0 + b, kk >> 4, kp) + (kk & 15)] = (uint8_t)(d >> (8 * b));
      d = ckb::mul_shoup(d, w, w256s, S.p);
    }
  }
  fence_async_smem();
  __syncthreads();
}

// One thread: the K steps of D = A . B^T over the n_mma columns.
__device__ __forceinline__ void tc_issue(uint32_t tmem, const uint8_t* A, const uint8_t* B,
                                         int kp, int n_mma) {
  const uint32_t a0 = su32(A), b0 = su32(B);
  const uint32_t sbo = (uint32_t)kp * 8;
  for (int ks = 0; ks < kp / 32; ++ks) {
    const uint64_t ad = sdesc(a0 + ks * 256, 128, sbo);
    for (int n0 = 0; n0 < n_mma; n0 += 256) {
      const int nn = n_mma - n0 < 256 ? n_mma - n0 : 256;
      const uint64_t bd = sdesc(b0 + (uint32_t)(n0 >> 3) * sbo + ks * 256, 128, sbo);
      mma_u8(tmem + (uint32_t)n0, ad, bd, idesc_u8(kTcRows, nn), ks > 0 ? 1u : 0u);
    }
  }
}

// v mod p for v < 2^56 (a narrow output's recombined columns).  With
// s = k - 1 and mu32 = floor(2^(32+s) / p): top = v >> s < 2^32 and
// q = hi32(top * mu32) underestimates floor(v / p) by at most 2
// (v / 2^(s+32) < 1/2 and 2^s / p <= 1), so v - q p lies in [0, 3p).
template <int FAST>
__device__ __forceinline__ uint64_t tc_reduce_narrow(uint64_t v, const TcSlot& S) {
  v += S.addc;
  if (!FAST && S.mu32 == 0) {  // primes below 2^26 (test chains): generic 128-bit reduction
    const Mod m{S.p, S.mu, S.k, S.two_p};
    return ckb::reduce128_any(0, v, S.r64, S.r64s, m);
  }
  const uint32_t top = (uint32_t)(v >> S.sh);
  const uint32_t q = __umulhi(top, S.mu32);
  uint64_t r = v - (uint64_t)q * S.p;
  if (FAST == 2) return r;  // lazy: [0, 3p), a forward-NTT input (CKB_RING_LAZY_BCONV)
  r = r >= S.p ? r - S.p : r;
  return r >= S.p ? r - S.p : r;
}

// One group of 8 narrow outputs (40 accumulator columns from 5g).  GUARD:
// the tail group (outputs past n_narrow are skipped); full groups run
// branch-free so the compiler interleaves the 8 independent reductions.
template <int FAST, bool GUARD>
__device__ __forceinline__ void tc_group8(uint32_t tl, int g, int n_narrow, const TcSlot* slots,
                                          uint64_t* __restrict__ out) {
  uint32_t v[40];
#pragma unroll
  for (int q = 0; q < 5; ++q) tmem_ld8(tl + (uint32_t)(5 * g + 8 * q), v + 8 * q);
  tmem_wait<40>(v);
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    if (!GUARD || g + o < n_narrow) {
      const TcSlot& S = slots[g + o];
      uint64_t x = (uint64_t)v[5 * o + 1] * 256u + v[5 * o];
      x += (uint64_t)v[5 * o + 2] * 65536u;
      x += (uint64_t)v[5 * o + 3] * 16777216u;
      x += (uint64_t)v[5 * o + 4] << 32;
      out[S.roff] = tc_reduce_narrow<FAST>(x, S);
    }
  }
}

// A wide output's 8 columns: v = lo + hi 2^32 < 2^80.  FAST (prime of 49..62
// bits): top = v >> (k-1) < 2^32 and q = hi32(top * mu32) is within 2 of
// floor(v / p) (v / 2^(k+31) < 0.82, 2^(k-1) / p <= 1); the remainder fits 64
// bits, so it is computed mod 2^64 from the low word.  Else 128-bit Barrett.
template <int FAST>
__device__ __forceinline__ void tc_wide1(uint32_t tl, const uint32_t* v, const TcSlot& S,
                                         uint64_t* __restrict__ out) {
  uint64_t lo = (uint64_t)v[1] * 256u + v[0];
  lo += (uint64_t)v[2] * 65536u;
  lo += (uint64_t)v[3] * 16777216u;
  lo += S.addc;
  uint64_t hi = (uint64_t)v[5] * 256u + v[4];
  hi += (uint64_t)v[6] * 65536u;
  hi += (uint64_t)v[7] * 16777216u;
  const uint64_t l = lo + (hi << 32);
  const uint64_t h = (hi >> 32) + (l < lo ? 1 : 0);
  if (FAST || S.mu32 != 0) {
    const uint32_t top = (uint32_t)__funnelshift_r((uint32_t)(l >> 32), (uint32_t)h, S.sh - 32);
    const uint32_t q = __umulhi(top, S.mu32);
    uint64_t r = l - (uint64_t)q * S.p;
    if (FAST != 2) {
      r = r >= S.p ? r - S.p : r;
      r = r >= S.p ? r - S.p : r;
    }
    out[S.roff] = r;
    return;
  }
  const Mod m{S.p, S.mu, S.k, S.two_p};
  out[S.roff] = ckb::barrett_reduce128(h, l, m);
}

// One group of 4 mid outputs (24 columns): v = sum_b<6 2^(8b) P_b < 2^64.
template <int FAST>
__device__ __forceinline__ void tc_group4_mid(uint32_t tl, int col, int g, int n_mid,
                                              const TcSlot* slots, uint64_t* __restrict__ out) {
  uint32_t v[24];
#pragma unroll
  for (int q = 0; q < 3; ++q) tmem_ld8(tl + (uint32_t)(col + 8 * q), v + 8 * q);
  tmem_wait<24>(v);
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    if (g + o < n_mid) {
      const TcSlot& S = slots[g + o];
      uint64_t x = (uint64_t)v[6 * o + 1] * 256u + v[6 * o];
      x += (uint64_t)v[6 * o + 2] * 65536u;
      x += (uint64_t)v[6 * o + 3] * 16777216u;
      x += ((uint64_t)v[6 * o + 5] * 256u + v[6 * o + 4]) << 32;
      out[S.roff] = tc_reduce_narrow<FAST>(x, S);
    }
  }
}

// Read this thread's TMEM lane and store its share of the outputs: the work
// units (narrow groups, mid groups, wide pairs, numbered in that order) with
// index = sub (mod H); out[slot.roff].  FAST: every output takes the 32-bit
// quotient path.
template <int FAST, int H>
__device__ __forceinline__ void tc_epilogue_t(uint32_t tl, TcCols cols, const TcSlot* slots,
                                              uint64_t* __restrict__ out, int sub) {
  const int un = cols.u_narrow, um = cols.u_mid, uw = cols.u_wide;
  for (int u = sub; u < un; u += H) {
    const int g = 8 * u;
    if (g + 8 <= cols.n_narrow)
      tc_group8<FAST, false>(tl, g, cols.n_narrow, slots, out);
    else
      tc_group8<FAST, true>(tl, g, cols.n_narrow, slots, out);
  }
  for (int u = un + ((sub - un) % H + H) % H; u < un + um; u += H) {
    const int g = 4 * (u - un);
    tc_group4_mid<FAST>(tl, cols.col_mid + 6 * g, g, cols.n_mid, slots + cols.n_narrow, out);
  }
  const TcSlot* ws = slots + cols.n_narrow + cols.n_mid;
  for (int u = un + um + ((sub - un - um) % H + H) % H; u < un + um + uw; u += H) {
    const int s = 2 * (u - un - um);
    uint32_t v[16];
    tmem_ld8(tl + (uint32_t)(cols.col_wide + 8 * s), v);
    tmem_ld8(tl + (uint32_t)(cols.col_wide + 8 * s + 8), v + 8);
    tmem_wait<16>(v);
    tc_wide1<FAST>(tl, v, ws[s], out);
    if (s + 1 < cols.n_wide) tc_wide1<FAST>(tl, v + 8, ws[s + 1], out);
  }
}

__device__ __forceinline__ void tc_epilogue(uint32_t tl, TcCols cols, const TcSlot* slots,
                                            uint64_t* __restrict__ out, bool fast, int sub,
                                            int h, bool lazy) {
  if (fast && lazy) {
    if (h == 1) tc_epilogue_t<2, 1>(tl, cols, slots, out, sub);
    else if (h == 2) tc_epilogue_t<2, 2>(tl, cols, slots, out, sub);
    else tc_epilogue_t<2, 4>(tl, cols, slots, out, sub);
  } else if (fast) {
    if (h == 1) tc_epilogue_t<1, 1>(tl, cols, slots, out, sub);
    else if (h == 2) tc_epilogue_t<1, 2>(tl, cols, slots, out, sub);
    else tc_epilogue_t<1, 4>(tl, cols, slots, out, sub);
  } else {
    if (h == 1) tc_epilogue_t<0, 1>(tl, cols, slots, out, sub);
    else if (h == 2) tc_epilogue_t<0, 2>(tl, cols, slots, out, sub);
    else tc_epilogue_t<0, 4>(tl, cols, slots, out, sub);
  }
}


__device__ inline void load_slot(TcSlot& s, const RingDev& R, int pi, int row, size_t N) {
  const uint64_t* mm = R.mods + (size_t)pi * kModStride;
  s.p = __ldg(mm);
  s.mu = __ldg(mm + 1);
  s.k = __ldg(mm + 2);
  s.two_p = __ldg(mm + 3);
  s.r64 = __ldg(mm + 8);
  s.r64s = __ldg(mm + 9);
  s.addc = 0;
  s.row = row;
  s.roff = (uint32_t)(row * N);
  s.key = row;
  s.pad = 0;
  s.sh = (uint32_t)s.k - 1;
  s.w256s = div_pow2(72, s.p);
  s.mu32 = 0;  // floor(2^(31+k) / p) in [2^31, 2^32) where the quotient path applies
  if (s.k >= 26 && s.k <= 48) {
    s.mu32 = (uint32_t)(s.k < 33 ? (1ull << (31 + s.k)) / s.p : div_pow2(31 + (int)s.k, s.p));
  } else if (s.k >= 49 && s.k <= 62) {
    s.mu32 = (uint32_t)div_pow2(31 + (int)s.k, s.p);
  }
}

// Split the output primes into the narrow / wide lists (thread 0).
struct TcShared {
  uint64_t bar;
  uint32_t tmem;
  int counts[3];  // outputs per class (narrow, mid, wide)
  int fast;       // every output takes the 32-bit quotient path
};

// Sort the n output slots (tmp, built in parallel) by class (narrow, mid,
// wide) into slots, stable; counts and the FAST flag into sh.  All threads.
__device__ inline void order_slots(TcSlot* slots, const TcSlot* tmp, int n, TcShared& sh) {
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int c = tc_class_of_bits((int)tmp[t].k);
    int pos = 0;
    for (int i = 0; i < n; ++i) {
      const int ci = tc_class_of_bits((int)tmp[i].k);
      pos += ci < c || (ci == c && i < t);
    }
    slots[pos] = tmp[t];
  }
  if (threadIdx.x == 0) {
    sh.counts[0] = sh.counts[1] = sh.counts[2] = 0;
    sh.fast = 1;
    for (int i = 0; i < n; ++i) {
      sh.counts[tc_class_of_bits((int)tmp[i].k)]++;
      sh.fast &= tmp[i].mu32 != 0;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// ModUp.  grid.y = digit j; persistent over (item, 128-coefficient tile).
// Values: y_i = [x_i qhat_i^-1]_{q_i} (i < cnt); constants C_ie = [qhat_i]_{p_e}
// from the bconv table.  Output rows as ckb_modup (digit_row, skip_own).
// Smem: A [128][kp] | B [n_alloc][kp] | slots [ext] | tmp slots [ext].
// ---------------------------------------------------------------------------
template <int AMAX>
__global__ void __launch_bounds__(kTcMaxThreads) k_modup_tc(
    uint64_t* __restrict__ out, const uint64_t* __restrict__ in, size_t in_bstride, int batch,
    int limbs, int ext, int alpha, int out_rows, int item_rows, int skip_own, int log_n,
    RingDev R, LimbMap lm, LimbMap em, const uint64_t* __restrict__ bconv, int kp_max,
    int nrows_max) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ TcShared sh;
  __shared__ uint64_t s_w[AMAX][3];
  const size_t N = (size_t)1 << log_n;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (kTcRows - 1), sub = tid >> 7, h = blockDim.x >> 7;
  const int j = blockIdx.y;
  const int first = j * alpha;
  const int cnt = min(alpha, limbs - first);
  const int kp = (8 * cnt + 31) & ~31;
  const size_t stride_i = 2 + 2 * (size_t)ext;
  const uint64_t* tab = bconv + (size_t)j * alpha * stride_i;
  uint8_t* A = smem;
  uint8_t* B = smem + kTcRows * kp_max;
  TcSlot* slots = reinterpret_cast<TcSlot*>(B + (size_t)nrows_max * kp_max);
  TcSlot* tmp = slots + ext;
  // output list (every ext limb outside the digit) and the digit constants
  // output list (every ext limb outside the digit, one per thread) and the
  // digit constants
  for (int e = tid; e < ext; e += blockDim.x) {
    if (e >= first && e < first + cnt) continue;
    const int idx = e < first ? e : e - cnt;
    load_slot(tmp[idx], R, em.p[e], skip_own ? idx : e, N);
    tmp[idx].key = e;  // ext index (constant lookup)
  }
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < cnt) {
    s_w[tid][0] = __ldg(tab + (size_t)tid * stride_i);
    s_w[tid][1] = __ldg(tab + (size_t)tid * stride_i + 1);
    s_w[tid][2] = __ldg(R.mods + (size_t)lm.p[first + tid] * kModStride);
  }
  __syncthreads();
  order_slots(slots, tmp, ext - cnt, sh);
  const TcCols cols = tc_cols(sh.counts[0], sh.counts[1], sh.counts[2]);
  if (cols.n_alloc > nrows_max) __trap();  // host masks disagree with the primes
  if (warp == 0) tmem_alloc(&sh.tmem, (uint32_t)cols.n_alloc);
  tc_build_b(B, kp, cols.n_alloc, slots, cols, cnt, [&](int u, int s) -> uint64_t {
    const TcSlot& S = slots[s];
    const uint64_t c = __ldg(tab + (size_t)u * stride_i + 2 + 2 * S.key);
    return c >= S.p ? c % S.p : c;
  });
  tc_after();
  const uint32_t tmem = sh.tmem;
  const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const bool fast = sh.fast;
  const bool lazy = (R.flags & CKB_RING_LAZY_BCONV) != 0;

  const int tpr = (int)(N / kTcRows);
  const int ntiles = batch * tpr;
  uint64_t x[AMAX];
  auto load = [&](int tile) {
    const int bi = tile / tpr;
    const size_t coef = (size_t)(tile % tpr) * kTcRows + row;
    const uint64_t* src = in + (size_t)bi * in_bstride + (size_t)first * N + coef;
#pragma unroll
    for (int i = 0; i < AMAX; ++i)  // this thread's 16-byte chunks: i/2 = sub (mod h)
      x[i] = i < cnt && ((i >> 1) & (h - 1)) == sub ? __ldcs(src + (size_t)i * N) : 0;
  };
  if ((int)blockIdx.x < ntiles) load(blockIdx.x);
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int bi = tile / tpr;
    const size_t coef = (size_t)(tile % tpr) * kTcRows + row;
    uint64_t* obase = out + ((size_t)bi * item_rows + (size_t)j * out_rows) * N + coef;
    // A row: y_i as raw little-endian bytes, two values per 16-byte chunk
#pragma unroll
    for (int c = 0; c < (8 * AMAX + 31) / 32 * 2; ++c) {
      if (c < kp / 16 && (c & (h - 1)) == sub) {
        uint64_t y[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 2 * c + h;
          y[h] = 0;
          if (i < AMAX && i < cnt) {
            y[h] = ckb::mul_shoup(x[i], s_w[i][0], s_w[i][1], s_w[i][2]);
            if (!skip_own) obase[(size_t)(first + i) * N] = x[i];
          }
        }
        *reinterpret_cast<ulonglong2*>(A + kmaj_off(row, c, kp)) = make_ulonglong2(y[0], y[1]);
      }
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (tid == 0) {
      tc_after();
      tc_issue(tmem, A, B, kp, cols.n_mma);
      mma_commit(&sh.bar);
    }
    if (tile + (int)gridDim.x < ntiles) load(tile + gridDim.x);  // overlaps the MMAs
    mbar_wait(&sh.bar, phase);
    phase ^= 1;
    tc_after();
    tc_epilogue(tl, cols, slots, obase, fast, sub, h, lazy);
    tc_before();
  }
  __syncthreads();
  if (warp == 0) tmem_free(tmem, (uint32_t)cols.n_alloc);
}

// ---------------------------------------------------------------------------
// ModDown correction (fast basis conversion), the tensor-core form of
// k_divround_corr_hps (ops.cu).  Per coefficient of poly pidx:
//   y_u = [x_u (P1/p_u)^-1]_{p_u} (u < n1, the dropped special limbs),
//   rho = round(sum y_u / p_u) (exact_rho near a tie),
//   r2_d: the centred mixed-radix remainders of the n2 rescale drops,
// then for every kept limb j:
//   E_j = -rho + sum_u y_u H_ju + sum_d r2_d Te_jd  (mod q_j)
// as one GEMM over the values (y_0..y_{n1-1}, rho, r2_d + q_{li_d}) with the
// constants (H_ju, q_j - 1, Te_jd); the shift of r2 is removed by addc_j.
// ---------------------------------------------------------------------------
constexpr int kTcMaxDrop = 16;

__device__ __forceinline__ int64_t centered_tc(uint64_t a, uint64_t p) {
  return a > (p >> 1) ? (int64_t)a - (int64_t)p : (int64_t)a;
}
__device__ __forceinline__ uint64_t sub_rm_tc(uint64_t acc, int64_t r, uint64_t M, uint64_t Ms,
                                              uint64_t p) {
  const uint64_t mag = (uint64_t)(r < 0 ? -r : r);
  const uint64_t t = ckb::mul_shoup(mag, M, Ms, p);
  return r < 0 ? ckb::add_mod(acc, t, p) : ckb::sub_mod(acc, t, p);
}


// exact rho (the rare tie path): same digits as ops.cu::exact_rho
__device__ __noinline__ uint64_t exact_rho_tc(const uint64_t* __restrict__ src, size_t N,
                                              int limbs, int m2, int n1, double f,
                                              const uint64_t* __restrict__ tab1, RingDev R,
                                              const LimbMap& lm) {
  int64_t r[kTcMaxDrop];
  const int s1 = 2 * (n1 + 1);
  int64_t top = 0;
  for (int d = 0; d < n1; ++d) {
    const int li = limbs - 1 - d;
    const uint64_t p = __ldg(R.mods + (size_t)lm.p[li] * kModStride);
    const uint64_t* Tb = tab1 + (size_t)li * s1;
    uint64_t a = src[(size_t)(li - m2) * N];
    for (int u = 0; u < d; ++u)
      a = sub_rm_tc(a, r[u], __ldg(Tb + 2 * u), __ldg(Tb + 2 * u + 1), p);
    r[d] = centered_tc(ckb::mul_shoup(a, __ldg(Tb + 2 * n1), __ldg(Tb + 2 * n1 + 1), p), p);
    if (r[d] != 0) top = r[d];
  }
  if (top == 0) return (uint64_t)rint(f);
  const uint64_t fl = (uint64_t)floor(f);
  return top > 0 ? fl : fl + 1;
}

template <int D1, int D2>
__global__ void __launch_bounds__(kTcMaxThreads) k_corr_tc(
    uint64_t* __restrict__ E, const uint64_t* __restrict__ T, int has_add, int polys, int limbs,
    int n1, int n2, int log_n, RingDev R, LimbMap lm, const uint64_t* __restrict__ tab1,
    const uint64_t* __restrict__ tab2, const uint64_t* __restrict__ tabE,
    const uint64_t* __restrict__ tabH, double margin, int kp, int nrows) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ TcShared sh;
  __shared__ uint64_t s_d[kTcMaxDrop][4];  // (P1/p_u)^-1, shoup, p_u, 1/p_u (bits)
  const size_t N = (size_t)1 << log_n;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (kTcRows - 1), sub = tid >> 7, h = blockDim.x >> 7;
  const int m1 = limbs - n1;
  const int m2 = m1 - n2;
  const int s1 = 2 * (n1 + 1), s2 = 2 * (n2 + 1), sE = 2 * (n1 + n2 + 1);
  constexpr int NVC = 1 + D2 + D1;  // value slots (see the A rows below)
  uint8_t* A = smem;
  uint8_t* B = smem + kTcRows * kp;
  TcSlot* slots = reinterpret_cast<TcSlot*>(B + (size_t)nrows * kp);
  TcSlot* tmp = slots + m2;
  for (int jj = tid; jj < m2; jj += blockDim.x) {  // one output slot per thread
    load_slot(tmp[jj], R, lm.p[jj], jj, N);
    // addc_j = -sum_d q_{li_d} Te_jd  (the shift making r2_d + q_{li_d} >= 0)
    const Mod m{tmp[jj].p, tmp[jj].mu, tmp[jj].k, tmp[jj].two_p};
    uint64_t a = 0;
    for (int d = 0; d < n2; ++d) {
      const uint64_t ql = __ldg(R.mods + (size_t)lm.p[m1 - 1 - d] * kModStride) % m.p;
      const uint64_t te = __ldg(tabE + (size_t)jj * sE + 2 * (n1 + d)) % m.p;
      a = ckb::add_mod(a, ckb::mul_mod(ql, te, m), m.p);
    }
    tmp[jj].addc = ckb::neg_mod(a, m.p);
  }
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < n1) {
    const uint64_t p = __ldg(R.mods + (size_t)lm.p[limbs - 1 - tid] * kModStride);
    s_d[tid][0] = __ldg(tabH + (size_t)m1 * n1 + 2 * tid);
    s_d[tid][1] = __ldg(tabH + (size_t)m1 * n1 + 2 * tid + 1);
    s_d[tid][2] = p;
    s_d[tid][3] = (uint64_t)__double_as_longlong(1.0 / (double)p);
  }
  __syncthreads();
  order_slots(slots, tmp, m2, sh);
  const TcCols cols = tc_cols(sh.counts[0], sh.counts[1], sh.counts[2]);
  if (cols.n_alloc > nrows) __trap();  // host masks disagree with the primes
  if (warp == 0) tmem_alloc(&sh.tmem, (uint32_t)cols.n_alloc);
  tc_build_b(B, kp, cols.n_alloc, slots, cols, NVC, [&](int u, int s) -> uint64_t {
    const TcSlot& S = slots[s];
    const int jj = S.key;
    uint64_t c = 0;
    if (u == 0) c = S.p - 1;  // -rho
    else if (u <= D2) c = u - 1 < n2 ? __ldg(tabE + (size_t)jj * sE + 2 * (n1 + u - 1)) : 0;
    else c = u - 1 - D2 < n1 ? __ldg(tabH + (size_t)jj * n1 + (u - 1 - D2)) : 0;
    return c >= S.p ? c % S.p : c;
  });
  tc_after();
  const uint32_t tmem = sh.tmem;
  const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const bool fast = sh.fast;
  const bool lazy = (R.flags & CKB_RING_LAZY_BCONV) != 0;
  const int trows = n1 + n2 + (has_add ? n2 : 0);
  const int tpr = (int)(N / kTcRows);
  const int ntiles = polys * tpr;
  uint64_t x[D1];
  auto load = [&](int tile) {
    const size_t pidx = tile / tpr;
    const size_t n = (size_t)(tile % tpr) * kTcRows + row;
    const uint64_t* src = T + pidx * trows * N + n;
#pragma unroll
    for (int u = 0; u < D1; ++u)
      x[u] = u < n1 && sub == 0 ? __ldcs(src + (size_t)(limbs - 1 - u - m2) * N) : 0;
  };
  if ((int)blockIdx.x < ntiles) load(blockIdx.x);
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t pidx = tile / tpr;
    const size_t n = (size_t)(tile % tpr) * kTcRows + row;
    const uint64_t* src = T + pidx * trows * N + n;
    if (sub == 0) {  // the row's values: one thread per row (rho and r2 need them all)
    uint64_t v[D1];
    double f = 0.0;
#pragma unroll
    for (int u = 0; u < D1; ++u) {
      v[u] = 0;
      if (u < n1) {
        v[u] = ckb::mul_shoup(x[u], s_d[u][0], s_d[u][1], s_d[u][2]);
        f = fma((double)v[u], __longlong_as_double((long long)s_d[u][3]), f);
      }
    }
    const double rho_d = rint(f);
    const uint64_t rho = fabs(f - rho_d) < margin
                             ? (uint64_t)rho_d
                             : exact_rho_tc(src, N, limbs, m2, n1, f, tab1, R, lm);
    // rescale drops (sequential; same integers as k_divround_corr_hps)
    int64_t r2[D2 > 0 ? D2 : 1];
#pragma unroll
    for (int d = 0; d < D2; ++d) {
      r2[d] = 0;
      if (d < n2) {
        const int li = m1 - 1 - d;
        const uint64_t* mm = R.mods + (size_t)lm.p[li] * kModStride;
        const Mod m{__ldg(mm), __ldg(mm + 1), __ldg(mm + 2), __ldg(mm + 3)};
        const uint64_t* Ta = tab1 + (size_t)li * s1;
        const uint64_t* H = tabH + (size_t)li * n1;
        const uint64_t* Tb = tab2 + (size_t)li * s2;
        const uint64_t xv = src[(size_t)(li - m2) * N];
        uint64_t w = ckb::mul_shoup(xv, __ldg(Ta + 2 * n1), __ldg(Ta + 2 * n1 + 1), m.p);
        uint64_t h = 0, l = (m.p << (__clzll((long long)m.p) - 4)) - rho;
#pragma unroll
        for (int u = 0; u < D1; ++u)
          if (u < n1) ckb::mac128(h, l, v[u], __ldg(H + u));
        w = ckb::sub_mod(w, ckb::reduce128_any(h, l, __ldg(mm + 8), __ldg(mm + 9), m), m.p);
        if (has_add) w = ckb::add_mod(w, src[(size_t)(n1 + n2 + li - m2) * N], m.p);
#pragma unroll
        for (int u = 0; u < D2; ++u)
          if (u < d) w = sub_rm_tc(w, r2[u], __ldg(Tb + 2 * u), __ldg(Tb + 2 * u + 1), m.p);
        r2[d] = centered_tc(ckb::mul_shoup(w, __ldg(Tb + 2 * n2), __ldg(Tb + 2 * n2 + 1), m.p),
                            m.p);
      }
    }
    // value list at compile-time positions: rho, r2_d + q_{li_d} (d < D2; 0
    // past n2), y_u (u < D1; 0 past n1) -- the constants of tc_build_b match
    constexpr int NV = 1 + D2 + D1;
    uint64_t vals[NV];
    vals[0] = rho;
#pragma unroll
    for (int d = 0; d < D2; ++d)
      vals[1 + d] = d < n2 ? (uint64_t)(r2[d] + (int64_t)__ldg(R.mods +
                                 (size_t)lm.p[m1 - 1 - d] * kModStride))
                           : 0;
#pragma unroll
    for (int u = 0; u < D1; ++u) vals[1 + D2 + u] = v[u];
#pragma unroll
    for (int c = 0; c < (8 * NV + 31) / 32 * 2; ++c) {
      const uint64_t a0 = 2 * c < NV ? vals[2 * c < NV ? 2 * c : 0] : 0;
      const uint64_t a1 = 2 * c + 1 < NV ? vals[2 * c + 1 < NV ? 2 * c + 1 : 0] : 0;
      *reinterpret_cast<ulonglong2*>(A + kmaj_off(row, c, kp)) = make_ulonglong2(a0, a1);
    }
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (tid == 0) {
      tc_after();
      tc_issue(tmem, A, B, kp, cols.n_mma);
      mma_commit(&sh.bar);
    }
    if (tile + (int)gridDim.x < ntiles) load(tile + gridDim.x);
    mbar_wait(&sh.bar, phase);
    phase ^= 1;
    tc_after();
    tc_epilogue(tl, cols, slots, E + pidx * m2 * N + n, fast, sub, h, lazy);
    tc_before();
  }
  __syncthreads();
  if (warp == 0) tmem_free(tmem, (uint32_t)cols.n_alloc);
}

// ---------------------------------------------------------------------------
// Self-test GEMM: D[128][n] = A[128][k] . B[n][k]^T (u8, s32), one tile.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTcThreads) k_tc_selftest(const uint8_t* __restrict__ Ag,
                                                            const uint8_t* __restrict__ Bg,
                                                            int32_t* __restrict__ D, int k,
                                                            int n, int n_alloc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ TcShared sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint8_t* A = smem;
  uint8_t* B = smem + kTcRows * k;
  for (int q = tid; q < kTcRows * k; q += blockDim.x) {
    const int r = q / k, kk = q % k;
    A[kmaj_off(r, kk >> 4, k) + (kk & 15)] = Ag[q];
  }
  for (int q = tid; q < n * k; q += blockDim.x) {
    const int r = q / k, kk = q % k;
    B[kmaj_off(r, kk >> 4, k) + (kk & 15)] = Bg[q];
  }
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  __syncthreads();
  if (warp == 0) tmem_alloc(&sh.tmem, (uint32_t)n_alloc);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sh.tmem;
  if (tid == 0) {
    tc_issue(tmem, A, B, k, n);
    mma_commit(&sh.bar);
  }
  mbar_wait(&sh.bar, 0);
  tc_after();
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < n; c += 8) {
    uint32_t v[8];
    tmem_ld8(tl + (uint32_t)c, v);
    tmem_wait<8>(v);
    for (int i = 0; i < 8; ++i) D[(size_t)tid * n + c + i] = (int32_t)v[i];
  }
  tc_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, (uint32_t)n_alloc);
}

// Tensor-pipe ceiling probe: each CTA issues `iters` back-to-back
// M=128 x N=256 x K=32 u8 MMAs (1 Mi MACs each) into one TMEM accumulator.
__global__ void __launch_bounds__(128) k_tc_probe(int iters, int32_t* __restrict__ sink) {
  __shared__ __align__(1024) uint8_t A[128 * 32];
  __shared__ __align__(1024) uint8_t B[256 * 32];
  __shared__ TcShared sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int q = tid; q < 128 * 32; q += blockDim.x) A[q] = (uint8_t)(q * 7 + blockIdx.x);
  for (int q = tid; q < 256 * 32; q += blockDim.x) B[q] = (uint8_t)(q * 13);
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  __syncthreads();
  if (warp == 0) tmem_alloc(&sh.tmem, 256);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = sh.tmem;
  if (tid == 0) {
    const uint64_t ad = sdesc(su32(A), 128, 32 * 8), bd = sdesc(su32(B), 128, 32 * 8);
    for (int it = 0; it < iters; ++it) mma_u8(tmem, ad, bd, idesc_u8(128, 256), it > 0);
    mma_commit(&sh.bar);
  }
  mbar_wait(&sh.bar, 0);
  tc_after();
  uint32_t v[8];
  tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16), v);
  tmem_wait<8>(v);
  if (v[0] == 0x7fffffffu) sink[0] = (int32_t)v[1];  // keep the result live
  tc_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 256);
}

inline int tc_alloc_cols(int n) {
  int a = 32;
  while (a < n) a <<= 1;
  return a;
}

// smem request that leaves room for exactly `ctas` resident CTAs per SM (so
// every resident CTA's TMEM allocation fits the 512 columns)
inline size_t tc_smem_request(size_t need, int n_alloc) {
  const int ctas = std::max(1, std::min(4, 512 / n_alloc));  // = tc_ctas
  return std::max(need, (size_t)(228 * 1024) / (ctas + 1));
}

}  // namespace

namespace ckb_internal {

// column class of prime index pi from the host-side masks (0 narrow, 1 mid, 2 wide)
int tc_class(const RingDev& R, int pi) {
  if ((R.wide_mask[pi >> 6] >> (pi & 63)) & 1) return 2;
  if ((R.mid_mask[pi >> 6] >> (pi & 63)) & 1) return 1;
  return 0;
}

// CTA shape: as many CTAs per SM as the 512 TMEM columns allow (<= 4), and
// 16 warps per SM in every case (h warps share each TMEM lane quarter).
inline int tc_ctas(int n_alloc) { return std::max(1, std::min(4, 512 / n_alloc)); }

// returns 1 when not applicable (caller falls back), else the launch status
int tc_modup(const RingDev& R, uint64_t* out, const uint64_t* in, size_t bstride, int batch,
             int limbs, const LimbMap& lm, int ext, const LimbMap& em, int alpha,
             const uint64_t* bconv, int skip_own, int out_rows, int item_rows, cudaStream_t st) {
  if (!(R.flags & CKB_RING_TC) || alpha < 2 || alpha > 16 || R.log_n < 7) return 1;
  const int nd = (limbs + alpha - 1) / alpha;
  int worst_rows = 0;
  for (int d = 0; d < nd; ++d) {
    const int first = d * alpha, cnt = std::min(alpha, limbs - first);
    int n3[3] = {0, 0, 0};
    for (int e = 0; e < ext; ++e) {
      if (e >= first && e < first + cnt) continue;
      n3[tc_class(R, em.p[e])]++;
    }
    const TcCols c = tc_cols(n3[0], n3[1], n3[2]);
    worst_rows = std::max(worst_rows, c.n_alloc);
  }
  if (worst_rows > 512) return 1;
  const int kp_max = (8 * alpha + 31) & ~31;
  const size_t need = (size_t)kTcRows * kp_max + (size_t)worst_rows * kp_max +
                      2 * (size_t)ext * sizeof(TcSlot);
  const size_t smem = tc_smem_request(need, worst_rows);
  const int ctas = tc_ctas(worst_rows);
  using K = decltype(&k_modup_tc<2>);
  K k = alpha <= 2 ? k_modup_tc<2> : alpha <= 4 ? k_modup_tc<4> : alpha <= 8 ? k_modup_tc<8>
      : alpha <= 12 ? k_modup_tc<12> : k_modup_tc<16>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int ntiles = batch * (int)((1u << R.log_n) / kTcRows);
  const int gx = std::max(1, std::min(ntiles, (148 * ctas + nd - 1) / nd));
  k<<<dim3((unsigned)gx, (unsigned)nd), kTcThreads * (4 / ctas), smem, st>>>(
      out, in, bstride, batch, limbs, ext, alpha, out_rows, item_rows, skip_own, (int)R.log_n, R,
      lm, em, bconv, kp_max, worst_rows);
  return finish();
}

int tc_corr(const RingDev& R, uint64_t* E, const uint64_t* T, int has_add, int polys, int limbs,
            const LimbMap& lm, int n1, int n2, const uint64_t* tab1, const uint64_t* tab2,
            const uint64_t* tabE, const uint64_t* tabH, double margin, cudaStream_t st) {
  if (!(R.flags & CKB_RING_TC) || R.log_n < 7 || !tabH || n1 < 1 || n1 > kTcMaxDrop || n2 > 2)
    return 1;
  const int m2 = limbs - n1 - n2;
  int n3[3] = {0, 0, 0};
  for (int jj = 0; jj < m2; ++jj) n3[tc_class(R, lm.p[jj])]++;
  const TcCols c = tc_cols(n3[0], n3[1], n3[2]);
  if (c.n_alloc > 512) return 1;
  const int d1 = n1 <= 6 ? 6 : n1 <= 8 ? 8 : n1 <= 11 ? 11 : n1 <= 13 ? 13 : 16;
  const int d2 = n2 == 0 ? 0 : n2 == 1 ? 1 : 2;
  const int kp = (8 * (1 + d1 + d2) + 31) & ~31;
  const size_t need = (size_t)kTcRows * kp + (size_t)c.n_alloc * kp + 2 * (size_t)m2 * sizeof(TcSlot);
  const size_t smem = tc_smem_request(need, c.n_alloc);
  const int ctas = std::max(1, std::min(4, 512 / c.n_alloc));
  using K = decltype(&k_corr_tc<6, 0>);
  K k = nullptr;
#define CKB_TCC(A_, B_) \
  if (d1 == A_ && d2 == B_) k = k_corr_tc<A_, B_>;
  CKB_TCC(6, 0) CKB_TCC(6, 1) CKB_TCC(6, 2) CKB_TCC(8, 0) CKB_TCC(8, 1) CKB_TCC(8, 2)
  CKB_TCC(11, 0) CKB_TCC(11, 1) CKB_TCC(11, 2) CKB_TCC(13, 0) CKB_TCC(13, 1) CKB_TCC(13, 2)
  CKB_TCC(16, 0) CKB_TCC(16, 1) CKB_TCC(16, 2)
#undef CKB_TCC
  if (!k) return 1;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int ntiles = polys * (int)((1u << R.log_n) / kTcRows);
  const int gx = std::max(1, std::min(ntiles, 148 * ctas));
  k<<<gx, kTcThreads * (4 / ctas), smem, st>>>(E, T, has_add, polys, limbs, n1, n2, (int)R.log_n, R, lm, tab1,
                                  tab2, tabE, tabH, margin, kp, c.n_alloc);
  return finish();
}

}  // namespace ckb_internal

extern "C" int ckb_tc_probe(int ctas, int iters, int32_t* sink, void* stream) {
  if (ctas < 1 || iters < 1 || !sink) return CKB_E_ARG;
  k_tc_probe<<<ctas, 128, 0, (cudaStream_t)stream>>>(iters, sink);
  return finish();
}

extern "C" int ckb_tc_selftest(const uint8_t* A, const uint8_t* B, int32_t* D, int k, int n,
                               void* stream) {
  if (k < 32 || k > 256 || (k & 31) || n < 16 || n > 256 || (n & 15) || !A || !B || !D)
    return CKB_E_ARG;
  const int n_alloc = tc_alloc_cols(n);
  const size_t smem = (size_t)kTcRows * k + (size_t)n * k;
  cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tc_selftest<<<1, kTcThreads, smem, (cudaStream_t)stream>>>(A, B, D, k, n, n_alloc);
  return finish();
}
