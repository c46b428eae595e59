/*
 * ckks_b200.h — C-ABI of the B200-native RNS-CKKS kernels (sm_100a).
 *
 * The reference (arxiv 2506.19693 "ReBoot", package `ciphermlp`) has no native
 * code and no FFI: its RNS-CKKS path is numpy inside `ciphermlp/ckks/*.py`.
 * Each entry point below replaces one numpy routine of that path; the
 * replaced reference function is cited beside it (paths relative to
 * /root/reference/pkg/src/ciphermlp/).  The Python host layer
 * (paper_2506_19693_b200/backend.py) binds these with ctypes — that binding is
 * the "reference-side FFI" documented in INTEGRATION.md.
 *
 * Conventions
 *  - Every polynomial is a run of `rows` limbs of N = 2^log_n uint64
 *    residues, row-major ([rows][N]); row r uses the prime
 *    `limb_prime[r % limbs]` (an index into the ring's prime table), so a
 *    batch [B][comps][limbs][N] is passed as rows = B*comps*limbs.
 *  - All data/table pointers are DEVICE pointers unless named *_host.
 *    `limb_prime`, `key_limb`, `scalars_host` are HOST arrays (copied into the
 *    kernel parameters; no allocation, no host<->device sync).
 *  - `stream` is a cudaStream_t passed as void*.  All calls are asynchronous
 *    on that stream and thread-safe (no global mutable state).
 *  - Return value: 0 on success, a positive cudaError_t on launch failure, or
 *    a negative CKB_E* code for bad arguments.
 *  - Residues are canonical ([0, p)) on input and output; primes < 2^60
 *    (ckb_build_tables rejects larger ones: lazy butterflies and the carry-free
 *    split dot products rely on it).
 */
#ifndef CKKS_B200_H
#define CKKS_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKB_MAX_LIMBS 128
#define CKB_E_ARG (-1)
#define CKB_E_LIMBS (-2)
#define CKB_E_LOGN (-3)

/* Device-resident tables for one ring degree and one prime chain.
 *   mods : [n_primes][16] {p, barrett_mu, bitlen, 2p, N^-1, shoup(N^-1),
 *                          psi_inv_brv[1]*N^-1, shoup(.), 2^64 mod p, shoup(.),
 *                          IEEE-754 bits of 1.0/p, 0...}
 *   ntt  : [n_primes][2][N][2] {psi_brv[j], shoup(.)} pairs, then {inv_psi_brv[j], shoup(.)};
 *          for primes < 2^46 (the FP64 butterfly path) each direction's 2N words
 *          are instead [N] doubles w (IEEE-754 bits) then the same [N] doubles with
 *          the entries of the two bottom stages interleaved inside each warp's
 *          block (contiguous vector loads in the row phase, csrc/ntt.cu)
 *   pair : [n_primes][n_primes][4] {p_i^-1 mod p_j, shoup(.), p_i mod p_j, 0}
 * Built on the host by ckb_build_tables, uploaded by the caller. */
typedef struct {
  uint32_t log_n;
  uint32_t n_primes;
  const uint64_t* mods;
  const uint64_t* ntt;
  const uint64_t* pair;
  /* bit i set: prime i is < 2^46 and its NTT rows may run the dedicated FP64
   * radix-16 kernel (host-side copy of the class the kernels derive from p;
   * all zero = one kernel choosing the path per row, same results). */
  uint64_t f64_mask[2];
  /* L2 budget of the two-phase transforms (N > 4096): rows are processed in
   * chunks of this many bytes so the intermediate stays in L2 between the
   * phases.  0 = 96 MB (one stream); give each of several concurrent streams a
   * share (the caller owns this struct; the library keeps no state). */
  uint64_t ntt_chunk_bytes;
  /* CKB_RING_* bits: configuration read at every call, never stored. */
  uint32_t flags;
  uint32_t reserved;
  /* Prime size classes of the tensor-core basis conversions (byte columns
   * per output): bit i of wide_mask: prime i >= 2^48 (8 columns); of
   * mid_mask: 2^40 <= prime i < 2^48 (6 columns); neither: < 2^40 (5).
   * Read only under CKB_RING_TC; a mismatch with the primes traps. */
  uint64_t wide_mask[2];
  uint64_t mid_mask[2];
} ckb_ring;

/* ckb_ring.flags */
#define CKB_RING_HPS_EXACT 1u /* test hook: settle every rho of the fast-conversion
                                 ModDown correction via the exact mixed-radix path */
#define CKB_RING_TC 4u        /* run ModUp and the fast-conversion ModDown
                                 correction on the tensor cores (tcgen05.mma
                                 kind::i8, byte-sliced; bit-identical results).
                                 Requires wide_mask. */
#define CKB_RING_LAZY_BCONV 8u /* with CKB_RING_TC: the tensor-core basis
                                 conversions (ckb_modup digits, the correction
                                 E of ckb_divround_ntt_corr) may leave outputs
                                 in [0, 3p) instead of [0, p) — valid inputs of
                                 ckb_ntt_forward*, their only consumer in a key
                                 switch; saves the final reductions */
#define CKB_RING_NTT_SPLIT 2u /* run FP64-class and integer-class NTT rows of one
                                 call as two kernels instead of one per-CTA-dispatch
                                 kernel (same integers; A/B measurements) */

/* Test hook: D[128][n] = A[128][k] . B[n][k]^T over u8 with s32 results on
 * the tensor cores (one tcgen05.mma kind::i8 tile; the operand layout of the
 * basis conversions).  k: multiple of 32 in [32, 256]; n: multiple of 16 in
 * [16, 256].  Device pointers. */
int ckb_tc_selftest(const uint8_t* A, const uint8_t* B, int32_t* D, int k, int n, void* stream);

/* Tensor-pipe ceiling probe (measurement): `ctas` CTAs each issue `iters`
 * back-to-back tcgen05.mma kind::i8 M=128 N=256 K=32 (2^20 u8 MACs each);
 * time it on `stream` for the int8 MAC/s roofline of the basis conversions.
 * sink: one device int32 (kept live, normally untouched). */
int ckb_tc_probe(int ctas, int iters, int32_t* sink, void* stream);

/* Library version (for load checks). */
int ckb_version(void);

/* Host-side table builder.  psi is chosen as in NttPlan/_primitive_2n_root
 * (ckks/ntt.py:81-89, :103-119): the smallest g>=2 with psi=g^((p-1)/2N),
 * psi^N = -1; tables are bit-reversed powers.  Outputs are HOST buffers of
 * the sizes documented for ckb_ring. */
int ckb_build_tables(uint32_t log_n, const uint64_t* primes_host, uint32_t n_primes,
                     uint64_t* mods_out, uint64_t* ntt_out, uint64_t* pair_out);

/* Negacyclic NTT, in place, natural order -> bit-reversed order.
 * Replaces NttPlan.forward (ckks/ntt.py:121-136) / RingElement.to_ntt (ring.py:109-115). */
int ckb_ntt_forward(const ckb_ring* ring, uint64_t* data, int rows, int limbs,
                    const int32_t* limb_prime, void* stream);
/* Inverse, bit-reversed -> natural order, times N^-1.
 * Replaces NttPlan.inverse (ckks/ntt.py:138-154) / RingElement.to_coeff (ring.py:117-123). */
int ckb_ntt_inverse(const ckb_ring* ring, uint64_t* data, int rows, int limbs,
                    const int32_t* limb_prime, void* stream);
/* Out-of-place forms: dst ([rows][N], contiguous) = NTT / iNTT of the rows of
 * src, row r = (item r / limbs, limb r % limbs) read at
 * src + item*src_item_stride + limb*N (0: limbs*N).  The transform's first pass
 * reads src, so a strided operand (one component of a [B][3][limbs][N] tensor
 * product) is transformed without a staging copy.  dst must not overlap src. */
int ckb_ntt_forward_from(const ckb_ring* ring, uint64_t* dst, const uint64_t* src,
                         int64_t src_item_stride, int rows, int limbs, const int32_t* limb_prime,
                         void* stream);
int ckb_ntt_inverse_from(const ckb_ring* ring, uint64_t* dst, const uint64_t* src,
                         int64_t src_item_stride, int rows, int limbs, const int32_t* limb_prime,
                         void* stream);

/* Key switching, steps 3-4 fused for N > 4096 (keys.py:88-97): the digits
 * written by ckb_modup with skip_own ([batch][item_rows][N], coefficient
 * domain; used as scratch) are forward-transformed — the column phase per
 * L2-resident chunk of items, then ONE kernel per chunk that finishes each
 * (item, extended limb, row tile) for every digit and accumulates the products
 * with the key rows — so acc ([batch][2][ext][N], NTT domain) is written
 * directly: replaces ckb_ntt_forward(digits) + ckb_ks_inner.  digit_prime: the
 * prime index of each digits row of one item (item_rows entries, the compact
 * skip_own order); the other arguments as ckb_ks_inner. */
int ckb_ks_ntt_mac(const ckb_ring* ring, uint64_t* acc, uint64_t* digits, int batch, int limbs,
                   int alpha, int ext_limbs, const int32_t* ext_prime, const int32_t* digit_prime,
                   const uint64_t* own, int64_t own_batch_stride, const uint64_t* key,
                   const uint64_t* const* key_ptrs, int key_limbs, const int32_t* key_limb,
                   void* stream);

/* Limb-wise arithmetic over rows*N residues.  Replace RingElement.add/sub/neg/
 * mul (ring.py:80-131).  op: 0 add, 1 sub, 2 mul (Hadamard), 3 neg (b unused),
 * 4 mul_add: out = a*b + c.  If 0 < b_rows < rows, b (and c) hold b_rows rows
 * that are broadcast periodically over a (e.g. one plaintext times both
 * ciphertext components, backend.py:147-151). */
int ckb_elementwise(const ckb_ring* ring, int op, uint64_t* out, const uint64_t* a,
                    const uint64_t* b, const uint64_t* c, int rows, int limbs,
                    const int32_t* limb_prime, int b_rows, void* stream);

/* Linear combination with per-limb integer scalars:
 *   out[poly][j][n] = sum_k scalars[k][j] * X_k[poly][j][n]  (mod p of limb j)
 * X_k = terms_host[k] (a HOST array of device pointers), polys of term_limbs[k]
 * >= limbs limbs each (read restricted to the first `limbs`); scalars: DEVICE
 * [n_terms][limbs] residues.  n_terms <= 16.  Multiplying by a constant slot
 * vector is multiplying by an integer, so the Chebyshev leaves of
 * bootstrapping's EvalMod become one pass (then one rescale). */
int ckb_scalar_mac(const ckb_ring* ring, uint64_t* out, const uint64_t* const* terms_host,
                   const int32_t* term_limbs, const uint64_t* scalars, int n_terms, int polys,
                   int limbs, const int32_t* limb_prime, void* stream);

/* Plaintext multiply-accumulate over the terms of a baby-step/giant-step row
 * (the CoeffToSlot / SlotToCoeff diagonals of bootstrapping):
 *   out[r][n] = sum_t X_t[r][n] * pts[t][r % limbs][n]  (mod p of limb r % limbs)
 * with X_t = x0 when term_idx[t] == -1, else stack + term_idx[t]*stack_stride
 * (elements), all X_t laid out like out: `rows` rows of N.  n_terms <= 64;
 * one 128-bit lazy sum and one reduction per coefficient.  Replaces a chain of
 * RingElement.mul / add (ring.py:80-131) with one pass over the operands. */
int ckb_pt_mac(const ckb_ring* ring, uint64_t* out, const uint64_t* x0, const uint64_t* stack,
               int64_t stack_stride, const int32_t* term_idx, const uint64_t* pts,
               int64_t pt_stride, int n_terms, int rows, int limbs, const int32_t* limb_prime,
               void* stream);
/* out = a * scalar[limb]; scalars_host is [limbs][2] {v, floor(v*2^64/p)} with v < p.
 * Replaces RingElement.scalar_mul (ring.py:110-115 of RingElement; backend.py:108-111). */
int ckb_scalar_mul(const ckb_ring* ring, uint64_t* out, const uint64_t* a, int rows,
                   int limbs, const int32_t* limb_prime, const uint64_t* scalars_host,
                   void* stream);

/* Ciphertext tensor product in the NTT domain (backend.py:136-140):
 * a,b: [batch][2][limbs][N]; out: [batch][3][limbs][N] = (a0b0, a0b1+a1b0, a1b1). */
int ckb_tensor(const ckb_ring* ring, uint64_t* out, const uint64_t* a, const uint64_t* b,
               int batch, int limbs, const int32_t* limb_prime, void* stream);

/* Key-switch ModUp (keys.py:84-90): split `in` (batch item b at
 * in + b*in_batch_stride, 0 meaning limbs*N; [limbs][N] coefficient domain,
 * basis limb_prime) into digits of `alpha` limbs and lift each digit into
 * the extended basis ext_prime (ext_limbs entries; the first `limbs` entries must
 * equal limb_prime).  alpha == 1 reproduces the reference's centered per-limb
 * digits exactly; alpha > 1 is the standard fast basis conversion using
 * bconv (device table [digits][alpha][2 + 2*ext_limbs]; see backend.py docs).
 * out: [batch][digits][ext_limbs][N], coefficient domain.  With skip_own a
 * digit's own limbs are not written and digit j keeps ext_limbs - width_j rows
 * (the ext basis without its own limbs) at row offset j*(ext_limbs - alpha) of
 * its item; a short last digit (limbs % alpha != 0) therefore has more rows and
 * an item holds (digits-1)*(ext_limbs-alpha) + ext_limbs - width_last rows.  The
 * skipped limbs' NTT is the NTT-domain input itself, which ckb_ks_inner reads
 * directly.  With CKB_RING_TC (alpha > 1, N >= 128) the per-output sums run on
 * the tensor cores (tcgen05.mma kind::i8, byte-sliced; csrc/tc.cu), same
 * integers. */
int ckb_modup(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int64_t in_batch_stride,
              int batch, int limbs, const int32_t* limb_prime, int ext_limbs,
              const int32_t* ext_prime, int alpha, const uint64_t* bconv, int skip_own,
              void* stream);

/* Key-switch inner product in the NTT domain (keys.py:91-97):
 *   acc[b][c][e] = sum_j digits[b][j][e] * key_b[j][c][key_limb[e]]
 * digits: [batch][n_digits][rows][N] with rows = ext_limbs, or (own != NULL)
 * the compact per-digit layout written by ckb_modup(skip_own), the own limbs then
 * read from `own` ([limbs][N] per item at b*own_batch_stride, NTT domain).
 * acc: [batch][2][ext_limbs][N].  key_ptrs: DEVICE array of `batch` pointers to
 * keys laid out [key_rows][2][key_limbs][N]; if NULL, `key` is used for every item. */
int ckb_ks_inner(const ckb_ring* ring, uint64_t* acc, const uint64_t* digits, int batch,
                 int n_digits, int ext_limbs, const int32_t* ext_prime, int alpha, int limbs,
                 const uint64_t* own, int64_t own_batch_stride, const uint64_t* key,
                 const uint64_t* const* key_ptrs, int key_limbs, const int32_t* key_limb,
                 void* stream);
/* The same with an addend folded in for ext limbs e < fold_limbs (the Q limbs):
 *   acc[b][0][e] += fold_b[b][e] * P_e,  acc[b][1][e] += fold_a[b][e] * P_e  (mod q_e)
 * fold_b / fold_a: DEVICE [limbs][N] per item at b*stride (NTT domain; fold_a may
 * be NULL), fold_mul: DEVICE [fold_limbs][2] {P mod q_e, shoup(.)} with P the
 * special modulus the following ModDown divides by.  That ModDown then yields
 * x P^-1 + addend directly (backend.py:136-143's d0/d1, :155-171's c0'), so it
 * reads no addend (and needs no addend rows for a fused rescale).  n_digits <= 8. */
int ckb_ks_inner_fold(const ckb_ring* ring, uint64_t* acc, const uint64_t* digits, int batch,
                      int n_digits, int ext_limbs, const int32_t* ext_prime, int alpha, int limbs,
                      const uint64_t* own, int64_t own_batch_stride, const uint64_t* key,
                      const uint64_t* const* key_ptrs, int key_limbs, const int32_t* key_limb,
                      const uint64_t* fold_b, int64_t fold_b_stride, const uint64_t* fold_a,
                      int64_t fold_a_stride, const uint64_t* fold_mul, int fold_limbs,
                      void* stream);

/* Exact divide-and-round chain (ring.py:165-189, keys.py:98-99, backend.py:86-112):
 *   x <- x * prescale[limb]              (optional; level adjust, backend.py:108-111)
 *   x <- divround(x, last n_drop1 limbs)  (dropped last-first, one prime at a time)
 *   x <- x + addend                      (optional; backend.py:142 / :171)
 *   x <- divround(x, last n_drop2 limbs)  (rescale, backend.py:86-92)
 * evaluated in mixed radix with host-precomputed constants (bit-identical to the
 * sequential reference; derivation in DESIGN.md):
 *   tab1: DEVICE [limbs][n_drop1+1][2]: for u < n_drop1 {M_u mod p_j, shoup} with
 *         M_u the product of the first u dropped primes, then {M_t^-1 mod p_j, shoup}
 *         (t = j's drop position, or n_drop1 = the whole product for kept limbs);
 *   tab2: DEVICE [limbs-n_drop1][n_drop2+1][2], the same for the second chain.
 * in: polys of `limbs` rows, poly p starting at in + p*in_poly_stride (0 means
 * limbs*N; a larger stride reads a limb prefix in place = RingElement.restrict);
 * addend: added to poly p when (p % addend_period) < addend_polys, reading addend row
 *   (p / addend_period) * addend_stride + p % addend_period of [.][limbs-n_drop1][N]; or NULL
 *   (mul_ct on [B][3] tensor products: period 2, polys 2, stride 3 -> d0,d1;
 *    rotate on [B][2] automorphed inputs: period 2, polys 1, stride 2 -> c0 only);
 * out: [polys][limbs-n_drop1-n_drop2][N]; prescale_host: [limbs][2] {v, shoup(v)} or NULL. */
int ckb_divround(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int64_t in_poly_stride,
                 const uint64_t* addend, int addend_polys, int addend_period, int addend_stride,
                 int polys, int limbs, const int32_t* limb_prime, int n_drop1, int n_drop2,
                 const uint64_t* prescale_host, const uint64_t* tab1, const uint64_t* tab2,
                 void* stream);

/* NTT-domain divide-and-round, step 1 (ring.py:165-189 / keys.py:98-99 /
 * backend.py:86-92 for ciphertexts kept in the NTT domain): from the
 * coefficient-domain dropped limbs T build the correction polynomial
 *   E_j = (sum_u r1_u M1_u) * P1^-1 + sum_u r2_u M2_u  (mod q_j), j < limbs-n_drop1-n_drop2
 * T per poly: rows [0, n1+n2) = x limbs [limbs-n1-n2, limbs), then (if has_addend)
 * n2 rows = addend limbs [limbs-n1-n2, limbs-n1); all coefficient domain.
 * tab1/tab2 as for ckb_divround; tabE: DEVICE [m2][n1+n2+1][2] {M1_u*P1^-1 mod q_j, shoup},
 * then {M2_u mod q_j, shoup}, then {C_j, 0} with C_j a multiple of q_j in [2^59, 2^61) (every r_u + C_j >= 0 and < 2^61).
 * E: [polys][m2][N], coefficient domain (NTT it next).
 * tabH (optional, used when n_drop1 >= 6 and n_drop2 <= 2): DEVICE [m1][n1]
 * {p_u^-1 mod q_j} for the kept limbs j < m1 = limbs - n_drop1, then [n1][2]
 * {(P1/p_u)^-1 mod p_u, shoup} for the dropped limbs u (drop order, u = 0 the
 * last limb).  The first chain's centred residue then comes from one fast
 * basis conversion, c1 = sum_u y_u (P1/p_u) - rho P1 with rho = round(sum y_u/p_u)
 * in FP64; coefficients whose rounding is within 2^-30 of ambiguous take the
 * mixed-radix path, so E is bit-identical either way.  With CKB_RING_TC the
 * fast-conversion form's sums over the dropped primes (and rho, r2) run as
 * one u8 GEMM on the tensor cores (csrc/tc.cu), same integers. */
/* (ckb_ring.flags & CKB_RING_HPS_EXACT sends every coefficient through the
 * exact path; default margin |frac - 1/2| < 2^-30.) */
int ckb_divround_ntt_corr(const ckb_ring* ring, uint64_t* E, const uint64_t* T, int has_addend,
                          int polys, int limbs, const int32_t* limb_prime, int n_drop1,
                          int n_drop2, const uint64_t* tab1, const uint64_t* tab2,
                          const uint64_t* tabE, const uint64_t* tabH, void* stream);
/* Steps 1b + 2 fused: forward-transform E ([polys][m2][N], coefficient domain,
 * used as scratch) and apply the combine below as the transform's last phase
 * stores, so the transformed E is never written back (same arguments as
 * ckb_divround_ntt_combine_acc; limb_prime is the full basis, whose first m2
 * entries are E's primes).  Replaces ckb_ntt_forward(E) + the combine. */
int ckb_ntt_forward_combine(const ckb_ring* ring, uint64_t* out, uint64_t* E, const uint64_t* x,
                            int64_t x_poly_stride, const uint64_t* addend, int addend_polys,
                            int addend_period, int addend_stride, int polys, int limbs,
                            const int32_t* limb_prime, int n_drop1, int n_drop2,
                            const uint64_t* tab1, const uint64_t* tab2, const uint64_t* post,
                            int64_t post_poly_stride, void* stream);
/* NTT-domain divide-and-round, step 2: out_j = (x_j * P1^-1 + add_j - E_j) * P2^-1 with x,
 * addend and E (after its forward NTT) in the NTT domain; addend addressing as ckb_divround. */
int ckb_divround_ntt_combine(const ckb_ring* ring, uint64_t* out, const uint64_t* x,
                             int64_t x_poly_stride, const uint64_t* addend, int addend_polys,
                             int addend_period, int addend_stride, const uint64_t* E, int polys,
                             int limbs, const int32_t* limb_prime, int n_drop1, int n_drop2,
                             const uint64_t* tab1, const uint64_t* tab2, void* stream);
/* ckb_divround_ntt_combine, then out += post (mod q_j) with post poly p at
 * post + p*post_poly_stride (0 means (limbs-n_drop1-n_drop2)*N), rows as out:
 * the accumulate of the rotate-and-sum schedules (packing.py:193-208,
 * linalg.py:60-82: s + rotate(s, k)) folded into the key switch's epilogue, so
 * the sum never makes a separate pass.  post may be NULL. */
int ckb_divround_ntt_combine_acc(const ckb_ring* ring, uint64_t* out, const uint64_t* x,
                                 int64_t x_poly_stride, const uint64_t* addend, int addend_polys,
                                 int addend_period, int addend_stride, const uint64_t* E,
                                 int polys, int limbs, const int32_t* limb_prime, int n_drop1,
                                 int n_drop2, const uint64_t* tab1, const uint64_t* tab2,
                                 const uint64_t* post, int64_t post_poly_stride, void* stream);
/* Galois automorphism on NTT-domain limbs (a permutation of the bit-reversed
 * evaluation slots; ring.py:222-232 transported to the evaluation domain).
 * galois_items (DEVICE, one galois per item of rows_per_item rows) or NULL. */
int ckb_automorphism_ntt(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int rows,
                         uint64_t galois, const uint64_t* galois_items, int rows_per_item,
                         void* stream);

/* Galois automorphism X -> X^galois, coefficient domain (ring.py:211-232).
 * If galois_inv_items (DEVICE, one galois^-1 mod 2N per item of rows_per_item
 * rows) is non-NULL, each item gets its own automorphism (batched rotations). */
int ckb_automorphism(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int rows,
                     int limbs, const int32_t* limb_prime, uint64_t galois,
                     const uint64_t* galois_inv_items, int rows_per_item, void* stream);

/* Canonicalise arbitrary 64-bit words per limb (x mod p): used after an
 * integer all-reduce of residue tensors across ranks (sum of <= 16 residues
 * below 2^60 cannot overflow), SURVEY §8(e). */
int ckb_reduce(const ckb_ring* ring, uint64_t* out, const uint64_t* in, int rows, int limbs,
               const int32_t* limb_prime, void* stream);

/* Device sampling (ring.py:148-158 distributions; counter-based Philox4x32-10):
 * a: [items][limbs][N] uniform residues mod each limb's prime (or NULL),
 * e: [items][N] rint(N(0, sigma^2)) int64 (or NULL); seeds: DEVICE [items] u64,
 * one independent stream per item, so batched and one-at-a-time sampling agree. */
int ckb_sample(const ckb_ring* ring, uint64_t* a, int64_t* e, const uint64_t* seeds, int items,
               int limbs, const int32_t* limb_prime, double sigma, void* stream);

/* Signed int64 coefficients -> residues (ring.py:139-145):
 * in: [polys][N] int64; out: [polys][limbs][N]. */
/* Packed residue transfer format for host <-> device copies of ciphertext
 * batches (no reference counterpart: the reference never leaves host memory;
 * RBCT, ckks/backend.py:210-247, stays the serialisation format).  Limb l of
 * each of `items` items ([items][limbs][N] uint64, canonical) is stored with
 * w_l bytes per residue — 5 for primes < 2^40, 6 below 2^48, else 8 (the
 * ckb_ring size masks) — little-endian, an item's limbs back to back.
 * ckb_packed_bytes: the packed size; ckb_pack / ckb_unpack: device buffers,
 * 8-byte aligned; unpack(pack(x)) == x for canonical x. */
int64_t ckb_packed_bytes(const ckb_ring* ring, int items, int limbs, const int32_t* limb_prime);
int ckb_pack(const ckb_ring* ring, uint8_t* out, const uint64_t* in, int items, int limbs,
             const int32_t* limb_prime, void* stream);
int ckb_unpack(const ckb_ring* ring, uint64_t* out, const uint8_t* in, int items, int limbs,
               const int32_t* limb_prime, void* stream);

int ckb_from_i64(const ckb_ring* ring, uint64_t* out, const int64_t* in, int polys, int limbs,
                 const int32_t* limb_prime, void* stream);

/* Encoder (encoding.py:34-49 + make_element, ring.py:139-145), around the
 * caller's forward FFT (cuFFT).  Step 1: spec ([batch][N] complex128,
 * interleaved) gets values[b][i] * scale (0 for i >= width) at bins[i] and at
 * bins[N/2 + i] (the conjugate bins); every entry is written.  Step 2: after
 * spec = FFT(spec), coefficient j = rint(Re(spec[j] / N * conj(twist_j))) with
 * twist ([N] complex128) = exp(i pi j / N), written as residues of every limb
 * to out ([batch][limbs][N]); if maxabs (one device u64) is non-NULL it is
 * raised to the bit pattern of max |coefficient| (the EncodingOverflow check). */
int ckb_embed_scatter(double* spec, const double* values, int batch, int width,
                      int64_t values_stride, double scale, const int32_t* bins, int log_n,
                      void* stream);
int ckb_embed_finish(const ckb_ring* ring, uint64_t* out, const double* spec, int batch,
                     int limbs, const int32_t* limb_prime, const double* twist, uint64_t* maxabs,
                     void* stream);
/* Centered CRT lift to float64 (ring.py:192-208 + encoding.py:67-69 astype):
 * in: [polys][limbs][N] coefficient domain; out: [polys][N] double. */
int ckb_to_f64(const ckb_ring* ring, double* out, const uint64_t* in, int polys, int limbs,
               const int32_t* limb_prime, void* stream);

/* ALU roofline probe (no reference counterpart; SURVEY §8(d) "measure the IMAD
 * pipe's peak with a microbenchmark"): blocks x 256 threads each run `iters`
 * radix-8 rounds (12 lazy CT butterflies, the NTT's own) on register-resident
 * residues mod p < 2^60, with the NTT's stage schedule (reducing and skipping
 * stages alternate, so `iters` must be even: CKB_E_ARG otherwise).
 * Butterflies launched = blocks * 256 * 12 * iters. */
int ckb_alu_probe(uint64_t p, uint64_t w, int iters, int blocks, uint64_t* sink, void* stream);

/* The same probe with the butterfly computed on the FP64 pipe (residues as exact
 * integers in doubles, p < 2^47): the ceiling of the FP64 NTT path. */
int ckb_alu_probe_f64(uint64_t p, uint64_t w, int iters, int blocks, uint64_t* sink,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CKKS_B200_H */
