#pragma once
// Shared internals of the B200 RNS-CKKS kernels (sm_100a); see include/ckks_b200.h.
//
// Every kernel replaces one numpy routine of the reference CKKS backend
// (/root/reference/pkg/src/ciphermlp/ckks/*.py); see the header for the map.
// The work is 64-bit modular integer arithmetic (IMAD / FP64 pipes); the one
// GEMM-shaped contraction, the basis conversion of ModUp and of the ModDown
// correction, runs on the tensor cores as a byte-sliced u8 GEMM (tc.cu).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>

#include "../../include/ckks_b200.h"
#include "modarith.cuh"

using ckb::Mod;

namespace ckb_internal {

constexpr int kMaxLimbs = CKB_MAX_LIMBS;
constexpr int kModStride = 16;  // u64 per prime in ckb_ring.mods

struct LimbMap {
  int16_t p[kMaxLimbs];
};

struct RingDev {
  const uint64_t* mods;  // [np][16]
  const uint64_t* ntt;   // [np][4][N]
  const uint64_t* pair;  // [np][np][4]
  uint32_t log_n;
  uint32_t np;
  uint64_t f64_mask[2];  // host-side prime classes (ckb_ring.f64_mask)
  uint64_t ntt_chunk_bytes;  // host-side (ckb_ring.ntt_chunk_bytes, 0 = default)
  uint32_t flags;            // host-side (ckb_ring.flags)
  uint64_t wide_mask[2];     // host-side (ckb_ring.wide_mask)
  uint64_t mid_mask[2];      // host-side (ckb_ring.mid_mask)
};

__device__ __forceinline__ Mod load_mod(const RingDev& R, int pi) {
  const uint64_t* m = R.mods + (size_t)pi * kModStride;
  Mod r;
  r.p = __ldg(m + 0);
  r.mu = __ldg(m + 1);
  r.k = __ldg(m + 2);
  r.two_p = __ldg(m + 3);
  return r;
}

inline bool make_map(LimbMap& m, const int32_t* src, int n) {
  if (n <= 0 || n > kMaxLimbs || src == nullptr) return false;
  for (int i = 0; i < n; ++i) m.p[i] = (int16_t)src[i];
  return true;
}

inline RingDev make_ring(const ckb_ring* r) {
  RingDev d;
  d.mods = r->mods;
  d.ntt = r->ntt;
  d.pair = r->pair;
  d.log_n = r->log_n;
  d.np = r->n_primes;
  d.f64_mask[0] = r->f64_mask[0];
  d.f64_mask[1] = r->f64_mask[1];
  d.ntt_chunk_bytes = r->ntt_chunk_bytes;
  d.flags = r->flags;
  d.wide_mask[0] = r->wide_mask[0];
  d.wide_mask[1] = r->wide_mask[1];
  d.mid_mask[0] = r->mid_mask[0];
  d.mid_mask[1] = r->mid_mask[1];
  return d;
}

// Tensor-core basis conversions (tc.cu).  Return 1 when not applicable (the
// caller runs its CUDA-core kernel), else the launch status.
int tc_modup(const RingDev& R, uint64_t* out, const uint64_t* in, size_t bstride, int batch,
             int limbs, const LimbMap& lm, int ext, const LimbMap& em, int alpha,
             const uint64_t* bconv, int skip_own, int out_rows, int item_rows, cudaStream_t st);
int tc_corr(const RingDev& R, uint64_t* E, const uint64_t* T, int has_add, int polys, int limbs,
            const LimbMap& lm, int n1, int n2, const uint64_t* tab1, const uint64_t* tab2,
            const uint64_t* tabE, const uint64_t* tabH, double margin, cudaStream_t st);

inline int finish() { return (int)cudaGetLastError(); }

inline int grid_for(size_t work, int block) {
  size_t g = (work + block - 1) / block;
  // persistent-ish cap: 148 SMs x 16 resident CTAs of 256 threads
  size_t cap = 148 * 16;
  return (int)std::max<size_t>(1, std::min(g, cap));
}

}  // namespace ckb_internal
