// dkss_arith.cuh -- multi-limb arithmetic mod p for the DKSS ring R = (Z/pZ)[alpha]/(alpha^m+1).
//
// Residues are canonical in [0, p), stored as L little-endian u32 limbs (L = ceil(d/32)).
// Modular reduction is Montgomery's (R = 2^(32L)) with a single-precision quotient
// estimate for the final canonicalisation, so every prime the planner can select works
// (d from 56 to 192 bits).  The ring product itself lives in dkss_kernels.cuh (ring_mul);
// twiddle tables are stored in Montgomery form (rho^s * R mod p) so twiddle products come
// out exact, and the pointwise product's R^-1 is undone by the final (2M)^-1 scaling.
#pragma once
#include <cstdint>

#include "dkss_carry.cuh"

#ifndef DKSS_MAXL
#define DKSS_MAXL 6
#endif

namespace dkss {

// ---------------------------------------------------------------------------
// per-plan modulus constants (passed by value to every kernel)
struct ModCtx {
  uint32_t p[DKSS_MAXL];
  uint32_t r2[DKSS_MAXL];      // R^2 mod p
  uint32_t kscale[DKSS_MAXL];  // (2M)^-1 * R^2 mod p  (undoes pointwise R^-1 and 2M)
  uint32_t kinv[DKSS_MAXL];    // (2M)^-1 * R mod p    (plain (2M)^-1 scaling)
  uint32_t pinv;               // -p^-1 mod 2^32
  float pf_inv;                // 2^(32(L-2)) / p  (quotient estimate)
  uint32_t cbias[DKSS_MAXL];   // -(2^(32L) - 1) * R mod p  (ring_mul bias correction)
  uint32_t proth;              // p = 1 + ptop * 2^(32(L-1)): p[0] = 1, middle limbs 0 (every
                               // table prime at the configs, 81 * 2^121 + 1); REDC specialises
  uint32_t qbias[2 * DKSS_MAXL + 1];  // p * 2^(32L + 5): keeps the pointwise bias removal >= 0
};

// r = (a + b) mod p and r = (a - b) mod p for canonical a, b (PTX carry chains, dkss_carry.cuh)
template <int L>
__device__ __forceinline__ void add_mod(uint32_t (&r)[L], const uint32_t (&a)[L], const uint32_t (&b)[L],
                                        const ModCtx& M) {
  Carry<L>::add_mod(r, a, b, M.p);
}

template <int L>
__device__ __forceinline__ void sub_mod(uint32_t (&r)[L], const uint32_t (&a)[L], const uint32_t (&b)[L],
                                        const ModCtx& M) {
  Carry<L>::sub_mod(r, a, b, M.p);
}

// r = p - a (a in [0, p]; the result p for a == 0 is never produced by callers that need
// canonical output -- see neg_mod_canon)
template <int L>
__device__ __forceinline__ void p_minus(uint32_t (&r)[L], const uint32_t (&a)[L], const ModCtx& M) {
  int64_t br = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    int64_t x = (int64_t)M.p[i] - a[i] + br;
    r[i] = (uint32_t)x;
    br = x >> 32;
  }
}

template <int L>
__device__ __forceinline__ void neg_mod_canon(uint32_t (&r)[L], const uint32_t (&a)[L], const ModCtx& M) {
  uint32_t nz = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) nz |= a[i];
  uint32_t t[L];
  p_minus<L>(t, a, M);
#pragma unroll
  for (int i = 0; i < L; ++i) r[i] = nz ? t[i] : 0u;
}

// Montgomery reduction of a (2L+1)-limb value T < 2^(32(2L+1)).  After the L REDC steps
// v = (T + q p)/R < T/R + p; the quotient floor(v/p) is estimated in single precision from
// the top three limbs, which is exact to +-1 while v/p < 2^20 (callers: ring products give
// T < m * 2^(32L) * p + p, i.e. v/p <= m + 1; mont_mul gives T < p^2).
// Returns the canonical residue T*R^-1 mod p.
template <int L>
__device__ __forceinline__ void redc(uint32_t (&r)[L], uint32_t (&t)[2 * L + 1], const ModCtx& M) {
  if (M.proth) {
    // p = 1 + ptop 2^(32(L-1)), -p^-1 = -1 mod 2^32: q = -t_i, and q p touches two limbs only
    // (t_i + q = 0 with carry t_i != 0; q ptop lands on limb i+L-1) -- one wide product per step
    const uint32_t ptop = M.p[L - 1];
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const uint32_t q = 0u - t[i];
      uint64_t c = t[i] != 0u;
#pragma unroll
      for (int j = i + 1; j < i + L - 1; ++j) {
        c += t[j];
        t[j] = (uint32_t)c;
        c >>= 32;
      }
      c += (uint64_t)q * ptop + t[i + L - 1];
      t[i + L - 1] = (uint32_t)c;
      c >>= 32;
#pragma unroll
      for (int j = i + L; j < 2 * L + 1; ++j) {
        c += t[j];
        t[j] = (uint32_t)c;
        c >>= 32;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const uint32_t q = t[i] * M.pinv;
      uint64_t c = 0;
#pragma unroll
      for (int j = 0; j < L; ++j) {
        c += (uint64_t)q * M.p[j] + t[i + j];
        t[i + j] = (uint32_t)c;
        c >>= 32;
      }
#pragma unroll
      for (int j = i + L; j < 2 * L + 1; ++j) {
        c += t[j];
        t[j] = (uint32_t)c;
        c >>= 32;
      }
    }
  }
  // v = t[L .. 2L] (L+1 limbs), v < (2^32 + 1) p.  Estimate floor(v/p) from the top limbs.
  const float vf = __uint2float_rz(t[2 * L]) * 18446744073709551616.0f + __uint2float_rz(t[2 * L - 1]) * 4294967296.0f +
                   __uint2float_rz(t[2 * L - 2]);
  const uint32_t qh = (uint32_t)__float2uint_rz(vf * M.pf_inv);
  // v -= qh * p
  uint32_t v[L + 1];
  if (M.proth) {
    const uint64_t qp = (uint64_t)qh * M.p[L - 1];
    int64_t br = 0;
#pragma unroll
    for (int j = 0; j <= L; ++j) {
      const uint32_t sub = j == 0 ? qh : j == L - 1 ? (uint32_t)qp : j == L ? (uint32_t)(qp >> 32) : 0u;
      int64_t x = (int64_t)t[L + j] - sub + br;
      v[j] = (uint32_t)x;
      br = x >> 32;
    }
  } else {
    uint64_t c = 0;
    int64_t br = 0;
#pragma unroll
    for (int j = 0; j <= L; ++j) {
      const uint64_t prod = (j < L ? (uint64_t)qh * M.p[j] : 0ull) + c;
      c = prod >> 32;
      int64_t x = (int64_t)t[L + j] - (uint32_t)prod + br;
      v[j] = (uint32_t)x;
      br = x >> 32;
    }
  }
  // qh overshoots by at most 1: negative -> add p once
  const bool neg = (int32_t)v[L] < 0;
  {
    uint64_t cc = 0;
    uint32_t w[L + 1];
#pragma unroll
    for (int j = 0; j <= L; ++j) {
      cc += (uint64_t)v[j] + (j < L ? M.p[j] : 0u);
      w[j] = (uint32_t)cc;
      cc >>= 32;
    }
#pragma unroll
    for (int j = 0; j <= L; ++j) v[j] = neg ? w[j] : v[j];
  }
  // undershoot by at most 1: v >= p -> subtract p
  {
    uint32_t w[L + 1];
    int64_t b2 = 0;
#pragma unroll
    for (int j = 0; j <= L; ++j) {
      int64_t x = (int64_t)v[j] - (j < L ? M.p[j] : 0u) + b2;
      w[j] = (uint32_t)x;
      b2 = x >> 32;
    }
    const bool ge = (b2 == 0);
#pragma unroll
    for (int j = 0; j < L; ++j) r[j] = ge ? w[j] : v[j];
  }
}

// canonical a*b mod p with a Montgomery factor: returns a*b*R^-1 mod p
template <int L>
__device__ __forceinline__ void mont_mul(uint32_t (&r)[L], const uint32_t (&a)[L], const uint32_t (&b)[L],
                                         const ModCtx& M) {
  uint32_t t[2 * L + 1];
#pragma unroll
  for (int i = 0; i < 2 * L + 1; ++i) t[i] = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    uint64_t c = 0;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      c += (uint64_t)a[i] * b[j] + t[i + j];
      t[i + j] = (uint32_t)c;
      c >>= 32;
    }
    t[i + L] = (uint32_t)c;
  }
  redc<L>(r, t, M);
}

}  // namespace dkss
