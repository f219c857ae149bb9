// dkss_arith.cuh -- multi-limb arithmetic mod p for the DKSS ring R = (Z/pZ)[alpha]/(alpha^m+1).
//
// Residues are canonical in [0, p), stored as L little-endian u32 limbs (L = ceil(d/32)).
// The ring product (reference r_mul, bigmul/dkss.py:401-420) is computed here as a
// negacyclic convolution
//     c_k = sum_i x_i * z_{k-i},   z_j = y_j (j >= 0),  z_j = p - y_{j+m} (j < 0)
// so every term is a plain non-negative product (the wrap alpha^m = -1 is folded into
// z).  Products are accumulated exactly in radix-2^28 column sums held in 64-bit
// registers: each 28x28-bit digit product is ONE IMAD.WIDE.U32 (a*b + c64) with no
// carry handling at all (measured ~100 IMAD.WIDE/clk/SM on B200, vs ~50 limb products
// per clk/SM for the radix-2^32 mad.lo.cc/madc.hi.cc chain; tools/microbench_imad.cu).
// Column capacity: m * ndig products of < 2^56 each <= 32*7*2^56 < 2^64.
//
// One Montgomery reduction (R = 2^(32L)) per output coefficient brings the
// <= 2d+log2(m)-bit sum back to a canonical residue; twiddle tables are stored in
// Montgomery form (rho^s * R mod p) so twiddle products come out exact.
#pragma once
#include <cstdint>

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
};

template <int L>
struct NDig {
  static constexpr int v = (32 * L + 27) / 28;  // radix-2^28 digits covering 32L bits
};

__device__ __forceinline__ uint32_t fshr(uint32_t lo, uint32_t hi, uint32_t sh) {
  return __funnelshift_r(lo, hi, sh);
}

// radix-2^32 limbs -> radix-2^28 digits
template <int L>
__device__ __forceinline__ void to_r28(const uint32_t (&w)[L], uint32_t (&d)[NDig<L>::v]) {
  constexpr int ND = NDig<L>::v;
#pragma unroll
  for (int j = 0; j < ND; ++j) {
    const int bit = 28 * j, q = bit >> 5, s = bit & 31;
    const uint32_t lo = q < L ? w[q] : 0u;
    const uint32_t hi = q + 1 < L ? w[q + 1] : 0u;
    d[j] = (s == 0 ? lo : fshr(lo, hi, s)) & 0x0FFFFFFFu;
  }
}

// acc[t] += x (x) z over digit columns: NDxND IMAD.WIDE.U32, no carries
template <int ND>
__device__ __forceinline__ void mac_cols(uint64_t (&acc)[2 * ND - 1], const uint32_t (&x)[ND],
                                         const uint32_t (&z)[ND]) {
#pragma unroll
  for (int a = 0; a < ND; ++a)
#pragma unroll
    for (int b = 0; b < ND; ++b) acc[a + b] += (uint64_t)x[a] * z[b];
}

// r (L limbs) = (a + b) mod p
template <int L>
__device__ __forceinline__ void add_mod(uint32_t (&r)[L], const uint32_t (&a)[L], const uint32_t (&b)[L],
                                        const ModCtx& M) {
  uint32_t s[L], t[L];
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    c += (uint64_t)a[i] + b[i];
    s[i] = (uint32_t)c;
    c >>= 32;
  }
  int64_t br = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    int64_t x = (int64_t)s[i] - M.p[i] + br;
    t[i] = (uint32_t)x;
    br = x >> 32;
  }
  // s + carry*2^(32L) >= p  <=>  carry || no borrow
  const bool ge = (c != 0) || (br == 0);
#pragma unroll
  for (int i = 0; i < L; ++i) r[i] = ge ? t[i] : s[i];
}

// r = (a - b) mod p
template <int L>
__device__ __forceinline__ void sub_mod(uint32_t (&r)[L], const uint32_t (&a)[L], const uint32_t (&b)[L],
                                        const ModCtx& M) {
  uint32_t s[L], t[L];
  int64_t br = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    int64_t x = (int64_t)a[i] - b[i] + br;
    s[i] = (uint32_t)x;
    br = x >> 32;
  }
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    c += (uint64_t)s[i] + M.p[i];
    t[i] = (uint32_t)c;
    c >>= 32;
  }
#pragma unroll
  for (int i = 0; i < L; ++i) r[i] = br ? t[i] : s[i];
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

// Montgomery reduction of a (2L+1)-limb value T < 2^(32(2L+1)) with T/R < 2^32 * p
// (true for every caller: T < m*p^2 + small).  Returns the canonical residue T*R^-1 mod p.
template <int L>
__device__ __forceinline__ void redc(uint32_t (&r)[L], uint32_t (&t)[2 * L + 1], const ModCtx& M) {
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
  // v = t[L .. 2L] (L+1 limbs), v < (2^32 + 1) p.  Estimate floor(v/p) from the top limbs.
  const float vf = __uint2float_rz(t[2 * L]) * 18446744073709551616.0f + __uint2float_rz(t[2 * L - 1]) * 4294967296.0f +
                   __uint2float_rz(t[2 * L - 2]);
  const uint32_t qh = (uint32_t)__float2uint_rz(vf * M.pf_inv);
  // v -= qh * p
  uint32_t v[L + 1];
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

// radix-2^28 column sums -> (2L+1) radix-2^32 limbs (value < 2^(32(2L+1)) by the bound)
template <int L>
__device__ __forceinline__ void cols_to_limbs(const uint64_t (&col)[2 * NDig<L>::v - 1], uint32_t (&t)[2 * L + 1]) {
  constexpr int ND = NDig<L>::v;
  constexpr int NC = 2 * ND - 1;
  constexpr int NT = 2 * L + 1;
  uint32_t dg[NC + 2];
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    c += col[k];
    dg[k] = (uint32_t)c & 0x0FFFFFFFu;
    c >>= 28;
  }
  dg[NC] = (uint32_t)c & 0x0FFFFFFFu;
  dg[NC + 1] = (uint32_t)(c >> 28);
#pragma unroll
  for (int i = 0; i < NT; ++i) t[i] = 0;
#pragma unroll
  for (int k = 0; k < NC + 2; ++k) {
    const int bit = 28 * k, q = bit >> 5, s = bit & 31;
    if (q < NT) t[q] |= dg[k] << s;
    if (s > 4 && q + 1 < NT) t[q + 1] |= dg[k] >> (32 - s);
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
