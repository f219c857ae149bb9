// smul_kernels.cuh -- sm_100a kernels for Schoenhage-Strassen multiplication (SMUL), the
// reference's comparison baseline for DKSS (bigmul/smul.py, bigmul/fermat.py; SURVEY.md
// §8(f) rank 3).  Outermost (cyclic) level: a*b = inverse FFT of the pointwise product of
// the length-n FFTs of the s-bit slices of a and b over Z/(2^K+1) with root 2^omega_exp
// (bigmul/smul.py:256-271), normalised by 2^-m and overlap-added at stride s
// (bigmul/smul.py:240-249).
//
// Data layout in HBM: an FFT vector is uint32[n][KW] (KW = K/32 limbs per element, little
// endian) plus uint32 top[n], the element's bit K -- elements are canonical in [0, 2^K]
// like the reference's (bigmul/fermat.py:1-8), so 2^K itself needs the extra word.
//
// Element arithmetic is warp-cooperative: lane l holds limbs [l*Q, l*Q+Q) of one element
// in registers (Q = ceil(KW/32)); a multi-limb add ripples inside the lane and resolves
// the carries between lanes with one (generate, propagate) ballot add.  Multiplying by a
// root power 2^e is a cyclic shift (bigmul/fermat.py:37-49): the limbs are read from the
// element's shared-memory copy at the shifted offset, the bits that wrap past 2^K are
// subtracted.  FFT passes hold 2^nlv elements of one transform per CTA in shared memory
// and run nlv radix-2 DIT levels of bigmul/fft.py:82-104 on them.
#pragma once
#include <cstdint>

namespace dkss {


struct SmulFftArgs {
  uint32_t* x;    // [npoly][n][KW]
  uint32_t* top;  // [npoly][n]
  int log_n, KW, K;
  int omega_fwd;  // forward root 2^omega_fwd of order n (= 2K/n on the outermost level)
  int inverse;    // 1: transform with the inverse root 2^(2K - omega_fwd)
  int lv0, nlv;   // DIT levels [lv0, lv0 + nlv): merges of length 2^(l+1)
  int post_e;     // >= 0: multiply every element by 2^post_e after the last level
  // encode fused into the first pass (enc_a non-null): polynomial q < enc_batch is the slices
  // of operand q of enc_a, q >= enc_batch of operand q - enc_batch of enc_b ([batch][enc_na])
  const uint32_t* enc_a;
  const uint32_t* enc_b;
  long long enc_na, enc_s;
  int enc_batch;
};

// limb i of the s-bit slice j of operand a (na limbs): bigmul/words.py:307-329
__device__ __forceinline__ uint32_t smul_slice_limb(const uint32_t* a, long long na, long long s, long long j, int i) {
  const long long rel = 32LL * i;  // bit offset inside the slice
  if (rel >= s) return 0u;
  const long long bit = j * s + rel;
  const long long wi = bit >> 5;
  const int sh = (int)(bit & 31);
  const uint32_t l0 = wi < na ? a[wi] : 0u, l1 = wi + 1 < na ? a[wi + 1] : 0u;
  uint32_t w = sh ? __funnelshift_r(l0, l1, sh) : l0;
  const long long keep = s - rel;
  if (keep < 32) w &= (1u << keep) - 1u;
  return w;
}

struct SmulPwArgs {
  const uint32_t* x;     // transforms of a: [batch][n][KW] + top
  const uint32_t* xtop;
  const uint32_t* y;     // transforms of b (== x for a square)
  const uint32_t* ytop;
  uint32_t* out;         // products, written at bit-reversed positions (input of the inverse)
  uint32_t* otop;
  int log_n, KW;
  long long count;       // batch * n products
};

// ---- warp-distributed multi-limb arithmetic ---------------------------------------------

// Shared-memory element layout: lane l touches limbs l*Q + j, a stride-Q pattern that is a
// Q-way bank conflict for Q a power of two; those layouts insert one pad word after every
// 32 limbs (limb i at i + i/32), which spreads the 32 lanes over 32 banks.
template <int Q>
__host__ __device__ constexpr bool smul_pad() { return Q >= 2 && (Q & (Q - 1)) == 0; }
template <int Q>
__device__ __forceinline__ int spos(int i) { return smul_pad<Q>() ? i + (i >> 5) : i; }
__host__ __device__ inline int smul_elem_stride(int KW, bool pad) { return KW + (pad ? (KW + 31) / 32 : 0); }

// r = x + (sub ? ~y : y) + cin over KW limbs; returns the carry out of limb KW-1
template <int Q, bool FULL = false>  // FULL: KW == 32*Q, every limb slot is live
__device__ __forceinline__ uint32_t w_add(uint32_t (&r)[Q], const uint32_t (&x)[Q], const uint32_t (&y)[Q], uint32_t cin,
                                          bool sub, int KW) {
  const int lane = threadIdx.x & 31, base = lane * Q;
  uint32_t c = 0;
  bool ones = true;
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    if (FULL || base + j < KW) {
      const unsigned long long s = (unsigned long long)x[j] + (sub ? ~y[j] : y[j]) + c;
      r[j] = (uint32_t)s;
      c = (uint32_t)(s >> 32);
      ones &= r[j] == 0xFFFFFFFFu;
    } else {
      r[j] = 0;
    }
  }
  const bool valid = FULL || base < KW;
  const unsigned G = __ballot_sync(0xFFFFFFFFu, valid && c), P = __ballot_sync(0xFFFFFFFFu, valid && ones && !c);
  const unsigned long long a = (unsigned long long)(G | P), b = G;
  const unsigned long long carries = (a + b + cin) ^ a ^ b;  // bit l: carry into lane l
  uint32_t ci = (uint32_t)(carries >> lane) & 1u;
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    if (FULL || base + j < KW) {
      const uint32_t t = r[j] + ci;
      ci = ci && t == 0u;
      r[j] = t;
    }
  }
  const int lk = FULL ? 31 : (KW - 1) / Q;  // lane holding limb KW-1
  return (uint32_t)(carries >> (lk + 1)) & 1u;
}

template <int Q>
__device__ __forceinline__ bool w_nonzero(const uint32_t (&x)[Q]) {
  uint32_t o = 0;
#pragma unroll
  for (int j = 0; j < Q; ++j) o |= x[j];
  return __any_sync(0xFFFFFFFFu, o != 0);
}

// (u + t) mod 2^K+1 for canonical u, t (bigmul/fermat.py:25-28)
template <int Q, bool FULL = false>
__device__ __forceinline__ int w_addmod(uint32_t (&r)[Q], const uint32_t (&u)[Q], int ut, const uint32_t (&t)[Q], int tt,
                                        int KW) {
  const uint32_t c = w_add<Q, FULL>(r, u, t, 0u, false, KW);
  int T = ut + tt + (int)c;
  const bool nz = w_nonzero<Q>(r);
  if (T >= 2 || (T == 1 && nz)) {  // value >= 2^K + 1: subtract it
    uint32_t z[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) z[j] = 0;
    const uint32_t nb = w_add<Q, FULL>(r, r, z, 0u, true, KW);  // r - 1
    T = T - 1 - (nb ? 0 : 1);
  }
  return T;
}

// (u - t) mod 2^K+1 for canonical u, t (bigmul/fermat.py:31-33)
template <int Q, bool FULL = false>
__device__ __forceinline__ int w_submod(uint32_t (&r)[Q], const uint32_t (&u)[Q], int ut, const uint32_t (&t)[Q], int tt,
                                        int KW) {
  const uint32_t c = w_add<Q, FULL>(r, u, t, 1u, true, KW);
  int T = ut - tt - (c ? 0 : 1);
  if (T < 0) {  // add 2^K + 1
    uint32_t z[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) z[j] = 0;
    const uint32_t c2 = w_add<Q, FULL>(r, r, z, 1u, false, KW);
    T += 1 + (int)c2;
  }
  return T;
}

// r = x * 2^e mod 2^K+1, x canonical in shared memory (limbs sx[0..KW), bit K = xtop),
// 0 <= e < 2K (bigmul/fermat.py:37-49)
template <int Q, bool FULL = false>
__device__ __forceinline__ int w_mulpow2(uint32_t (&r)[Q], const uint32_t* sx, int xtop, int e, int KW) {
  const int lane = threadIdx.x & 31, base = lane * Q;
  const int K = 32 * KW;
  bool neg = false;
  if (e >= K) {
    e -= K;
    neg = true;
  }
  if (e == 0 && !neg) {
#pragma unroll
    for (int j = 0; j < Q; ++j) r[j] = (FULL || base + j < KW) ? sx[spos<Q>(base + j)] : 0u;
    return xtop;
  }
  const int ew = e >> 5, eb = e & 31;
  uint32_t lo[Q], hi[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    const int i = base + j;
    lo[j] = hi[j] = 0;
    if (!FULL && i >= KW) continue;
    if (xtop) {  // x = 2^K = -1: x * 2^e = -2^e
      hi[j] = i == ew ? (1u << eb) : 0u;
      continue;
    }
    const int s1 = i - ew;  // limb i of (x << e) mod 2^K
    const uint32_t a1 = s1 >= 0 ? sx[spos<Q>(s1)] : 0u, a0 = s1 >= 1 ? sx[spos<Q>(s1 - 1)] : 0u;
    lo[j] = eb ? __funnelshift_l(a0, a1, eb) : a1;
    const int s2 = i + KW - ew;  // limb i of (x << e) >> K
    const uint32_t b1 = s2 < KW ? sx[spos<Q>(s2)] : 0u, b0 = s2 - 1 < KW ? sx[spos<Q>(s2 - 1)] : 0u;
    hi[j] = eb ? __funnelshift_l(b0, b1, eb) : b1;
  }
  // lo - hi (or hi - lo for e >= K: 2^K == -1 negates)
  return neg ? w_submod<Q, FULL>(r, hi, 0, lo, 0, KW) : w_submod<Q, FULL>(r, lo, 0, hi, 0, KW);
}

// SMEM: sx is an element in the padded shared-memory layout (else plain limbs in HBM)
template <int Q, bool SMEM = false, bool FULL = false>
__device__ __forceinline__ void w_store(uint32_t* sx, const uint32_t (&r)[Q], int KW) {
  const int base = (threadIdx.x & 31) * Q;
#pragma unroll
  for (int j = 0; j < Q; ++j)
    if (FULL || base + j < KW) sx[SMEM ? spos<Q>(base + j) : base + j] = r[j];
}

// ---- kernels ----------------------------------------------------------------------------

// nlv radix-2 DIT levels of bigmul/fft.py:82-104 on the 2^nlv elements
// hi | (j << lv0) | lo of one transform, held in shared memory; a warp per butterfly.  The
// first forward pass reads the operand limbs directly: element p is the s-bit slice
// bitrev(p) (bit_slices + the shuffle, bigmul/smul.py:260-261)
template <int Q, bool FULL>
__global__ void __launch_bounds__(1024) k_smul_fft(SmulFftArgs A) {
  griddep_wait();
  griddep_launch();
  extern __shared__ uint32_t smem[];
  const int G = 1 << A.nlv, KW = A.KW, K = A.K;
  uint32_t* sx = smem;
  const int ES = smul_elem_stride(KW, smul_pad<Q>());
  uint32_t* stop = smem + (long long)G * ES;
  const long long n = 1LL << A.log_n;
  uint32_t* X = A.x + (long long)blockIdx.y * n * KW;
  uint32_t* T = A.top + (long long)blockIdx.y * n;
  const long long g = blockIdx.x;
  const long long lo = g & ((1LL << A.lv0) - 1), hi = (g >> A.lv0) << (A.lv0 + A.nlv);
  auto gidx = [&](int j) { return hi | ((long long)j << A.lv0) | lo; };
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  if (A.enc_a) {  // first forward pass: the shuffled slices straight from the operand limbs
    const int q = blockIdx.y;
    const uint32_t* op = q < A.enc_batch ? A.enc_a + (long long)q * A.enc_na : A.enc_b + (long long)(q - A.enc_batch) * A.enc_na;
    for (int j = warp; j < G; j += nw) {
      const long long sl = __brev((unsigned)gidx(j)) >> (32 - A.log_n);
      for (int i = lane; i < KW; i += 32) sx[j * ES + spos<Q>(i)] = smul_slice_limb(op, A.enc_na, A.enc_s, sl, i);
      if (lane == 0) stop[j] = 0u;
    }
  } else {
    // a warp per element (contiguous KW-limb rows), copied global -> shared with cp.async so
    // every load of the tile is in flight at once (a register round trip serialised them)
    for (int j = warp; j < G; j += nw) {
      const uint32_t* src = X + gidx(j) * KW;
      for (int i = lane; i < KW; i += 32) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(sx + j * ES + spos<Q>(i));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src + i) : "memory");
      }
      if (lane == 0) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(stop + j);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(T + gidx(j)) : "memory");
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  __syncthreads();
  for (int l = A.lv0; l < A.lv0 + A.nlv; ++l) {
    const int lb = l - A.lv0;
    const long long half = 1LL << l;
    for (int pr = warp; pr < G / 2; pr += nw) {
      const int ja = ((pr >> lb) << (lb + 1)) | (pr & ((1 << lb) - 1)), jb = ja | (1 << lb);
      // root power k * n/len; omega^(n/2) = -1 = 2^K, so the exponent k * (n/len) * omega_exp
      // stays below K for the forward root 2^(2K/n); the inverse root 2^(2K - 2K/n) gives
      // 2K minus that (bigmul/fermat.py:91-93) -- 32-bit arithmetic, no modulo
      const int k = (int)(gidx(ja) & (half - 1));
      const int ef = (k << (A.log_n - l - 1)) * A.omega_fwd;
      const int e = A.inverse && ef ? 2 * K - ef : ef;
      uint32_t* pa = sx + ja * ES;
      uint32_t* pb = sx + jb * ES;
      uint32_t t[Q], u[Q], s[Q], d[Q];
      const int tt = w_mulpow2<Q, FULL>(t, pb, (int)stop[jb], e, KW);
      const int base = lane * Q;
#pragma unroll
      for (int q = 0; q < Q; ++q) u[q] = (FULL || base + q < KW) ? pa[spos<Q>(base + q)] : 0u;
      const int ut = (int)stop[ja];
      const int st = w_addmod<Q, FULL>(s, u, ut, t, tt, KW);
      const int dt = w_submod<Q, FULL>(d, u, ut, t, tt, KW);
      __syncwarp();
      w_store<Q, true, FULL>(pa, s, KW);
      w_store<Q, true, FULL>(pb, d, KW);
      if (lane == 0) {
        stop[ja] = (uint32_t)st;
        stop[jb] = (uint32_t)dt;
      }
      __syncwarp();
    }
    __syncthreads();
  }
  if (A.post_e >= 0) {  // normalisation by 2^-m (bigmul/smul.py:268-270)
    for (int j = warp; j < G; j += nw) {
      uint32_t r[Q];
      const int rt = w_mulpow2<Q, FULL>(r, sx + j * ES, (int)stop[j], A.post_e, KW);
      __syncwarp();
      w_store<Q, true, FULL>(sx + j * ES, r, KW);
      if (lane == 0) stop[j] = (uint32_t)rt;
      __syncwarp();
    }
    __syncthreads();
  }
  for (int j = warp; j < G; j += nw) {
    uint32_t* dst = X + gidx(j) * KW;
    for (int i = lane; i < KW; i += 32) dst[i] = sx[j * ES + spos<Q>(i)];
    if (lane == 0) T[gidx(j)] = stop[j];
  }
}

// pointwise products in Z/(2^K+1) (bigmul/smul.py:206-216 at the outermost level; the
// product is the same residue whichever multiplier computes it): schoolbook column sums,
// carry resolution, fold hi*2^K == -hi.  One warp per product; smem per warp:
// x, y (2*KW limbs), column sums (2*KW x 96 bit), product limbs (2*KW).
template <int WPP>
__device__ __forceinline__ void group_sync() {
  if (WPP == 1)
    __syncwarp();
  else
    __syncthreads();  // WPP > 1: the group is the whole CTA
}

template <int Q, int WPP, bool FULL>
__global__ void __launch_bounds__(WPP == 1 ? 128 : 32 * WPP) k_smul_pointwise(SmulPwArgs A) {
  griddep_wait();
  griddep_launch();
  extern __shared__ uint32_t smem[];
  const int KW = A.KW, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp / WPP, gw = warp % WPP, ngrp = (blockDim.x >> 5) / WPP, gt = gw * 32 + lane;
  const int per = 10 * KW + 8;
  uint32_t* sa = smem + (long long)grp * per;
  uint32_t* sb = sa + KW + 2;      // b with two zero limbs on either side
  uint32_t* scol = sb + KW + 2;    // [2KW][3]: low, mid, high words of the column sum
  uint32_t* sp = scol + 6 * KW;    // product limbs
  const long long n = 1LL << A.log_n;
  for (long long pk = (long long)blockIdx.x * ngrp + grp; pk < A.count; pk += (long long)gridDim.x * ngrp) {
    const long long bidx = pk >> A.log_n, k = pk & (n - 1);
    const uint32_t* xa = A.x + pk * KW;
    const uint32_t* yb = A.y + pk * KW;
    const int at = (int)A.xtop[pk], bt = (int)A.ytop[pk];
    const long long opos = bidx * n + (__brev((unsigned)k) >> (32 - A.log_n));
    if (!(at | bt)) {
      for (int i = gt; i < KW; i += 32 * WPP) {
        sa[i] = xa[i];
        sb[i] = yb[i];
      }
      if (gt < 2) {  // zero pads: the column windows run one limb off either end of b
        sb[-1 - gt] = 0u;
        sb[KW + gt] = 0u;
      }
      group_sync<WPP>();
      // two adjacent columns per thread: a[i] is loaded once for both, the b window slides by
      // one limb per step (one shared load per limb product); each column's 96-bit sum is a
      // mad.lo.cc / madc.hi.cc / addc chain, three instructions per limb product
      for (int c0 = 2 * gt; c0 < 2 * KW - 1; c0 += 2 * 32 * WPP) {
        uint32_t x0 = 0, x1 = 0, x2 = 0, y0 = 0, y1 = 0, y2 = 0;
        const int i0 = c0 - KW + 1 > 0 ? c0 - KW + 1 : 0, i1 = c0 + 1 < KW - 1 ? c0 + 1 : KW - 1;
        uint32_t bl = sb[c0 - i0], bh = sb[c0 + 1 - i0];  // b[c0 - i], b[c0 + 1 - i]
        for (int i = i0; i <= i1; ++i) {
          const uint32_t ai = sa[i];
          asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
              : "+r"(x0), "+r"(x1), "+r"(x2) : "r"(ai), "r"(bl));
          asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
              : "+r"(y0), "+r"(y1), "+r"(y2) : "r"(ai), "r"(bh));
          bh = bl;
          bl = sb[c0 - i - 1];
        }
        scol[3 * c0] = x0;
        scol[3 * c0 + 1] = x1;
        scol[3 * c0 + 2] = x2;
        if (c0 + 1 < 2 * KW) {
          scol[3 * c0 + 3] = y0;
          scol[3 * c0 + 4] = y1;
          scol[3 * c0 + 5] = y2;
        }
      }
      group_sync<WPP>();
    }
    if (gw == 0) {
      uint32_t r[Q];
      int rt;
      if (at | bt) {  // 2^K == -1
        uint32_t z[Q], v[Q];
        const int base = lane * Q;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          z[j] = 0;
          v[j] = (FULL || base + j < KW) ? (at ? yb[base + j] : xa[base + j]) : 0u;
        }
        if (at && bt) {
#pragma unroll
          for (int j = 0; j < Q; ++j) r[j] = (base + j == 0) ? 1u : 0u;
          rt = 0;
        } else {
          rt = w_submod<Q, FULL>(r, z, 0, v, at ? bt : at, KW);
        }
      } else {
        // limb c = low(C_c) + mid(C_(c-1)) + high(C_(c-2)) + carries; lane owns 2Q limbs
        const int b2 = lane * 2 * Q;
        uint32_t w[2 * Q];
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < 2 * Q; ++j) {
          const int i = b2 + j;
          unsigned long long v = c;
          if (FULL || i < 2 * KW) {
            v += scol[3 * i];
            if (i >= 1) v += scol[3 * (i - 1) + 1];
            if (i >= 2) v += scol[3 * (i - 2) + 2];
          }
          w[j] = (uint32_t)v;
          c = (uint32_t)(v >> 32);
        }
        // the lane's small carry-out goes to the next lane's first limb
        uint32_t cin = __shfl_up_sync(0xFFFFFFFFu, c, 1);
        if (lane == 0) cin = 0;
        uint32_t g = 0;
        bool ones = true;
#pragma unroll
        for (int j = 0; j < 2 * Q; ++j) {
          const unsigned long long v = (unsigned long long)w[j] + cin;
          w[j] = (uint32_t)v;
          cin = (uint32_t)(v >> 32);
          ones &= w[j] == 0xFFFFFFFFu;
        }
        g = cin;
        const unsigned GG = __ballot_sync(0xFFFFFFFFu, g != 0), PP = __ballot_sync(0xFFFFFFFFu, ones && !g);
        const unsigned long long a2 = (unsigned long long)(GG | PP), bb = GG;
        uint32_t ci = (uint32_t)((((a2 + bb) ^ a2 ^ bb)) >> lane) & 1u;
#pragma unroll
        for (int j = 0; j < 2 * Q; ++j) {
          const uint32_t t = w[j] + ci;
          ci = ci && t == 0u;
          w[j] = t;
          if (FULL || b2 + j < 2 * KW) sp[b2 + j] = w[j];
        }
        __syncwarp();
        uint32_t plo[Q], phi[Q];
        const int base = lane * Q;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          plo[j] = (FULL || base + j < KW) ? sp[base + j] : 0u;
          phi[j] = (FULL || base + j < KW) ? sp[KW + base + j] : 0u;
        }
        rt = w_submod<Q, FULL>(r, plo, 0, phi, 0, KW);
      }
      w_store<Q, false, FULL>(A.out + opos * KW, r, KW);
      if (lane == 0) A.otop[opos] = (uint32_t)rt;
    }
    group_sync<WPP>();  // the group's shared memory is reused by the next product
  }
}

struct SmulDecodeArgs {
  const uint32_t* x;  // [batch][n][KW] normalised coefficients (natural order)
  int log_n, KW;
  long long s;        // slice stride in bits
  int s_log;          // log2(s) when s is a power of two (shifts instead of 64-bit divisions), else -1
};

// sum of the 32-bit windows of coefficients k*s landing on product limb t
// (bigmul/smul.py:244-249: total = sum cv[k] << (k*s))
__device__ __forceinline__ unsigned long long smul_window_sum(const SmulDecodeArgs& D, int pidx, long long t) {
  const long long n = 1LL << D.log_n, K = 32LL * D.KW;
  const uint32_t* v = D.x + (long long)pidx * n * D.KW;
  long long k0 = 32 * t - K + 1, k1;
  if (D.s_log >= 0) {
    k0 = k0 <= 0 ? 0 : (k0 + D.s - 1) >> D.s_log;
    k1 = (32 * t + 31) >> D.s_log;
  } else {
    k0 = k0 <= 0 ? 0 : (k0 + D.s - 1) / D.s;
    k1 = (32 * t + 31) / D.s;
  }
  if (k1 > n - 1) k1 = n - 1;
  unsigned long long S = 0;
  for (long long k = k0; k <= k1; ++k) {
    const long long off = 32 * t - k * D.s;
    const uint32_t* c = v + k * D.KW;
    uint32_t w;
    if (off >= 0) {
      const int q = (int)(off >> 5), sh = (int)(off & 31);
      const uint32_t l0 = q < D.KW ? __ldg(c + q) : 0u, l1 = q + 1 < D.KW ? __ldg(c + q + 1) : 0u;
      w = sh ? __funnelshift_r(l0, l1, sh) : l0;
    } else {
      w = __ldg(c) << (int)(-off);
    }
    S += w;
  }
  return S;
}

__global__ void __launch_bounds__(kDecThreads) k_smul_decode1(DecodeArgs A, SmulDecodeArgs D) {
  griddep_wait();
  griddep_launch();
  decode1_body(A, [&](int pidx, long long t) { return smul_window_sum(D, pidx, t); });
}

}  // namespace dkss
