// dkss_kernels.cuh -- sm_100a kernels for the DKSS multiply (reference: bigmul/dkss.py).
//
// Data layout in HBM: a polynomial is uint32[2M][m][L] (element-major, L limbs per
// canonical residue).  A batch of polynomials is contiguous.
//
// Transform structure.  The reference's dkss_fft (bigmul/dkss.py:443-495) is a radix-2m
// decimation in time: for every column l, a length-2m DFT with root alpha over the
// elements j*mu + l, then twiddles rho^(vv*l*base_pow), then 2m recursive row
// transforms, finally a length-b base DFT with root alpha^(2m/b).  We run it IN PLACE:
// every level is one "column pass" kernel that reads a column and writes its DFT outputs
// (twiddled) back to the same positions, so after all passes the output sits in
// digit-reversed order (position of natural index i = f*2m + vv is vv*mu + pos_sub(f)).
// The product never needs natural order: the pointwise product is elementwise, and the
// third transform (the reference computes F(a_hat . b_hat), dkss.py:546) is evaluated as
// the TRANSPOSE of our forward pass sequence, F P^-1 = (P F)^T: the same passes in
// reverse order with "twiddle, then column DFT" (the DFT and twiddle matrices are
// symmetric).  Only stage-level parity checks permute back to natural order.
//
// Kernel shape.  Every pass kernel is persistent: a CTA walks tiles (NE elements = COLS
// columns, or NE contiguous elements for the bottom kernel) with a 2-stage pipeline --
// TMA bulk copies (cp.async.bulk, mbarrier completion) bring tile k+1's elements and
// twiddle rows into shared memory while tile k is transformed and multiplied.
#pragma once
#include <cstdint>
#include <type_traits>
#ifdef DKSS_EXP_TRACE
#include <cstdio>
#endif
#include "dkss_arith.cuh"

namespace dkss {


__host__ __device__ constexpr int pad_4mod8(int w) { return ((w + 3) / 8) * 8 + 4; }

// shared-memory strides (words).  Elements are L-limb residues x MM coefficients, padded
// so the elements touched by one warp start on different banks.  A twiddle row holds
// [rho~_s (MM residues) | W_s (MM residues)]; a W row holds MM residues.
template <int MM, int L>
struct Smem {
  static constexpr int ES = ((MM * L + 31) / 32) * 32 + 4;
  static constexpr int EST = pad_4mod8(2 * MM * L);
  static constexpr int ESW = ES;  // W rows double as the DFT's ping-pong buffer
};

// CTA shape per inner length m: NT threads, NE elements (COLS columns of 2m) per tile; a
// ring-product work item is T consecutive output coefficients of one element.  Registers
// are capped by MINB CTAs per SM.  TWS: twiddle rows staged in shared memory by TMA
// (m = 32 reads them through L1 instead -- the shared-memory budget of a 64-element column).
template <int MM>
struct Cfg;
template <>
struct Cfg<8> {
  static constexpr int NT = 256, COLS = 4, NE = 64, MINB = 2, T = 2;
  static constexpr bool TWS = true;
};
#ifndef DKSS_CFG16_NT  // experiment overrides (tools/exp_run.sh)
#define DKSS_CFG16_NT 256
#endif
#ifndef DKSS_CFG16_MINB
#define DKSS_CFG16_MINB 2
#endif
#ifndef DKSS_CFG16_T
#define DKSS_CFG16_T 2
#endif
template <>
#ifndef DKSS_CFG16_COLS
#define DKSS_CFG16_COLS 1
#endif
struct Cfg<16> {
  static constexpr int NT = DKSS_CFG16_NT, COLS = DKSS_CFG16_COLS, NE = 32 * DKSS_CFG16_COLS, MINB = DKSS_CFG16_MINB,
                       T = DKSS_CFG16_T;
#ifdef DKSS_EXP_NOTWS
  static constexpr bool TWS = false;
#else
  static constexpr bool TWS = true;
#endif
};
template <>
struct Cfg<32> {
  static constexpr int NT = 256, COLS = 1, NE = 64, MINB = 2, T = 2;
  static constexpr bool TWS = false;
};

// column-pass shape: Cfg<MM>, except the DFT-only passes (table twiddles on the tensor cores,
// DO) at m = 16 take four columns per tile -- 128 elements, 32 KB: a 32-element tile kept too few
// bytes in flight (the 1024 x 2^18 batch's passes ran at 0.9-2.1 TB/s) -- and run the column DFT
// in registers (dft32x4_regs)
template <int MM, bool DO>
struct PCfg : Cfg<MM> {};
template <>
struct PCfg<16, true> {
  static constexpr int NT = 256, COLS = 4, NE = 128, MINB = 3, T = 2;
  static constexpr bool TWS = false;
};

// shared-memory words per CTA, by kernel kind (host uses the same formulas)
template <int MM, int L>
struct SmemPlan {
  using S = Smem<MM, L>;
  using C = Cfg<MM>;
  static constexpr int STAGE_PASS = C::NE * S::ES + (C::TWS ? C::NE * S::EST : 0);
  static constexpr int PASS = 2 * STAGE_PASS + C::NE * S::ES;  // + DFT ping-pong buffer
  static constexpr int BOT_STAGES = (MM == 32) ? 1 : 2;
  static constexpr int STAGE_BOT = 2 * C::NE * S::ES;
  static constexpr int BOT = BOT_STAGES * STAGE_BOT + C::NE * S::ESW;
  static constexpr int RMUL = 2 * C::NE * S::ES + C::NE * S::ESW;
};

// programmatic dependent launch: kernels of one multiply are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs may become resident
// while its predecessor drains; griddep_wait() blocks until the predecessor grid has
// completed and its memory is visible (a no-op without the attribute)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Tiles of a persistent CTA kernel: handed out from a per-launch counter (ctr[0]) when one
// is given, so CTAs that finish early take more tiles and the SMs run out of work together
// (static round-robin leaves one CTA per SM working alone at the end); ctr[1] counts CTAs
// that ran dry, and the last of them re-zeroes both for the next launch.
__device__ __forceinline__ long long grab_tile(unsigned* ctr, long long prev, long long* s_slot) {
  if (!ctr) return prev < 0 ? (long long)blockIdx.x : prev + gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) *s_slot = atomicAdd(ctr, 1u);
  __syncthreads();
  return *s_slot;
}
__device__ __forceinline__ void release_tiles(unsigned* ctr) {
  if (!ctr) return;
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
    ctr[0] = 0u;
    ctr[1] = 0u;
  }
}

__device__ __forceinline__ int bitrev_n(int x, int bits) { return bits ? (int)(__brev((unsigned)x) >> (32 - bits)) : 0; }

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk global -> shared, completion on an mbarrier)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// generic-proxy accesses of this thread are ordered before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int L>
__device__ __forceinline__ void ld_res(uint32_t (&r)[L], const uint32_t* p) {
  if constexpr (L == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
  } else if constexpr (L == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    r[0] = v.x; r[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < L; ++i) r[i] = p[i];
  }
}

template <int L>
__device__ __forceinline__ void ld_res_g(uint32_t (&r)[L], const uint32_t* __restrict__ p) {
  if constexpr (L == 4) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
  } else if constexpr (L == 2) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    r[0] = v.x; r[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < L; ++i) r[i] = __ldg(p + i);
  }
}

template <int L>
__device__ __forceinline__ void st_res(uint32_t* p, const uint32_t (&r)[L]) {
  if constexpr (L == 4) {
    *reinterpret_cast<uint4*>(p) = make_uint4(r[0], r[1], r[2], r[3]);
  } else if constexpr (L == 2) {
    *reinterpret_cast<uint2*>(p) = make_uint2(r[0], r[1]);
  } else {
#pragma unroll
    for (int i = 0; i < L; ++i) p[i] = r[i];
  }
}

// residue loaders used as ring-product operands
template <int L>
struct ResS {  // shared memory, L words per coefficient
  const uint32_t* p;
  __device__ __forceinline__ void operator()(int i, uint32_t (&d)[L]) const { ld_res<L>(d, p + i * L); }
};
template <int L>
struct ResG {  // global memory through the read-only path
  const uint32_t* p;
  __device__ __forceinline__ void operator()(int i, uint32_t (&d)[L]) const { ld_res_g<L>(d, p + i * L); }
};

// ---------------------------------------------------------------------------
// Ring product core (reference r_mul, bigmul/dkss.py:401-420):
//   out[t] = ((y * x) mod (alpha^MM + 1))_{k0+t} * R^-1 mod p,  t < kT,
//   c_k = sum_i y_i X_{k-i},  X_j = x_j (j >= 0),  X_j = -x_{j+MM} (j < 0)   (alpha^MM = -1).
// y (yl(i, r), the outer operand -- the twiddle in the transforms) is read once per step; x
// (xl(j, r), j in [0, MM)) forms a sliding window of kT residues.  A wrapped window entry is
// complemented, x' = ~x = B - x with B = 2^(32L) - 1, so every product is non-negative and
// the accumulated value is c_k + B * sum_{i>k} y_i; wl(k, r) supplies the residue
// W_k = -B * sum_{i>k} y_i mod p that cancels the bias.  Each 32x32 limb product is
// accumulated into a column (64-bit sum, 32-bit carry counter) with mad.lo.cc / madc.hi.cc /
// addc, which ptxas maps to one IMAD.WIDE.U32 with carry-out plus a shared IADD3.X:
// L^2 wide products per residue pair (the IMAD.WIDE pipe sustains ~30/clk/SM on B200,
// tools/microbench_imad.cu).
__device__ __forceinline__ void mac_limb(uint32_t& lo, uint32_t& hi, uint32_t& cy, uint32_t a, uint32_t b) {
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
      : "+r"(lo), "+r"(hi), "+r"(cy)
      : "r"(a), "r"(b));
}

#ifndef DKSS_R32_UNROLL
#define DKSS_R32_UNROLL 4
#endif

// wl argument of ring_mul for products where y is not a table twiddle (the pointwise
// products): the bias B * sum_{i>k} y_i is removed exactly instead of through a W residue --
// value = acc + S_k + Q - S_k 2^(32L) with S_k = sum_{i>k} y_i as an integer and
// Q = p 2^(32L+5) (a multiple of p keeping the value non-negative), then REDC as usual
struct BiasFromY {};
template <int MM, int L, class YL, class XL, class WL, int kT = Cfg<MM>::T>
__device__ __forceinline__ void ring_mul(YL yl, XL xl, WL wl, int k0, const ModCtx& mc, uint32_t (&out)[kT][L]) {
  constexpr int NCOL = 2 * L - 1;
  constexpr int UNR = DKSS_R32_UNROLL;
  uint32_t lo[kT][NCOL], hi[kT][NCOL], cy[kT][NCOL];
#pragma unroll
  for (int t = 0; t < kT; ++t)
#pragma unroll
    for (int c = 0; c < NCOL; ++c) lo[t][c] = hi[t][c] = cy[t][c] = 0;
  uint32_t win[kT][L];
#pragma unroll
  for (int t = 1; t < kT; ++t) xl(k0 + t, win[t]);
#pragma unroll(UNR)
  for (int i0 = 0; i0 < MM; i0 += kT) {
#pragma unroll
    for (int s = 0; s < kT; ++s) {
      const int i = i0 + s;
      uint32_t yg[L], xg[L];
      yl(i, yg);
      const int j = k0 - i;
      xl(j & (MM - 1), xg);
      const uint32_t msk = (uint32_t)(j >> 31);
#pragma unroll
      for (int q = 0; q < L; ++q) win[(kT - s) % kT][q] = xg[q] ^ msk;
#pragma unroll
      for (int t = 0; t < kT; ++t)
#pragma unroll
        for (int a = 0; a < L; ++a)
#pragma unroll
          for (int b = 0; b < L; ++b)
            mac_limb(lo[t][a + b], hi[t][a + b], cy[t][a + b], yg[a], win[(t - s + kT) % kT][b]);
    }
  }
  if constexpr (std::is_same_v<WL, BiasFromY>) {
    // S = sum_{i > k0+kT-1} y_i, then walk t down adding y_{k0+t+1}
    uint32_t S[L + 1];
#pragma unroll
    for (int q = 0; q <= L; ++q) S[q] = 0;
    for (int i = MM - 1; i > k0 + kT - 1; --i) {
      uint32_t yg[L];
      yl(i, yg);
      uint64_t c = 0;
#pragma unroll
      for (int q = 0; q < L; ++q) {
        c += (uint64_t)S[q] + yg[q];
        S[q] = (uint32_t)c;
        c >>= 32;
      }
      S[L] += (uint32_t)c;
    }
#pragma unroll
    for (int t = kT - 1; t >= 0; --t) {
      uint32_t tl[2 * L + 1];
      int64_t acc = 0;
#pragma unroll
      for (int q = 0; q < 2 * L + 1; ++q) {
        uint64_t col = 0;
        if (q < NCOL) col += lo[t][q];
        if (q >= 1 && q - 1 < NCOL) col += hi[t][q - 1];
        if (q >= 2 && q - 2 < NCOL) col += cy[t][q - 2];
        acc += (int64_t)col + mc.qbias[q];
        if (q <= L) acc += S[q];
        if (q >= L) acc -= S[q - L];
        tl[q] = (uint32_t)acc;
        acc >>= 32;  // arithmetic: carries and borrows
      }
      redc<L>(out[t], tl, mc);
      if (t > 0) {
        uint32_t yg[L];
        yl(k0 + t, yg);
        uint64_t c = 0;
#pragma unroll
        for (int q = 0; q < L; ++q) {
          c += (uint64_t)S[q] + yg[q];
          S[q] = (uint32_t)c;
          c >>= 32;
        }
        S[L] += (uint32_t)c;
      }
    }
  } else {
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      // value = sum_c (lo_c + hi_c 2^32 + cy_c 2^64) 2^(32c) + W_k  ->  2L+1 limbs
      uint32_t wv[L];
      wl(k0 + t, wv);
      uint32_t tl[2 * L + 1];
      uint64_t acc = 0;
#pragma unroll
      for (int q = 0; q < 2 * L + 1; ++q) {
        if (q < NCOL) acc += lo[t][q];
        if (q >= 1 && q - 1 < NCOL) acc += hi[t][q - 1];
        if (q >= 2 && q - 2 < NCOL) acc += cy[t][q - 2];
        if (q < L) acc += wv[q];
        tl[q] = (uint32_t)acc;
        acc >>= 32;
      }
      redc<L>(out[t], tl, mc);
    }
  }
}

// store kT consecutive output coefficients k0.. of (alpha^r * w) into element dst
template <int MM, int L, int kT>
__device__ __forceinline__ void store_rot(uint32_t* dst, const uint32_t (&w)[kT][L], int k0, int r,
                                          const ModCtx& mc) {
#pragma unroll
  for (int t = 0; t < kT; ++t) {
    int kk = (k0 + t + r) & (2 * MM - 1);
    uint32_t v[L];
    if (kk >= MM) {
      kk -= MM;
      neg_mod_canon<L>(v, w[t], mc);
    } else {
#pragma unroll
      for (int q = 0; q < L; ++q) v[q] = w[t][q];
    }
    st_res<L>(dst + kk * L, v);
  }
}


// ---------------------------------------------------------------------------
// radix-2 DIT over NE elements in shared memory, split into groups of n = 2^logn
// (<= 2MM) already in bit-reversed order; ping-pongs between `buf` and `alt` (one barrier
// per stage) and returns the buffer holding the result.  Butterfly root for block size
// `size`: alpha^(kk * 2MM/size) -- the reference's fft_eval merge with PolyAlphaRing,
// bigmul/fft.py:87-94 and bigmul/dkss.py:64-91 (any transform length n uses
// scale*step = 2m/size).  alpha^e is a rotation with negation of wrapped slots
// (poly_mul_xpow, bigmul/dkss.py:46-61): a negated slot just swaps the two outputs.
template <int MM, int L, int NE>
__device__ __forceinline__ uint32_t* dft_pingpong(uint32_t* buf, uint32_t* alt, int logn, const ModCtx& mc) {
  constexpr int ES = Smem<MM, L>::ES, NT = Cfg<MM>::NT;
  constexpr int ITEMS = (NE / 2) * MM;
  uint32_t* src = buf;
  uint32_t* dst = alt;
  for (int ls = 1; ls <= logn; ++ls) {
    const int half = 1 << (ls - 1);
    const int rootstep = (2 * MM) >> ls;  // 2MM / size
    for (int it = threadIdx.x; it < ITEMS; it += NT) {
      const int bf = it / MM, k = it % MM;
      const int blk = bf >> (ls - 1), kk = bf & (half - 1);
      const int a = (blk << ls) + kk, b = a + half;
      int sk = k - kk * rootstep;  // source coefficient of alpha^e * x_b
      const bool neg = sk < 0;
      if (neg) sk += MM;
      uint32_t u[L], x[L], s[L], d[L];
      ld_res<L>(u, src + a * ES + k * L);
      ld_res<L>(x, src + b * ES + sk * L);
      add_mod<L>(s, u, x, mc);
      sub_mod<L>(d, u, x, mc);
      const int oa = a * ES + k * L, ob = b * ES + k * L;
      st_res<L>(dst + (neg ? ob : oa), s);
      st_res<L>(dst + (neg ? oa : ob), d);
    }
    __syncthreads();
    uint32_t* tmp = src;
    src = dst;
    dst = tmp;
  }
  return src;
}

// ---------------------------------------------------------------------------
// The same 2m-point DFT for m = 32 with the data in registers: lane k of a warp holds
// coefficient k of 8 elements, the rotation by alpha^r of a butterfly's second operand is a warp
// shuffle (lane k reads lane (k - r) mod m) and its negation of the wrapped lanes (k < r) swaps
// the two outputs.  Eight warps: stages 1-3 on slots [8w, 8w + 8), one exchange through shared
// memory, stages 4-6 on slots {w + 8i}; in place in `buf` (NE = 64 elements in bit-reversed
// slots, as dft_pingpong), two shared-memory round trips instead of six and no per-item index
// arithmetic.
template <int L, bool R0>
__device__ __forceinline__ void bfly_reg(uint32_t (&u)[L], uint32_t (&v)[L], int r, int k, const ModCtx& mc) {
  uint32_t x[L], sm[L], df[L];
  if constexpr (R0) {
#pragma unroll
    for (int q = 0; q < L; ++q) x[q] = v[q];
  } else {
    const int src = (k - r) & 31;
#pragma unroll
    for (int q = 0; q < L; ++q) x[q] = __shfl_sync(0xFFFFFFFFu, v[q], src);
  }
  add_mod<L>(sm, u, x, mc);
  sub_mod<L>(df, u, x, mc);
  const bool neg = !R0 && k < r;
#pragma unroll
  for (int q = 0; q < L; ++q) {
    u[q] = neg ? df[q] : sm[q];
    v[q] = neg ? sm[q] : df[q];
  }
}

template <int L>
__device__ __forceinline__ void dft64_regs(uint32_t* buf, const ModCtx& mc) {
  constexpr int ES = Smem<32, L>::ES;
  const int w = threadIdx.x >> 5, k = threadIdx.x & 31;
  uint32_t x[8][L];
  // stages 1-3: butterflies inside the slot block [8w, 8w + 8); root alpha^(kk * 64 / size)
#pragma unroll
  for (int i = 0; i < 8; ++i) ld_res<L>(x[i], buf + (8 * w + i) * ES + k * L);
#pragma unroll
  for (int a = 0; a < 8; a += 2) bfly_reg<L, true>(x[a], x[a + 1], 0, k, mc);  // size 2: kk = 0
#pragma unroll
  for (int a = 0; a < 8; a += 4) {  // size 4: kk in {0, 1}, rootstep 16
    bfly_reg<L, true>(x[a], x[a + 2], 0, k, mc);
    bfly_reg<L, false>(x[a + 1], x[a + 3], 16, k, mc);
  }
  bfly_reg<L, true>(x[0], x[4], 0, k, mc);  // size 8: kk in 0..3, rootstep 8
  bfly_reg<L, false>(x[1], x[5], 8, k, mc);
  bfly_reg<L, false>(x[2], x[6], 16, k, mc);
  bfly_reg<L, false>(x[3], x[7], 24, k, mc);
#pragma unroll
  for (int i = 0; i < 8; ++i) st_res<L>(buf + (8 * w + i) * ES + k * L, x[i]);
  __syncthreads();
  // stages 4-6: slots w + 8i; size 16 (rootstep 4): kk = w; size 32 (rootstep 2): kk = w + 8 (i & 1);
  // size 64 (rootstep 1): kk = w + 8 (i & 3)
#pragma unroll
  for (int i = 0; i < 8; ++i) ld_res<L>(x[i], buf + (w + 8 * i) * ES + k * L);
#pragma unroll
  for (int i = 0; i < 8; i += 2) bfly_reg<L, false>(x[i], x[i + 1], 4 * w, k, mc);
#pragma unroll
  for (int i = 0; i < 8; i += 4) {
    bfly_reg<L, false>(x[i], x[i + 2], 2 * w, k, mc);
    bfly_reg<L, false>(x[i + 1], x[i + 3], 2 * (w + 8), k, mc);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) bfly_reg<L, false>(x[i], x[i + 4], w + 8 * i, k, mc);
#pragma unroll
  for (int i = 0; i < 8; ++i) st_res<L>(buf + (w + 8 * i) * ES + k * L, x[i]);
  __syncthreads();
}

// The first level's column DFT of a freshly encoded operand (m = 32): its inputs are u-bit slices
// (u <= 56), so every intermediate value is an integer of magnitude < 2^(u + 6) and the whole DFT
// runs on signed 64-bit integers -- a butterfly is two 64-bit adds instead of an add and a
// subtract mod p on four limbs -- converted to canonical residues (v or p + v) at the end.
// Values travel in the low two words of a residue slot.
template <bool R0>
__device__ __forceinline__ void bfly_s64(long long& u, long long& v, int r, int k) {
  long long x = v;
  if constexpr (!R0) x = __shfl_sync(0xFFFFFFFFu, v, (k - r) & 31);
  const long long sm = u + x, df = u - x;
  const bool neg = !R0 && k < r;
  u = neg ? df : sm;
  v = neg ? sm : df;
}

template <int L>
__device__ __forceinline__ void dft64_regs_enc(uint32_t* buf, const ModCtx& mc) {
  constexpr int ES = Smem<32, L>::ES;
  const int w = threadIdx.x >> 5, k = threadIdx.x & 31;
  long long x[8];
  auto ld64 = [&](int slot) {
    const uint2 v = *reinterpret_cast<const uint2*>(buf + slot * ES + k * L);
    return (long long)(((unsigned long long)v.y << 32) | v.x);
  };
  auto st64 = [&](int slot, long long v) {
    *reinterpret_cast<uint2*>(buf + slot * ES + k * L) = make_uint2((uint32_t)v, (uint32_t)((unsigned long long)v >> 32));
  };
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = ld64(8 * w + i);
#pragma unroll
  for (int a = 0; a < 8; a += 2) bfly_s64<true>(x[a], x[a + 1], 0, k);
#pragma unroll
  for (int a = 0; a < 8; a += 4) {
    bfly_s64<true>(x[a], x[a + 2], 0, k);
    bfly_s64<false>(x[a + 1], x[a + 3], 16, k);
  }
  bfly_s64<true>(x[0], x[4], 0, k);
  bfly_s64<false>(x[1], x[5], 8, k);
  bfly_s64<false>(x[2], x[6], 16, k);
  bfly_s64<false>(x[3], x[7], 24, k);
#pragma unroll
  for (int i = 0; i < 8; ++i) st64(8 * w + i, x[i]);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = ld64(w + 8 * i);
#pragma unroll
  for (int i = 0; i < 8; i += 2) bfly_s64<false>(x[i], x[i + 1], 4 * w, k);
#pragma unroll
  for (int i = 0; i < 8; i += 4) {
    bfly_s64<false>(x[i], x[i + 2], 2 * w, k);
    bfly_s64<false>(x[i + 1], x[i + 3], 2 * (w + 8), k);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) bfly_s64<false>(x[i], x[i + 4], w + 8 * i, k);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    // canonical residue of the integer x[i]: x[i] or p + x[i] (|x[i]| < 2^62 << p)
    const bool ng = x[i] < 0;
    const uint32_t ext = ng ? 0xFFFFFFFFu : 0u;
    uint32_t res[L];
    unsigned long long c = 0;
#pragma unroll
    for (int q = 0; q < L; ++q) {
      const uint32_t xv = q == 0 ? (uint32_t)x[i] : q == 1 ? (uint32_t)((unsigned long long)x[i] >> 32) : ext;
      c += (unsigned long long)xv + (ng ? mc.p[q] : 0u);
      res[q] = (uint32_t)c;
      c >>= 32;
    }
    st_res<L>(buf + (w + 8 * i) * ES + k * L, res);
  }
  __syncthreads();
}

// the base-case DFT of the bottom kernel for m = 32, b = 16 (2^24: four groups of 16 elements per
// 64-element tile, root alpha^4): stages 1-3 exactly as dft64_regs's (same roots), then stage 4
// (pairs (16g + i, 16g + 8 + i), root alpha^(4i)) after one exchange through shared memory
template <int L>
__device__ __forceinline__ void dft16x4_regs(uint32_t* buf, const ModCtx& mc) {
  constexpr int ES = Smem<32, L>::ES;
  const int w = threadIdx.x >> 5, k = threadIdx.x & 31;
  uint32_t x[8][L];
#pragma unroll
  for (int i = 0; i < 8; ++i) ld_res<L>(x[i], buf + (8 * w + i) * ES + k * L);
#pragma unroll
  for (int a = 0; a < 8; a += 2) bfly_reg<L, true>(x[a], x[a + 1], 0, k, mc);
#pragma unroll
  for (int a = 0; a < 8; a += 4) {
    bfly_reg<L, true>(x[a], x[a + 2], 0, k, mc);
    bfly_reg<L, false>(x[a + 1], x[a + 3], 16, k, mc);
  }
  bfly_reg<L, true>(x[0], x[4], 0, k, mc);
  bfly_reg<L, false>(x[1], x[5], 8, k, mc);
  bfly_reg<L, false>(x[2], x[6], 16, k, mc);
  bfly_reg<L, false>(x[3], x[7], 24, k, mc);
#pragma unroll
  for (int i = 0; i < 8; ++i) st_res<L>(buf + (8 * w + i) * ES + k * L, x[i]);
  __syncthreads();
  // warp w: group g = w >> 1, i in [4 (w & 1), 4 (w & 1) + 4): x[2t] = slot 16g + i, x[2t+1] = +8
  const int g = w >> 1, i0 = 4 * (w & 1);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    ld_res<L>(x[2 * t], buf + (16 * g + i0 + t) * ES + k * L);
    ld_res<L>(x[2 * t + 1], buf + (16 * g + 8 + i0 + t) * ES + k * L);
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) bfly_reg<L, false>(x[2 * t], x[2 * t + 1], 4 * (i0 + t), k, mc);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    st_res<L>(buf + (16 * g + i0 + t) * ES + k * L, x[2 * t]);
    st_res<L>(buf + (16 * g + 8 + i0 + t) * ES + k * L, x[2 * t + 1]);
  }
  __syncthreads();
}

// base-case DFT of a bottom tile: registers where a version exists (m = 32, b = 64 or 16), else
// the shared-memory ping-pong; returns the buffer holding the result
template <int MM, int L, int NE>
__device__ __forceinline__ uint32_t* base_dft(uint32_t* buf, uint32_t* alt, int logb, const ModCtx& mc) {
  if constexpr (MM == 32 && NE == 64 && Cfg<MM>::NT == 256) {
    if (logb == 6) {
      dft64_regs<L>(buf, mc);
      return buf;
    }
    if (logb == 4) {
      dft16x4_regs<L>(buf, mc);
      return buf;
    }
  }
  return dft_pingpong<MM, L, NE>(buf, alt, logb, mc);
}

// m = 16, four 32-element columns per tile (PCfg<16, true>): half-warp h of warp w holds
// coefficient k = lane & 15 of 8 elements of column c = 2 (w >> 2) + h; rotations are shuffles
// inside the half-warp.  Stages 1-3 on slots [8b, 8b + 8), b = w & 3; one exchange through shared
// memory; stages 4-5 on slots {b' + 8i}, b' in {2 (w & 3), 2 (w & 3) + 1}, i < 4.
template <int L, bool R0>
__device__ __forceinline__ void bfly_reg16(uint32_t (&u)[L], uint32_t (&v)[L], int r, int k, int h,
                                           const ModCtx& mc) {
  uint32_t x[L], sm[L], df[L];
  if constexpr (R0) {
#pragma unroll
    for (int q = 0; q < L; ++q) x[q] = v[q];
  } else {
    const int src = (h << 4) | ((k - r) & 15);
#pragma unroll
    for (int q = 0; q < L; ++q) x[q] = __shfl_sync(0xFFFFFFFFu, v[q], src);
  }
  add_mod<L>(sm, u, x, mc);
  sub_mod<L>(df, u, x, mc);
  const bool neg = !R0 && k < r;
#pragma unroll
  for (int q = 0; q < L; ++q) {
    u[q] = neg ? df[q] : sm[q];
    v[q] = neg ? sm[q] : df[q];
  }
}

template <int L>
__device__ __forceinline__ void dft32x4_regs(uint32_t* buf, const ModCtx& mc) {
  constexpr int ES = Smem<16, L>::ES;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, k = lane & 15;
  uint32_t* col = buf + (2 * (w >> 2) + h) * 32 * ES;
  const int b = w & 3;
  uint32_t x[8][L];
#pragma unroll
  for (int i = 0; i < 8; ++i) ld_res<L>(x[i], col + (8 * b + i) * ES + k * L);
  // size 2: kk = 0; size 4 (rootstep 8): kk in {0, 1}; size 8 (rootstep 4): kk in 0..3
#pragma unroll
  for (int a = 0; a < 8; a += 2) bfly_reg16<L, true>(x[a], x[a + 1], 0, k, h, mc);
#pragma unroll
  for (int a = 0; a < 8; a += 4) {
    bfly_reg16<L, true>(x[a], x[a + 2], 0, k, h, mc);
    bfly_reg16<L, false>(x[a + 1], x[a + 3], 8, k, h, mc);
  }
  bfly_reg16<L, true>(x[0], x[4], 0, k, h, mc);
  bfly_reg16<L, false>(x[1], x[5], 4, k, h, mc);
  bfly_reg16<L, false>(x[2], x[6], 8, k, h, mc);
  bfly_reg16<L, false>(x[3], x[7], 12, k, h, mc);
#pragma unroll
  for (int i = 0; i < 8; ++i) st_res<L>(col + (8 * b + i) * ES + k * L, x[i]);
  __syncthreads();
  // x[2 g + i'] = slot b' + 8 i', b' = 2 b + g: size 16 (rootstep 2): pairs i' (0, 1), (2, 3), kk =
  // b'; size 32 (rootstep 1): pairs i' (0, 2), (1, 3), kk = b' + 8 i'
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) ld_res<L>(x[4 * g + i], col + (2 * b + g + 8 * i) * ES + k * L);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int bp = 2 * b + g;
    bfly_reg16<L, false>(x[4 * g + 0], x[4 * g + 1], 2 * bp, k, h, mc);
    bfly_reg16<L, false>(x[4 * g + 2], x[4 * g + 3], 2 * bp, k, h, mc);
    bfly_reg16<L, false>(x[4 * g + 0], x[4 * g + 2], bp, k, h, mc);
    bfly_reg16<L, false>(x[4 * g + 1], x[4 * g + 3], bp + 8, k, h, mc);
  }
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) st_res<L>(col + (2 * b + g + 8 * i) * ES + k * L, x[4 * g + i]);
  __syncthreads();
}

// dft32x4_regs for the first level of a freshly encoded operand, on signed 64-bit integers (see
// dft64_regs_enc)
template <bool R0>
__device__ __forceinline__ void bfly_s64_16(long long& u, long long& v, int r, int k, int h) {
  long long x = v;
  if constexpr (!R0) x = __shfl_sync(0xFFFFFFFFu, v, (h << 4) | ((k - r) & 15));
  const long long sm = u + x, df = u - x;
  const bool neg = !R0 && k < r;
  u = neg ? df : sm;
  v = neg ? sm : df;
}

template <int L>
__device__ __forceinline__ void dft32x4_regs_enc(uint32_t* buf, const ModCtx& mc) {
  constexpr int ES = Smem<16, L>::ES;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, k = lane & 15;
  uint32_t* col = buf + (2 * (w >> 2) + h) * 32 * ES;
  const int b = w & 3;
  long long x[8];
  auto ld64 = [&](int slot) {
    const uint2 v = *reinterpret_cast<const uint2*>(col + slot * ES + k * L);
    return (long long)(((unsigned long long)v.y << 32) | v.x);
  };
  auto st64 = [&](int slot, long long v) {
    *reinterpret_cast<uint2*>(col + slot * ES + k * L) = make_uint2((uint32_t)v, (uint32_t)((unsigned long long)v >> 32));
  };
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = ld64(8 * b + i);
#pragma unroll
  for (int a = 0; a < 8; a += 2) bfly_s64_16<true>(x[a], x[a + 1], 0, k, h);
#pragma unroll
  for (int a = 0; a < 8; a += 4) {
    bfly_s64_16<true>(x[a], x[a + 2], 0, k, h);
    bfly_s64_16<false>(x[a + 1], x[a + 3], 8, k, h);
  }
  bfly_s64_16<true>(x[0], x[4], 0, k, h);
  bfly_s64_16<false>(x[1], x[5], 4, k, h);
  bfly_s64_16<false>(x[2], x[6], 8, k, h);
  bfly_s64_16<false>(x[3], x[7], 12, k, h);
#pragma unroll
  for (int i = 0; i < 8; ++i) st64(8 * b + i, x[i]);
  __syncthreads();
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) x[4 * g + i] = ld64(2 * b + g + 8 * i);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int bp = 2 * b + g;
    bfly_s64_16<false>(x[4 * g + 0], x[4 * g + 1], 2 * bp, k, h);
    bfly_s64_16<false>(x[4 * g + 2], x[4 * g + 3], 2 * bp, k, h);
    bfly_s64_16<false>(x[4 * g + 0], x[4 * g + 2], bp, k, h);
    bfly_s64_16<false>(x[4 * g + 1], x[4 * g + 3], bp + 8, k, h);
  }
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long v = x[4 * g + i];
      const bool ng = v < 0;
      const uint32_t ext = ng ? 0xFFFFFFFFu : 0u;
      uint32_t res[L];
      unsigned long long c = 0;
#pragma unroll
      for (int q = 0; q < L; ++q) {
        const uint32_t xv = q == 0 ? (uint32_t)v : q == 1 ? (uint32_t)((unsigned long long)v >> 32) : ext;
        c += (unsigned long long)xv + (ng ? mc.p[q] : 0u);
        res[q] = (uint32_t)c;
        c >>= 32;
      }
      st_res<L>(col + (2 * b + g + 8 * i) * ES + k * L, res);
    }
  __syncthreads();
}

// the column DFT of a pass tile: registers for m = 32 (one 64-element column, 8 warps), the
// shared-memory ping-pong otherwise; returns the buffer holding the result
template <int MM, int L, int NE>
__device__ __forceinline__ uint32_t* column_dft(uint32_t* buf, uint32_t* alt, int logn, const ModCtx& mc) {
  if constexpr (MM == 32 && NE == 64 && Cfg<MM>::NT == 256) {
    dft64_regs<L>(buf, mc);
    return buf;
  } else if constexpr (MM == 16 && NE == 128) {
    dft32x4_regs<L>(buf, mc);
    return buf;
  } else {
    return dft_pingpong<MM, L, NE>(buf, alt, logn, mc);
  }
}

// ---------------------------------------------------------------------------
// timing experiments only (tools/exp_build.sh): drop the column DFT or the twiddle products
#ifdef DKSS_EXP_NODFT
constexpr bool kExpNoDft = true;
#else
constexpr bool kExpNoDft = false;
#endif
#ifdef DKSS_EXP_NOSPREAD
constexpr bool kSpreadIssue = false;
#else
constexpr bool kSpreadIssue = true;
#endif
#ifdef DKSS_EXP_NOMAC
constexpr bool kExpNoMac = true;
#else
constexpr bool kExpNoMac = false;
#endif

#ifdef DKSS_EXP_TRACE
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE_DECL unsigned long long tr_[12]; int trn_ = 0; tr_[trn_++] = gtime();
#define TRACE_MARK if (trn_ < 12) tr_[trn_++] = gtime();
#define TRACE_DUMP(name)                                                                                 \
  if (threadIdx.x == 0 && (blockIdx.x % 37 == 0 || blockIdx.x == gridDim.x - 1)) {                        \
    for (int q_ = trn_; q_ < 12; ++q_) tr_[q_] = tr_[0];                                                 \
    printf("TRACE %s blk %d t0 %llu : %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", name, blockIdx.x, \
           tr_[0] % 1000000000ull, tr_[1] - tr_[0], tr_[2] - tr_[0], tr_[3] - tr_[0], tr_[4] - tr_[0],        \
           tr_[5] - tr_[0], tr_[6] - tr_[0], tr_[7] - tr_[0], tr_[8] - tr_[0], tr_[9] - tr_[0],             \
           tr_[10] - tr_[0], tr_[11] - tr_[0]);                                                            \
  }
#else
#define TRACE_DECL
#define TRACE_MARK
#define TRACE_DUMP(name)
#endif

struct PassArgs {
  uint32_t* poly;        // first polynomial of the launch
  long long poly_words;  // 2M * MM * L
  int log_mu;            // column stride mu = 2^log_mu (elements)
  int log_top_mu;        // log2(M/m): twiddle exponents are split at this bit (alpha shift | row)
  int log_cpp;           // log2 columns per polynomial in this launch's layout (log_top_mu unless sharded)
  long long l_off;       // global column offset of local column 0 (sharded first level; else 0)
  int log_mu_enc;        // fused encode: log2 of the global column count mu_0 (operand position stride)
  long long base_pow;    // (2m)^level
  const uint32_t* twr;   // [M/m][2MM][L]: rho~_s = rho^s R mod p, then W_s (see ring_mul)
  int scale;             // inverse pass: 1 multiply outputs by mc.kscale; 2 the twiddle rows are
                         // pre-scaled, untwiddled elements are multiplied before the DFT
  long long total_cols;  // columns in the launch (npoly * M/m)
  // fused encode (first forward level): elements are sliced from the operands instead of
  // loaded -- poly q < enc_split takes operand q of ops_a, others operand q-enc_split of ops_b
  const uint32_t* ops_a;
  const uint32_t* ops_b;
  long long na;          // limbs per operand
  int enc_split;
  int u;                 // bits per inner coefficient
  int M;                 // outer length (elements e >= M are zero)
  int wpc;               // warp-per-column kernels: warps sharing one column (power of 2)
  unsigned* ctr;         // CTA kernels: tile tickets of this launch (null: static round-robin)
  int tw_skip;           // CTA kernels: elements with a table twiddle (s != 0) pass through
                         // untouched -- the tensor-core kernel (dkss_tc.cuh) multiplies them
  // four-step split with the exchange fused into the stores (CTA kernels):
  // every output element goes straight to the rank that owns it next, through the peer base
  // pointers peer[world] (CUDA IPC mappings over NVLink, or plain pointers for emulated ranks)
  //   peer_mode 1 (first forward level, launch layout [2][E][C]): element (q, j, c) -> rank
  //     j >> peer_log_r, at ((q R + (j & (R-1))) mu0 + l_off + c) in that rank's [2][R][mu0] rows
  //   peer_mode 2 (last inverse level of the rows, launch layout [R][mu0], one row per launch
  //     polynomial jr): element (jr, global column l) -> rank l >> peer_log_c, at
  //     ((peer_row0 + jr) C + (l & (C-1))) in that rank's [E][C] columns
  const unsigned long long* peer;
  int peer_mode;
  int peer_log_r, peer_log_c, peer_log_mu0;
  long long peer_row0;
};

// destination of output element `pos` (element index inside launch polynomial `poly`) under a
// fused-exchange store (peer_mode != 0); elem_words per element
__device__ __forceinline__ uint32_t* peer_dst(const PassArgs& A, long long poly, long long pos, int elem_words) {
  const long long C = 1LL << A.peer_log_c;
  if (A.peer_mode == 1) {
    const long long j = pos >> A.peer_log_c, c = pos & (C - 1);
    const long long R = 1LL << A.peer_log_r;
    uint32_t* base = reinterpret_cast<uint32_t*>(A.peer[j >> A.peer_log_r]);
    return base + (((poly * R + (j & (R - 1))) << A.peer_log_mu0) + A.l_off + c) * elem_words;
  }
  uint32_t* base = reinterpret_cast<uint32_t*>(A.peer[pos >> A.peer_log_c]);
  return base + ((A.peer_row0 + poly) * C + (pos & (C - 1))) * elem_words;
}

// the global word offset col_elem gives, or the fused-exchange destination
__device__ __forceinline__ uint32_t* out_elem(const PassArgs& A, long long cg, int j, int loge, int elem_words) {
  const long long poly = cg >> A.log_cpp, cc = cg & ((1LL << A.log_cpp) - 1);
  const long long inst = cc >> A.log_mu, l = cc & ((1LL << A.log_mu) - 1);
  const long long pos = (inst << (A.log_mu + loge)) + ((long long)j << A.log_mu) + l;
  if (A.peer_mode) return peer_dst(A, poly, pos, elem_words);
  return A.poly + poly * A.poly_words + pos * elem_words;
}

template <int MM>
struct Geo {
  static constexpr int E = 2 * MM;
  static constexpr int LOGE = (E == 16) ? 4 : (E == 32) ? 5 : (E == 64) ? 6 : (E == 8) ? 3 : 7;
};

// element j of launch column cg: global word offset, and the column index l in its row
__device__ __forceinline__ long long col_elem(const PassArgs& A, long long cg, int j, int loge, int elem_words,
                                              long long* l_out) {
  const long long poly = cg >> A.log_cpp, cc = cg & ((1LL << A.log_cpp) - 1);
  const long long inst = cc >> A.log_mu, l = cc & ((1LL << A.log_mu) - 1);
  *l_out = l + A.l_off;
  return poly * A.poly_words + ((inst << (A.log_mu + loge)) + ((long long)j << A.log_mu) + l) * elem_words;
}

// twiddle row of element (j, l): s = (j*l*base_pow) mod (M/m), r = its alpha shift
__device__ __forceinline__ long long tw_exp(const PassArgs& A, int j, long long l, int* r) {
  const long long e = (long long)j * l * A.base_pow;
  *r = (int)(e >> A.log_top_mu);
  return e & ((1LL << A.log_top_mu) - 1);
}

// TMA-load the NE column elements of tile `tile` (FWD: bit-reversed slots) and, when staged,
// the twiddle row of every element needing a ring product.  Warp 0 counts the bytes and
// arms the barrier; the copies themselves are issued by the calling threads (one warp, or
// spread over the whole CTA when kSpreadIssue: a bulk copy's issue is serialised per
// warp, so 2*NE copies from one warp cost microseconds)
// part: 3 = everything; 1 = arm the barrier + twiddle rows (independent of the previous
// kernel's output, issued before griddep_wait); 2 = the column elements
template <int MM, int L, bool FWD, class C = Cfg<MM>>
__device__ __forceinline__ void issue_pass_tile(const PassArgs& A, long long tile, uint64_t* bar, uint32_t* buf,
                                                uint32_t* tws, bool load_elems = true, int part = 3) {
  constexpr int ES = Smem<MM, L>::ES, EST = Smem<MM, L>::EST;
  constexpr int NE = C::NE, COLS = C::COLS, E = 2 * MM, LOGE = Geo<MM>::LOGE;
  constexpr int NW = kSpreadIssue ? C::NT / 32 : 1;
  constexpr uint32_t EB = MM * L * 4, TB = 2 * MM * L * 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0 && (part & 1)) {
    uint32_t bytes = 0;
    for (int e = lane; e < NE; e += 32) {
      const long long cg = tile * COLS + e / E;
      if (cg >= A.total_cols) continue;
      if (load_elems) bytes += EB;
      if constexpr (C::TWS) {
        long long l;
        col_elem(A, cg, 0, LOGE, 0, &l);
        int r;
        if (!A.tw_skip && tw_exp(A, e % E, l, &r)) bytes += TB;
      }
    }
    bytes = __reduce_add_sync(0xFFFFFFFFu, bytes);
    if (lane == 0) mbar_expect_tx(bar, bytes);
    __syncwarp();
  }
  for (int q = warp + NW * lane; q < 2 * NE; q += NW * 32) {
    const int e = q % NE;
    const int c = e / E, j = e % E;
    const long long cg = tile * COLS + c;
    if (cg >= A.total_cols) continue;
    long long l;
    const long long off = col_elem(A, cg, j, LOGE, MM * L, &l);
    if (q < NE) {
      const int slot = FWD ? c * E + bitrev_n(j, LOGE) : e;
      if (load_elems && (part & 2)) bulk_g2s(buf + slot * ES, A.poly + off, EB, bar);
    } else if constexpr (C::TWS) {
      if (!(part & 1) || A.tw_skip) continue;
      int r;
      const long long s = tw_exp(A, j, l, &r);
      if (s) bulk_g2s(tws + e * EST, A.twr + s * (2 * MM * L), TB, bar);
    }
  }
}

// twiddle product of element `el` (x in `xs`) with row s: rho~ from tws (staged) or global
template <int MM, int L, int kT>
__device__ __forceinline__ void twiddle_mul(const PassArgs& A, const uint32_t* xs, const uint32_t* tws_el, long long s,
                                            int k0, const ModCtx& mc, uint32_t (&w)[kT][L]) {
  if constexpr (Cfg<MM>::TWS) {
    ring_mul<MM, L>(ResS<L>{tws_el}, ResS<L>{xs}, ResS<L>{tws_el + MM * L}, k0, mc, w);
  } else {
    const uint32_t* row = A.twr + s * (2 * MM * L);
    ring_mul<MM, L>(ResG<L>{row}, ResS<L>{xs}, ResG<L>{row + MM * L}, k0, mc, w);
  }
}

// fused dkss_encode (bigmul/dkss.py:381-398) for the first forward level: coefficient k of
// element pos is bits [u(pos*m/2 + k), +u) of the operand for pos < M, k < m/2, else 0;
// written straight into the column buffer at the bit-reversed slot
template <int MM, int L, class C = Cfg<MM>>
__device__ __forceinline__ void cta_encode_tile(const PassArgs& A, long long tile, uint32_t* buf) {
  constexpr int ES = Smem<MM, L>::ES, NT = C::NT, NE = C::NE, COLS = C::COLS;
  constexpr int E = 2 * MM, LOGE = Geo<MM>::LOGE, HALF = MM / 2;
  // only the lower m/2 coefficients of an element carry operand bits: those items are spread over
  // all threads and unrolled, so a thread's operand loads are in flight together; the upper
  // halves are zero-filled
  constexpr int ITEMS = NE * HALF;
#pragma unroll
  for (int it0 = 0; it0 < ITEMS; it0 += NT) {
    const int it = it0 + threadIdx.x;
    if (ITEMS % NT != 0 && it >= ITEMS) break;
    const int el = it / HALF, k = it % HALF;
    const int c = el / E, j = el % E;
    const long long cg = tile * COLS + c;
    uint32_t out[L];
#pragma unroll
    for (int q = 0; q < L; ++q) out[q] = 0;
    if (cg < A.total_cols) {
      const long long q = cg >> A.log_cpp, cc = cg & ((1LL << A.log_cpp) - 1);
      const long long inst = cc >> A.log_mu, l = cc & ((1LL << A.log_mu) - 1);
      const long long pos = (inst << (A.log_mu_enc + LOGE)) + ((long long)j << A.log_mu_enc) + l + A.l_off;
      if (pos < A.M) {
        const uint32_t* op = q < A.enc_split ? A.ops_a + q * A.na : A.ops_b + (q - A.enc_split) * A.na;
        const long long bit = (long long)A.u * (pos * HALF + k);
        const long long w0 = bit >> 5;
        const int sh = (int)(bit & 31);
        uint32_t src[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) src[w] = (w0 + w < A.na && 32 * w < sh + A.u) ? __ldg(op + w0 + w) : 0u;
        int rem = A.u;
#pragma unroll
        for (int w = 0; w < 3 && w < L; ++w) {
          const uint32_t v = sh ? __funnelshift_r(src[w], src[w + 1], sh) : src[w];
          out[w] = rem >= 32 ? v : (rem > 0 ? v & ((1u << rem) - 1u) : 0u);
          rem -= 32;
        }
      }
    }
    uint32_t* slot = buf + (c * E + bitrev_n(j, LOGE)) * ES;
    st_res<L>(slot + k * L, out);
    uint32_t zero[L];
#pragma unroll
    for (int q = 0; q < L; ++q) zero[q] = 0;
    st_res<L>(slot + (HALF + k) * L, zero);
  }
}

// forward column pass (one level of dkss_fft): column DFT, then twiddle ring product
// rho^(vv*l*base_pow) = alpha^r * rho_table[s] (bigmul/dkss.py:480-492)
// DO (DFT only): the table twiddles are the tensor cores' (tw_skip), so no ring products are
// compiled in -- fewer registers, three CTAs per SM (m = 32: the column DFT in registers needs
// no ping-pong buffer either)
template <int MM, int L, bool DO = false>
__global__ void __launch_bounds__(Cfg<MM>::NT, DO ? 3 : Cfg<MM>::MINB) k_fwd_pass(PassArgs A, ModCtx mc) {
  griddep_launch();
  using C = PCfg<MM, DO>;
  constexpr int kT = C::T;
  constexpr int ES = Smem<MM, L>::ES, EST = Smem<MM, L>::EST;
  constexpr int NT = C::NT, NE = C::NE, COLS = C::COLS, E = 2 * MM, LOGE = Geo<MM>::LOGE;
  constexpr int STAGE = NE * ES + (C::TWS ? NE * EST : 0);
  constexpr int TPE = MM / kT;
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ __align__(8) uint64_t bar[2];
  TRACE_DECL
  const long long ntiles = (A.total_cols + COLS - 1) / COLS;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  __shared__ long long s_tile;
  long long tile = grab_tile(A.ctr, -1, &s_tile);
  const bool enc = A.ops_a != nullptr;
  // PDL: the twiddle rows do not depend on the previous kernel; the elements (and, for the
  // fused encode, the operands) do
  if (tile < ntiles && (kSpreadIssue || threadIdx.x < 32))
    issue_pass_tile<MM, L, true, C>(A, tile, &bar[0], smem, smem + NE * ES, !enc, 1);
  griddep_wait();
  if (tile < ntiles && (kSpreadIssue || threadIdx.x < 32))
    issue_pass_tile<MM, L, true, C>(A, tile, &bar[0], smem, smem + NE * ES, !enc, 2);
  for (int k = 0; tile < ntiles; ++k) {
    const int st = k & 1;
    uint32_t* buf = smem + st * STAGE;
    uint32_t* tws = buf + NE * ES;
    const long long nxt = grab_tile(A.ctr, tile, &s_tile);
    if (nxt < ntiles && (kSpreadIssue || threadIdx.x < 32))
      issue_pass_tile<MM, L, true, C>(A, nxt, &bar[st ^ 1], smem + (st ^ 1) * STAGE, smem + (st ^ 1) * STAGE + NE * ES,
                                   !enc);
    if (enc) {
      cta_encode_tile<MM, L, C>(A, tile, buf);
      __syncthreads();
    }
    TRACE_MARK
    mbar_wait(&bar[st], (k >> 1) & 1);
    TRACE_MARK
    const uint32_t* xv;
    if constexpr (MM == 32 && NE == 64 && C::NT == 256) {
      if (enc && A.u <= 56 && !kExpNoDft) {
        dft64_regs_enc<L>(buf, mc);
        xv = buf;
      } else {
        xv = kExpNoDft ? buf : column_dft<MM, L, NE>(buf, smem + 2 * STAGE, LOGE, mc);
      }
    } else if constexpr (MM == 16 && NE == 128) {
      if (enc && A.u <= 56 && !kExpNoDft) {
        dft32x4_regs_enc<L>(buf, mc);
        xv = buf;
      } else {
        xv = kExpNoDft ? buf : column_dft<MM, L, NE>(buf, smem + 2 * STAGE, LOGE, mc);
      }
    } else {
      xv = kExpNoDft ? buf : column_dft<MM, L, NE>(buf, smem + 2 * STAGE, LOGE, mc);
    }
    TRACE_MARK
    for (int it = threadIdx.x; it < NE * TPE; it += NT) {
      const int el = it / TPE, k0 = (it % TPE) * kT;
      const int c = el / E, vv = el % E;
      const long long cg = tile * COLS + c;
      if (cg >= A.total_cols) continue;
      long long l;
      const long long off = col_elem(A, cg, vv, LOGE, MM * L, &l);
      int r;
      const long long s = tw_exp(A, vv, l, &r);
      // fused exchange: elements the tensor-core kernel still multiplies stay local (it stores
      // them to their owners)
      uint32_t* dst = (A.peer_mode && !(A.tw_skip && s != 0)) ? out_elem(A, cg, vv, LOGE, MM * L) : A.poly + off;
      uint32_t w[kT][L];
      if (DO || s == 0 || kExpNoMac || A.tw_skip) {
        if (s != 0) r = 0;  // tw_skip: the tensor-core kernel applies rho^e (rotation included)
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(w[t], xv + el * ES + (k0 + t) * L);
      } else if constexpr (!DO) {
        twiddle_mul<MM, L, kT>(A, xv + el * ES, tws + el * EST, s, k0, mc, w);
      }
      store_rot<MM, L, kT>(dst, w, k0, r, mc);
    }
    fence_proxy_async();
    __syncthreads();
    TRACE_MARK
    tile = nxt;
  }
  if (A.peer_mode) __threadfence_system();  // fused exchange: stores to other GPUs performed
  release_tiles(A.ctr);
  TRACE_DUMP(enc ? "fwd0" : "fwd")
}

// inverse (transposed) column pass: twiddle ring product, then column DFT
template <int MM, int L, bool DO = false>
__global__ void __launch_bounds__(Cfg<MM>::NT, DO ? 3 : Cfg<MM>::MINB) k_inv_pass(PassArgs A, ModCtx mc) {
  griddep_launch();
  using C = PCfg<MM, DO>;
  constexpr int kT = C::T;
  constexpr int ES = Smem<MM, L>::ES, EST = Smem<MM, L>::EST;
  constexpr int NT = C::NT, NE = C::NE, COLS = C::COLS, E = 2 * MM, LOGE = Geo<MM>::LOGE;
  constexpr int STAGE = NE * ES + (C::TWS ? NE * EST : 0);
  constexpr int TPE = MM / kT;
  constexpr int PER = (NE * TPE + NT - 1) / NT;
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ __align__(8) uint64_t bar[2];
  TRACE_DECL
  const long long ntiles = (A.total_cols + COLS - 1) / COLS;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  __shared__ long long s_tile;
  long long tile = grab_tile(A.ctr, -1, &s_tile);
  if (tile < ntiles && (kSpreadIssue || threadIdx.x < 32))
    issue_pass_tile<MM, L, false, C>(A, tile, &bar[0], smem, smem + NE * ES, true, 1);
  griddep_wait();  // PDL: twiddle rows above are independent of the previous kernel
  if (tile < ntiles && (kSpreadIssue || threadIdx.x < 32))
    issue_pass_tile<MM, L, false, C>(A, tile, &bar[0], smem, smem + NE * ES, true, 2);
  for (int k = 0; tile < ntiles; ++k) {
    const int st = k & 1;
    uint32_t* buf = smem + st * STAGE;
    uint32_t* tws = buf + NE * ES;
    const long long nxt = grab_tile(A.ctr, tile, &s_tile);
    if (nxt < ntiles && (kSpreadIssue || threadIdx.x < 32))
      issue_pass_tile<MM, L, false, C>(A, nxt, &bar[st ^ 1], smem + (st ^ 1) * STAGE, smem + (st ^ 1) * STAGE + NE * ES);
    TRACE_MARK
    mbar_wait(&bar[st], (k >> 1) & 1);
    TRACE_MARK
    uint32_t res[PER][kT][L];
    int dsl[PER], rot[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int it = threadIdx.x + q * NT;
      dsl[q] = -1;
      if (it >= NE * TPE) continue;
      const int el = it / TPE, k0 = (it % TPE) * kT;
      const int c = el / E, j = el % E;
      const long long cg = tile * COLS + c;
      if (cg >= A.total_cols) continue;
      long long l;
      col_elem(A, cg, 0, LOGE, 0, &l);
      const long long s = tw_exp(A, j, l, &rot[q]);
      if (s != 0 && (DO || A.tw_skip)) {  // already multiplied (and rotated) by the tensor-core kernel
        rot[q] = 0;
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(res[q][t], buf + el * ES + (k0 + t) * L);
      } else if (s == 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(res[q][t], buf + el * ES + (k0 + t) * L);
        if (A.scale == 2) {
          uint32_t ks[L];
#pragma unroll
          for (int qq = 0; qq < L; ++qq) ks[qq] = mc.kscale[qq];
#pragma unroll
          for (int t = 0; t < kT; ++t) mont_mul<L>(res[q][t], res[q][t], ks, mc);
        }
      } else if constexpr (!DO) {
        twiddle_mul<MM, L, kT>(A, buf + el * ES, tws + el * EST, s, k0, mc, res[q]);
      }
      dsl[q] = (c * E + bitrev_n(j, LOGE)) * ES;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (dsl[q] >= 0) store_rot<MM, L, kT>(buf + dsl[q], res[q], ((threadIdx.x + q * NT) % TPE) * kT, rot[q], mc);
    __syncthreads();
    TRACE_MARK
    const uint32_t* ov = column_dft<MM, L, NE>(buf, smem + 2 * STAGE, LOGE, mc);
    for (int it = threadIdx.x; it < NE * MM; it += NT) {
      const int el = it / MM, kk = it % MM;
      const int c = el / E, vv = el % E;
      const long long cg = tile * COLS + c;
      if (cg >= A.total_cols) continue;
      uint32_t* dst = out_elem(A, cg, vv, LOGE, MM * L);
      uint32_t v[L];
      ld_res<L>(v, ov + el * ES + kk * L);
      if (A.scale == 1) {
        uint32_t ks[L];
#pragma unroll
        for (int q = 0; q < L; ++q) ks[q] = mc.kscale[q];
        mont_mul<L>(v, v, ks, mc);
      }
      st_res<L>(dst + kk * L, v);
    }
    fence_proxy_async();
    __syncthreads();
    TRACE_MARK
    tile = nxt;
  }
  if (A.peer_mode) __threadfence_system();  // fused exchange: stores to other GPUs performed
  release_tiles(A.ctr);
  TRACE_DUMP("inv")
}

// ---------------------------------------------------------------------------
// bottom of the transform: groups of b = 2^logb contiguous elements.
//   mode 0: base DFT of `a` only (stage API)
//   mode 1: base DFT a, base DFT b, pointwise b*a (Montgomery, *R^-1), base DFT -> a
// `scale` multiplies the final outputs by mc.kscale (used when the whole transform is
// one base DFT, levels == 0).
struct BottomArgs {
  uint32_t* a;
  const uint32_t* b;
  long long poly_words;  // 2M*MM*L
  long long elems_per_poly;
  int logb;
  int mode;
  int scale;
  long long total_elems;  // elements in the launch (npoly * 2M)
  unsigned* ctr;          // tile tickets of this launch (null: static round-robin)
};

template <int MM, int L>
__device__ __forceinline__ void issue_bottom_tile(const BottomArgs& A, long long tile, uint64_t* bar, uint32_t* sa,
                                                  uint32_t* sb) {
  constexpr int ES = Smem<MM, L>::ES, NE = Cfg<MM>::NE;
  constexpr uint32_t EB = MM * L * 4;
  constexpr int NW = kSpreadIssue ? Cfg<MM>::NT / 32 : 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool two = A.mode != 0;
  const long long e0 = tile * NE;
  const int bmask = (1 << A.logb) - 1;
  if (warp == 0) {
    const long long n = A.total_elems - e0 < NE ? A.total_elems - e0 : NE;
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)n * (two ? 2 * EB : EB));
    __syncwarp();
  }
  // copies spread over the calling warps (see issue_pass_tile)
  for (int q = warp + NW * lane; q < 2 * NE; q += NW * 32) {
    const int el = q % NE;
    if (e0 + el >= A.total_elems || (q >= NE && !two)) continue;
    const int slot = (el & ~bmask) | bitrev_n(el & bmask, A.logb);
    if (q < NE)
      bulk_g2s(sa + slot * ES, A.a + (e0 + el) * (MM * L), EB, bar);
    else
      bulk_g2s(sb + slot * ES, A.b + (e0 + el) * (MM * L), EB, bar);
  }
}

template <int MM, int L>
__global__ void __launch_bounds__(Cfg<MM>::NT, Cfg<MM>::MINB) k_bottom(BottomArgs A, ModCtx mc) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  constexpr int kT = Cfg<MM>::T;
  constexpr int ES = Smem<MM, L>::ES, ESW = Smem<MM, L>::ESW;
  constexpr int NT = Cfg<MM>::NT, NE = Cfg<MM>::NE;
  constexpr int NS = SmemPlan<MM, L>::BOT_STAGES, STAGE = SmemPlan<MM, L>::STAGE_BOT;
  constexpr int TPE = MM / kT;
  constexpr int PER = (NE * TPE + NT - 1) / NT;
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ __align__(8) uint64_t bar[2];
  uint32_t* wr = smem + NS * STAGE;
  const long long ntiles = (A.total_elems + NE - 1) / NE;
  const int bmask = (1 << A.logb) - 1;
  const bool two = A.mode != 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  __shared__ long long s_tile;
  long long tile = grab_tile(A.ctr, -1, &s_tile);
  if (tile < ntiles && (kSpreadIssue || threadIdx.x < 32))
    issue_bottom_tile<MM, L>(A, tile, &bar[0], smem, smem + NE * ES);
  for (int k = 0; tile < ntiles; ++k) {
    const int st = NS == 2 ? (k & 1) : 0;
    uint32_t* sa = smem + st * STAGE;
    uint32_t* sb = sa + NE * ES;
    const long long nxt = grab_tile(A.ctr, tile, &s_tile);
    if (NS == 2 && nxt < ntiles && (kSpreadIssue || threadIdx.x < 32))
      issue_bottom_tile<MM, L>(A, nxt, &bar[st ^ 1], smem + (st ^ 1) * STAGE, smem + (st ^ 1) * STAGE + NE * ES);
    mbar_wait(&bar[st], NS == 2 ? ((k >> 1) & 1) : (k & 1));
    const long long e0 = tile * NE;
    // three NE-element buffers {sa, sb, wr} serve as DFT ping-pong space and results
    uint32_t* ra = base_dft<MM, L, NE>(sa, wr, A.logb, mc);
    uint32_t* out = ra;
    if (two) {
      uint32_t* rb = base_dft<MM, L, NE>(sb, ra == sa ? wr : sa, A.logb, mc);
      __syncthreads();
      uint32_t res[PER][kT][L];
      int dsts[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int it = threadIdx.x + q * NT;
        dsts[q] = -1;
        if (it < NE * TPE) {
          const int el = it / TPE, k0 = (it % TPE) * kT;
          ring_mul<MM, L>(ResS<L>{rb + el * ES}, ResS<L>{ra + el * ES}, BiasFromY{}, k0, mc, res[q]);
          const int slot = (el & ~bmask) | bitrev_n(el & bmask, A.logb);
          dsts[q] = slot * ES + k0 * L;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < PER; ++q)
        if (dsts[q] >= 0) {
#pragma unroll
          for (int t = 0; t < kT; ++t) st_res<L>(ra + dsts[q] + t * L, res[q][t]);
        }
      __syncthreads();
      out = base_dft<MM, L, NE>(ra, rb, A.logb, mc);
    }
    for (int it = threadIdx.x; it < NE * MM; it += NT) {
      const int el = it / MM, kk = it % MM;
      if (e0 + el >= A.total_elems) continue;
      uint32_t v[L];
      ld_res<L>(v, out + el * ES + kk * L);
      if (A.scale) {
        uint32_t ks[L];
#pragma unroll
        for (int q = 0; q < L; ++q) ks[q] = mc.kscale[q];
        mont_mul<L>(v, v, ks, mc);
      }
      st_res<L>(A.a + (e0 + el) * (MM * L) + kk * L, v);
    }
    fence_proxy_async();
    __syncthreads();
    if (NS == 1 && nxt < ntiles && (kSpreadIssue || threadIdx.x < 32)) issue_bottom_tile<MM, L>(A, nxt, &bar[0], smem, smem + NE * ES);
    tile = nxt;
  }
  release_tiles(A.ctr);
}

// standalone batched ring product (stage API r_mul / pointwise): out = y*x (exact)
template <int MM, int L>
__global__ void __launch_bounds__(Cfg<MM>::NT, Cfg<MM>::MINB) k_rmul(const uint32_t* __restrict__ x,
                                                                     const uint32_t* __restrict__ y, uint32_t* out,
                                                                     long long count, ModCtx mc) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  constexpr int kT = Cfg<MM>::T;
  constexpr int ES = Smem<MM, L>::ES, ESW = Smem<MM, L>::ESW;
  constexpr int NT = Cfg<MM>::NT, NE = Cfg<MM>::NE;
  constexpr int TPE = MM / kT;
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sx = smem;
  uint32_t* sy = smem + NE * ES;
  const long long e0 = (long long)blockIdx.x * NE;
  constexpr int V4 = MM * L / 4;
  for (int it = threadIdx.x; it < NE * V4; it += NT) {
    const int el = it / V4, w4 = it % V4;
    uint4 vx = make_uint4(0, 0, 0, 0), vy = vx;
    if (e0 + el < count) {
      const long long off = (e0 + el) * (MM * L) + w4 * 4;
      vx = *reinterpret_cast<const uint4*>(x + off);
      vy = *reinterpret_cast<const uint4*>(y + off);
    }
    *reinterpret_cast<uint4*>(sx + el * ES + w4 * 4) = vx;
    *reinterpret_cast<uint4*>(sy + el * ES + w4 * 4) = vy;
  }
  __syncthreads();

  __syncthreads();
  for (int it = threadIdx.x; it < NE * TPE; it += NT) {
    const int el = it / TPE, k0 = (it % TPE) * kT;
    if (e0 + el >= count) continue;
    uint32_t w[kT][L];
    ring_mul<MM, L>(ResS<L>{sy + el * ES}, ResS<L>{sx + el * ES}, BiasFromY{}, k0, mc, w);
    uint32_t r2[L];
#pragma unroll
    for (int q = 0; q < L; ++q) r2[q] = mc.r2[q];
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      mont_mul<L>(w[t], w[t], r2, mc);
      st_res<L>(out + (e0 + el) * (MM * L) + (k0 + t) * L, w[t]);
    }
  }
}

// twiddle rows [top_mu][2MM][L] from the Montgomery-form table [top_mu][MM][L]:
// first MM residues = rho~_s, next MM = W_s[k] = -(2^(32L)-1) sum_{i>k} rho~_s[i] mod p
template <int L>
__global__ void k_build_twr(const uint32_t* __restrict__ tw, uint32_t* twr, long long top_mu, int MM, ModCtx mc) {
  const long long total = top_mu * MM;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long s = i / MM;
    const int k = (int)(i % MM);
    const uint32_t* row = tw + s * MM * L;
    uint32_t* dst = twr + s * 2LL * MM * L;
    uint32_t y[L], acc[L];
#pragma unroll
    for (int q = 0; q < L; ++q) {
      y[q] = row[k * L + q];
      acc[q] = 0;
    }
    st_res<L>(dst + k * L, y);
    for (int j = k + 1; j < MM; ++j) {
#pragma unroll
      for (int q = 0; q < L; ++q) y[q] = row[j * L + q];
      add_mod<L>(acc, acc, y, mc);
    }
    uint32_t c[L];
#pragma unroll
    for (int q = 0; q < L; ++q) c[q] = mc.cbias[q];
    mont_mul<L>(acc, acc, c, mc);
    st_res<L>(dst + (MM + k) * L, acc);
  }
}

// ---------------------------------------------------------------------------
// elementwise helpers (templated on L only)

// v <- v * c * R^-1 for every residue (c = R^2 gives Montgomery form; c = kinv gives /2M)
template <int L>
__global__ void k_mont_scale(uint32_t* v, long long nres, int which, ModCtx mc) {
  uint32_t c[L];
#pragma unroll
  for (int q = 0; q < L; ++q) c[q] = which == 0 ? mc.r2[q] : which == 1 ? mc.kinv[q] : mc.kscale[q];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nres; i += (long long)gridDim.x * blockDim.x) {
    uint32_t x[L];
#pragma unroll
    for (int q = 0; q < L; ++q) x[q] = v[i * L + q];
    mont_mul<L>(x, x, c, mc);
#pragma unroll
    for (int q = 0; q < L; ++q) v[i * L + q] = x[q];
  }
}

#ifdef DKSS_COMMON_KERNELS  // non-template kernels: compiled only in dkss_capi.cu
// dkss_encode (bigmul/dkss.py:381-398): poly[e][k] = bits [u(e*m/2+k), +u) of the operand
// for e < M, k < m/2; zero elsewhere.  One thread per (poly, element, coefficient).
struct EncodeArgs {
  const uint32_t* ops;  // npoly operands, each `na` limbs
  long long na;
  uint32_t* poly;
  long long poly_words;
  int npoly, M, MM, L, u;
};

__global__ void k_encode(EncodeArgs A) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  const long long per = 2LL * A.M * A.MM;
  const long long total = per * A.npoly;
  const int half = A.MM / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long pidx = i / per, r = i % per;
    const long long e = r / A.MM;
    const int k = (int)(r % A.MM);
    uint32_t out[DKSS_MAXL] = {0, 0, 0, 0, 0, 0};
    if (e < A.M && k < half) {
      const long long bit = (long long)A.u * (e * half + k);
      const uint32_t* op = A.ops + pidx * A.na;
      const long long q = bit >> 5;
      const int s = (int)(bit & 31);
      // gather up to 4 source limbs (u <= 96)
      uint32_t src[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) src[w] = (q + w < A.na) ? op[q + w] : 0u;
      uint32_t sh[3];
#pragma unroll
      for (int w = 0; w < 3; ++w) sh[w] = s ? __funnelshift_r(src[w], src[w + 1], s) : src[w];
      int rem = A.u;
#pragma unroll
      for (int w = 0; w < 3; ++w) {
        if (rem >= 32) out[w] = sh[w];
        else if (rem > 0) out[w] = sh[w] & ((1u << rem) - 1u);
        rem -= 32;
      }
    }
    uint32_t* dst = A.poly + pidx * A.poly_words + r * A.L;
    for (int w = 0; w < A.L; ++w) dst[w] = out[w];
  }
}

// natural index i -> in-place position after the forward passes (digit reversal)
__device__ __forceinline__ long long fwd_position(long long i, int logE, int levels, int logb) {
  // i = f*2m + vv at each level (least-significant digit first); position = vv*mu + pos_sub(f)
  long long pos = 0;
  int remaining = levels * logE + logb;  // log2(2M)
  for (int lv = 0; lv < levels; ++lv) {
    const long long vv = i & ((1LL << logE) - 1);
    i >>= logE;
    remaining -= logE;
    pos += vv << remaining;
  }
  return pos + i;  // base-case block is in natural order
}

// out[i] = in[position(i)] (to natural order) or out[position(i)] = in[i] (inverse)
__global__ void k_permute(const uint32_t* in, uint32_t* out, long long elems, int elem_words, int logE, int levels,
                          int logb, int to_natural, long long poly_words, int npoly) {
  const long long total = elems * npoly * elem_words;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long w = t % elem_words;
    const long long gi = t / elem_words;
    const long long pidx = gi / elems, i = gi % elems;
    const long long pos = fwd_position(i, logE, levels, logb);
    const long long base = pidx * poly_words;
    if (to_natural) out[base + i * elem_words + w] = in[base + pos * elem_words + w];
    else out[base + pos * elem_words + w] = in[base + i * elem_words + w];
  }
}

// ---------------------------------------------------------------------------
// decode (bigmul/dkss.py:498-513): overlap-add of the (scaled, canonical) coefficients at
// bit offsets u*(l*m/2 + k), coefficient l read from index (-l) mod 2M, then a
// device-wide carry propagation.
//
// phase 1: one thread per output limb t computes S_t = sum of the 32-bit windows of every
// coefficient overlapping [32t, 32t+32); then w_t = lo32(S_t) + hi(S_{t-1}) < 2^32 + 2^6,
// so every limb's carry-out is 0/1.  Warp and block (generate, propagate) masks are
// resolved with the add-trick: carries = ((G|P) + G + cin) ^ (G|P) ^ G.
constexpr int kDecThreads = 256;
constexpr int kDecWarps = kDecThreads / 32;

struct DecodeArgs {
  const uint32_t* v;   // natural-order coefficients, npoly polys
  long long poly_words;
  uint32_t* out;       // npoly products, nout limbs each
  long long nout;
  uint32_t* gmask;     // per warp: generate bits   [npoly][nout/32]
  uint32_t* pmask;     // per warp: propagate bits
  uint32_t* bstat;     // per block: bit0 = cout(cin=0), bit1 = cout(cin=1)
  int blocks_per_poly;
  int M, MM, L, u;
  const unsigned long long* sglob;  // non-null: per-limb window sums precomputed (distributed decode)
};

__device__ __forceinline__ unsigned long long window_sum(const DecodeArgs& A, const uint32_t* v, long long t) {
  if (t < 0) return 0ull;
  const long long twoM = 2LL * A.M;
  const int half = A.MM / 2;
  const int lh = __ffs(half) - 1;
  unsigned long long S = 0;
  if (A.u == 32) {
    // slot s = t - q contributes limb q of its two coefficients (l = s/half, l - 1)
#pragma unroll 1
    for (int q = 0; q < A.L; ++q) {
      const long long s = t - q;
      if (s < 0) break;
      const long long lq = s >> lh;
      const int kk = (int)(s & (half - 1));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long l = lq - h;
        const int k = kk + h * half;
        if (l < 0 || l >= twoM) continue;
        const long long src = (twoM - l) & (twoM - 1);
        S += __ldg(v + (src * A.MM + k) * A.L + q);
      }
    }
    return S;
  }
  const long long wbits = 32LL * A.L;
  long long s_lo = (32 * t - wbits) / A.u + 1;
  if (32 * t - wbits < 0) s_lo = 0;
  const long long s_hi = (32 * t + 31) / A.u;
  for (long long s = s_lo; s <= s_hi; ++s) {
    const long long off = 32 * t - (long long)A.u * s;  // bit offset of window inside coefficient
    const long long lq = s >> lh;
    for (int h = 0; h < 2; ++h) {
      const long long l = lq - h;
      const long long k = s - l * half;
      if (l < 0 || l >= twoM || k < 0 || k >= A.MM) continue;
      const long long src = (twoM - l) & (twoM - 1);
      const uint32_t* c = v + (src * A.MM + k) * A.L;
      uint32_t word;
      if (off >= 0) {
        const int q = (int)(off >> 5), sh = (int)(off & 31);
        const uint32_t lo = q < A.L ? __ldg(c + q) : 0u, hi = q + 1 < A.L ? __ldg(c + q + 1) : 0u;
        word = sh ? __funnelshift_r(lo, hi, sh) : lo;
      } else {
        word = __ldg(c) << (int)(-off);
      }
      S += word;
    }
  }
  return S;
}

// phase 1: per-limb sums, per-warp (generate, propagate) masks, per-block carry function.
// `sum(pidx, t)` is the 64-bit sum of the 32-bit windows that land on limb t (every
// window sum is < 2^35, so limb t = low(S_t) + high(S_(t-1)) carries at most one bit).
template <class SumFn>
__device__ __forceinline__ void decode1_body(const DecodeArgs& A, SumFn sum) {
  const int pidx = blockIdx.x / A.blocks_per_poly;
  const int blk = blockIdx.x % A.blocks_per_poly;
  const long long t = (long long)blk * kDecThreads + threadIdx.x;
  __shared__ unsigned long long sS[kDecThreads + 1];
  __shared__ uint32_t wg[kDecWarps], wp[kDecWarps];
  unsigned long long S = t < A.nout ? sum(pidx, t) : 0ull;
  sS[threadIdx.x + 1] = S;
  if (threadIdx.x == 0) sS[0] = (t < A.nout && t > 0) ? sum(pidx, t - 1) : 0ull;
  __syncthreads();
  unsigned long long w = (S & 0xFFFFFFFFull) + (sS[threadIdx.x] >> 32);
  if (t >= A.nout) w = 0;
  const bool g = w >> 32;
  const bool p = (uint32_t)w == 0xFFFFFFFFu && !g;
  const unsigned G = __ballot_sync(0xFFFFFFFFu, g), P = __ballot_sync(0xFFFFFFFFu, p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (t < A.nout) A.out[(long long)pidx * A.nout + t] = (uint32_t)w;
  if (lane == 0) {
    const long long wi = ((long long)pidx * A.blocks_per_poly + blk) * kDecWarps + warp;
    A.gmask[wi] = G;
    A.pmask[wi] = P;
    // warp carry-out for cin = 0 / 1
    const unsigned long long a = (unsigned long long)(G | P), b = G;
    wg[warp] = (unsigned)((a + b) >> 32);
    wp[warp] = (unsigned)((a + b + 1) >> 32);
  }
  __syncthreads();
  if (warp == 0) {
    const bool c0 = lane < kDecWarps && wg[lane], c1 = lane < kDecWarps && wp[lane];
    const unsigned WG = __ballot_sync(0xFFFFFFFFu, c0), WP = __ballot_sync(0xFFFFFFFFu, c1 && !c0);
    if (lane == 0) {
      const unsigned long long a = (unsigned long long)(WG | WP), b = WG;
      const unsigned co0 = (unsigned)((a + b) >> kDecWarps) & 1u, co1 = (unsigned)((a + b + 1) >> kDecWarps) & 1u;
      A.bstat[(long long)pidx * A.blocks_per_poly + blk] = co0 | (co1 << 1);
    }
  }
}

__global__ void __launch_bounds__(kDecThreads) k_decode1(DecodeArgs A) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  decode1_body(A, [&](int pidx, long long t) {
    return A.sglob ? A.sglob[t] : window_sum(A, A.v + (long long)pidx * A.poly_words, t);
  });
}

// decode1 for u = 32 with the residues staged: slot s = l*m/2 + k holds residue k of element l
// and residue k + m/2 of element l - 1, and limb q of slot s lands on output limb s + q.  The
// block's 256 + L slots are read once, each residue as one vector load (consecutive slots are
// consecutive residues: coalesced), their per-limb pair sums go to shared memory, and
// S_t = sum_q P[t - q][q] is summed from there -- instead of L dependent strided scalar loads
// per limb (window_sum)
template <int L>
__global__ void __launch_bounds__(kDecThreads) k_decode1_u32(DecodeArgs A) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  __shared__ unsigned long long sP[(kDecThreads + L) * L];
  const int pidx = blockIdx.x / A.blocks_per_poly;
  const long long t0 = (long long)(blockIdx.x % A.blocks_per_poly) * kDecThreads;
  const uint32_t* v = A.v + (long long)pidx * A.poly_words;
  const long long twoM = 2LL * A.M;
  const int half = A.MM / 2, lh = __ffs(half) - 1;
  for (int i = threadIdx.x; i < kDecThreads + L; i += kDecThreads) {
    const long long s = t0 - L + i;
    unsigned long long acc[L];
#pragma unroll
    for (int q = 0; q < L; ++q) acc[q] = 0;
    if (s >= 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long l = (s >> lh) - h;
        if (l < 0 || l >= twoM) continue;
        const long long src = (twoM - l) & (twoM - 1);
        const uint32_t* c = v + (src * A.MM + (s & (half - 1)) + h * half) * L;
        uint32_t w[L];
        if constexpr (L == 4) {
          const uint4 x = __ldg(reinterpret_cast<const uint4*>(c));
          w[0] = x.x, w[1] = x.y, w[2] = x.z, w[3] = x.w;
        } else if constexpr (L % 2 == 0) {
#pragma unroll
          for (int q = 0; q < L; q += 2) {
            const uint2 x = __ldg(reinterpret_cast<const uint2*>(c + q));
            w[q] = x.x, w[q + 1] = x.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < L; ++q) w[q] = __ldg(c + q);
        }
#pragma unroll
        for (int q = 0; q < L; ++q) acc[q] += w[q];
      }
    }
#pragma unroll
    for (int q = 0; q < L; ++q) sP[i * L + q] = acc[q];
  }
  __syncthreads();
  decode1_body(A, [&](int, long long t) {
    const int i = (int)(t - t0) + L;  // slot index of t inside sP (t >= t0 - 1)
    unsigned long long S = 0;
#pragma unroll
    for (int q = 0; q < L; ++q) S += sP[(i - q) * L + q];
    return S;
  });
}

// phase 2: one CTA per product turns the block carry functions into block carry-ins
// (bit 2 of bstat).  Carry functions of a block are kill (c0=c1=0), propagate (c0=0,c1=1)
// or generate (c0=c1=1); thread chunks are composed sequentially, the 1024 chunk results
// with the (generate | propagate) + generate add trick at warp and CTA level.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) k_decode_scan(DecodeArgs A) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  const int B = A.blocks_per_poly;
  uint32_t* st = A.bstat + (long long)blockIdx.x * B;
  const int per = (B + kScanThreads - 1) / kScanThreads;
  const int b0 = threadIdx.x * per, b1 = min(B, b0 + per);
  // compose this thread's chunk: f(cin) = cout
  unsigned f0 = 0, f1 = 1;  // identity
  for (int b = b0; b < b1; ++b) {
    const unsigned s = st[b];
    const unsigned c0 = s & 1u, c1 = (s >> 1) & 1u;
    f0 = f0 ? c1 : c0;
    f1 = f1 ? c1 : c0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool g = f0, p = f1 && !f0;
  const unsigned G = __ballot_sync(0xFFFFFFFFu, g), P = __ballot_sync(0xFFFFFFFFu, p);
  __shared__ unsigned wg[32], wp[32], wcin[32];
  if (lane == 0) {
    const unsigned long long a = (unsigned long long)(G | P), b = G;
    wg[warp] = (unsigned)((a + b) >> 32);
    wp[warp] = (unsigned)((a + b + 1) >> 32);
  }
  __syncthreads();
  if (warp == 0) {
    const bool c0 = wg[lane], c1 = wp[lane];
    const unsigned WG = __ballot_sync(0xFFFFFFFFu, c0), WP = __ballot_sync(0xFFFFFFFFu, c1 && !c0);
    const unsigned long long a = (unsigned long long)(WG | WP), b = WG;
    const unsigned long long carries = (a + b) ^ a ^ b;  // carry into each warp, product cin = 0
    wcin[lane] = (unsigned)((carries >> lane) & 1ull);
  }
  __syncthreads();
  const unsigned long long a = (unsigned long long)(G | P), b = G;
  const unsigned long long carries = (a + b + wcin[warp]) ^ a ^ b;
  unsigned cin = (unsigned)((carries >> lane) & 1ull);
  for (int bb = b0; bb < b1; ++bb) {
    const unsigned s = st[bb];
    st[bb] = (s & 3u) | (cin << 2);
    cin = cin ? (s >> 1) & 1u : s & 1u;
  }
}

// phase 3: apply carries inside each block
__device__ __forceinline__ void decode2_body(const DecodeArgs& A, int pidx, int blk, unsigned cin) {
  const long long t = (long long)blk * kDecThreads + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ unsigned s_wcin[kDecWarps];
  if (warp == 0) {
    const long long wi = ((long long)pidx * A.blocks_per_poly + blk) * kDecWarps + lane;
    const unsigned G = lane < kDecWarps ? A.gmask[wi] : 0u, P = lane < kDecWarps ? A.pmask[wi] : 0u;
    const unsigned long long a = (unsigned long long)(G | P), b = G;
    const bool c0 = (unsigned)((a + b) >> 32), c1 = (unsigned)((a + b + 1) >> 32);
    const unsigned WG = __ballot_sync(0xFFFFFFFFu, c0), WP = __ballot_sync(0xFFFFFFFFu, c1 && !c0);
    const unsigned long long wa = (unsigned long long)(WG | WP), wb = WG;
    const unsigned long long carries = (wa + wb + cin) ^ wa ^ wb;  // bit i = carry into warp i
    if (lane < kDecWarps) s_wcin[lane] = (unsigned)((carries >> lane) & 1ull);
  }
  __syncthreads();
  if (t >= A.nout) return;
  const long long wi = ((long long)pidx * A.blocks_per_poly + blk) * kDecWarps + warp;
  const unsigned G = A.gmask[wi], P = A.pmask[wi];
  const unsigned long long a = (unsigned long long)(G | P), b = G;
  const unsigned long long carries = (a + b + s_wcin[warp]) ^ a ^ b;
  // a carry into a limb is rare (w_t's high word is set only when lo(S_t) + hi(S_(t-1))
  // overflows), so the limbs decode1 wrote are rewritten only where one arrives
  if ((carries >> lane) & 1ull) A.out[(long long)pidx * A.nout + t] += 1u;
}

__global__ void __launch_bounds__(kDecThreads) k_decode2(DecodeArgs A) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  const int pidx = blockIdx.x / A.blocks_per_poly;
  const int blk = blockIdx.x % A.blocks_per_poly;
  decode2_body(A, pidx, blk, (A.bstat[(long long)pidx * A.blocks_per_poly + blk] >> 2) & 1u);
}

// phases 2 + 3 in one kernel for products of at most kSelfScanBlocks blocks: warp 0 of every
// block composes the carry functions of the blocks before it (each lane a contiguous chunk,
// then the (generate | propagate) + generate add across lanes) -- no scan launch.  Measured:
// 2^20 (256 blocks) -2%, 2^22 (1024 blocks) +1%, so only up to 256 blocks
constexpr int kSelfScanBlocks = 256;
__global__ void __launch_bounds__(kDecThreads) k_decode2s(DecodeArgs A) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  const int pidx = blockIdx.x / A.blocks_per_poly;
  const int blk = blockIdx.x % A.blocks_per_poly;
  __shared__ unsigned s_cin;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const uint32_t* st = A.bstat + (long long)pidx * A.blocks_per_poly;
    const int per = (blk + 31) / 32;
    const int b0 = lane * per, b1 = min(blk, b0 + per);
    unsigned f0 = 0, f1 = 1;  // identity: cout(cin = 0), cout(cin = 1)
    for (int b = b0; b < b1; ++b) {
      const unsigned sv = st[b];
      const unsigned c0 = sv & 1u, c1 = (sv >> 1) & 1u;
      f0 = f0 ? c1 : c0;
      f1 = f1 ? c1 : c0;
    }
    const unsigned G = __ballot_sync(0xFFFFFFFFu, f0), P = __ballot_sync(0xFFFFFFFFu, f1 && !f0);
    const unsigned long long a = (unsigned long long)(G | P), b = G;
    if (lane == 0) s_cin = (unsigned)((a + b) >> 32) & 1u;  // carry out of all predecessors (product cin 0)
  }
  __syncthreads();
  decode2_body(A, pidx, blk, s_cin);
}

// ---------------------------------------------------------------------------
// distributed decode of a four-step split (u = 32).  Rank r holds the product coefficients of
// physical elements g = j*mu0 + r*C + c (its columns of every row j); the decode reads
// logical element l at physical (2M - l) mod 2M, so row j of rank r is the logical run
// [2M - j*mu0 - r*C - C + 1, 2M - j*mu0 - r*C] (rank 0 / row 0: [2M - C + 1, 2M) plus the lone
// element 0, run E).  For every run, k_decode_partial writes the window sums of the output
// limbs [l_a*half, l_b*half + half + L - 1) using only this rank's coefficients; runs of
// different ranks overlap by half + L - 1 limbs, and k_decode_assemble adds the gathered runs
// into the global per-limb sums that k_decode1 then turns into limbs and carries.
struct PartialArgs {
  const uint32_t* x;          // [E][C] local elements (m*L words each)
  unsigned long long* s_out;  // [E + 1][seg] window sums
  long long seg;              // limbs per run segment: C*half + half + L - 1
  long long C, mu0, twoM;
  int rank, E, MM, L;
};

__device__ __forceinline__ void run_bounds(long long r, long long j, long long C, long long mu0, long long twoM, int E,
                                           long long* la, long long* lb) {
  if (j == E) {  // the lone element 0 (rank 0 only)
    *la = 0;
    *lb = r == 0 ? 1 : 0;
    return;
  }
  const long long hi = twoM - j * mu0 - r * C;  // logical index of physical column r*C (row j)
  *la = hi - C + 1;
  *lb = (hi == twoM) ? twoM : hi + 1;  // physical element 0 is the lone run
}

__global__ void k_decode_partial(PartialArgs A) {
  griddep_wait();
  griddep_launch();
  const int half = A.MM / 2;
  const long long total = (long long)(A.E + 1) * A.seg;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx / A.seg, tl = idx % A.seg;
    long long la, lb;
    run_bounds(A.rank, j, A.C, A.mu0, A.twoM, A.E, &la, &lb);
    unsigned long long S = 0;
    if (lb > la) {
      const long long t = la * half + tl;
      for (int q = 0; q < A.L; ++q) {
        const long long sl = t - q;
        if (sl < 0) break;
        const long long lq = sl / half;
        const int kk = (int)(sl % half);
        for (int h = 0; h < 2; ++h) {
          const long long l = lq - h;
          if (l < la || l >= lb) continue;
          const long long g = (A.twoM - l) % A.twoM;  // physical element
          const long long jj = g / A.mu0, cc = g % A.mu0 - (long long)A.rank * A.C;
          const int k = kk + h * half;
          S += __ldg(A.x + ((jj * A.C + cc) * A.MM + k) * A.L + q);
        }
      }
    }
    A.s_out[idx] = S;
  }
  __threadfence_system();  // s_out may be rank 0's gather buffer on another GPU (fused exchange)
}

struct AssembleArgs {
  const unsigned long long* parts;  // [G][E + 1][seg] gathered window sums
  unsigned long long* sglob;        // [nout] zeroed
  long long seg, nout, C, mu0, twoM;
  int world, E, half;
};

__global__ void k_decode_assemble(AssembleArgs A) {
  griddep_wait();
  griddep_launch();
  const long long total = (long long)A.world * (A.E + 1) * A.seg;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const unsigned long long v = A.parts[idx];
    if (!v) continue;
    const long long tl = idx % A.seg, rj = idx / A.seg;
    const long long r = rj / (A.E + 1), j = rj % (A.E + 1);
    long long la, lb;
    run_bounds(r, j, A.C, A.mu0, A.twoM, A.E, &la, &lb);
    const long long t = la * A.half + tl;
    if (lb > la && t < A.nout) atomicAdd(A.sglob + t, v);
  }
}

// ---------------------------------------------------------------------------
// block transpose for the four-step exchange: src [n][A][B][run] -> dst [n][B][A][run]
// (run = contiguous uint4 per block); blockIdx.y walks the (n, a, b) blocks of src
__global__ void k_block_transpose(const uint4* __restrict__ src, uint4* __restrict__ dst, int A, int B,
                                  long long run) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  const int blk = blockIdx.y;
  const int b = blk % B, t = blk / B;
  const int a = t % A, n = t / A;
  const uint4* s = src + (long long)blk * run;
  uint4* d = dst + (((long long)n * B + b) * A + a) * run;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < run; i += (long long)gridDim.x * blockDim.x)
    d[i] = s[i];
}

// ---------------------------------------------------------------------------
// radix change of little-endian digit strings: `sbits`-bit digits (stored one per u32,
// 8 <= sbits <= 32; e.g. CPython's 30-bit int digits) -> 32-bit limbs.  Operand q
// (blockIdx.y) is digits [off[q], off[q+1]) of `stage` and becomes limbs
// dst[q*ndst, (q+1)*ndst); limb i holds bits [32i, 32i+32), gathered from at most five
// consecutive digits.
struct RepackArgs {
  const uint32_t* stage;
  const long long* off;
  uint32_t* dst;
  long long ndst;
  int sbits;
};

__global__ void k_repack_bits(RepackArgs A) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  const int q = blockIdx.y;
  const long long o0 = A.off[q], ns = A.off[q + 1] - o0;
  const uint32_t* src = A.stage + o0;
  uint32_t* dst = A.dst + (long long)q * A.ndst;
  const uint64_t mask = A.sbits == 32 ? 0xFFFFFFFFull : ((1ull << A.sbits) - 1);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < A.ndst; i += (long long)gridDim.x * blockDim.x) {
    const long long bit = 32 * i;
    const long long d = bit / A.sbits;
    const int o = (int)(bit - d * A.sbits);
    uint64_t acc = 0;
    int sh = -o;
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      if (sh >= 32) break;
      const uint64_t dig = (d + t < ns) ? (src[d + t] & mask) : 0;
      acc |= sh >= 0 ? dig << sh : dig >> (-sh);
      sh += A.sbits;
    }
    dst[i] = (uint32_t)acc;
  }
}

// ---------------------------------------------------------------------------
// Lucas-Lehmer step tail (bigmul/bench.py:187-194, 214-216): s = (c - 2) mod (2^p - 1)
// for a product c < 2^(2p), canonical in [0, 2^p - 1).  One CTA of kMersThreads threads;
// n = ceil(p/32) limbs of s, thread t owns a contiguous chunk; every multi-limb add
// resolves its carries with a block-wide (generate, propagate) scan.
constexpr int kMersThreads = 1024;

struct MersArgs {
  const uint32_t* c;  // product limbs
  long long nc;
  long long p;
  uint32_t* s;        // n = ceil(p/32) limbs out (limbs of s beyond n are left untouched)
};

// carry-in of this thread's chunk given its (g, p) and the carry into chunk 0; also
// returns the carry out of the last chunk in *cout (all threads)
__device__ __forceinline__ uint32_t block_carry(uint32_t g, uint32_t pr, uint32_t c0, uint32_t* cout) {
  __shared__ uint32_t wg[32], wp[32], s_out;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // inclusive warp scan of (g, p): combine earlier (g', p') into later: g |= p & g'; p &= p'
  uint32_t G = g, Pp = pr;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t g2 = __shfl_up_sync(0xFFFFFFFFu, G, d), p2 = __shfl_up_sync(0xFFFFFFFFu, Pp, d);
    if (lane >= d) {
      G |= Pp & g2;
      Pp &= p2;
    }
  }
  if (lane == 31) {
    wg[warp] = G;
    wp[warp] = Pp;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t g1 = lane < (int)(blockDim.x >> 5) ? wg[lane] : 0u, p1 = lane < (int)(blockDim.x >> 5) ? wp[lane] : 1u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t g2 = __shfl_up_sync(0xFFFFFFFFu, g1, d), p2 = __shfl_up_sync(0xFFFFFFFFu, p1, d);
      if (lane >= d) {
        g1 |= p1 & g2;
        p1 &= p2;
      }
    }
    // exclusive carry into warp `lane`, with the external carry c0
    const uint32_t ge = __shfl_up_sync(0xFFFFFFFFu, g1, 1), pe = __shfl_up_sync(0xFFFFFFFFu, p1, 1);
    const uint32_t cin_w = lane == 0 ? c0 : (ge | (pe & c0));
    wg[lane] = cin_w;
    if (lane == 31) s_out = g1 | (p1 & c0);
  }
  __syncthreads();
  const uint32_t cw = wg[warp];
  const uint32_t ge = __shfl_up_sync(0xFFFFFFFFu, G, 1), pe = __shfl_up_sync(0xFFFFFFFFu, Pp, 1);
  const uint32_t cin = lane == 0 ? cw : (ge | (pe & cw));
  *cout = s_out;
  __syncthreads();
  return cin;
}

// limb i of (c >> sh) restricted to bits below 32*n (sh = bit offset)
__device__ __forceinline__ uint32_t limb_at(const uint32_t* c, long long nc, long long bit) {
  const long long w = bit >> 5;
  const int o = (int)(bit & 31);
  const uint32_t lo = w < nc ? c[w] : 0u, hi = (w + 1) < nc ? c[w + 1] : 0u;
  return o ? __funnelshift_r(lo, hi, o) : lo;
}

__global__ void __launch_bounds__(kMersThreads) k_mersenne_sub2(MersArgs A) {
  griddep_wait();
  griddep_launch();
  const long long p = A.p, n = (p + 31) >> 5;
  const int topb = (int)(p - 32 * (n - 1));  // bits used in limb n-1 (1..32)
  const uint32_t topmask = topb == 32 ? 0xFFFFFFFFu : ((1u << topb) - 1u);
  const long long K = (n + blockDim.x - 1) / blockDim.x;
  const long long i0 = threadIdx.x * K, i1 = min(n, i0 + K);
  __shared__ uint32_t s_flag[2];
  uint32_t cout;
  // (1) t = lo + hi, lo = c mod 2^p, hi = c >> p
  auto lo_at = [&](long long i) { return i < A.nc ? (i == n - 1 ? A.c[i] & topmask : A.c[i]) : 0u; };
  auto hi_at = [&](long long i) { return limb_at(A.c, A.nc, p + 32 * i) & (i == n - 1 ? topmask : 0xFFFFFFFFu); };
  uint32_t g = 0, pr = 1;
  {
    uint32_t cy = 0;
    for (long long i = i0; i < i1; ++i) {
      const uint64_t v = (uint64_t)lo_at(i) + hi_at(i) + cy;
      cy = (uint32_t)(v >> 32);
      pr &= ((uint32_t)v == 0xFFFFFFFFu);
    }
    g = cy;
  }
  uint32_t cin = block_carry(g, pr, 0u, &cout);
  for (long long i = i0; i < i1; ++i) {
    const uint64_t v = (uint64_t)lo_at(i) + hi_at(i) + cin;
    cin = (uint32_t)(v >> 32);
    A.s[i] = (uint32_t)v;
  }
  __syncthreads();
  // (2) fold the bit at position p (t < 2^(p+1)): t = (t mod 2^p) + (t >> p)
  uint32_t fold = cout;  // carry out of limb n-1 (bit 32n)
  if (topb < 32) fold = (A.s[n - 1] >> topb) & 1u;
  __syncthreads();
  if (threadIdx.x == 0 && topb < 32) A.s[n - 1] &= topmask;
  __syncthreads();
  g = 0;
  pr = 1;
  for (long long i = i0; i < i1; ++i) pr &= (A.s[i] == 0xFFFFFFFFu);
  cin = block_carry(0u, pr, fold, &cout);
  for (long long i = i0; i < i1 && cin; ++i) {
    const uint64_t v = (uint64_t)A.s[i] + cin;
    cin = (uint32_t)(v >> 32);
    A.s[i] = (uint32_t)v;
  }
  __syncthreads();
  // (3) t - 2 mod (2^p - 1), t in [0, 2^p - 1]: t >= 2 -> t - 2, else t + 2^p - 3
  if (threadIdx.x == 0) s_flag[0] = 0;
  __syncthreads();
  uint32_t any_hi = 0;
  for (long long i = max(i0, 1LL); i < i1; ++i) any_hi |= A.s[i];
  if (any_hi) atomicOr(&s_flag[0], 1u);
  __syncthreads();
  if (threadIdx.x == 0) s_flag[1] = !s_flag[0] && A.s[0] < 2;
  __syncthreads();
  if (s_flag[1]) {
    const uint32_t t0 = A.s[0];
    for (long long i = i0; i < i1; ++i) A.s[i] = i == n - 1 ? topmask : 0xFFFFFFFFu;
    __syncthreads();
    if (threadIdx.x == 0) A.s[0] = (n == 1 ? topmask : 0xFFFFFFFFu) - 2u + t0;  // 2^p - 3 + t0
    return;
  }
  // borrow chain of t - 2 (t >= 2 here): chunk 0 generates a borrow if its own limbs
  // underflow; a later chunk passes a borrow on iff all its limbs are zero
  g = 0;
  pr = 1;
  if (i0 == 0) {
    uint32_t b = 0;
    for (long long i = i0; i < i1; ++i) {
      const uint32_t sub = (i == 0 ? 2u : 0u) + b;
      b = (uint32_t)(A.s[i] < sub);
    }
    g = b;
    pr = 0;
  } else {
    for (long long i = i0; i < i1; ++i) pr &= (A.s[i] == 0u);
  }
  cin = block_carry(g, pr, 0u, &cout);
  for (long long i = i0; i < i1; ++i) {
    const uint32_t sub = (i == 0 ? 2u : 0u) + cin;
    const uint32_t v = A.s[i];
    cin = (uint32_t)(v < sub);
    A.s[i] = v - sub;
  }
}

#endif  // DKSS_COMMON_KERNELS

}  // namespace dkss
