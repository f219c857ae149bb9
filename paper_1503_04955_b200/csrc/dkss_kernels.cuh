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
#pragma once
#include <cstdint>
#include "dkss_arith.cuh"

namespace dkss {

constexpr int kThreads = 256;
constexpr int kT = 4;  // output coefficients per thread in a ring product

// words per element in shared memory: padded so that 8 elements read by one warp
// (4 threads each) land on distinct banks
template <int MM, int L>
struct Smem {
  static constexpr int ES = ((MM * L + 31) / 32) * 32 + 4;
};

template <int MM>
struct Cfg {
  // elements per CTA: enough ring-product work items (elements * MM/kT) for kThreads
  static constexpr int NE = (kThreads * kT / MM) >= 2 * MM ? (kThreads * kT / MM) : 2 * MM;
  static constexpr int COLS = NE / (2 * MM);
};

__device__ __forceinline__ int bitrev_n(int x, int bits) { return bits ? (int)(__brev((unsigned)x) >> (32 - bits)) : 0; }

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

// ---------------------------------------------------------------------------
// ring product core: out[t] = (x * y)_{k0+t} for t < kT, canonical, times R^-1
// (Montgomery).  x: element in shared memory (stride L per coefficient).
// y: loader functor giving the plain coefficient y_j, j in [0, MM).
template <int MM, int L, class YL>
__device__ __forceinline__ void ring_mul_rows(const uint32_t* xs, YL yl, int k0, const ModCtx& mc,
                                              uint32_t (&out)[kT][L]) {
  constexpr int ND = NDig<L>::v;
  constexpr int NC = 2 * ND - 1;
  uint64_t acc[kT][NC];
#pragma unroll
  for (int t = 0; t < kT; ++t)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[t][c] = 0;
  uint32_t win[kT][ND];
#pragma unroll
  for (int t = 1; t < kT; ++t) {
    uint32_t zw[L];
    yl(k0 + t, zw);
    to_r28<L>(zw, win[t]);
  }
#pragma unroll(MM <= 16 ? MM / kT : 1)
  for (int i0 = 0; i0 < MM; i0 += kT) {
#pragma unroll
    for (int s = 0; s < kT; ++s) {
      const int i = i0 + s;
      uint32_t xw[L], xd[ND];
      ld_res<L>(xw, xs + i * L);
      to_r28<L>(xw, xd);
      // new window entry: z_{k0 - i}; negative index wraps with a sign (alpha^m = -1)
      const int j = k0 - i;
      uint32_t yw[L], nw[L];
      yl(j & (MM - 1), yw);
      p_minus<L>(nw, yw, mc);
      const bool wrap = j < 0;
#pragma unroll
      for (int q = 0; q < L; ++q) yw[q] = wrap ? nw[q] : yw[q];
      to_r28<L>(yw, win[(kT - s) % kT]);
#pragma unroll
      for (int t = 0; t < kT; ++t) mac_cols<ND>(acc[t], xd, win[(t - s + kT) % kT]);
    }
  }
#pragma unroll
  for (int t = 0; t < kT; ++t) {
    uint32_t tl[2 * L + 1];
    cols_to_limbs<L>(acc[t], tl);
    redc<L>(out[t], tl, mc);
  }
}

// store T consecutive output coefficients k0.. of (alpha^r * w) into element dst
template <int MM, int L>
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
// in-place radix-2 DIT over NE elements in shared memory, split into groups of n
// (power of two <= 2MM) already in bit-reversed order.  Butterfly root for block size
// `size`: alpha^(kk * 2MM/size) -- the reference's fft_eval merge with PolyAlphaRing,
// bigmul/fft.py:87-94 and bigmul/dkss.py:64-91 (any transform length n uses
// scale*step = 2m/size).  alpha^e is a rotation with negation of wrapped slots
// (poly_mul_xpow, bigmul/dkss.py:46-61), folded into the add/sub choice.
template <int MM, int L, int NE>
__device__ __forceinline__ void dft_inplace(uint32_t* buf, int logn, const ModCtx& mc) {
  constexpr int ES = Smem<MM, L>::ES;
  constexpr int ITEMS = (NE / 2) * MM;
  constexpr int PER = (ITEMS + kThreads - 1) / kThreads;
  for (int ls = 1; ls <= logn; ++ls) {
    const int half = 1 << (ls - 1);
    const int rootstep = (2 * MM) >> ls;  // 2MM / size
    uint32_t oa[PER][L], ob[PER][L];
    int ia[PER], ib[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int it = threadIdx.x + q * kThreads;
      ia[q] = -1;
      if (it < ITEMS) {
        const int bf = it / MM, k = it % MM;
        const int blk = bf >> (ls - 1), kk = bf & (half - 1);
        const int a = (blk << ls) + kk, b = a + half;
        const int e = kk * rootstep;  // < 2MM
        int src = k - e;
        bool neg = false;
        if (src < 0) { src += MM; neg = true; }
        if (src < 0) { src += MM; neg = false; }
        uint32_t u[L], x[L];
        ld_res<L>(u, buf + a * ES + k * L);
        ld_res<L>(x, buf + b * ES + src * L);
        uint32_t s[L], d[L];
        add_mod<L>(s, u, x, mc);
        sub_mod<L>(d, u, x, mc);
#pragma unroll
        for (int w = 0; w < L; ++w) {
          oa[q][w] = neg ? d[w] : s[w];
          ob[q][w] = neg ? s[w] : d[w];
        }
        ia[q] = a * ES + k * L;
        ib[q] = b * ES + k * L;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (ia[q] >= 0) {
        st_res<L>(buf + ia[q], oa[q]);
        st_res<L>(buf + ib[q], ob[q]);
      }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
struct PassArgs {
  uint32_t* poly;        // first polynomial of the launch
  long long poly_words;  // 2M * MM * L
  int log_mu;            // column stride mu = 2^log_mu (elements)
  int log_top_mu;        // log2(M/m)
  long long base_pow;    // (2m)^level
  const uint32_t* tw;    // [M/m][MM][L] Montgomery-form rho^s
  int scale;             // inverse pass: multiply outputs by mc.kscale
  long long total_cols;  // columns in the launch (npoly * M/m)
};

// forward column pass (one level of dkss_fft): column DFT, then twiddle ring product
template <int MM, int L>
__global__ void __launch_bounds__(kThreads) k_fwd_pass(PassArgs A, ModCtx mc) {
  constexpr int ES = Smem<MM, L>::ES;
  constexpr int NE = Cfg<MM>::NE, COLS = Cfg<MM>::COLS, E = 2 * MM;
  constexpr int LOGE = (E == 16) ? 4 : (E == 32) ? 5 : (E == 64) ? 6 : (E == 8) ? 3 : 7;
  extern __shared__ __align__(16) uint32_t smem[];
  const long long cols_per_poly = 1LL << A.log_top_mu;  // M/m columns
  const long long col0 = (long long)blockIdx.x * COLS;
  const int mu_mask = (1 << A.log_mu) - 1;
  // load: element j of column c -> smem slot c*E + bitrev(j)
  constexpr int V4 = MM * L / 4;
  for (int it = threadIdx.x; it < NE * V4; it += kThreads) {
    const int el = it / V4, w4 = it % V4;
    const int c = el / E, j = el % E;
    const long long cg = col0 + c;
    if (cg >= A.total_cols) continue;
    const long long poly = cg / cols_per_poly, cc = cg % cols_per_poly;
    const long long inst = cc >> A.log_mu, l = cc & mu_mask;
    const long long pos = (inst << (A.log_mu + LOGE)) + ((long long)j << A.log_mu) + l;
    const uint4 v = *reinterpret_cast<const uint4*>(A.poly + poly * A.poly_words + pos * (MM * L) + w4 * 4);
    *reinterpret_cast<uint4*>(smem + (c * E + bitrev_n(j, LOGE)) * ES + w4 * 4) = v;
  }
  __syncthreads();
  dft_inplace<MM, L, NE>(smem, LOGE, mc);
  // twiddles rho^(vv*l*base_pow) = alpha^r * rho_table[s] (bigmul/dkss.py:480-492)
  constexpr int TPE = MM / kT;
  const long long top_mask = cols_per_poly - 1;
  for (int it = threadIdx.x; it < NE * TPE; it += kThreads) {
    const int el = it / TPE, tg = it % TPE, k0 = tg * kT;
    const int c = el / E, vv = el % E;
    const long long cg = col0 + c;
    if (cg >= A.total_cols) continue;
    const long long poly = cg / cols_per_poly, cc = cg % cols_per_poly;
    const long long inst = cc >> A.log_mu, l = cc & mu_mask;
    const long long pos = (inst << (A.log_mu + LOGE)) + ((long long)vv << A.log_mu) + l;
    uint32_t* dst = A.poly + poly * A.poly_words + pos * (MM * L);
    const uint32_t* xs = smem + el * ES;
    const long long e = (long long)vv * l * A.base_pow;
    const long long s = e & top_mask;
    const int r = (int)(e >> A.log_top_mu);
    uint32_t w[kT][L];
    if (s == 0) {
#pragma unroll
      for (int t = 0; t < kT; ++t) ld_res<L>(w[t], xs + (k0 + t) * L);
    } else {
      const uint32_t* tws = A.tw + s * (MM * L);
      ring_mul_rows<MM, L>(xs, [&](int j, uint32_t(&y)[L]) { ld_res_g<L>(y, tws + j * L); }, k0, mc, w);
    }
    store_rot<MM, L>(dst, w, k0, r, mc);
  }
}

// inverse (transposed) column pass: twiddle ring product, then column DFT
template <int MM, int L>
__global__ void __launch_bounds__(kThreads) k_inv_pass(PassArgs A, ModCtx mc) {
  constexpr int ES = Smem<MM, L>::ES;
  constexpr int NE = Cfg<MM>::NE, COLS = Cfg<MM>::COLS, E = 2 * MM;
  constexpr int LOGE = (E == 16) ? 4 : (E == 32) ? 5 : (E == 64) ? 6 : (E == 8) ? 3 : 7;
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* raw = smem;
  uint32_t* tw_buf = smem + NE * ES;
  const long long cols_per_poly = 1LL << A.log_top_mu;
  const long long col0 = (long long)blockIdx.x * COLS;
  const int mu_mask = (1 << A.log_mu) - 1;
  constexpr int V4 = MM * L / 4;
  for (int it = threadIdx.x; it < NE * V4; it += kThreads) {
    const int el = it / V4, w4 = it % V4;
    const int c = el / E, j = el % E;
    const long long cg = col0 + c;
    if (cg >= A.total_cols) continue;
    const long long poly = cg / cols_per_poly, cc = cg % cols_per_poly;
    const long long inst = cc >> A.log_mu, l = cc & mu_mask;
    const long long pos = (inst << (A.log_mu + LOGE)) + ((long long)j << A.log_mu) + l;
    const uint4 v = *reinterpret_cast<const uint4*>(A.poly + poly * A.poly_words + pos * (MM * L) + w4 * 4);
    *reinterpret_cast<uint4*>(raw + el * ES + w4 * 4) = v;
  }
  __syncthreads();
  constexpr int TPE = MM / kT;
  const long long top_mask = cols_per_poly - 1;
  for (int it = threadIdx.x; it < NE * TPE; it += kThreads) {
    const int el = it / TPE, tg = it % TPE, k0 = tg * kT;
    const int c = el / E, j = el % E;
    if (col0 + c >= A.total_cols) continue;
    const long long cc = (col0 + c) % cols_per_poly;
    const long long l = cc & mu_mask;
    const uint32_t* xs = raw + el * ES;
    const long long e = (long long)j * l * A.base_pow;
    const long long s = e & top_mask;
    const int r = (int)(e >> A.log_top_mu);
    uint32_t w[kT][L];
    if (s == 0) {
#pragma unroll
      for (int t = 0; t < kT; ++t) ld_res<L>(w[t], xs + (k0 + t) * L);
    } else {
      const uint32_t* tws = A.tw + s * (MM * L);
      ring_mul_rows<MM, L>(xs, [&](int jj, uint32_t(&y)[L]) { ld_res_g<L>(y, tws + jj * L); }, k0, mc, w);
    }
    store_rot<MM, L>(tw_buf + (c * E + bitrev_n(j, LOGE)) * ES, w, k0, r, mc);
  }
  __syncthreads();
  dft_inplace<MM, L, NE>(tw_buf, LOGE, mc);
  for (int it = threadIdx.x; it < NE * MM; it += kThreads) {
    const int el = it / MM, k = it % MM;
    const int c = el / E, vv = el % E;
    const long long cg = col0 + c;
    if (cg >= A.total_cols) continue;
    const long long poly = cg / cols_per_poly, cc = cg % cols_per_poly;
    const long long inst = cc >> A.log_mu, l = cc & mu_mask;
    const long long pos = (inst << (A.log_mu + LOGE)) + ((long long)vv << A.log_mu) + l;
    uint32_t v[L];
    ld_res<L>(v, tw_buf + el * ES + k * L);
    if (A.scale) {
      uint32_t ks[L];
#pragma unroll
      for (int q = 0; q < L; ++q) ks[q] = mc.kscale[q];
      mont_mul<L>(v, v, ks, mc);
    }
    st_res<L>(A.poly + poly * A.poly_words + pos * (MM * L) + k * L, v);
  }
}

// ---------------------------------------------------------------------------
// bottom of the transform: groups of b = 2^logb contiguous elements.
//   mode 0: base DFT of `a` only (stage API)
//   mode 1: base DFT a, base DFT b, pointwise a*b (Montgomery, *R^-1), base DFT -> a
//   mode 2: like 1 but the pointwise product is exact (extra * R^2 R^-1) -- stage API
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
};

template <int MM, int L>
__global__ void __launch_bounds__(kThreads) k_bottom(BottomArgs A, ModCtx mc) {
  constexpr int ES = Smem<MM, L>::ES;
  constexpr int NE = Cfg<MM>::NE;
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sa = smem;
  uint32_t* sb = smem + NE * ES;
  const long long e0 = (long long)blockIdx.x * NE;  // global element index over the batch
  const int bmask = (1 << A.logb) - 1;
  constexpr int V4 = MM * L / 4;
  const bool two = A.mode != 0;
  for (int it = threadIdx.x; it < NE * V4; it += kThreads) {
    const int el = it / V4, w4 = it % V4;
    const long long ge = e0 + el;
    if (ge >= A.total_elems) continue;
    const int slot = (el & ~bmask) | bitrev_n(el & bmask, A.logb);
    const long long off = ge * (MM * L) + w4 * 4;
    *reinterpret_cast<uint4*>(sa + slot * ES + w4 * 4) = *reinterpret_cast<const uint4*>(A.a + off);
    if (two) *reinterpret_cast<uint4*>(sb + slot * ES + w4 * 4) = *reinterpret_cast<const uint4*>(A.b + off);
  }
  __syncthreads();
  dft_inplace<MM, L, NE>(sa, A.logb, mc);
  if (two) {
    dft_inplace<MM, L, NE>(sb, A.logb, mc);
    constexpr int TPE = MM / kT;
    constexpr int PER = (NE * TPE + kThreads - 1) / kThreads;
    uint32_t res[PER][kT][L];
    int dsts[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int it = threadIdx.x + q * kThreads;
      dsts[q] = -1;
      if (it < NE * TPE) {
        const int el = it / TPE, tg = it % TPE, k0 = tg * kT;
        const uint32_t* ys = sb + el * ES;
        ring_mul_rows<MM, L>(sa + el * ES, [&](int j, uint32_t(&y)[L]) { ld_res<L>(y, ys + j * L); }, k0, mc,
                             res[q]);
        if (A.mode == 2) {
          uint32_t r2[L];
#pragma unroll
          for (int w = 0; w < L; ++w) r2[w] = mc.r2[w];
#pragma unroll
          for (int t = 0; t < kT; ++t) mont_mul<L>(res[q][t], res[q][t], r2, mc);
        }
        const int slot = (el & ~bmask) | bitrev_n(el & bmask, A.logb);
        dsts[q] = slot * ES + k0 * L;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (dsts[q] >= 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) st_res<L>(sa + dsts[q] + t * L, res[q][t]);
      }
    __syncthreads();
    dft_inplace<MM, L, NE>(sa, A.logb, mc);
  }
  for (int it = threadIdx.x; it < NE * MM; it += kThreads) {
    const int el = it / MM, k = it % MM;
    if (e0 + el >= A.total_elems) continue;
    uint32_t v[L];
    ld_res<L>(v, sa + el * ES + k * L);
    if (A.scale) {
      uint32_t ks[L];
#pragma unroll
      for (int q = 0; q < L; ++q) ks[q] = mc.kscale[q];
      mont_mul<L>(v, v, ks, mc);
    }
    st_res<L>(A.a + (e0 + el) * (MM * L) + k * L, v);
  }
}

// standalone batched ring product (stage API r_mul / pointwise): out = x*y (exact)
template <int MM, int L>
__global__ void __launch_bounds__(kThreads) k_rmul(const uint32_t* __restrict__ x, const uint32_t* __restrict__ y,
                                                   uint32_t* out, long long count, ModCtx mc) {
  constexpr int ES = Smem<MM, L>::ES;
  constexpr int NE = Cfg<MM>::NE;
  constexpr int TPE = MM / kT;
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sx = smem;
  uint32_t* sy = smem + NE * ES;
  const long long e0 = (long long)blockIdx.x * NE;
  constexpr int V4 = MM * L / 4;
  for (int it = threadIdx.x; it < NE * V4; it += kThreads) {
    const int el = it / V4, w4 = it % V4;
    if (e0 + el < count) {
      const long long off = (e0 + el) * (MM * L) + w4 * 4;
      *reinterpret_cast<uint4*>(sx + el * ES + w4 * 4) = *reinterpret_cast<const uint4*>(x + off);
      *reinterpret_cast<uint4*>(sy + el * ES + w4 * 4) = *reinterpret_cast<const uint4*>(y + off);
    }
  }
  __syncthreads();
  for (int it = threadIdx.x; it < NE * TPE; it += kThreads) {
    const int el = it / TPE, tg = it % TPE, k0 = tg * kT;
    if (e0 + el >= count) continue;
    const uint32_t* ys = sy + el * ES;
    uint32_t w[kT][L];
    ring_mul_rows<MM, L>(sx + el * ES, [&](int j, uint32_t(&yy)[L]) { ld_res<L>(yy, ys + j * L); }, k0, mc, w);
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
constexpr int kDecThreads = 1024;

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
};

__device__ __forceinline__ unsigned long long window_sum(const DecodeArgs& A, const uint32_t* v, long long t) {
  if (t < 0) return 0ull;
  const long long twoM = 2LL * A.M;
  const int half = A.MM / 2;
  const long long wbits = 32LL * A.L;
  long long s_lo = (32 * t - wbits) / A.u + 1;
  if (32 * t - wbits < 0) s_lo = 0;
  const long long s_hi = (32 * t + 31) / A.u;
  unsigned long long S = 0;
  for (long long s = s_lo; s <= s_hi; ++s) {
    const long long off = 32 * t - (long long)A.u * s;  // bit offset of window inside coefficient
    const long long lq = s / half;
    for (int h = 0; h < 2; ++h) {
      const long long l = lq - h;
      const long long k = s - l * half;
      if (l < 0 || l >= twoM || k < 0 || k >= A.MM) continue;
      const long long src = (twoM - l) & (twoM - 1);
      const uint32_t* c = v + (src * A.MM + k) * A.L;
      uint32_t word;
      if (off >= 0) {
        const int q = (int)(off >> 5), sh = (int)(off & 31);
        const uint32_t lo = q < A.L ? c[q] : 0u, hi = q + 1 < A.L ? c[q + 1] : 0u;
        word = sh ? __funnelshift_r(lo, hi, sh) : lo;
      } else {
        word = c[0] << (int)(-off);
      }
      S += word;
    }
  }
  return S;
}

__global__ void __launch_bounds__(kDecThreads) k_decode1(DecodeArgs A) {
  const int pidx = blockIdx.x / A.blocks_per_poly;
  const int blk = blockIdx.x % A.blocks_per_poly;
  const long long t = (long long)blk * kDecThreads + threadIdx.x;
  const uint32_t* v = A.v + (long long)pidx * A.poly_words;
  __shared__ unsigned long long sS[kDecThreads + 1];
  __shared__ uint32_t wg[32], wp[32];
  unsigned long long S = t < A.nout ? window_sum(A, v, t) : 0ull;
  sS[threadIdx.x + 1] = S;
  if (threadIdx.x == 0) sS[0] = (t < A.nout && t > 0) ? window_sum(A, v, t - 1) : 0ull;
  __syncthreads();
  unsigned long long w = (S & 0xFFFFFFFFull) + (sS[threadIdx.x] >> 32);
  if (t >= A.nout) w = 0;
  const bool g = w >> 32;
  const bool p = (uint32_t)w == 0xFFFFFFFFu && !g;
  const unsigned G = __ballot_sync(0xFFFFFFFFu, g), P = __ballot_sync(0xFFFFFFFFu, p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (t < A.nout) A.out[(long long)pidx * A.nout + t] = (uint32_t)w;
  if (lane == 0) {
    const long long wi = ((long long)pidx * A.blocks_per_poly + blk) * 32 + warp;
    A.gmask[wi] = G;
    A.pmask[wi] = P;
    // warp carry-out for cin = 0 / 1
    const unsigned long long a = (unsigned long long)(G | P), b = G;
    wg[warp] = (unsigned)((a + b) >> 32);
    wp[warp] = (unsigned)((a + b + 1) >> 32);
  }
  __syncthreads();
  if (warp == 0) {
    const bool c0 = wg[lane], c1 = wp[lane];
    const unsigned WG = __ballot_sync(0xFFFFFFFFu, c0), WP = __ballot_sync(0xFFFFFFFFu, c1 && !c0);
    if (lane == 0) {
      const unsigned long long a = (unsigned long long)(WG | WP), b = WG;
      const unsigned co0 = (unsigned)((a + b) >> 32), co1 = (unsigned)((a + b + 1) >> 32);
      A.bstat[(long long)pidx * A.blocks_per_poly + blk] = co0 | (co1 << 1);
    }
  }
}

__global__ void __launch_bounds__(kDecThreads) k_decode2(DecodeArgs A) {
  const int pidx = blockIdx.x / A.blocks_per_poly;
  const int blk = blockIdx.x % A.blocks_per_poly;
  const long long t = (long long)blk * kDecThreads + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ unsigned s_cin_block;
  __shared__ unsigned s_wcin[32];
  if (warp == 0) {
    // carry into this block: scan the statuses of blocks 0..blk-1 of this poly
    unsigned cin = 0;
    const uint32_t* st = A.bstat + (long long)pidx * A.blocks_per_poly;
    for (int base = 0; base < blk; base += 32) {
      const int bi = base + lane;
      const unsigned sv = bi < blk ? st[bi] : 0u;
      const bool c0 = sv & 1u, c1 = (sv >> 1) & 1u;
      const unsigned G = __ballot_sync(0xFFFFFFFFu, bi < blk && c0);
      const unsigned P = __ballot_sync(0xFFFFFFFFu, bi < blk && c1 && !c0);
      const int n = min(32, blk - base);
      const unsigned long long a = (unsigned long long)(G | P), b = G;
      const unsigned long long sum = a + b + cin;
      cin = (unsigned)((sum >> n) & 1ull);
    }
    // carries into each warp of this block
    const long long wi = ((long long)pidx * A.blocks_per_poly + blk) * 32 + lane;
    const unsigned G = A.gmask[wi], P = A.pmask[wi];
    const unsigned long long a = (unsigned long long)(G | P), b = G;
    const bool c0 = (unsigned)((a + b) >> 32), c1 = (unsigned)((a + b + 1) >> 32);
    const unsigned WG = __ballot_sync(0xFFFFFFFFu, c0), WP = __ballot_sync(0xFFFFFFFFu, c1 && !c0);
    const unsigned long long wa = (unsigned long long)(WG | WP), wb = WG;
    const unsigned long long carries = (wa + wb + cin) ^ wa ^ wb;  // bit i = carry into warp i
    s_wcin[lane] = (unsigned)((carries >> lane) & 1ull);
    if (lane == 0) s_cin_block = cin;
  }
  __syncthreads();
  if (t >= A.nout) return;
  const long long wi = ((long long)pidx * A.blocks_per_poly + blk) * 32 + warp;
  const unsigned G = A.gmask[wi], P = A.pmask[wi];
  const unsigned long long a = (unsigned long long)(G | P), b = G;
  const unsigned long long carries = (a + b + s_wcin[warp]) ^ a ^ b;
  const unsigned c = (unsigned)((carries >> lane) & 1ull);
  A.out[(long long)pidx * A.nout + t] += c;
}

#endif  // DKSS_COMMON_KERNELS

}  // namespace dkss
