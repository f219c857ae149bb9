// dkss_warp.cuh -- warp-per-column transform passes for m = 8 / 16.
//
// The CTA-wide column DFT of dkss_kernels.cuh needs a block barrier per radix-2 stage and
// leaves the IMAD pipe idle while it runs.  Here one warp owns a whole 2m-element column:
// lane = (element group g, coefficient c), each lane holds coefficient c of EPT = 2m/G
// consecutive slots in registers, and the length-2m DFT over R (root alpha) runs entirely in
// registers -- the alpha^e rotations are __shfl_sync from lane (g, (c - e) mod m), the
// negation of wrapped coefficients swaps the butterfly outputs.  No block barriers: a warp
// loads its column with TMA (per-warp mbarrier), transforms it, writes it back to its own
// shared-memory slice and runs the column's twiddle ring products (ring_mul) itself.
// `wpc` warps may share a column at small sizes (each redoes the cheap DFT and takes every
// wpc-th element's products) so that enough warps issue IMADs.
#pragma once
#include "dkss_kernels.cuh"

namespace dkss {

constexpr int kWarpsPerCta = 4;
// resident CTAs per SM the warp-per-column kernels are register-capped for: the forward
// kernel (one column slice per warp) fits 4 per SM, the inverse (two slices) 3
#ifndef DKSS_WARP_MINB_FWD
#define DKSS_WARP_MINB_FWD 4
#endif
#ifndef DKSS_WARP_MINB_INV
#define DKSS_WARP_MINB_INV 3
#endif

template <int MM>
struct WG {
  static constexpr int E = 2 * MM, G = 32 / MM, EPT = E / G, LOGE = Geo<MM>::LOGE;
};

// in-register length-2MM DIT DFT: X[i] holds coefficient c = lane % MM of slot g*EPT + i
// (g = lane / MM); input slots are in bit-reversed order, output slots in natural order.
// Butterfly root for block size `size` is alpha^(kk * 2MM/size) as in dft_pingpong.
template <int MM, int L>
__device__ __forceinline__ void warp_dft(uint32_t (&X)[WG<MM>::EPT][L], const ModCtx& mc) {
  constexpr int EPT = WG<MM>::EPT, LOGE = WG<MM>::LOGE;
  const int lane = threadIdx.x & 31, c = lane & (MM - 1), g = lane / MM;
#pragma unroll
  for (int ls = 1; ls <= LOGE; ++ls) {
    const int half = 1 << (ls - 1);
    const int rootstep = (2 * MM) >> ls;
    if (half < EPT) {
      // both slots of every butterfly live in this thread: i and i + half
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        if (i & half) continue;
        const int kk = i & (half - 1);
        const int e = kk * rootstep;  // static
        uint32_t xb[L], s[L], d[L];
        bool neg = false;
        if (e == 0) {
#pragma unroll
          for (int q = 0; q < L; ++q) xb[q] = X[i + half][q];
        } else {
          const int src = g * MM + ((c - e) & (MM - 1));
#pragma unroll
          for (int q = 0; q < L; ++q) xb[q] = __shfl_sync(0xFFFFFFFFu, X[i + half][q], src);
          neg = c < e;
        }
        add_mod<L>(s, X[i], xb, mc);
        sub_mod<L>(d, X[i], xb, mc);
#pragma unroll
        for (int q = 0; q < L; ++q) {
          X[i][q] = neg ? d[q] : s[q];
          X[i + half][q] = neg ? s[q] : d[q];
        }
      }
    } else {
      // partner slot sits in group g ^ D: lower group keeps the sum, upper the difference
      const int D = half / EPT;
      const bool lower = (g & D) == 0;
      const int glo = g & ~D, ghi = g | D;
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int kk = (glo * EPT + i) & (half - 1);
        const int e = kk * rootstep;
        const int usrc = glo * MM + c;
        const int xsrc = ghi * MM + ((c - e) & (MM - 1));
        uint32_t u[L], xb[L], s[L], d[L];
#pragma unroll
        for (int q = 0; q < L; ++q) {
          u[q] = __shfl_sync(0xFFFFFFFFu, X[i][q], usrc);
          xb[q] = __shfl_sync(0xFFFFFFFFu, X[i][q], xsrc);
        }
        const bool neg = c < e;
        add_mod<L>(s, u, xb, mc);
        sub_mod<L>(d, u, xb, mc);
        const bool take_s = lower != neg;
#pragma unroll
        for (int q = 0; q < L; ++q) X[i][q] = take_s ? s[q] : d[q];
      }
    }
  }
}

// lane 0..31: TMA-load the 2MM elements of column cg into buf (FWD: bit-reversed slots)
template <int MM, int L, bool FWD>
__device__ __forceinline__ void warp_issue_column(const PassArgs& A, long long cg, uint64_t* bar, uint32_t* buf) {
  constexpr int ES = Smem<MM, L>::ES, E = 2 * MM, LOGE = Geo<MM>::LOGE;
  constexpr uint32_t EB = MM * L * 4;
  const int lane = threadIdx.x & 31;
  if (lane == 0) mbar_expect_tx(bar, E * EB);
  __syncwarp();
  for (int j = lane; j < E; j += 32) {
    long long l;
    const long long off = col_elem(A, cg, j, LOGE, MM * L, &l);
    bulk_g2s(buf + (FWD ? bitrev_n(j, LOGE) : j) * ES, A.poly + off, EB, bar);
  }
}

// fused encode of one coefficient (see cta_encode_tile)
template <int MM, int L>
__device__ __forceinline__ void encode_coef(const PassArgs& A, long long cg, int j, int k, uint32_t (&out)[L]) {
  constexpr int HALF = MM / 2, LOGE = Geo<MM>::LOGE;
#pragma unroll
  for (int q = 0; q < L; ++q) out[q] = 0;
  if (k >= HALF) return;
  const long long qp = cg >> A.log_cpp, cc = cg & ((1LL << A.log_cpp) - 1);
  const long long inst = cc >> A.log_mu, l = cc & ((1LL << A.log_mu) - 1);
  const long long pos = (inst << (A.log_mu_enc + LOGE)) + ((long long)j << A.log_mu_enc) + l + A.l_off;
  if (pos >= A.M) return;
  const uint32_t* op = qp < A.enc_split ? A.ops_a + qp * A.na : A.ops_b + (qp - A.enc_split) * A.na;
  const long long bit = (long long)A.u * (pos * HALF + k);
  const long long w0 = bit >> 5;
  const int sh = (int)(bit & 31);
  uint32_t src[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) src[w] = (w0 + w < A.na) ? __ldg(op + w0 + w) : 0u;
  int rem = A.u;
#pragma unroll
  for (int w = 0; w < 3 && w < L; ++w) {
    const uint32_t v = sh ? __funnelshift_r(src[w], src[w + 1], sh) : src[w];
    out[w] = rem >= 32 ? v : (rem > 0 ? v & ((1u << rem) - 1u) : 0u);
    rem -= 32;
  }
}

// forward column pass, warp per column (A.wpc warps per column)
template <int MM, int L>
__global__ void __launch_bounds__(kWarpsPerCta * 32, DKSS_WARP_MINB_FWD) k_fwd_warp(PassArgs A, ModCtx mc) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  constexpr int kT = Cfg<MM>::T;
  constexpr int ES = Smem<MM, L>::ES, E = 2 * MM, EPT = WG<MM>::EPT, TPE = MM / kT;
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ __align__(8) uint64_t bars[kWarpsPerCta];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = lane & (MM - 1), g = lane / MM;
  uint32_t* buf = smem + warp * E * ES;
  uint64_t* bar = &bars[warp];
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  const long long gw = (long long)blockIdx.x * kWarpsPerCta + warp;
  const long long nw = (long long)gridDim.x * kWarpsPerCta;
  const int wpc = A.wpc, part = (int)(gw % wpc);
  const bool enc = A.ops_a != nullptr;
  uint32_t phase = 0;
  for (long long cg = gw / wpc; cg < A.total_cols; cg += nw / wpc) {
    uint32_t X[EPT][L];
    if (enc) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) encode_coef<MM, L>(A, cg, bitrev_n(g * EPT + i, WG<MM>::LOGE), c, X[i]);
    } else {
      warp_issue_column<MM, L, true>(A, cg, bar, buf);
      mbar_wait(bar, phase);
      phase ^= 1;
#pragma unroll
      for (int i = 0; i < EPT; ++i) ld_res<L>(X[i], buf + (g * EPT + i) * ES + c * L);
    }
    warp_dft<MM, L>(X, mc);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < EPT; ++i) st_res<L>(buf + (g * EPT + i) * ES + c * L, X[i]);
    __syncwarp();
    long long l;
    col_elem(A, cg, 0, Geo<MM>::LOGE, 0, &l);
    // elements vv = part, part + wpc, ...: (E / wpc) * TPE work items over 32 lanes
    const int nitems = (E / wpc) * TPE;
    for (int it = lane; it < nitems; it += 32) {
      const int vv = (it / TPE) * wpc + part, k0 = (it % TPE) * kT;
      uint32_t* dst = A.poly + col_elem(A, cg, vv, Geo<MM>::LOGE, MM * L, &l);
      int r;
      const long long s = tw_exp(A, vv, l, &r);
      uint32_t w[kT][L];
      if (s == 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(w[t], buf + vv * ES + (k0 + t) * L);
      } else {
        const uint32_t* row = A.twr + s * (2 * MM * L);
        ring_mul<MM, L>(ResG<L>{row}, ResS<L>{buf + vv * ES}, ResG<L>{row + MM * L}, k0, mc, w);
      }
      store_rot<MM, L, kT>(dst, w, k0, r, mc);
    }
    fence_proxy_async();
    __syncwarp();
  }
}

// inverse (transposed) column pass, warp per column: twiddle products into a result slice at
// bit-reversed slots, then the register DFT, then the store (optionally scaled by kscale)
template <int MM, int L>
__global__ void __launch_bounds__(kWarpsPerCta * 32, DKSS_WARP_MINB_INV) k_inv_warp(PassArgs A, ModCtx mc) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  constexpr int kT = Cfg<MM>::T;
  constexpr int ES = Smem<MM, L>::ES, E = 2 * MM, EPT = WG<MM>::EPT, TPE = MM / kT, LOGE = Geo<MM>::LOGE;
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ __align__(8) uint64_t bars[kWarpsPerCta];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = lane & (MM - 1), g = lane / MM;
  uint32_t* buf = smem + warp * 2 * E * ES;
  uint32_t* res = buf + E * ES;
  uint64_t* bar = &bars[warp];
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  const long long gw = (long long)blockIdx.x * kWarpsPerCta + warp;
  const long long nw = (long long)gridDim.x * kWarpsPerCta;
  uint32_t phase = 0;
  long long cg = gw;
  if (cg < A.total_cols) warp_issue_column<MM, L, false>(A, cg, bar, buf);
  for (; cg < A.total_cols; cg += nw) {
    mbar_wait(bar, phase);
    phase ^= 1;
    long long l;
    col_elem(A, cg, 0, LOGE, 0, &l);
    for (int it = lane; it < E * TPE; it += 32) {
      const int j = it / TPE, k0 = (it % TPE) * kT;
      int r;
      const long long s = tw_exp(A, j, l, &r);
      uint32_t w[kT][L];
      if (s == 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(w[t], buf + j * ES + (k0 + t) * L);
      } else {
        const uint32_t* row = A.twr + s * (2 * MM * L);
        ring_mul<MM, L>(ResG<L>{row}, ResS<L>{buf + j * ES}, ResG<L>{row + MM * L}, k0, mc, w);
      }
      store_rot<MM, L, kT>(res + bitrev_n(j, LOGE) * ES, w, k0, r, mc);
    }
    fence_proxy_async();
    __syncwarp();
    // the input slice is free: prefetch the next column while this one is transformed
    if (cg + nw < A.total_cols) warp_issue_column<MM, L, false>(A, cg + nw, bar, buf);
    uint32_t X[EPT][L];
#pragma unroll
    for (int i = 0; i < EPT; ++i) ld_res<L>(X[i], res + (g * EPT + i) * ES + c * L);
    warp_dft<MM, L>(X, mc);
    uint32_t ks[L];
#pragma unroll
    for (int q = 0; q < L; ++q) ks[q] = mc.kscale[q];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      if (A.scale) mont_mul<L>(X[i], X[i], ks, mc);
      st_res<L>(A.poly + col_elem(A, cg, g * EPT + i, LOGE, MM * L, &l) + c * L, X[i]);
    }
    __syncwarp();
  }
}

}  // namespace dkss

namespace dkss {

// ---------------------------------------------------------------------------
// Split passes: column DFT kernel + elementwise twiddle kernel.
//
// k_dft_cols: one warp per 2m-element column (m <= 16), register DFT, in place.  Input
// slots are read in bit-reversed order (TMA into the warp's slice), output element vv is
// written back to position vv of the column.  Optional fused encode (first forward level)
// and (2M)^-1 scaling (last inverse level).
template <int MM, int L>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_dft_cols(PassArgs A, ModCtx mc) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  constexpr int ES = Smem<MM, L>::ES, E = 2 * MM, EPT = WG<MM>::EPT, LOGE = Geo<MM>::LOGE;
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ __align__(8) uint64_t bars[kWarpsPerCta];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = lane & (MM - 1), g = lane / MM;
  uint32_t* buf = smem + warp * E * ES;
  uint64_t* bar = &bars[warp];
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  const long long gw = (long long)blockIdx.x * kWarpsPerCta + warp;
  const long long nw = (long long)gridDim.x * kWarpsPerCta;
  const bool enc = A.ops_a != nullptr;
  uint32_t phase = 0;
  long long cg = gw;
  if (!enc && cg < A.total_cols) warp_issue_column<MM, L, true>(A, cg, bar, buf);
  uint32_t ks[L];
#pragma unroll
  for (int q = 0; q < L; ++q) ks[q] = mc.kscale[q];
  for (; cg < A.total_cols; cg += nw) {
    uint32_t X[EPT][L];
    if (enc) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) encode_coef<MM, L>(A, cg, bitrev_n(g * EPT + i, LOGE), c, X[i]);
    } else {
      mbar_wait(bar, phase);
      phase ^= 1;
#pragma unroll
      for (int i = 0; i < EPT; ++i) ld_res<L>(X[i], buf + (g * EPT + i) * ES + c * L);
      fence_proxy_async();
      __syncwarp();
      if (cg + nw < A.total_cols) warp_issue_column<MM, L, true>(A, cg + nw, bar, buf);
    }
    warp_dft<MM, L>(X, mc);
    long long l;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      if (A.scale) mont_mul<L>(X[i], X[i], ks, mc);
      st_res<L>(A.poly + col_elem(A, cg, g * EPT + i, LOGE, MM * L, &l) + c * L, X[i]);
    }
  }
}

// k_twiddle: elementwise twiddle ring products of one level, in place.  Work item = (element
// position (j, l) of a column, kT output coefficients); the MM/kT items of an element are
// adjacent lanes of one warp, so the element is read completely before any lane stores
// (warp-synchronous in-place update).  Exponent j*l*base_pow (bigmul/dkss.py:480-492);
// forward levels run it after k_dft_cols, inverse levels before.
template <int MM, int L>
__global__ void __launch_bounds__(256, 2) k_twiddle(PassArgs A, ModCtx mc) {
  griddep_wait();  // PDL: predecessor grid complete, its writes visible
  griddep_launch();
  constexpr int kT = Cfg<MM>::T, TPE = MM / kT, E = 2 * MM, LOGE = Geo<MM>::LOGE;
  static_assert(32 % TPE == 0, "an element's work items must share a warp");
  const long long total = A.total_cols * E * TPE;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // all lanes iterate the same number of times (warp-synchronous stores below)
  const long long iters = (total + stride - 1) / stride;
  long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long n = 0; n < iters; ++n, it += stride) {
    const bool live = it < total;
    const long long el = it / TPE;
    const int k0 = (int)(it % TPE) * kT;
    const long long cg = el / E;
    const int j = (int)(el % E);
    uint32_t w[kT][L];
    int r = 0;
    uint32_t* dst = nullptr;
    if (live) {
      long long l;
      dst = A.poly + col_elem(A, cg, j, LOGE, MM * L, &l);
      const long long s = tw_exp(A, j, l, &r);
      if (s == 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(w[t], dst + (k0 + t) * L);
      } else {
        const uint32_t* row = A.twr + s * (2 * MM * L);
        ring_mul<MM, L>(ResG<L>{row}, ResG<L>{dst}, ResG<L>{row + MM * L}, k0, mc, w);
      }
    }
    __syncwarp();
    if (live) store_rot<MM, L, kT>(dst, w, k0, r, mc);
  }
}

}  // namespace dkss
