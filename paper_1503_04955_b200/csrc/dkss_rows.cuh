// dkss_rows.cuh -- the row phase of a two-level transform in one cluster kernel.
//
// With E = 2m, a plan whose transform length is 2M = E^2 * b (two column levels and a
// base case of length b) splits every polynomial into E rows of mu0 = E*b elements after
// the first column level.  Everything that follows -- the second forward level of a and b
// (bigmul/dkss.py:471-495 one recursion down), the base-case DFTs and the pointwise ring
// products (:458-463, :544-545), and the second level of the inverse -- stays inside one
// row.  k_rows gives each (a-row, b-row) pair a thread-block cluster of CS = b CTAs, one
// second-level column per CTA, kept in shared memory from the first load to the last
// store: the base-case groups (one element from every column) are gathered through
// distributed shared memory, and the product is scattered back the same way.  This
// replaces three launches (forward level 1, bottom, inverse level 1) and their global
// round trips; it is the on-chip form of the four-step split of fourstep.py.
#pragma once
#include <cooperative_groups.h>

#include "dkss_kernels.cuh"

namespace dkss {

struct RowsArgs {
  uint32_t* a;           // a polynomials (product rows are written back here)
  const uint32_t* b;     // b polynomials (== a for squaring)
  long long poly_words;  // 2M * MM * L
  long long rows;        // row pairs in the launch (pairs * E)
  int log_top_mu;        // log2(M/m): twiddle split
  const uint32_t* twr;   // twiddle rows (see PassArgs)
};

template <int MM, int L>
struct RowsSmem {
  using S = Smem<MM, L>;
  static constexpr int E = 2 * MM;
  static constexpr int BUF = E * S::ES;                        // one column / one group set
  static constexpr int TW = Cfg<MM>::TWS ? E * S::EST : 0;     // staged twiddle rows
  static constexpr int WORDS = 5 * BUF + TW;                   // A, B, T, X0, X1 + twiddles
};

template <int MM, int L, int CS>
__global__ void __launch_bounds__(Cfg<MM>::NT, Cfg<MM>::MINB) k_rows(RowsArgs R, ModCtx mc) {
  namespace cg = cooperative_groups;
  griddep_launch();
  constexpr int kT = Cfg<MM>::T, NT = Cfg<MM>::NT;
  constexpr int ES = Smem<MM, L>::ES, EST = Smem<MM, L>::EST;
  constexpr int E = 2 * MM, LOGE = Geo<MM>::LOGE, TPE = MM / kT;
  constexpr int PER = (E * TPE + NT - 1) / NT;
  constexpr int LOGB = CS == 2 ? 1 : CS == 4 ? 2 : CS == 8 ? 3 : 4;
  constexpr int GP = E / CS;  // base-case groups per CTA
  constexpr uint32_t EB = MM * L * 4, TB = 2 * MM * L * 4;
  constexpr int BUF = RowsSmem<MM, L>::BUF;
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sA = smem;            // a column (TMA), later: gathered a groups
  uint32_t* sB = smem + BUF;      // b column (TMA), later: gathered b groups
  uint32_t* sT = smem + 2 * BUF;  // DFT ping-pong
  uint32_t* x0 = smem + 3 * BUF;  // a after the forward level (read by the cluster)
  uint32_t* x1 = smem + 4 * BUF;  // b after the forward level, later: product column
  uint32_t* tws = smem + 5 * BUF;
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();  // second-level column l1 of this CTA
  const long long row = blockIdx.x / CS;
  const long long q = row / E, j0 = row % E;
  const long long mu0 = (long long)E * CS, EW = MM * L;
  uint32_t* arow = R.a + q * R.poly_words + j0 * mu0 * EW;
  const uint32_t* brow = R.b + q * R.poly_words + j0 * mu0 * EW;
  PassArgs A{};  // twiddle exponents of level 1: s = j * l1 * E mod (M/m)
  A.base_pow = E;
  A.log_top_mu = R.log_top_mu;
  A.twr = R.twr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  // twiddle rows (independent of the previous kernel), then the two columns
  if (warp == 0) {
    uint32_t twb = 0;
    if constexpr (Cfg<MM>::TWS) {
      for (int v = lane; v < E; v += 32) {
        int r;
        if (tw_exp(A, v, c, &r)) twb += TB;
      }
      twb = __reduce_add_sync(0xFFFFFFFFu, twb);
    }
    if (lane == 0) {
      mbar_expect_tx(&bar[0], E * EB + twb);
      mbar_expect_tx(&bar[1], E * EB);
    }
    __syncwarp();
  }
  __syncthreads();
  if constexpr (Cfg<MM>::TWS) {
    for (int v = threadIdx.x; v < E; v += NT) {
      int r;
      const long long s = tw_exp(A, v, c, &r);
      if (s) bulk_g2s(tws + v * EST, R.twr + s * (2 * MM * L), TB, &bar[0]);
    }
  }
  griddep_wait();
  for (int i = threadIdx.x; i < 2 * E; i += NT) {
    const int j = i % E;
    const long long pos = (long long)j * CS + c;
    if (i < E)
      bulk_g2s(sA + bitrev_n(j, LOGE) * ES, arow + pos * EW, EB, &bar[0]);
    else
      bulk_g2s(sB + bitrev_n(j, LOGE) * ES, brow + pos * EW, EB, &bar[1]);
  }
  // ---- forward level 1 of a, then b: column DFT + twiddle, results kept in x0 / x1
  for (int pl = 0; pl < 2; ++pl) {
    mbar_wait(&bar[pl], 0);
    uint32_t* in = pl ? sB : sA;
    const uint32_t* xv = dft_pingpong<MM, L, E>(in, sT, LOGE, mc);
    uint32_t* dstc = pl ? x1 : x0;
    for (int it = threadIdx.x; it < E * TPE; it += NT) {
      const int vv = it / TPE, k0 = (it % TPE) * kT;
      int r;
      const long long s = tw_exp(A, vv, c, &r);
      uint32_t w[kT][L];
      if (s == 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(w[t], xv + vv * ES + (k0 + t) * L);
      } else {
        twiddle_mul<MM, L, kT>(A, xv + vv * ES, tws + vv * EST, s, k0, mc, w);
      }
      store_rot<MM, L, kT>(dstc + vv * ES, w, k0, r, mc);
    }
    __syncthreads();
  }
  // ---- gather the base-case groups of this CTA: group g = element g of every column
  cl.sync();
  {
    constexpr int N4 = MM * L / 4;
    for (int it = threadIdx.x; it < 2 * GP * CS * N4; it += NT) {
      const int part = it % N4, rest = it / N4;
      const int pl = rest / (GP * CS), el = rest % (GP * CS);
      const int gl = el / CS, e = el % CS;
      const int g = c * GP + gl;
      const uint32_t* src = cl.map_shared_rank(pl ? x1 : x0, e) + g * ES;
      uint32_t* dst = (pl ? sB : sA) + (gl * CS + bitrev_n(e, LOGB)) * ES;
      reinterpret_cast<uint4*>(dst)[part] = reinterpret_cast<const uint4*>(src)[part];
    }
  }
  cl.sync();  // every peer has its groups: x0 / x1 are free
  // ---- base case: DFT(a), DFT(b), pointwise b * a, DFT (k_bottom, mode 1)
  uint32_t* out;
  {
    uint32_t* ra = dft_pingpong<MM, L, E>(sA, sT, LOGB, mc);
    uint32_t* rb = dft_pingpong<MM, L, E>(sB, ra == sA ? sT : sA, LOGB, mc);
    __syncthreads();
    uint32_t res[PER][kT][L];
    int dsts[PER];
#pragma unroll
    for (int qq = 0; qq < PER; ++qq) {
      const int it = threadIdx.x + qq * NT;
      dsts[qq] = -1;
      if (it < E * TPE) {
        const int el = it / TPE, k0 = (it % TPE) * kT;
        ring_mul<MM, L>(ResS<L>{rb + el * ES}, ResS<L>{ra + el * ES}, BiasFromY{}, k0, mc, res[qq]);
        const int slot = (el & ~(CS - 1)) | bitrev_n(el & (CS - 1), LOGB);
        dsts[qq] = slot * ES + k0 * L;
      }
    }
    __syncthreads();
#pragma unroll
    for (int qq = 0; qq < PER; ++qq)
      if (dsts[qq] >= 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) st_res<L>(ra + dsts[qq] + t * L, res[qq][t]);
      }
    __syncthreads();
    out = dft_pingpong<MM, L, E>(ra, rb, LOGB, mc);
  }
  // ---- scatter the product back to the column owners: element (g, e) -> CTA e, x1[g]
  {
    constexpr int N4 = MM * L / 4;
    for (int it = threadIdx.x; it < GP * CS * N4; it += NT) {
      const int part = it % N4, el = it / N4;
      const int gl = el / CS, e = el % CS;
      uint32_t* dst = cl.map_shared_rank(x1, e) + (c * GP + gl) * ES;
      reinterpret_cast<uint4*>(dst)[part] = reinterpret_cast<const uint4*>(out + el * ES)[part];
    }
  }
  cl.sync();
  // ---- inverse level 1 of the product column: twiddle, then DFT; write the row back
  {
    uint32_t res[PER][kT][L];
    int dsl[PER], rot[PER];
#pragma unroll
    for (int qq = 0; qq < PER; ++qq) {
      const int it = threadIdx.x + qq * NT;
      dsl[qq] = -1;
      if (it >= E * TPE) continue;
      const int j = it / TPE, k0 = (it % TPE) * kT;
      const long long s = tw_exp(A, j, c, &rot[qq]);
      if (s == 0) {
#pragma unroll
        for (int t = 0; t < kT; ++t) ld_res<L>(res[qq][t], x1 + j * ES + (k0 + t) * L);
      } else {
        twiddle_mul<MM, L, kT>(A, x1 + j * ES, tws + j * EST, s, k0, mc, res[qq]);
      }
      dsl[qq] = bitrev_n(j, LOGE) * ES;
    }
    __syncthreads();
#pragma unroll
    for (int qq = 0; qq < PER; ++qq)
      if (dsl[qq] >= 0) store_rot<MM, L, kT>(sA + dsl[qq], res[qq], ((threadIdx.x + qq * NT) % TPE) * kT, rot[qq], mc);
    __syncthreads();
    const uint32_t* ov = dft_pingpong<MM, L, E>(sA, sT, LOGE, mc);
    for (int it = threadIdx.x; it < E * MM; it += NT) {
      const int vv = it / MM, kk = it % MM;
      uint32_t v[L];
      ld_res<L>(v, ov + vv * ES + kk * L);
      st_res<L>(arow + ((long long)vv * CS + c) * EW + kk * L, v);
    }
  }
}

}  // namespace dkss
