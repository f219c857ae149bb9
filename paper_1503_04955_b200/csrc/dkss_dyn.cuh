// dkss_dyn.cuh -- the row phase of a two-level transform as one persistent kernel with
// dependency-driven work items.
//
// With E = 2m and 2M = E^2 * b, every polynomial has E rows of mu0 = E*b elements after the
// first column level, and everything up to the last inverse level stays inside a row
// (bigmul/dkss.py:493-495 one recursion down; :458-463 base case; :544-545 pointwise).  The
// three launches that walk the rows (second forward level, base case + pointwise, second
// inverse level) become one grid of persistent CTAs that take work items from a ticket
// counter, in row order:
//   F (pair, row, a|b, column): forward level-1 column DFT + twiddles,
//   B (pair, row, tile):        base DFTs of a and b, pointwise r_mul, base DFT (NE elements),
//   I (pair, row, column):      inverse level-1 twiddles + column DFT of the product.
// A B item waits until every F item of its row has finished, an I item until every B item of
// its row has (per-row completion counters).  Tickets are handed out in that order, so a CTA
// only ever waits on items already held by running CTAs.  What this buys over three launches:
// no launch boundaries (each one costs a start-up and a tail where SMs run out of tiles), and
// rows flow through the phases as soon as they are ready, so the SMs stay busy.
//
// Element data produced by other CTAs is read with ordinary loads after an acquire on the
// row counter; twiddle rows (written at plan creation) are staged with TMA.
#pragma once
#include "dkss_kernels.cuh"

namespace dkss {

struct DynArgs {
  uint32_t* a;             // a polynomials (products are written here)
  const uint32_t* b;       // b polynomials (== a when squaring)
  long long poly_words;    // 2M * MM * L
  int batch;               // pairs
  int rows_pp;             // rows per pair (E; E/G for a four-step row shard)
  int npolys_fwd;          // 1 (squaring) or 2 polynomials transformed per pair
  int log_mu0, log_mu1;    // row length, level-1 columns per row
  int log_top_mu;          // twiddle split (log2 M/m)
  int logb;                // base length
  const uint32_t* twr;     // twiddle rows
  unsigned* fwd_done;      // [batch * E]: F items finished per row
  unsigned* bot_done;      // [batch * E]: B items finished per row
  unsigned* ticket;        // next work item; ticket[1] counts exited CTAs
  unsigned n_f, n_b, n_i;  // items per phase
  unsigned rows;           // batch * E (counters to reset)
};

template <int MM, int L>
struct DynSmem {
  using S = Smem<MM, L>;
  static constexpr int NE = Cfg<MM>::NE;  // elements per item (one column = 2m for m >= 16)
  static constexpr int WORDS = 3 * NE * S::ES + (Cfg<MM>::TWS ? NE * S::EST : 0);
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// all threads: wait until *ctr >= target (thread 0 polls, the CTA then synchronises)
__device__ __forceinline__ void wait_count(const unsigned* ctr, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned ns = 32;
    while (ld_acquire_u32(ctr) < target) {
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
    }
  }
  __syncthreads();
}

// all threads: count one finished item of a row after the CTA's global stores
__device__ __forceinline__ void signal_done(unsigned* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
  }
}

// copy NE elements (data words) from global into padded shared slots, 16 bytes per access
template <int MM, int L, int NE, class SlotFn, class SrcFn>
__device__ __forceinline__ void load_elems(uint32_t* dst, SlotFn slot, SrcFn src) {
  constexpr int ES = Smem<MM, L>::ES, N4 = MM * L / 4, NT = Cfg<MM>::NT;
  for (int it = threadIdx.x; it < NE * N4; it += NT) {
    const int e = it / N4, part = it % N4;
    // L2 only (ld.global.cg): the data were written by other SMs during this kernel
    reinterpret_cast<uint4*>(dst + slot(e) * ES)[part] = __ldcg(reinterpret_cast<const uint4*>(src(e)) + part);
  }
}

template <int MM, int L>
__global__ void __launch_bounds__(Cfg<MM>::NT, Cfg<MM>::MINB) k_rows_dyn(DynArgs R, ModCtx mc) {
  griddep_launch();
  constexpr int kT = Cfg<MM>::T, NT = Cfg<MM>::NT, NE = Cfg<MM>::NE;
  constexpr int ES = Smem<MM, L>::ES, EST = Smem<MM, L>::EST;
  constexpr int E = 2 * MM, LOGE = Geo<MM>::LOGE, TPE = MM / kT;
  constexpr int PER = (NE * TPE + NT - 1) / NT;
  constexpr long long EW = MM * L;
  constexpr uint32_t TB = 2 * MM * L * 4;
  static_assert(NE == E, "one column per work item");
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* s0 = smem;
  uint32_t* s1 = smem + NE * ES;
  uint32_t* s2 = smem + 2 * NE * ES;
  uint32_t* tws = smem + 3 * NE * ES;
  __shared__ __align__(8) uint64_t bar;
  __shared__ unsigned s_item;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  const long long mu0 = 1LL << R.log_mu0, mu1 = 1LL << R.log_mu1;
  const int bmask = (1 << R.logb) - 1;
  const unsigned n_all = R.n_f + R.n_b + R.n_i;
  PassArgs A{};  // level-1 twiddle exponents: s = j * l * E mod (M/m)
  A.base_pow = E;
  A.log_top_mu = R.log_top_mu;
  A.twr = R.twr;
  uint32_t phase = 0;
  griddep_wait();  // the first column level (previous kernel) is complete
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(R.ticket, 1u);
    __syncthreads();
    const unsigned item = s_item;
    __syncthreads();
    if (item >= n_all) {
      // the last CTA out leaves the counters zeroed for the next launch (every other CTA has
      // stopped reading them: it took a ticket past the end)
      if (threadIdx.x == 0) s_item = atomicAdd(R.ticket + 1, 1u) == gridDim.x - 1;
      __syncthreads();
      if (s_item) {
        for (unsigned i = threadIdx.x; i < R.rows; i += NT) R.fwd_done[i] = R.bot_done[i] = 0u;
        if (threadIdx.x == 0) R.ticket[0] = R.ticket[1] = 0u;
      }
      break;
    }
    if (item < R.n_f) {
      // ---- F: forward level-1 column l of row (pair, row) of polynomial w
      const unsigned l = item & (unsigned)(mu1 - 1);
      const unsigned rest = item >> R.log_mu1;
      const unsigned w = rest % R.npolys_fwd, prow = rest / R.npolys_fwd;  // prow = pair * E + row
      const unsigned pair = prow / R.rows_pp, row = prow % R.rows_pp;
      uint32_t* poly = (w ? const_cast<uint32_t*>(R.b) : R.a) + pair * R.poly_words + row * mu0 * EW;
      // twiddle rows first (TMA, independent), then the column (plain loads)
      if constexpr (Cfg<MM>::TWS) {
        if (threadIdx.x == 0) {
          uint32_t bytes = 0;
          for (int v = 0; v < E; ++v) {
            int r;
            if (tw_exp(A, v, l, &r)) bytes += TB;
          }
          mbar_expect_tx(&bar, bytes);
        }
        __syncthreads();
        for (int v = threadIdx.x; v < E; v += NT) {
          int r;
          const long long s = tw_exp(A, v, l, &r);
          if (s) bulk_g2s(tws + v * EST, R.twr + s * (2 * MM * L), TB, &bar);
        }
      }
      load_elems<MM, L, NE>(s0, [](int j) { return bitrev_n(j, LOGE); },
                            [&](int j) { return poly + ((long long)j * mu1 + l) * EW; });
      if constexpr (Cfg<MM>::TWS) {
        mbar_wait(&bar, phase);
        phase ^= 1;
      }
      __syncthreads();
      const uint32_t* xv = dft_pingpong<MM, L, NE>(s0, s1, LOGE, mc);
      for (int it = threadIdx.x; it < NE * TPE; it += NT) {
        const int vv = it / TPE, k0 = (it % TPE) * kT;
        int r;
        const long long s = tw_exp(A, vv, l, &r);
        uint32_t wv[kT][L];
        if (s == 0) {
#pragma unroll
          for (int t = 0; t < kT; ++t) ld_res<L>(wv[t], xv + vv * ES + (k0 + t) * L);
        } else {
          twiddle_mul<MM, L, kT>(A, xv + vv * ES, tws + vv * EST, s, k0, mc, wv);
        }
        store_rot<MM, L, kT>(poly + ((long long)vv * mu1 + l) * EW, wv, k0, r, mc);
      }
      fence_proxy_async();
      signal_done(R.fwd_done + prow);
    } else if (item < R.n_f + R.n_b) {
      // ---- B: base case + pointwise products of NE contiguous elements of a row
      const unsigned bi = item - R.n_f;
      const unsigned tpr = (unsigned)(mu0 / NE);  // tiles per row
      const unsigned prow = bi / tpr, t = bi % tpr;
      const unsigned pair = prow / R.rows_pp, row = prow % R.rows_pp;
      wait_count(R.fwd_done + prow, (unsigned)(R.npolys_fwd * mu1));
      const long long base = pair * R.poly_words + (row * mu0 + (long long)t * NE) * EW;
      uint32_t* pa = R.a + base;
      const uint32_t* pb = R.b + base;
      auto slot = [&](int el) { return (el & ~bmask) | bitrev_n(el & bmask, R.logb); };
      load_elems<MM, L, NE>(s0, slot, [&](int el) { return pa + el * EW; });
      load_elems<MM, L, NE>(s1, slot, [&](int el) { return pb + el * EW; });
      __syncthreads();
      uint32_t* ra = dft_pingpong<MM, L, NE>(s0, s2, R.logb, mc);
      uint32_t* rb = dft_pingpong<MM, L, NE>(s1, ra == s0 ? s2 : s0, R.logb, mc);
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
          dsts[q] = slot(el) * ES + k0 * L;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < PER; ++q)
        if (dsts[q] >= 0) {
#pragma unroll
          for (int tt = 0; tt < kT; ++tt) st_res<L>(ra + dsts[q] + tt * L, res[q][tt]);
        }
      __syncthreads();
      const uint32_t* out = dft_pingpong<MM, L, NE>(ra, rb, R.logb, mc);
      for (int it = threadIdx.x; it < NE * MM; it += NT) {
        const int el = it / MM, kk = it % MM;
        uint32_t v[L];
        ld_res<L>(v, out + el * ES + kk * L);
        st_res<L>(pa + el * EW + kk * L, v);
      }
      signal_done(R.bot_done + prow);
    } else {
      // ---- I: inverse level-1 column l of the product row: twiddles, then the column DFT
      const unsigned ii = item - R.n_f - R.n_b;
      const unsigned l = ii & (unsigned)(mu1 - 1), prow = ii >> R.log_mu1;
      const unsigned pair = prow / R.rows_pp, row = prow % R.rows_pp;
      uint32_t* poly = R.a + pair * R.poly_words + row * mu0 * EW;
      if constexpr (Cfg<MM>::TWS) {
        if (threadIdx.x == 0) {
          uint32_t bytes = 0;
          for (int v = 0; v < E; ++v) {
            int r;
            if (tw_exp(A, v, l, &r)) bytes += TB;
          }
          mbar_expect_tx(&bar, bytes);
        }
        __syncthreads();
        for (int v = threadIdx.x; v < E; v += NT) {
          int r;
          const long long s = tw_exp(A, v, l, &r);
          if (s) bulk_g2s(tws + v * EST, R.twr + s * (2 * MM * L), TB, &bar);
        }
      }
      wait_count(R.bot_done + prow, (unsigned)(mu0 / NE));
      load_elems<MM, L, NE>(s0, [](int j) { return j; }, [&](int j) { return poly + ((long long)j * mu1 + l) * EW; });
      if constexpr (Cfg<MM>::TWS) {
        mbar_wait(&bar, phase);
        phase ^= 1;
      }
      __syncthreads();
      uint32_t res[PER][kT][L];
      int dsl[PER], rot[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int it = threadIdx.x + q * NT;
        dsl[q] = -1;
        if (it >= NE * TPE) continue;
        const int j = it / TPE, k0 = (it % TPE) * kT;
        const long long s = tw_exp(A, j, l, &rot[q]);
        if (s == 0) {
#pragma unroll
          for (int tt = 0; tt < kT; ++tt) ld_res<L>(res[q][tt], s0 + j * ES + (k0 + tt) * L);
        } else {
          twiddle_mul<MM, L, kT>(A, s0 + j * ES, tws + j * EST, s, k0, mc, res[q]);
        }
        dsl[q] = bitrev_n(j, LOGE) * ES;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < PER; ++q)
        if (dsl[q] >= 0) store_rot<MM, L, kT>(s0 + dsl[q], res[q], ((threadIdx.x + q * NT) % TPE) * kT, rot[q], mc);
      __syncthreads();
      const uint32_t* ov = dft_pingpong<MM, L, NE>(s0, s1, LOGE, mc);
      for (int it = threadIdx.x; it < NE * MM; it += NT) {
        const int vv = it / MM, kk = it % MM;
        uint32_t v[L];
        ld_res<L>(v, ov + vv * ES + kk * L);
        st_res<L>(poly + ((long long)vv * mu1 + l) * EW + kk * L, v);
      }
      fence_proxy_async();
      __syncthreads();
    }
  }
}

}  // namespace dkss
