// dkss_tc.cuh -- the twiddle products of a transform level on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).
//
// A level multiplies element (j, l) of every column by rho^e, e = j * l * base_pow
// (bigmul/dkss.py:480-492), = alpha^r * rho_table[s] with s = e mod (M/m).  Every element with
// the same s is multiplied by the SAME ring element t = rho_table[s], and over bytes that is a
// dense integer matrix product:
//
//   x_i = sum_k X[i][k] 256^k          -- u8 digits: the element's own little-endian bytes
//   T_l = t_l 2^160 mod p              -- balanced signed base-256 digits D_l[0..16] (s8)
//   Z[j][d] = sum_{i,k} X[i][k] D_{+-(j-i) mod m}[d-k]      (|Z| < 2^25)
//   z_j = (sum_d Z[j][d] 256^d) 2^-160 mod p = (x t)_j        (negacyclic: the wrapped terms use
//                                                              p - T, alpha^m = -1)
//
// One CTA tile = up to 128 elements sharing s: D[128][32m] (s32, TMEM) += A[128][16m] (u8)
// x B[32m][16m] (s8).  B is never materialised: with A's 16-byte K chunks in reversed
// coefficient order (chunk i' holds x_{m-1-i'}), B row (j, d), K chunk i' is the 16-byte unit
// V[j + i'][d] of a per-s table V[2m-1][32][16], so the UMMA descriptor of B is just V read with
// strides (SBO 128 B between 8-row groups, LBO 512 B between K chunks): 32 KB of shared memory
// for the whole 32m x 16m Toeplitz operand (m = 32).
//
// Epilogue (CUDA cores, one thread per element row): tcgen05.ld of the 32 byte-position sums of
// a coefficient, one 288-bit signed integer, + p 2^160, five Montgomery REDC steps with
// R = 2^160 using p = 1 + P3 2^96 (Proth: -p^-1 = -1 mod 2^32, q p touches limbs 0, 3, 4),
// canonical, then stored at (j + r) mod 2m with the negation of alpha^m = -1 -- the same
// element the CUDA-core kernels' ring_mul + store_rot produce (tests/test_gpu_parity.py).
#pragma once
#include <cstdint>
#include "dkss_kernels.cuh"

namespace dkss {

constexpr int kTcRows = 128;     // UMMA M
constexpr int kTcNChunk = 256;   // UMMA N per instruction and per TMEM buffer
constexpr int kTcThreads = 256;  // 8 warps: loads and epilogue; thread 0 issues the MMAs

struct TcArgs {
  uint32_t* poly;            // element index 0 of the launch (elements of MM * 4 words)
  const uint32_t* tiles;     // [ntiles][3]: s, first entry, entry count (<= 128)
  const uint32_t* entries;   // (element index << 6) | alpha shift r (mod 2m)
  const uint8_t* vtab;       // [M/m][2m - 1][32][16] s8 digits, from the (scaled) twiddle rows
  int ntiles;
  uint32_t p3;               // p = 1 + p3 * 2^96
};

template <int MM>
struct TcSmem {
  static constexpr int K = MM * 16;                    // bytes per element (A row)
  static constexpr int ABYTES = kTcRows * K;           // A tile
  static constexpr int VBYTES = (2 * MM - 1) * 32 * 16;
  static constexpr int VPAD = (VBYTES + 1023) / 1024 * 1024;
  static constexpr int STAGE = ABYTES + VPAD + kTcRows * 4;  // + entries
  static constexpr int BYTES = 2 * STAGE + 1024;             // two stages + alignment slack
};

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major, no swizzle (cute/arch/mma_sm100_desc.hpp)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1
  return d;
}

// kind::i8 instruction descriptor: D s32 (bits 4-5 = 2), A u8 (7-9 = 0), B s8 (10-12 = 1),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "TC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra TC_WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(valid ? 16 : 0)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// z = (sum_d Z[d] 256^d + p 2^160) 2^-160 mod p, canonical, for p = 1 + p3 2^96 (L = 4)
__device__ __forceinline__ void reduce_coeff(const int32_t (&Z)[32], uint32_t p3, uint32_t (&out)[4]) {
  long long acc[9];
#pragma unroll
  for (int w = 0; w < 9; ++w) acc[w] = 0;
#pragma unroll
  for (int d = 0; d < 32; ++d) acc[d >> 2] += (long long)Z[d] << (8 * (d & 3));
  uint32_t t[10];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    acc[w + 1] += acc[w] >> 32;  // arithmetic shift: carries and borrows
    t[w] = (uint32_t)acc[w];
  }
  // + p 2^160 = 2^160 + p3 2^256 (limb 5 += 1, limb 8 += p3): non-negative, < 2^288
  long long top = acc[8] + (long long)p3;
  {
    unsigned long long s = (unsigned long long)t[5] + 1u;
    t[5] = (uint32_t)s;
    unsigned long long c = s >> 32;
    s = (unsigned long long)t[6] + c;
    t[6] = (uint32_t)s;
    c = s >> 32;
    s = (unsigned long long)t[7] + c;
    t[7] = (uint32_t)s;
    top += (long long)(s >> 32);
  }
  t[8] = (uint32_t)top;
  t[9] = (uint32_t)((unsigned long long)top >> 32);
#pragma unroll
  for (int step = 0; step < 5; ++step) {  // REDC: q = -t0, t += q p, t >>= 32
    const uint32_t q = 0u - t[0];
    unsigned long long c = (t[0] != 0u) ? 1ull : 0ull;
    const unsigned long long hq = (unsigned long long)q * p3;
    unsigned long long s = (unsigned long long)t[1] + c;
    t[1] = (uint32_t)s;
    c = s >> 32;
    s = (unsigned long long)t[2] + c;
    t[2] = (uint32_t)s;
    c = s >> 32;
    s = (unsigned long long)t[3] + (uint32_t)hq + c;
    t[3] = (uint32_t)s;
    c = s >> 32;
    s = (unsigned long long)t[4] + (hq >> 32) + c;
    t[4] = (uint32_t)s;
    c = s >> 32;
#pragma unroll
    for (int w = 5; w < 10; ++w) {
      s = (unsigned long long)t[w] + c;
      t[w] = (uint32_t)s;
      c = s >> 32;
    }
#pragma unroll
    for (int w = 0; w < 9; ++w) t[w] = t[w + 1];
    t[9] = 0;
  }
  // t < 2^128 + p < 3p: subtract p while that does not borrow
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    uint32_t r[5], b;
    r[0] = t[0] - 1u;
    b = t[0] < 1u;
    r[1] = t[1] - b;
    b = t[1] < b;
    r[2] = t[2] - b;
    b = t[2] < b;
    r[3] = t[3] - p3 - b;
    b = (unsigned long long)t[3] < (unsigned long long)p3 + b;
    r[4] = t[4] - b;
    b = t[4] < b;
    if (!b) {
#pragma unroll
      for (int q = 0; q < 5; ++q) t[q] = r[q];
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) out[q] = t[q];
}

// p - z (z canonical; 0 stays 0)
__device__ __forceinline__ void neg_p(uint32_t (&z)[4], uint32_t p3) {
  if ((z[0] | z[1] | z[2] | z[3]) == 0u) return;
  uint32_t b;
  const uint32_t r0 = 1u - z[0];
  b = z[0] > 1u;
  const uint32_t r1 = 0u - z[1] - b;
  b = (z[1] | b) != 0u;
  const uint32_t r2 = 0u - z[2] - b;
  b = (z[2] | b) != 0u;
  const uint32_t r3 = p3 - z[3] - b;
  z[0] = r0;
  z[1] = r1;
  z[2] = r2;
  z[3] = r3;
}

}  // namespace tc

// Grouped twiddle products of one level, in place (see the file comment).  Persistent CTAs
// walk the tile list; tile t + 1's elements, V table and entries are prefetched (cp.async)
// while tile t multiplies; within a tile the N chunks alternate between two TMEM buffers so
// the epilogue of chunk c overlaps the MMAs of chunk c + 1.
template <int MM>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_twiddle(TcArgs A) {
  griddep_wait();  // PDL: the column pass that produced the elements has completed
  griddep_launch();
  using S = TcSmem<MM>;
  constexpr int K = S::K, NCH = MM * 32 / kTcNChunk, KSTEPS = K / 32;
  constexpr int SBO_A = MM * 128;  // bytes between 8-row groups of A
  constexpr int CPC = kTcNChunk / 32;  // coefficients per N chunk
  constexpr int EW = MM * 4;           // words per element
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc::smem_u32(&tmem_sh)),
                 "r"(2 * kTcNChunk));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(tc::smem_u32(&mbar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(tc::smem_u32(&mbar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t idesc = tc::make_idesc(kTcRows, kTcNChunk);
  uint32_t ph[2] = {0u, 0u};

  // stage `st` <- tile t: the elements (reversed coefficient chunks, zero rows past the count),
  // the tile's V table and its entries
  auto prefetch = [&](int t, int st) {
    uint8_t* sA = smem + st * S::STAGE;
    uint8_t* sV = sA + S::ABYTES;
    uint32_t* sE = reinterpret_cast<uint32_t*>(sV + S::VPAD);
    const uint32_t s = A.tiles[3 * t], first = A.tiles[3 * t + 1], cnt = A.tiles[3 * t + 2];
    for (int i = threadIdx.x; i < kTcRows / 4; i += kTcThreads)
      tc::cp16(sE + 4 * i, A.entries + first + 4 * i, (uint32_t)(4 * i) < cnt);
    const uint8_t* vsrc = A.vtab + (size_t)s * S::VBYTES;
    for (int i = threadIdx.x; i < S::VBYTES / 16; i += kTcThreads) tc::cp16(sV + 16 * i, vsrc + 16 * i, true);
    for (int i = threadIdx.x; i < kTcRows * MM; i += kTcThreads) {
      const int r = i / MM, c = i % MM;
      const bool live = (uint32_t)r < cnt;
      const uint32_t e = live ? __ldg(A.entries + first + r) >> 6 : 0u;
      tc::cp16(sA + (r >> 3) * SBO_A + (MM - 1 - c) * 128 + (r & 7) * 16, A.poly + (size_t)e * EW + c * 4, live);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  int t = blockIdx.x;
  if (t < A.ntiles) prefetch(t, 0);
  for (int k = 0; t < A.ntiles; ++k, t += gridDim.x) {
    const int st = k & 1;
    const int tn = t + gridDim.x;
    if (tn < A.ntiles) {
      prefetch(tn, st ^ 1);  // the other stage's MMAs all completed in the previous tile
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic-proxy writes -> tensor core
    __syncthreads();
    tc::fence_after();
    uint8_t* sA = smem + st * S::STAGE;
    uint8_t* sV = sA + S::ABYTES;
    const uint32_t* sE = reinterpret_cast<const uint32_t*>(sV + S::VPAD);
    const uint32_t cnt = A.tiles[3 * t + 2];
    const uint32_t a_base = tc::smem_u32(sA), v_base = tc::smem_u32(sV);
    auto issue = [&](int ch) {
      const uint32_t tbuf = tmem + (uint32_t)((ch & 1) * kTcNChunk);
#pragma unroll
      for (int ks = 0; ks < KSTEPS; ++ks) {
        const uint64_t da = tc::make_desc(a_base + ks * 256, 128, SBO_A);
        const uint64_t db = tc::make_desc(v_base + (ch * kTcNChunk / 8) * 128 + ks * 1024, 512, 128);
        tc::mma_i8(tbuf, da, db, idesc, ks > 0 ? 1u : 0u);
      }
      tc::mma_commit(&mbar[ch & 1]);
    };
    if (threadIdx.x == 0) {
      issue(0);
      if (NCH > 1) issue(1);
    }
    const int row = 32 * (warp & 3) + lane;
    const bool live = (uint32_t)row < cnt;
    const uint32_t ent = live ? sE[row] : 0u;
    uint32_t* dst = A.poly + (size_t)(ent >> 6) * EW;
    const int rot = (int)(ent & 63u);
    for (int ch = 0; ch < NCH; ++ch) {
      tc::mbar_wait_parity(&mbar[ch & 1], ph[ch & 1]);
      ph[ch & 1] ^= 1u;
      tc::fence_after();
      const uint32_t lane_addr = tmem + (uint32_t)((ch & 1) * kTcNChunk) + ((uint32_t)(32 * (warp & 3)) << 16);
      for (int cj = warp >> 2; cj < CPC; cj += 2) {
        int32_t Zv[32];
        tc::tmem_ld32(lane_addr + cj * 32, Zv);
        if (live) {
          uint32_t o[4];
          tc::reduce_coeff(Zv, A.p3, o);
          int pos = (ch * CPC + cj + rot) & (2 * MM - 1);
          if (pos >= MM) {
            pos -= MM;
            tc::neg_p(o, A.p3);
          }
          *reinterpret_cast<uint4*>(dst + pos * 4) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      tc::fence_before();
      __syncthreads();  // TMEM buffer (ch & 1) drained
      if (threadIdx.x == 0 && ch + 2 < NCH) {
        tc::fence_after();
        issue(ch + 2);
      }
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * kTcNChunk));
}

// V tables of the tensor-core twiddle products: for every table row s, the effective twiddle
// t = w R^-1 of the stored (Montgomery-form) row w (ring_mul computes REDC(x w)), scaled to
// T = t 2^160 = w 2^32 = mont_mul(w, 2^160 mod p); V[s][l'][d] = 16 bytes k = 0..15 of the digit
// at position d - k of (l' >= m-1 ? T_{l'-m+1} : p - T_{l'+1}) in balanced base 256.
template <int MM>
__global__ void k_tc_build_v(const uint32_t* __restrict__ twr, long long nrows, uint8_t* __restrict__ vtab, ModCtx mc,
                             const uint32_t* __restrict__ c160) {
  constexpr int L = 4, LP = 2 * MM - 1;
  const long long n = nrows * LP;
  for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < n; it += (long long)gridDim.x * blockDim.x) {
    const long long s = it / LP;
    const int lp = (int)(it % LP);
    const bool pos = lp >= MM - 1;
    const int l = pos ? lp - (MM - 1) : lp + 1;
    uint32_t w[L], K[L], T[L];
#pragma unroll
    for (int q = 0; q < L; ++q) {
      w[q] = twr[(s * 2 * MM + l) * L + q];
      K[q] = c160[q];
    }
    mont_mul<L>(T, w, K, mc);  // canonical
    if (!pos) neg_mod_canon<L>(T, T, mc);
    int8_t dig[17];
    int carry = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      int v = (int)((T[k >> 2] >> (8 * (k & 3))) & 0xFFu) + carry;
      carry = v >= 128;
      dig[k] = (int8_t)(v - (carry ? 256 : 0));
    }
    dig[16] = (int8_t)carry;
    uint8_t* out = vtab + (size_t)it * 32 * 16;
    for (int d = 0; d < 32; ++d) {
      uint32_t wd[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int k = 4 * q + b, x = d - k;
          const uint32_t byte = (x >= 0 && x <= 16) ? (uint8_t)dig[x] : 0u;
          v |= byte << (8 * b);
        }
        wd[q] = v;
      }
      *reinterpret_cast<uint4*>(out + d * 16) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
  }
}

}  // namespace dkss
