// dkss_tc.cuh -- the twiddle products of a transform level on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).
//
// A level multiplies element (j, l) of every column by rho^e, e = j * l * base_pow
// (bigmul/dkss.py:480-492), = alpha^r * rho_table[s] with s = e mod (M/m).  Every element with
// the same s is multiplied by the SAME ring element t = rho_table[s], and over bytes that is a
// dense integer matrix product.  Multiplication by a constant mod p is
// linear in the bytes of the other factor, so the constant is spread over them:
//
//   x_i = sum_k X[i][k] 256^k                 -- u8 digits: the element's own little-endian bytes
//   C_l,k = +-t_l 256^k 2^32 mod p            -- in (-p/2, p/2), balanced signed base-256 digits
//                                                D_l,k[0..15] (s8); the wrapped terms of the
//                                                negacyclic product are negated (alpha^m = -1)
//   Z[j][d] = sum_{i,k} X[i][k] D_{j-i,k}[d]  (|Z| < 16 m 255 128 <= 2^24)
//   z_j = (sum_d Z[j][d] 256^d) 2^-32 mod p = (x t)_j
//
// so one ring product is a 16m x 16m byte matrix with no structural zeros (a byte Toeplitz
// formulation with T = t 2^160 needs 32m output positions, half of them zero bands).
//
// One CTA tile = up to 128 elements sharing s: D[128][16m] (s32, TMEM) += A[128][16m] (u8)
// x B[16m][16m] (s8).  B is never materialised: with A's 16-byte K chunks in reversed
// coefficient order (chunk i' holds x_{m-1-i'}), B row (j, d), K chunk i' is the 16-byte unit
// V[j + i'][d] = (D_{j+i'-m+1,k}[d])_{k<16} of a per-s table V[2m-1][16][16], so the UMMA
// descriptor of B is just V read with strides (SBO 128 B between 8-row groups, LBO 256 B between
// K chunks): 16 KB of shared memory for the whole 16m x 16m operand (m = 32).
//
// Epilogue (CUDA cores, one thread per element row and coefficient): tcgen05.ld of the 16
// byte-position sums of a coefficient, folded into a signed five-limb integer with three
// IMAD.WIDE per limb, + p 2^17 (non-negative), one Montgomery REDC step with R = 2^32 using
// p = 1 + P3 2^96 (Proth: -p^-1 = -1 mod 2^32, q p touches limbs 0, 3, 4), one conditional
// subtraction, then stored at (j + r) mod 2m with the negation of alpha^m = -1 -- the same
// element the CUDA-core kernels' ring_mul + store_rot produce (tests/test_gpu_parity.py).
#pragma once
#include <cstdint>
#include "dkss_kernels.cuh"

namespace dkss {

constexpr int kTcRows = 128;     // UMMA M
constexpr int kTcNChunk = 256;   // UMMA N per instruction and per TMEM buffer
constexpr int kTcEpiWarps = 16;  // epilogue: 4 per TMEM lane quadrant
constexpr int kTcProdWarps = 2;  // smem producers (element gather + V bulk copy)
constexpr int kTcThreads = (kTcEpiWarps + kTcProdWarps + 1) * 32;  // + one MMA-issue warp

struct TcArgs {
  uint32_t* poly;            // element index 0 of the launch (elements of MM * 4 words)
  const uint32_t* tiles;     // [ntiles][3]: s, first entry, entry count (<= 128)
  const uint32_t* entries;   // (element index << 6) | alpha shift r (mod 2m)
  const uint8_t* vtab;       // [M/m][2m - 1][16][16] s8 digits, from the (scaled) twiddle rows
  int ntiles;
  uint32_t p3;               // p = 1 + p3 * 2^96
  // fused four-step exchange of the first level (PassArgs::peer_mode 1): element el = q E C + pos
  // (q = el >> peer_log_poly) is stored into its row owner's [2][R][mu0] buffer
  const unsigned long long* peer = nullptr;
  int peer_log_r = 0, peer_log_c = 0, peer_log_mu0 = 0, peer_log_poly = 0;
  long long l_off = 0;
};

__device__ __forceinline__ uint32_t* tc_dst(const TcArgs& A, uint32_t el, int ew) {
  if (!A.peer) return A.poly + (size_t)el * ew;
  const long long q = (long long)el >> A.peer_log_poly, pos = (long long)el & ((1LL << A.peer_log_poly) - 1);
  const long long j = pos >> A.peer_log_c, c = pos & ((1LL << A.peer_log_c) - 1);
  const long long R = 1LL << A.peer_log_r;
  uint32_t* base = reinterpret_cast<uint32_t*>(A.peer[j >> A.peer_log_r]);
  return base + (((q * R + (j & (R - 1))) << A.peer_log_mu0) + A.l_off + c) * ew;
}

template <int MM>
struct TcSmem {
  static constexpr int K = MM * 16;                    // bytes per element (A row)
  static constexpr int ABYTES = kTcRows * K;           // A tile
  static constexpr int VBYTES = (2 * MM - 1) * 16 * 16;
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

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(bytes)
               : "memory");
}

// bulk copy global -> shared (TMA engine), completion counted in bytes on mbar
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}

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

// the same load without the wait (several loads, then one tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, int32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

// z = (sum_{d<16} Z[d] 256^d) 2^-32 mod p, canonical, for p = 1 + p3 2^96 (L = 4) with
// 2^31 <= p3 < 2^32 - 2^17 (p in (2^127, 2^128 - 2^113)).  |Z[d]| <= 16 m 255 128, so
// |sum| <= 16 m 128 (256^16 - 1) < m 2^139 <= 2^144 < p 2^17: adding p 2^17 makes it
// non-negative and < 2^145 (five limbs).  One REDC step (q = -t0, since -p^-1 = -1 mod 2^32;
// q p = q + q p3 2^96) gives r = (V + q p) / 2^32 < 2^113 + p < min(2p, 2^128), so one
// conditional subtraction makes r canonical.  `Z` points at 16 consecutive sums.
template <class Arr>
__device__ __forceinline__ void reduce_coeff16(const Arr& Z, int z0, uint32_t p3, bool neg, uint32_t (&out)[4]) {
  uint32_t t0, t1, t2, t3, t4;
  {
    long long c = 0;
    uint32_t t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // 64-bit sums of four byte positions, carried into 32-bit limbs
      long long a = (long long)Z[z0 + 4 * k];
      asm("mad.wide.s32 %0, %1, 256, %0;" : "+l"(a) : "r"(Z[z0 + 4 * k + 1]));
      asm("mad.wide.s32 %0, %1, 65536, %0;" : "+l"(a) : "r"(Z[z0 + 4 * k + 2]));
      asm("mad.wide.s32 %0, %1, 16777216, %0;" : "+l"(a) : "r"(Z[z0 + 4 * k + 3]));
      a += c;
      t[k] = (uint32_t)a;
      c = a >> 32;
    }
    t0 = t[0], t1 = t[1], t2 = t[2], t3 = t[3];
    t4 = (uint32_t)c;  // two's complement top limb (|c| < 2^16)
  }
  // + p 2^17 = 2^17 + p3 2^113: limbs (2^17, 0, 0, p3 << 17, p3 >> 15); then the REDC step
  const uint32_t q = 0u - (t0 + 0x20000u);
  asm("add.cc.u32 %0, %0, 0x20000;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.cc.u32 %2, %2, 0;\n\t"
      "addc.cc.u32 %3, %3, %5;\n\taddc.u32 %4, %4, %6;\n\t"
      "add.cc.u32 %0, %0, %7;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.cc.u32 %2, %2, 0;\n\t"
      "madc.lo.cc.u32 %3, %7, %8, %3;\n\tmadc.hi.u32 %4, %7, %8, %4;\n"
      : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4)
      : "r"(p3 << 17), "r"(p3 >> 15), "r"(q), "r"(p3));
  // r = t1..t4 < 2^113 + p: subtract p once if r >= p; then p - r when `neg` (alpha^m = -1 wrap)
  uint32_t r0, r1, r2, r3, bo;
  asm("sub.cc.u32 %0, %5, 1;\n\tsubc.cc.u32 %1, %6, 0;\n\tsubc.cc.u32 %2, %7, 0;\n\t"
      "subc.cc.u32 %3, %8, %9;\n\tsubc.u32 %4, 0, 0;\n"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(bo)
      : "r"(t1), "r"(t2), "r"(t3), "r"(t4), "r"(p3));
  const bool keep = bo != 0u;  // borrow: r < p
  const uint32_t c0 = keep ? t1 : r0, c1 = keep ? t2 : r1, c2 = keep ? t3 : r2, c3 = keep ? t4 : r3;
  uint32_t e0, e1, e2, e3;
  asm("sub.cc.u32 %0, 1, %4;\n\tsubc.cc.u32 %1, 0, %5;\n\tsubc.cc.u32 %2, 0, %6;\n\tsubc.u32 %3, %8, %7;\n"
      : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3)
      : "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(p3));
  const bool flip = neg && ((c0 | c1 | c2 | c3) != 0u);
  out[0] = flip ? e0 : c0;
  out[1] = flip ? e1 : c1;
  out[2] = flip ? e2 : c2;
  out[3] = flip ? e3 : c3;
}

}  // namespace tc

// Grouped twiddle products of one level, in place (see the file comment).  Persistent CTAs walk
// the tile list with warp-specialised roles and mbarrier pipelines (no CTA-wide barriers in the
// loop):
//   producer warps (kTcProdWarps): gather tile k's elements into smem stage k & 1 with 16-byte
//     cp.async (8 rows x 64 contiguous bytes per instruction: coalesced reads, conflict-free
//     writes), the tile's V table with one bulk copy; stage reuse waits on the MMA's commit;
//   MMA warp (one thread): per N chunk, waits for a free TMEM buffer, issues the K steps,
//     commits to the buffer's "full" barrier, and after the tile's last chunk to the stage's
//     "empty" barrier;
//   epilogue warps (kTcEpiWarps): per chunk, tcgen05.ld of their coefficient columns, release the
//     TMEM buffer, then reduce (tc::reduce_coeff16) and store.
template <int MM>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_twiddle(TcArgs A) {
  // PDL: the set-up, the first tile's schedule entries and V table (constants of the plan) overlap
  // the tail of the column pass; only the element gather waits for it (griddep_wait below)
  griddep_launch();
  using S = TcSmem<MM>;
  constexpr int K = S::K, NCH = MM * 16 / kTcNChunk, KSTEPS = K / 32;
  constexpr int SBO_A = MM * 128;      // bytes between 8-row groups of A
  constexpr int CPC = kTcNChunk / 16;  // coefficients per N chunk (16 byte positions each)
  constexpr int EW = MM * 4;           // words per element
  constexpr int CPE = CPC / 4;         // coefficients per epilogue warp per chunk (4 lane quadrants)
  static_assert(kTcEpiWarps == 16 && CPC == 16 && CPE == 4, "two coefficient pairs per epilogue warp per chunk");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // full[2], empty[2] (smem stages), tfull[2], tempty[2] (TMEM buffers)
  __shared__ __align__(8) uint64_t bars[8];
  __shared__ uint32_t tmem_sh;
  uint64_t* full = bars;
  uint64_t* empty = bars + 2;
  uint64_t* tfull = bars + 4;
  uint64_t* tempty = bars + 6;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc::smem_u32(&tmem_sh)),
                 "r"(2 * kTcNChunk));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&full[i], kTcProdWarps * 32 + 1);  // every producer lane + the V expect-tx
      tc::mbar_init(&empty[i], 1);
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], kTcEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_sh;
  const int G = gridDim.x;

  if (warp >= kTcEpiWarps && warp < kTcEpiWarps + kTcProdWarps) {
    // ===== producers =====
    // Each lane gathers rows g8 * 8 + (lane & 7) of the tile (g8 = pw, pw + kTcProdWarps, ...),
    // 16-byte chunks c = 4 i + (lane >> 3).  The tile header and row entries of tile k + 1 are
    // loaded while tile k's copies are in flight; a tile's "full" barrier is signalled as soon as
    // its own copies have landed (wait_group 0, proxy fence, arrive).
    constexpr int GPW = kTcRows / 8 / kTcProdWarps;  // row groups per producer warp
    const int pw = warp - kTcEpiWarps;
    const int rr = lane & 7, cc = lane >> 3;
    uint32_t hs = 0, hcnt = 0, ent[GPW];
    auto load_tile = [&](int t) {
      const uint32_t first = __ldg(A.tiles + 3 * t + 1);
      hs = __ldg(A.tiles + 3 * t);
      hcnt = __ldg(A.tiles + 3 * t + 2);
#pragma unroll
      for (int i = 0; i < GPW; ++i) ent[i] = __ldg(A.entries + first + (pw + i * kTcProdWarps) * 8 + rr) >> 6;
    };
    int k = 0;
    if ((int)blockIdx.x < A.ntiles) load_tile(blockIdx.x);
    for (int t = blockIdx.x; t < A.ntiles; t += G, ++k) {
      const int st = k & 1;
      if (k >= 2) tc::mbar_wait_parity(&empty[st], ((k >> 1) - 1) & 1);
      uint8_t* sA = smem + st * S::STAGE;
      uint8_t* sV = sA + S::ABYTES;
      if (pw == 0 && lane == 0) {
        tc::mbar_arrive_tx(&full[st], S::VBYTES);
        tc::bulk_g2s(sV, A.vtab + (size_t)hs * S::VBYTES, S::VBYTES, &full[st]);
      }
      if (k == 0) griddep_wait();  // the column pass that produced the elements has completed
#ifndef DKSS_TC_EXP_NOLOAD  // experiment builds only: time the pipeline without the element gather
#pragma unroll
      for (int i = 0; i < GPW; ++i) {
        const int g8 = pw + i * kTcProdWarps;
        const bool live = (uint32_t)(g8 * 8 + rr) < hcnt;  // rows past the count: zero-filled
        const uint32_t* src = A.poly + (size_t)(live ? ent[i] : 0u) * EW;
        uint8_t* dst = sA + g8 * SBO_A + rr * 16;
#pragma unroll
        for (int c0 = 0; c0 < MM; c0 += 4) {
          const int c = c0 + cc;
          tc::cp16(dst + (MM - 1 - c) * 128, src + c * 4, live);
        }
      }
#endif
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      if (t + G < A.ntiles) load_tile(t + G);  // next tile's header and rows, under this tile's copies
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic-proxy writes -> tensor core
      tc::mbar_arrive(&full[st]);
    }
  } else if (warp == kTcEpiWarps + kTcProdWarps) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc = tc::make_idesc(kTcRows, kTcNChunk);
      int k = 0, g = 0;
      for (int t = blockIdx.x; t < A.ntiles; t += G, ++k) {
        const int st = k & 1;
        tc::mbar_wait_parity(&full[st], (k >> 1) & 1);
        tc::fence_after();
        const uint32_t a_base = tc::smem_u32(smem + st * S::STAGE);
        const uint32_t v_base = a_base + S::ABYTES;
        for (int ch = 0; ch < NCH; ++ch, ++g) {
          const int b = g & 1;
          if (g >= 2) {
            tc::mbar_wait_parity(&tempty[b], ((g >> 1) - 1) & 1);
            tc::fence_after();
          }
          const uint32_t tbuf = tmem + (uint32_t)(b * kTcNChunk);
#pragma unroll
          for (int ks = 0; ks < KSTEPS; ++ks) {
            const uint64_t da = tc::make_desc(a_base + ks * 256, 128, SBO_A);
            const uint64_t db = tc::make_desc(v_base + (ch * kTcNChunk / 8) * 128 + ks * 512, 256, 128);
            tc::mma_i8(tbuf, da, db, idesc, ks > 0 ? 1u : 0u);
          }
          tc::mma_commit(&tfull[b]);
        }
        tc::mma_commit(&empty[st]);
      }
    }
  } else if (warp < kTcEpiWarps) {
    // ===== epilogue =====
    griddep_wait();  // its stores overwrite elements the previous kernel wrote
    const int quad = warp & 3;
    const int row = 32 * quad + lane;
    int g = 0;
    for (int t = blockIdx.x; t < A.ntiles; t += G) {
      const uint32_t first = __ldg(A.tiles + 3 * t + 1), cnt = __ldg(A.tiles + 3 * t + 2);
      const bool live = (uint32_t)row < cnt;
      const bool warp_live = (uint32_t)(32 * quad) < cnt;  // warp-uniform
      const uint32_t ent = live ? __ldg(A.entries + first + row) : 0u;
      uint32_t* dst = tc_dst(A, ent >> 6, EW);
      const int rot = (int)(ent & 63u);
      for (int ch = 0; ch < NCH; ++ch, ++g) {
        const int b = g & 1;
        tc::mbar_wait_parity(&tfull[b], (g >> 1) & 1);
        tc::fence_after();
        int32_t Z0[32], Z1[32];
        const uint32_t lane_addr = tmem + (uint32_t)(b * kTcNChunk) + ((uint32_t)(32 * quad) << 16);
        const int pp0 = warp >> 2, pp1 = pp0 + 4;  // coefficient pairs (2 x 16 columns) of this warp
        if (warp_live) {
          tc::tmem_ld32_nowait(lane_addr + pp0 * 32, Z0);
          tc::tmem_ld32_nowait(lane_addr + pp1 * 32, Z1);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[b]);  // this warp's columns of buffer b are read
#ifdef DKSS_TC_EXP_NOEPI  // experiment builds only: time the pipeline without the reduction
        if (live && Z0[0] == 0x7fffffff && Z1[0] == 0x7fffffff) dst[0] = 0u;
#else
        if (live) {
#pragma unroll
          for (int h = 0; h < CPE; ++h) {
            const int cj = 2 * (h < 2 ? pp0 : pp1) + (h & 1);
            const int pos = (ch * CPC + cj + rot) & (2 * MM - 1);
            uint32_t o[4];
            if (h < 2)
              tc::reduce_coeff16(Z0, 16 * (h & 1), A.p3, pos >= MM, o);
            else
              tc::reduce_coeff16(Z1, 16 * (h & 1), A.p3, pos >= MM, o);
            *reinterpret_cast<uint4*>(dst + (pos & (MM - 1)) * 4) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
#endif
      }
    }
  }
  if (A.peer) __threadfence_system();  // fused exchange: stores to other GPUs performed
  tc::fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * kTcNChunk));
}

// V tables of the tensor-core twiddle products: for every table row s, the effective twiddle
// t = w R^-1 of the stored (Montgomery-form) row w (ring_mul computes REDC(x w)); with
// ck[k] = 2^(32 + 8k) mod p, C_l,k = t_l 256^k 2^32 = mont_mul(w_l, ck[k]).  V[s][l'][d] = the
// 16 bytes k = 0..15 of digit d of (l' >= m-1 ? C_{l'-m+1,k} : p - C_{l'+1,k}) written in
// (-p/2, p/2) with balanced base-256 digits (16 suffice: p/2 < 127 (256^16 - 1) / 255).
template <int MM>
__global__ void k_tc_build_v(const uint32_t* __restrict__ twr, long long nrows, uint8_t* __restrict__ vtab, ModCtx mc,
                             const uint32_t* __restrict__ ck) {
  constexpr int L = 4, LP = 2 * MM - 1;
  const long long n = nrows * LP;
  for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < n; it += (long long)gridDim.x * blockDim.x) {
    const long long s = it / LP;
    const int lp = (int)(it % LP);
    const bool pos = lp >= MM - 1;
    const int l = pos ? lp - (MM - 1) : lp + 1;
    uint32_t w[L];
#pragma unroll
    for (int q = 0; q < L; ++q) w[q] = twr[(s * 2 * MM + l) * L + q];
    uint32_t unit[16][4];  // unit[d] = bytes k = 0..15 of digit d
#pragma unroll
    for (int d = 0; d < 16; ++d)
#pragma unroll
      for (int q = 0; q < 4; ++q) unit[d][q] = 0;
#pragma unroll 1
    for (int k = 0; k < 16; ++k) {
      uint32_t K[L], T[L];
#pragma unroll
      for (int q = 0; q < L; ++q) K[q] = ck[4 * k + q];
      mont_mul<L>(T, w, K, mc);  // canonical
      if (!pos) neg_mod_canon<L>(T, T, mc);
      // 2T > p (T > (p - 1) / 2): write T - p (two's complement) instead
      bool gt = (T[L - 1] >> 31) != 0u, decided = gt;  // 2T >= 2^128 > p
#pragma unroll
      for (int q = L - 1; q >= 0; --q) {
        const uint32_t t2 = (T[q] << 1) | (q ? T[q - 1] >> 31 : 0u);  // limb q of 2T
        if (!decided && t2 != mc.p[q]) {
          gt = t2 > mc.p[q];
          decided = true;
        }
      }
      if (gt) {  // T - p mod 2^128
        unsigned long long br = 0;
#pragma unroll
        for (int q = 0; q < L; ++q) {
          const unsigned long long v = (unsigned long long)T[q] - mc.p[q] - br;
          T[q] = (uint32_t)v;
          br = (v >> 63) & 1ull;
        }
      }
      int carry = 0;
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        int v = (int)((T[d >> 2] >> (8 * (d & 3))) & 0xFFu) + carry;
        carry = v >= 128;
        const uint32_t byte = (uint8_t)(int8_t)(v - (carry ? 256 : 0));
        unit[d][k >> 2] |= byte << (8 * (k & 3));
      }
    }
    uint4* out = reinterpret_cast<uint4*>(vtab + (size_t)it * 16 * 16);
#pragma unroll
    for (int d = 0; d < 16; ++d) out[d] = make_uint4(unit[d][0], unit[d][1], unit[d][2], unit[d][3]);
  }
}

}  // namespace dkss
