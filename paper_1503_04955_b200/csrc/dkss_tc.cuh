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
// x B[16m][16m] (s8).
//   A: the elements' own bytes, K = (coefficient c, byte k) in memory order, fetched by TMA row
//      gathers (tile::gather4: 4 rows x 128 B per instruction) into the 128-byte-swizzle K-major
//      layout (K blocks of [128 rows][128 B]).
//   B is never materialised: B row (jj, d), K chunk c is the 16-byte unit W[jj + c][d] of a per-s
//      table W[2m-1][16][16], W[t] = (D_{m-1-t,k}[d])_{k<16} (negated for the wrapped part), so
//      the UMMA descriptor of B is just W read with strides (SBO 128 B between 8-row groups, LBO
//      256 B between K chunks): 16 KB of shared memory for the whole 16m x 16m operand (m = 32).
//      TMEM column block jj holds coefficient m - 1 - jj.
//
// Epilogue (CUDA cores, one thread per element row and coefficient): tcgen05.ld of the 16
// byte-position sums of a coefficient, folded into a signed five-limb integer with one IMAD.WIDE
// per position (the multipliers +-256^k carry the negation of the rotation's alpha^m = -1 wrap),
// + p 2^17 (non-negative), one Montgomery REDC step with R = 2^32 using p = 1 + P3 2^96 (Proth:
// -p^-1 = -1 mod 2^32, q p touches limbs 0, 3, 4), one conditional subtraction, then stored at
// (j + r) mod 2m -- the same element the CUDA-core kernels' ring_mul + store_rot produce
// (tests/test_gpu_parity.py).
#pragma once
#include <cstdint>
#include "dkss_kernels.cuh"

namespace dkss {

constexpr int kTcRows = 128;     // UMMA M
constexpr int kTcNChunk = 256;   // UMMA N per instruction and per TMEM buffer
constexpr int kTcEpiWarps = 16;  // epilogue: 4 per TMEM lane quadrant
constexpr int kTcProdWarps = 4;  // smem producers (TMA row gather of the elements + V bulk copy)
constexpr int kTcThreads = (kTcEpiWarps + kTcProdWarps + 1) * 32;  // + one MMA-issue warp

// CUtensorMap of the launch's elements as a 2-D byte tensor [elements][16 m], box 128 B x 1 row,
// 128-byte swizzle (encoded on the host, csrc/dkss_capi.cu tc_tensor_map)
struct alignas(64) TcTensorMap {
  unsigned long long v[16];
};

struct TcArgs {
  TcTensorMap tmap;          // over `poly`
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
  static constexpr int KBLOCKS = K / 128;              // 128-byte K blocks of [128 rows][128 B], swizzled
  static constexpr int KBBYTES = kTcRows * 128;
  static constexpr int ABYTES = kTcRows * K;           // A tile
  static constexpr int VBYTES = (2 * MM - 1) * 16 * 16;
  static constexpr int VPAD = (VBYTES + 1023) / 1024 * 1024;
  // three A stages (a gather is issued two tiles ahead of its MMAs: its latency is longer than one
  // tile's MMAs), two V stages (a table is 1/4 of an A tile and arrives by one bulk copy)
  static constexpr int ASTAGES = 3, VSTAGES = 2;
  static constexpr int VOFF = ASTAGES * ABYTES;
  static constexpr int BYTES = ASTAGES * ABYTES + VSTAGES * VPAD + 1024;  // + alignment slack
};

#ifdef DKSS_TC_TRACE  // experiment builds only: SM-clock stamps of CTA 0's roles (tools/tc_trace.py)
// [launch % 8][role: 0 producer, 1 MMA, 2 epilogue warp 0][event]
static __device__ unsigned long long g_tc_trace[8][3][512];
static __device__ unsigned int g_tc_launch;
#define TC_STAMP(role, idx)                                                            \
  do {                                                                                 \
    if (blockIdx.x == 0 && (idx) < 512) g_tc_trace[trace_slot][role][idx] = clock64(); \
  } while (0)
#else
#define TC_STAMP(role, idx) \
  do {                      \
  } while (0)
#endif

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

// K-major operand in the 128-byte-swizzle layout (rows of 128 B, 8-row atoms of 1024 B)
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                  // leading byte offset: unused with a swizzled K-major operand
  d |= (uint64_t)(1024 >> 4) << 32;        // stride between 8-row atoms
  d |= (uint64_t)1 << 46;                  // descriptor version 1
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// TMA row gather: rows r0..r3 of the 2-D tensor, 128 bytes each starting at byte column c0, into
// four consecutive 128-byte rows of a swizzled K block
__device__ __forceinline__ void tma_gather4(void* sdst, const void* tmap, int c0, int r0, int r1, int r2, int r3,
                                            uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n" ::"r"(smem_u32(sdst)),
      "l"(tmap), "r"(smem_u32(mbar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
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

// 32 columns (two coefficients' byte-position sums) of this lane's row; completed by tmem_ld_wait
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

// 32-byte store (one full sector; a 16-byte store of a 32-byte sector is a partial write)
__device__ __forceinline__ void st256(uint32_t* p, const uint32_t (&lo)[4], const uint32_t (&hi)[4]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"l"(p), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]),
               "r"(lo[3]), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3])
               : "memory");
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// z = (sum_{d<16} Z[d] 256^d) 2^-32 mod p, canonical, for p = 1 + p3 2^96 (L = 4) with
// 2^31 <= p3 < 2^32 - 2^17 (p in (2^127, 2^128 - 2^113)).  |Z[d]| <= 16 m 255 128, so
// |sum| <= 16 m 128 (256^16 - 1) < m 2^139 <= 2^144 < p 2^17: adding p 2^17 makes it
// non-negative and < 2^145 (five limbs).  One REDC step (q = -t0, since -p^-1 = -1 mod 2^32;
// q p = q + q p3 2^96) gives r = (V + q p) / 2^32 < 2^113 + p < min(2p, 2^128), so one
// conditional subtraction makes r canonical.  `Z` points at 16 consecutive sums.
template <class Arr>
__device__ __forceinline__ void reduce_coeff16(const Arr& Z, int z0, uint32_t p3, bool neg, uint32_t (&out)[4]) {
  // signed fold with the negation of the alpha^m = -1 wrap in the multipliers (+-256^k): one
  // IMAD.WIDE per byte position (register multipliers, so ptxas cannot split them into shift +
  // high-product + two adds), 64-bit sums of four positions carried into 32-bit limbs
  const int m0 = neg ? -1 : 1, m1 = m0 * 256, m2 = m0 * 65536, m3 = m0 * 16777216;
  long long a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    asm("mul.wide.s32 %0, %1, %2;" : "=l"(a[k]) : "r"(Z[z0 + 4 * k]), "r"(m0));
    asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(a[k]) : "r"(Z[z0 + 4 * k + 1]), "r"(m1));
    asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(a[k]) : "r"(Z[z0 + 4 * k + 2]), "r"(m2));
    asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(a[k]) : "r"(Z[z0 + 4 * k + 3]), "r"(m3));
  }
  a[1] += a[0] >> 32;
  a[2] += a[1] >> 32;
  a[3] += a[2] >> 32;
  uint32_t t0 = (uint32_t)a[0], t1 = (uint32_t)a[1], t2 = (uint32_t)a[2], t3 = (uint32_t)a[3];
  uint32_t t4 = (uint32_t)(a[3] >> 32);  // two's complement top limb (|.| < 2^16)
  // + p 2^17 = 2^17 + p3 2^113: limbs (2^17, 0, 0, p3 << 17, p3 >> 15); then the REDC step
  const uint32_t q = 0u - (t0 + 0x20000u);
  asm("add.cc.u32 %0, %0, 0x20000;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.cc.u32 %2, %2, 0;\n\t"
      "addc.cc.u32 %3, %3, %5;\n\taddc.u32 %4, %4, %6;\n\t"
      "add.cc.u32 %0, %0, %7;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.cc.u32 %2, %2, 0;\n\t"
      "madc.lo.cc.u32 %3, %7, %8, %3;\n\tmadc.hi.u32 %4, %7, %8, %4;\n"
      : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4)
      : "r"(p3 << 17), "r"(p3 >> 15), "r"(q), "r"(p3));
  // r = t1..t4 < 2^113 + p: subtract p once if r >= p (a zero sum gives r = p -> 0)
  uint32_t r0, r1, r2, r3, bo;
  asm("sub.cc.u32 %0, %5, 1;\n\tsubc.cc.u32 %1, %6, 0;\n\tsubc.cc.u32 %2, %7, 0;\n\t"
      "subc.cc.u32 %3, %8, %9;\n\tsubc.u32 %4, 0, 0;\n"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(bo)
      : "r"(t1), "r"(t2), "r"(t3), "r"(t4), "r"(p3));
  const bool keep = bo != 0u;  // borrow: r < p
  out[0] = keep ? t1 : r0;
  out[1] = keep ? t2 : r1;
  out[2] = keep ? t3 : r2;
  out[3] = keep ? t4 : r3;
}

}  // namespace tc

// Grouped twiddle products of one level, in place (see the file comment).  Persistent CTAs walk
// the tile list with warp-specialised roles and mbarrier pipelines (no CTA-wide barriers in the
// loop):
//   producer warps (kTcProdWarps): TMA row gathers of tile k's elements into A stage k % 3, the
//     tile's W table with one bulk copy into V stage k % 2; stage reuse waits on the MMA's commit;
//   MMA warp (one thread): per N chunk, waits for a free TMEM buffer, issues the K steps,
//     commits to the buffer's "full" barrier, and after the tile's last chunk to the stage's
//     "empty" barrier;
//   epilogue warps (kTcEpiWarps): per chunk, tcgen05.ld of their coefficient columns (two
//     coefficients ahead of the reduction), release the TMEM buffer, reduce (tc::reduce_coeff16)
//     and store adjacent coefficients as 32-byte sectors.
template <int MM>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_twiddle(const __grid_constant__ TcArgs A) {
  // PDL: the set-up, the first tile's schedule entries and V table (constants of the plan) overlap
  // the tail of the column pass; only the element gather waits for it (griddep_wait below)
  griddep_launch();
  using S = TcSmem<MM>;
  constexpr int K = S::K, NCH = MM * 16 / kTcNChunk, KSTEPS = K / 32;
  constexpr int CPC = kTcNChunk / 16;  // coefficients per N chunk (16 byte positions each)
  constexpr int EW = MM * 4;           // words per element
  constexpr int CPE = CPC / 4;         // coefficients per epilogue warp per chunk (4 lane quadrants)
  static_assert(kTcEpiWarps == 16 && CPC == 16 && CPE == 4, "four coefficients per epilogue warp per chunk");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // full[AS], empty[AS] (A stages; a tile's V table arrives on the same "full"), tfull[2],
  // tempty[2] (TMEM buffers)
  constexpr int AS = S::ASTAGES;
  __shared__ __align__(8) uint64_t bars[2 * AS + 4];
  __shared__ uint32_t tmem_sh;
  uint64_t* full = bars;
  uint64_t* empty = bars + AS;
  uint64_t* tfull = bars + 2 * AS;
  uint64_t* tempty = bars + 2 * AS + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc::smem_u32(&tmem_sh)),
                 "r"(2 * kTcNChunk));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < AS; ++i) {
      tc::mbar_init(&full[i], 1);  // one arrival carrying the expected bytes (elements + V table)
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
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
#ifdef DKSS_TC_TRACE
  const unsigned int trace_slot = g_tc_launch & 7u;
  int ev = 0;
  TC_STAMP(warp < kTcEpiWarps ? 2 : warp - kTcEpiWarps == 0 ? 0 : 1, ev++);
#endif

  if (warp >= kTcEpiWarps && warp < kTcEpiWarps + kTcProdWarps) {
    // ===== producers =====
    // One TMA row-gather instruction moves 4 rows x 128 B (one K block) into the swizzled tile at
    // full shared-memory width (16-byte cp.async copies cost one shared-memory wavefront each and
    // starved the MMAs' operand reads).  A tile needs 32 row groups x KBLOCKS of them and a warp
    // issues one about every 60 clocks, so they are spread over all producer lanes: lane idx =
    // 32 pw + lane takes row group idx / KBLOCKS, K block idx % KBLOCKS (m = 16: half the lanes).
    // Rows past the tile's count repeat its first row (their products are never stored); row
    // groups past the count are skipped.  The tile header and row entries of tile k + 1 are
    // loaded while tile k's copies fly.
    const int pw = warp - kTcEpiWarps;
    const int pidx = pw * 32 + lane;
    const uint32_t pgroup = pidx / S::KBLOCKS;
    const int pkb = pidx % S::KBLOCKS;
    uint32_t hs = 0, hcnt = 0;
    int r[4] = {0, 0, 0, 0};
    auto load_tile = [&](int t) {
      const uint32_t first = __ldg(A.tiles + 3 * t + 1);
      hs = __ldg(A.tiles + 3 * t);
      hcnt = __ldg(A.tiles + 3 * t + 2);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t row = 4 * pgroup + i;
        r[i] = (int)(__ldg(A.entries + first + (row < hcnt ? row : 0u)) >> 6);
      }
    };
    int k = 0, sa = 0, ua = 0;  // tile count, its A stage k % AS and that stage's use count k / AS
    int sp = AS - 2, up = -1;   // stage and use count of tile k - 2
    if ((int)blockIdx.x < A.ntiles) load_tile(blockIdx.x);
    for (int t = blockIdx.x; t < A.ntiles; t += G, ++k) {
#ifdef DKSS_TC_TRACE
      if (pidx == 0) TC_STAMP(0, ev++);  // before the stage wait
#endif
      if (k >= AS) tc::mbar_wait_parity(&empty[sa], (ua - 1) & 1);
#ifdef DKSS_TC_TRACE
      if (pidx == 0) TC_STAMP(0, ev++);  // stage free
#endif
      uint8_t* sA = smem + sa * S::ABYTES;
      const uint32_t groups = (hcnt + 3) >> 2;
      if (k == 0) griddep_wait();  // the column pass that produced the elements has completed
#ifndef DKSS_TC_EXP_NOLOAD  // experiment builds only: time the pipeline without the element gather
      if (pgroup < groups)
        tc::tma_gather4(sA + pkb * S::KBBYTES + pgroup * 512, &A.tmap, pkb * 128, r[0], r[1], r[2], r[3], &full[sa]);
#endif
      if (pidx == 0) {
        // V stage k & 1 was read by tile k - 2: its MMAs have completed when that tile's A stage
        // is released (the same event the next tile's gather waits for); the expected byte count
        // may be posted after some of the gathers have completed (tx-count is signed)
        if (k >= 2) tc::mbar_wait_parity(&empty[sp], up & 1);
#ifdef DKSS_TC_EXP_NOLOAD
        tc::mbar_arrive_tx(&full[sa], S::VBYTES);
#else
        tc::mbar_arrive_tx(&full[sa], S::VBYTES + groups * 4 * S::K);
#endif
        tc::bulk_g2s(smem + S::VOFF + (k & 1) * S::VPAD, A.vtab + (size_t)hs * S::VBYTES, S::VBYTES, &full[sa]);
      }
      if (t + G < A.ntiles) load_tile(t + G);  // next tile's header and rows, under this tile's copies
#ifdef DKSS_TC_TRACE
      if (pidx == 0) TC_STAMP(0, ev++);  // copies issued
#endif
      if (++sa == AS) sa = 0, ++ua;
      if (++sp == AS) sp = 0, ++up;
    }
  } else if (warp == kTcEpiWarps + kTcProdWarps) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc = tc::make_idesc(kTcRows, kTcNChunk);
      int k = 0, g = 0, sa = 0, ua = 0;
      for (int t = blockIdx.x; t < A.ntiles; t += G, ++k) {
        TC_STAMP(1, ev++);  // before the "full" wait
        tc::mbar_wait_parity(&full[sa], ua & 1);
        tc::fence_after();
        TC_STAMP(1, ev++);  // tile in shared memory
        const uint32_t a_base = tc::smem_u32(smem + sa * S::ABYTES);
        const uint32_t v_base = tc::smem_u32(smem + S::VOFF + (k & 1) * S::VPAD);
        for (int ch = 0; ch < NCH; ++ch, ++g) {
          const int b = g & 1;
          if (g >= 2) {
            tc::mbar_wait_parity(&tempty[b], ((g >> 1) - 1) & 1);
            tc::fence_after();
          }
          TC_STAMP(1, ev++);  // TMEM buffer free
          const uint32_t tbuf = tmem + (uint32_t)(b * kTcNChunk);
#pragma unroll
          for (int ks = 0; ks < KSTEPS; ++ks) {
            const uint64_t da = tc::make_desc_sw128(a_base + (ks >> 2) * S::KBBYTES + (ks & 3) * 32);
            const uint64_t db = tc::make_desc(v_base + (ch * kTcNChunk / 8) * 128 + ks * 512, 256, 128);
            tc::mma_i8(tbuf, da, db, idesc, ks > 0 ? 1u : 0u);
          }
          tc::mma_commit(&tfull[b]);
          TC_STAMP(1, ev++);  // chunk issued
        }
        tc::mma_commit(&empty[sa]);
        if (++sa == AS) sa = 0, ++ua;
      }
    }
  } else if (warp < kTcEpiWarps) {
    // ===== epilogue =====
    // Warp (quad, q) owns the four coefficients 4q .. 4q+3 of every chunk (64 TMEM columns) for
    // the 32 rows of lane quadrant `quad`.
    griddep_wait();  // its stores overwrite elements the previous kernel wrote
    const int quad = warp & 3, q = warp >> 2;
    const int row = 32 * quad + lane;
    int g = 0;
    // tile headers are loaded two tiles ahead and row entries one tile ahead, so neither of the
    // dependent loads is waited for
    uint32_t cnt1 = 0, ent1 = 0, first2 = 0, cnt2 = 0;
    {
      const int t0 = blockIdx.x;
      if (t0 < A.ntiles) {
        const uint32_t first1 = __ldg(A.tiles + 3 * t0 + 1);
        cnt1 = __ldg(A.tiles + 3 * t0 + 2);
        ent1 = (uint32_t)row < cnt1 ? __ldg(A.entries + first1 + row) : 0u;
      }
      if (t0 + G < A.ntiles) {
        first2 = __ldg(A.tiles + 3 * (t0 + G) + 1);
        cnt2 = __ldg(A.tiles + 3 * (t0 + G) + 2);
      }
    }
    for (int t = blockIdx.x; t < A.ntiles; t += G) {
      const uint32_t cnt = cnt1, ent = ent1;
      ent1 = (t + G < A.ntiles && (uint32_t)row < cnt2) ? __ldg(A.entries + first2 + row) : 0u;
      cnt1 = cnt2;
      if (t + 2 * G < A.ntiles) {
        first2 = __ldg(A.tiles + 3 * (t + 2 * G) + 1);
        cnt2 = __ldg(A.tiles + 3 * (t + 2 * G) + 2);
      }
      const bool live = (uint32_t)row < cnt;
      const bool warp_live = (uint32_t)(32 * quad) < cnt;  // warp-uniform
      const int rot = (int)(ent & 63u);
      uint32_t* dst = tc_dst(A, ent >> 6, EW);
      // column blocks c0 .. c0 + 3 of a chunk hold coefficients m-1-c0 .. m-4-c0: positions P, P-1,
      // P-2, P-3 (mod 2m) of the rotated element, c0 a multiple of 4.  P odd: (P-1, P) and (P-3, P-2)
      // are 32-byte sectors; P even: (P-2, P-1) is one, P and P-3 are stored alone.
      const bool podd = ((MM - 1 + rot) & 1) != 0;
      for (int ch = 0; ch < NCH; ++ch, ++g) {
        const int b = g & 1;
#ifdef DKSS_TC_TRACE
        if (warp == 0 && lane == 0) TC_STAMP(2, ev++);  // before the accumulator wait
#endif
        tc::mbar_wait_parity(&tfull[b], (g >> 1) & 1);
        tc::fence_after();
#ifdef DKSS_TC_TRACE
        if (warp == 0 && lane == 0) TC_STAMP(2, ev++);  // accumulators ready
#endif
        // the four coefficients are loaded one ahead: coefficient h + 1's tcgen05.ld is in flight
        // while coefficient h is reduced (the TMEM read of a chunk takes about as long as its MMAs,
        // so it must overlap the reduction, not precede it)
        int32_t Za[32], Zb[32];
        const uint32_t caddr = tmem + (uint32_t)(b * kTcNChunk) + ((uint32_t)(32 * quad) << 16) + q * 64;
        const int c0 = ch * CPC + 4 * q;  // first column block of this warp's four
        const int P = (MM - 1 - c0 + rot) & (2 * MM - 1);
        uint32_t o0[4], o1[4], o2[4], o3[4];
        auto reduce = [&](const int32_t(&Z)[32], int z0, int h, uint32_t(&o)[4]) {
          tc::reduce_coeff16(Z, z0, A.p3, ((P - h) & (2 * MM - 1)) >= MM, o);
        };
        auto at = [&](int h) { return dst + ((P - h) & (MM - 1)) * 4; };
#if defined(DKSS_TC_EXP_NOEPI) || defined(DKSS_TC_EXP_NOSTORE)  // experiment builds only
        const bool st = live && P == 0x7fffffff;
#else
        const bool st = live;
#endif
        if (warp_live) {
          tc::tmem_ld32_nowait(caddr, Za);
          tc::tmem_ld_wait();
          tc::tmem_ld32_nowait(caddr + 32, Zb);  // in flight while the first two are reduced
          reduce(Za, 0, 0, o0);
          reduce(Za, 16, 1, o1);
          if (st) {
            if (podd)
              tc::st256(at(1), o1, o0);
            else
              *reinterpret_cast<uint4*>(at(0)) = make_uint4(o0[0], o0[1], o0[2], o0[3]);
          }
          tc::tmem_ld_wait();
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[b]);  // this warp's columns of buffer b are read
#ifdef DKSS_TC_TRACE
        if (warp == 0 && lane == 0) TC_STAMP(2, ev++);  // buffer released
#endif
        if (warp_live) {
          reduce(Zb, 0, 2, o2);
          if (st && !podd) tc::st256(at(2), o2, o1);
          reduce(Zb, 16, 3, o3);
          if (st) {
            if (podd)
              tc::st256(at(3), o3, o2);
            else
              *reinterpret_cast<uint4*>(at(3)) = make_uint4(o3[0], o3[1], o3[2], o3[3]);
          }
        }
#ifdef DKSS_TC_TRACE
        if (warp == 0 && lane == 0) TC_STAMP(2, ev++);  // chunk stored
#endif
      }
    }
  }
  if (A.peer) __threadfence_system();  // fused exchange: stores to other GPUs performed
  tc::fence_before();
  __syncthreads();
#ifdef DKSS_TC_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_tc_trace[trace_slot][0][511] = clock64();
    g_tc_launch = g_tc_launch + 1;
  }
#endif
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * kTcNChunk));
}

// W tables of the tensor-core twiddle products: for every table row s, the effective twiddle
// t = w R^-1 of the stored (Montgomery-form) row w (ring_mul computes REDC(x w)); with
// ck[k] = 2^(32 + 8k) mod p, C_l,k = t_l 256^k 2^32 = mont_mul(w_l, ck[k]).  With l' = 2m-2-t:
// W[s][t][d] = the 16 bytes k = 0..15 of digit d of (l' >= m-1 ? C_{l'-m+1,k} : p - C_{l'+1,k})
// written in (-p/2, p/2) with balanced base-256 digits (16 suffice: p/2 < 127 (256^16 - 1) / 255).
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
    uint4* out = reinterpret_cast<uint4*>(vtab + (size_t)(s * LP + (LP - 1 - lp)) * 16 * 16);
#pragma unroll
    for (int d = 0; d < 16; ++d) out[d] = make_uint4(unit[d][0], unit[d][1], unit[d][2], unit[d][3]);
  }
}

}  // namespace dkss
