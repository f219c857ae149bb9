// tc_ring.cu -- prototype: the DKSS twiddle product on the 5th-generation tensor cores.
//
// A twiddle step multiplies many ring elements x (R = (Z/p)[alpha]/(alpha^m + 1), m coefficients
// of L = 4 u32 limbs) by ONE table entry t = rho^s (bigmul/dkss.py:480-492: every (vv, l) with the
// same s uses the same rho^s).  Over bytes that is a dense integer GEMM:
//
//   x_i = sum_k X[i][k] 256^k  (u8 digits: the element's own little-endian bytes),
//   T_l = t_l * 2^160 mod p written in balanced signed base-256 digits e[l][0..16] (s8),
//   Z[j][d] = sum_{i,k} X[i][k] * B[(j,d)][(i,k)],   B[(j,d)][(i,k)] = digit d-k of (+-T_{(j-i) mod m})
//             (sign -1 where the negacyclic product wraps, i > j),
//   z_j = (sum_d Z[j][d] 256^d) * 2^-160 mod p = x * t  (coefficient j)
//
// so ONE CTA tile is D[128 rows][m*32] += A[128][m*16] (u8, the elements) x B^T (s8, the twiddle's
// Toeplitz expansion), tcgen05.mma kind::i8 with int32 accumulators in TMEM (|Z| < 2^25), and the
// epilogue (tcgen05.ld, 32 byte-position sums -> one 288-bit integer -> Montgomery REDC with
// R = 2^160 using the Proth form of p) runs on the CUDA cores.
//
// This file is the isolated-core benchmark of VERDICT r1 item 7: tc_ring_run() multiplies `rows`
// elements by one twiddle `reps` times and reports the time; tools/tc_ring_check.py checks the
// products bit-exactly against the C oracle's r_mul and compares ring products/s with the
// IMAD.WIDE core (tools/bench_core.cu).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared
//        -Xcompiler -fPIC -o tools/libtc_ring.so tools/tc_ring.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace {

constexpr int kL = 4;            // u32 limbs per residue (p = 81 * 2^121 + 1)
constexpr int kRows = 128;       // UMMA M
constexpr int kNChunk = 256;     // UMMA N per instruction / per TMEM buffer
constexpr int kThreads = 256;    // 8 warps: warp 0 lane 0 issues MMA; all 8 run the epilogue

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows x 16 bytes stored
// as 128 contiguous bytes; LBO = byte distance between the two 16-byte K halves of one MMA step,
// SBO = byte distance between 8-row groups (cute/arch/mma_sm100_desc.hpp SmemDescriptor)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor kind::i8: D s32, A u8, B s8, both K-major, N, M
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 32 consecutive TMEM columns of this thread's lane
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

// z = (sum_d Z[d] 256^d + p 2^160) * 2^-160 mod p, canonical (p = 81 * 2^121 + 1: -p^-1 = -1 mod 2^32
// and q * p touches limbs 0, 3, 4)
__device__ __forceinline__ void reduce_coeff(const int32_t (&Z)[32], uint32_t (&out)[kL]) {
  long long acc[9];
#pragma unroll
  for (int w = 0; w < 9; ++w) acc[w] = 0;
#pragma unroll
  for (int d = 0; d < 32; ++d) acc[d >> 2] += (long long)Z[d] << (8 * (d & 3));
  uint32_t t[10];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    acc[w + 1] += acc[w] >> 32;  // arithmetic: carries and borrows
    t[w] = (uint32_t)acc[w];
  }
  // + p * 2^160 (limb 5 += 1, limb 8 += 81 << 25) makes the value non-negative (|v| < 2^276)
  long long top = acc[8] + (81LL << 25);
  {
    unsigned long long s = (unsigned long long)t[5] + 1u;
    t[5] = (uint32_t)s;
    unsigned long long c = s >> 32;
    s = (unsigned long long)t[6] + c;
    t[6] = (uint32_t)s;
    c = s >> 32;
    s = (unsigned long long)t[7] + c;
    t[7] = (uint32_t)s;
    c = s >> 32;
    top += (long long)c;
  }
  t[8] = (uint32_t)top;
  t[9] = (uint32_t)(top >> 32);
  // 5 REDC steps: q = -t0 mod 2^32, t += q p, t >>= 32
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    const uint32_t q = 0u - t[0];
    // t0 + q = 0 mod 2^32 with carry (t0 != 0)
    unsigned long long c = (t[0] != 0u) ? 1ull : 0ull;
    const unsigned long long hq = (unsigned long long)q * 81ull << 25;  // q * 81 * 2^121 at limb 3 (bit 25)
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
  // t < 2^128 + p < 3p: subtract p (limbs 1, 0, 0, 81 << 25) while that does not borrow
  const uint32_t P3 = 81u << 25;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    uint32_t r[5], b;
    r[0] = t[0] - 1u;
    b = t[0] < 1u;
    r[1] = t[1] - b;
    b = t[1] < b;
    r[2] = t[2] - b;
    b = t[2] < b;
    r[3] = t[3] - P3 - b;
    b = (unsigned long long)t[3] < (unsigned long long)P3 + b;
    r[4] = t[4] - b;
    b = t[4] < b;
    if (!b) {
#pragma unroll
      for (int q = 0; q < 5; ++q) t[q] = r[q];
    }
  }
#pragma unroll
  for (int q = 0; q < kL; ++q) out[q] = t[q];
}

// Each CTA walks tiles of 128 elements; B (the twiddle's Toeplitz expansion, s8, K-major core
// layout, NTOT x K bytes) is read from global per N-chunk.  A tile = the elements' bytes.
template <int MM>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_twiddle(const uint32_t* __restrict__ x, const int8_t* __restrict__ bmat, uint32_t* __restrict__ z,
                 int rows, int reps) {
  constexpr int K = MM * 16;          // bytes per element
  constexpr int NTOT = MM * 32;       // (coefficient, byte position) columns
  constexpr int NCHUNKS = NTOT / kNChunk;
  constexpr int KSTEPS = K / 32;      // one MMA step covers 32 bytes of K
  constexpr int SBO = (K / 16) * 128; // bytes between 8-row groups
  constexpr int ABYTES = kRows * K;
  constexpr int BBYTES = kNChunk * K;
  constexpr int COEF_PER_CHUNK = kNChunk / 32;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + ABYTES;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(2 * kNChunk));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t idesc = make_idesc(kRows, kNChunk);
  uint32_t phase = 0;
  const int ntiles = (rows + kRows - 1) / kRows;

  for (int rep = 0; rep < reps; ++rep) {
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int row0 = tile * kRows;
      // A tile: row r, 16-byte chunk c -> (r / 8) * SBO + c * 128 + (r % 8) * 16
      for (int i = threadIdx.x; i < kRows * (K / 16); i += kThreads) {
        const int r = i / (K / 16), c = i % (K / 16);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row0 + r < rows) v = *reinterpret_cast<const uint4*>(x + (size_t)(row0 + r) * MM * kL + c * 4);
        *reinterpret_cast<uint4*>(sA + (r / 8) * SBO + c * 128 + (r % 8) * 16) = v;
      }
      for (int ch = 0; ch < NCHUNKS; ++ch) {
        // B chunk (already in core layout in global): 256 rows n x K bytes
        const uint4* src = reinterpret_cast<const uint4*>(bmat + (size_t)ch * BBYTES);
        for (int i = threadIdx.x; i < BBYTES / 16; i += kThreads) reinterpret_cast<uint4*>(sB)[i] = src[i];
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        const uint32_t tbuf = tmem + (uint32_t)((ch & 1) * kNChunk);
        if (warp == 0 && lane == 0) {
#pragma unroll
          for (int ks = 0; ks < KSTEPS; ++ks) {
            const uint64_t da = make_desc(smem_u32(sA) + ks * 256, 128, SBO);
            const uint64_t db = make_desc(smem_u32(sB) + ks * 256, 128, SBO);
            mma_i8(tbuf, da, db, idesc, ks > 0 ? 1u : 0u);
          }
          mma_commit(&mbar);
        }
        mbar_wait(&mbar, phase);
        phase ^= 1;
        tc_fence_after();
        // epilogue: warp w reads lanes 32 (w % 4) .. +31 (its rows); warps w and w + 4 split the
        // chunk's coefficients
        const int r = 32 * (warp % 4) + lane;
        const uint32_t lane_addr = tbuf + ((uint32_t)(32 * (warp % 4)) << 16);
        for (int cj = warp / 4; cj < COEF_PER_CHUNK; cj += 2) {
          int32_t Zv[32];
          tmem_ld32(lane_addr + cj * 32, Zv);
          uint32_t o[kL];
          reduce_coeff(Zv, o);
          const int j = ch * COEF_PER_CHUNK + cj;
          if (row0 + r < rows)
            *reinterpret_cast<uint4*>(z + (size_t)(row0 + r) * MM * kL + j * kL) = make_uint4(o[0], o[1], o[2], o[3]);
        }
        tc_fence_before();
        __syncthreads();  // smem B / TMEM buffer free for the next chunk
        tc_fence_after();
      }
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * kNChunk));
}

template <int MM>
int run(const uint32_t* hx, const int8_t* hb, uint32_t* hz, int rows, int reps, int grid, float* ms) {
  constexpr int K = MM * 16, NTOT = MM * 32;
  const size_t xbytes = (size_t)rows * MM * kL * 4, bbytes = (size_t)NTOT * K;
  uint32_t *dx, *dz;
  int8_t* db;
  if (cudaMalloc(&dx, xbytes) || cudaMalloc(&dz, xbytes) || cudaMalloc(&db, bbytes)) return -1;
  cudaMemcpy(dx, hx, xbytes, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, bbytes, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)kRows * K + (size_t)kNChunk * K;
  auto k = k_tc_twiddle<MM>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -2;
  k<<<grid, kThreads, smem>>>(dx, db, dz, rows, 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "tc_ring: %s\n", cudaGetErrorString(e));
    return -3;
  }
  cudaMemcpy(hz, dz, xbytes, cudaMemcpyDeviceToHost);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, kThreads, smem>>>(dx, db, dz, rows, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  e = cudaGetLastError();
  cudaFree(dx);
  cudaFree(dz);
  cudaFree(db);
  return e == cudaSuccess ? 0 : -4;
}

}  // namespace

extern "C" int tc_ring_run(int m, const uint32_t* x, const int8_t* bmat, uint32_t* z, int rows, int reps, int grid,
                           float* ms) {
  if (m == 16) return run<16>(x, bmat, z, rows, reps, grid, ms);
  if (m == 32) return run<32>(x, bmat, z, rows, reps, grid, ms);
  return -10;
}
