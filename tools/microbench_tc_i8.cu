// microbench_tc_i8.cu -- dense int8 tensor-core issue rate on this GPU (the roofline peak of the
// tensor-core twiddle kernel, csrc/dkss_tc.cuh): one CTA per SM, one thread issues back-to-back
// tcgen05.mma.cta_group::1.kind::i8 (M = 128, N = 256, K = 32: u8 x s8 -> s32 in TMEM) from
// shared-memory operands with the same descriptors as the product kernel, alternating two TMEM
// accumulators; CUDA events around the launch, NVML-free (the caller samples clocks).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench_tc_i8 tools/microbench_tc_i8.cu
// run:   tools/microbench_tc_i8 [iters]   -> one JSON line
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

constexpr int kN = 256, kK = 32;

template <int kM>
__global__ void __launch_bounds__(128, 1) k_mma_i8(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + kN) * kK / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_sh)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_sh;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
    const uint32_t a = smem_u32(smem), b = a + 128 * kK;
    const uint64_t da = make_desc(a, 128, 256), db = make_desc(b, 128, 256);
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (uint32_t)((it & 1) * kN);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
          "l"(da), "l"(db), "r"(idesc), "r"(it > 1 ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred done;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t@!done bra W;\n\t}\n" ::"r"(
            smem_u32(&mbar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (threadIdx.x == 0) sink[blockIdx.x] = (int)v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

template <int kM>
int run(int iters, int sms, int clk) {
  const size_t smem = (size_t)(128 + kN) * kK + 1024;
  cudaFuncSetAttribute(k_mma_i8<kM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int* sink;
  cudaMalloc(&sink, sms * 4);
  k_mma_i8<kM><<<sms, 128, smem>>>(1000, sink);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mma_i8<kM><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * kM * kN * kK * (double)iters * sms;
  const double per_clk_sm = ops / 2 / (ms * 1e-3) / sms / (clk * 1e3);
  printf("{\"instr\": \"tcgen05.mma.cta_group::1.kind::i8 M%d N256 K32, u8 x s8 -> s32, smem operands\", \"M\": %d, "
         "\"iters_per_sm\": %d, \"sms\": %d, \"kernel_ms\": %.3f, \"ns_per_mma\": %.2f, \"ops_per_s\": %.4e, \"tops\": %.1f, "
         "\"macs_per_clk_per_sm_at_max_clock\": %.1f, \"max_clock_mhz\": %d}\n",
         kM, kM, iters, sms, ms, ms * 1e6 / iters, ops / (ms * 1e-3), ops / (ms * 1e-3) / 1e12, per_clk_sm, clk / 1000);
  cudaFree(sink);
  return 0;
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 200000;
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  // M = 128 first: the line bench.py reads (profiles/tc_i8_peak.json) is the first one
  return run<128>(iters, sms, clk) | run<64>(iters, sms, clk);
}
