// microbench_tmem_ld.cu -- tcgen05.ld (TMEM -> registers) throughput on this GPU: the read rate the
// tensor-core twiddle kernel's epilogue (csrc/dkss_tc.cuh) is held against in DESIGN.md section 3b.
// One CTA per SM allocates all 512 TMEM columns; W warps (W/4 per lane quadrant) loop over
// back-to-back 32x32b loads of X columns (x16 or x32) from their quadrant, one tcgen05.wait::ld per
// load or per two loads (two register sets).  CUDA events around the launch.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench_tmem_ld tools/microbench_tmem_ld.cu
// run:   tools/microbench_tmem_ld [iters]   -> one JSON line per shape
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, int32_t (&v)[32]) {
  if constexpr (X == 32) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
  }
}

template <int X, int PER_WAIT>
__global__ void __launch_bounds__(512, 1) k_ld(int iters, int warps, int* sink) {
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_sh)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_sh;
  int acc = 0;
  if (warp < warps) {
    const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    int32_t v[32], w[32];
#pragma unroll 1
    for (int it = 0; it < iters; it += PER_WAIT) {
      ld<X>(base + (uint32_t)((it * X + (warp >> 2) * 64) & 511), v);
      if (PER_WAIT == 2) ld<X>(base + (uint32_t)(((it + 1) * X + (warp >> 2) * 64) & 511), w);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      acc += v[0];
      if (PER_WAIT == 2) acc += w[0];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = acc;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int X, int PER_WAIT>
void run(int iters, int warps, int sms, int clk_khz, int* sink) {
  k_ld<X, PER_WAIT><<<sms, 512>>>(1000, warps, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_ld<X, PER_WAIT><<<sms, 512>>>(iters, warps, sink);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  if (e != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    exit(1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes_per_sm = (double)warps * iters * 32.0 * X * 4.0;
  const double clocks = ms * 1e-3 * clk_khz * 1e3;
  printf("{\"instr\": \"tcgen05.ld.32x32b.x%d\", \"warps\": %d, \"loads_per_wait\": %d, \"iters_per_warp\": %d, \"kernel_ms\": %.3f, "
         "\"bytes_per_clk_per_sm_at_max_clock\": %.1f, \"clocks_per_load_per_warp\": %.1f, \"max_clock_mhz\": %d}\n",
         X, warps, PER_WAIT, iters, ms, bytes_per_sm / clocks, clocks / iters, clk_khz / 1000);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 200000;
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int* sink;
  cudaMalloc(&sink, sms * 4);
  for (int w : {4, 8, 16}) {
    run<32, 1>(iters, w, sms, clk, sink);
    run<16, 1>(iters, w, sms, clk, sink);
    run<32, 2>(iters, w, sms, clk, sink);
    run<16, 2>(iters, w, sms, clk, sink);
  }
  return 0;
}
