// Integer-pipe microbenchmark for the DKSS ring-product roofline (SURVEY.md §8(d) asks for a
// measured IMAD peak, which MEASURED_PEAKS.json does not hold).  Each kernel keeps ILP
// independent accumulator chains per thread and issues one instruction class in a tight loop.
// Output: one JSON line per instruction class with ops/clk/SM and ops/s at the observed clock.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_imad tools/microbench_imad.cu -lnvidia-ml
// SM clocks are sampled with NVML while each kernel runs (~0.3 s per kernel).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvml.h>
#include <thread>
#include <atomic>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ILP = 8;

__global__ void k_imad_wide(uint64_t* out, long long* cyc, int iters) {
  uint64_t acc[ILP];
  uint32_t a[ILP], b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { a[j] = threadIdx.x * 7 + j; b[j] = blockIdx.x * 13 + j * 3 + 1; acc[j] = j; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(a[j]), "r"(b[j]));
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imad_lo(uint64_t* out, long long* cyc, int iters) {
  uint32_t acc[ILP], a[ILP], b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { a[j] = threadIdx.x * 7 + j; b[j] = blockIdx.x * 13 + j * 3 + 1; acc[j] = j; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[j]) : "r"(a[j]), "r"(b[j]));
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imad_hi(uint64_t* out, long long* cyc, int iters) {
  uint32_t acc[ILP], a[ILP], b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { a[j] = threadIdx.x * 7 + j; b[j] = blockIdx.x * 13 + j * 3 + 1; acc[j] = j; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(acc[j]) : "r"(a[j]), "r"(b[j]));
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// lo/hi pair with carry into a 3-word column accumulator (classic product scanning step)
__global__ void k_madc_chain(uint64_t* out, long long* cyc, int iters) {
  uint32_t c0[ILP], c1[ILP], c2[ILP], a[ILP], b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { a[j] = threadIdx.x * 7 + j; b[j] = blockIdx.x * 13 + j * 3 + 1; c0[j] = j; c1[j] = 0; c2[j] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j)
        asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                     : "+r"(c0[j]), "+r"(c1[j]), "+r"(c2[j]) : "r"(a[j]), "r"(b[j]));
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += c0[j] + c1[j] + c2[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_iadd3(uint64_t* out, long long* cyc, int iters) {
  uint32_t acc[ILP], a[ILP], b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { a[j] = threadIdx.x * 7 + j; b[j] = blockIdx.x * 13 + j * 3 + 1; acc[j] = j; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) asm volatile("add.u32 %0, %0, %1;" : "+r"(acc[j]) : "r"(a[j]));
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j] + b[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(uint64_t*, long long*, int);

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  const int threads = 256, blocks_per_sm = 4, blocks = sms * blocks_per_sm, iters = 4096 * 48;
  uint64_t* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(uint64_t) * blocks * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * blocks));
  struct { const char* name; kfn f; int ops_per_inner; } ks[] = {
      {"IMAD.WIDE.U32 (mad.wide.u32, 64-bit acc)", k_imad_wide, 1},
      {"IMAD (mad.lo.u32)", k_imad_lo, 1},
      {"IMAD.HI (mad.hi.u32)", k_imad_hi, 1},
      {"mad.lo.cc+madc.hi.cc+addc (1 limb product)", k_madc_chain, 1},
      {"IADD (add.u32)", k_iadd3, 1},
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  long long* hc = new long long[blocks];
  nvmlDevice_t nvdev;
  bool nv = nvmlInit() == NVML_SUCCESS && nvmlDeviceGetHandleByIndex(0, &nvdev) == NVML_SUCCESS;
  for (auto& k : ks) {
    for (int rep = 0; rep < 2; ++rep) {  // first pass = warm-up
      std::atomic<bool> stop(false);
      std::vector<unsigned> clk;
      std::thread sampler([&] {
        while (nv && !stop.load()) {
          unsigned c = 0;
          if (nvmlDeviceGetClockInfo(nvdev, NVML_CLOCK_SM, &c) == NVML_SUCCESS) clk.push_back(c);
          std::this_thread::sleep_for(std::chrono::milliseconds(5));
        }
      });
      CK(cudaEventRecord(e0));
      k.f<<<blocks, threads>>>(out, cyc, iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      stop = true;
      sampler.join();
      CK(cudaGetLastError());
      if (rep == 0) continue;
      std::sort(clk.begin(), clk.end());
      unsigned med = clk.empty() ? 0 : clk[clk.size() / 2];
      float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
      CK(cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
      double avgc = 0; for (int i = 0; i < blocks; ++i) avgc += hc[i]; avgc /= blocks;
      double ops = (double)blocks * threads * iters * 8 * ILP * k.ops_per_inner;
      double ops_per_clk_sm = ops / sms / avgc;
      double ghz = avgc / (ms * 1e-3) / 1e9;  // SM cycles per wall second (all blocks concurrent)
      printf("{\"instr\": \"%s\", \"ops_per_clk_per_sm\": %.2f, \"ops_per_s\": %.4e, \"kernel_ms\": %.4f, \"sm_ghz_est\": %.3f, \"nvml_sm_mhz_median\": %u, \"nvml_samples\": %zu, \"sms\": %d}\n",
             k.name, ops_per_clk_sm, ops / (ms * 1e-3), ms, ghz, med, clk.size(), sms);
    }
  }
  printf("{\"clock_rate_attr_mhz\": %d}\n", clk_khz / 1000);
  return 0;
}
