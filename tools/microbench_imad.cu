// Integer-pipe microbenchmark for the DKSS ring-product roofline (SURVEY.md §8(d) asks for a
// measured IMAD peak, which MEASURED_PEAKS.json does not hold).
//
// Each thread runs ILP independent dependency chains; every step of a chain uses the previous
// result as a multiplier operand, so ptxas can neither hoist nor strength-reduce the products
// (an earlier version with loop-invariant operands was reduced to 64-bit adds).  1024 threads
// per SM, SM clock sampled with NVML while each kernel runs.  One JSON line per instruction.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_imad tools/microbench_imad.cu -lnvidia-ml
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nvml.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));            \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

constexpr int ILP = 8;
constexpr int UNR = 8;

// acc = lo(acc) * b + acc  (IMAD.WIDE.U32 with a 64-bit addend)
__global__ void k_imad_wide_u32(uint64_t* out, int iters) {
  uint64_t acc[ILP];
  uint32_t b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { acc[j] = threadIdx.x * 7 + j + 1; b[j] = blockIdx.x * 13 + j * 3 + 1; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) {
        uint32_t lo = (uint32_t)acc[j];
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(lo), "r"(b[j]));
      }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_wide_s32(uint64_t* out, int iters) {
  int64_t acc[ILP];
  int32_t b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { acc[j] = threadIdx.x * 7 + j + 1; b[j] = -(int)(blockIdx.x * 13 + j * 3 + 1); }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) {
        int32_t lo = (int32_t)acc[j];
        asm volatile("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(lo), "r"(b[j]));
      }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 16 independent 64-bit accumulators += x * y_j; x changes every step through one LOP3
// (ALU pipe) so nothing can be hoisted or reassociated across steps
__global__ void k_imad_wide_clean(uint64_t* out, int iters) {
  constexpr int N = 16;
  uint64_t acc[N];
  uint32_t y[N];
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
#pragma unroll
  for (int j = 0; j < N; ++j) { acc[j] = j; y[j] = blockIdx.x * 13 + j * 0x9E3779B9u + 1; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < N; ++j) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(x), "r"(y[j]));
      x ^= (uint32_t)acc[u];
    }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < N; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// as above with a carry-out into a per-accumulator counter (radix-2^32 product scanning)
__global__ void k_imad_wide_cc(uint64_t* out, int iters) {
  constexpr int N = 12;
  uint32_t lo[N], hi[N], cy[N], y[N];
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
#pragma unroll
  for (int j = 0; j < N; ++j) { lo[j] = j; hi[j] = 0; cy[j] = 0; y[j] = blockIdx.x * 13 + j * 0x9E3779B9u + 1; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < N; ++j)
        asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                     : "+r"(lo[j]), "+r"(hi[j]), "+r"(cy[j])
                     : "r"(x), "r"(y[j]));
      x ^= lo[u];
    }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < N; ++j) s += lo[j] + hi[j] + cy[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// acc = acc * b + c  (32-bit IMAD)
__global__ void k_imad_lo(uint64_t* out, int iters) {
  uint32_t acc[ILP], b[ILP], c[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { acc[j] = threadIdx.x * 7 + j + 1; b[j] = blockIdx.x * 13 + j * 3 + 1; c[j] = j * 5 + 3; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(acc[j]) : "r"(b[j]), "r"(c[j]));
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// acc = hi(acc * b) + c
__global__ void k_imad_hi(uint64_t* out, int iters) {
  uint32_t acc[ILP], b[ILP], c[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { acc[j] = threadIdx.x * 7 + j + 1; b[j] = 0x9E3779B9u + blockIdx.x * 13 + j; c[j] = j * 5 + 3; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(acc[j]) : "r"(b[j]), "r"(c[j]));
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// one 32x32 limb product into a 3-word column accumulator (product scanning), multiplier
// taken from the running low word
__global__ void k_madc_chain(uint64_t* out, int iters) {
  uint32_t c0[ILP], c1[ILP], c2[ILP], b[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { c0[j] = threadIdx.x * 7 + j + 1; c1[j] = 0; c2[j] = 0; b[j] = blockIdx.x * 13 + j * 3 + 1; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int j = 0; j < ILP; ++j) {
        uint32_t a = c0[j];
        asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                     : "+r"(c0[j]), "+r"(c1[j]), "+r"(c2[j])
                     : "r"(a), "r"(b[j]));
      }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += c0[j] + c1[j] + c2[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef void (*kfn)(uint64_t*, int);

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int threads = 256, blocks_per_sm = 4, blocks = sms * blocks_per_sm, iters = 4096 * 24;
  uint64_t* out;
  CK(cudaMalloc(&out, sizeof(uint64_t) * blocks * threads));
  struct {
    const char* name;
    kfn f;
  } ks[] = {
      {"IMAD.WIDE.U32 clean (16 acc, x varies)", k_imad_wide_clean},
      {"IMAD.WIDE.U32 + carry-out (12 col pairs, x varies)", k_imad_wide_cc},
      {"IMAD.WIDE.U32 (mad.wide.u32, 64-bit acc)", k_imad_wide_u32},
      {"IMAD.WIDE (mad.wide.s32, 64-bit acc)", k_imad_wide_s32},
      {"IMAD (mad.lo.u32)", k_imad_lo},
      {"IMAD.HI (mad.hi.u32)", k_imad_hi},
      {"mad.lo.cc+madc.hi.cc+addc (1 limb product)", k_madc_chain},
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
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
      k.f<<<blocks, threads>>>(out, iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      stop = true;
      sampler.join();
      CK(cudaGetLastError());
      if (rep == 0) continue;
      std::sort(clk.begin(), clk.end());
      const unsigned med = clk.empty() ? 0 : clk[clk.size() / 2];
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double per_iter = (k.f == k_imad_wide_clean) ? 64.0 : (k.f == k_imad_wide_cc) ? 48.0 : (double)UNR * ILP;
      const double ops = (double)blocks * threads * iters * per_iter;
      const double per_s = ops / (ms * 1e-3);
      printf("{\"instr\": \"%s\", \"ops_per_s\": %.4e, \"per_clk_per_sm_at_nvml_clock\": %.2f, \"kernel_ms\": %.3f, "
             "\"nvml_sm_mhz_median\": %u, \"nvml_samples\": %zu, \"sms\": %d}\n",
             k.name, per_s, med ? per_s / sms / (med * 1e6) : 0.0, ms, med, clk.size(), sms);
    }
  }
  return 0;
}
