// Isolated throughput of the ring-product core (ring_mul_rows) with operands resident in
// shared memory: each CTA repeatedly multiplies NE elements (x digits, y digits) and folds the
// results into a checksum.  Reports ring products/s and 32x32 limb products/s (m^2 L^2 per
// ring product, SURVEY.md §8(d) work unit) for m = 16 / 32, L = 4, and T = 2 / 4.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -o tools/bench_core tools/bench_core.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1503_04955_b200/csrc/dkss_kernels.cuh"

using namespace dkss;

template <int MM, int L, int T, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_core(const uint32_t* __restrict__ seed, uint32_t* out, int reps, ModCtx mc) {
  constexpr int ES = Smem<MM, L>::ES;
  constexpr int TPE = MM / T;
  constexpr int NE = NT / TPE;
  __shared__ __align__(16) uint32_t sx[NE * ES], sy[NE * ES];
  for (int i = threadIdx.x; i < NE * ES; i += NT) {
    sx[i] = seed[(blockIdx.x * 7 + i) & 4095];
    sy[i] = seed[(blockIdx.x * 13 + i + 77) & 4095] & 0x7FFFFFFF;
  }
  __syncthreads();
  const int el = threadIdx.x / TPE, k0 = (threadIdx.x % TPE) * T;
  uint32_t chk = 0;
  for (int r = 0; r < reps; ++r) {
    uint32_t w[T][L];
    const uint32_t* xp = sx + el * ES;
    const uint32_t rr = (uint32_t)r & 1u;
    auto xl = [&](int i, uint32_t(&d)[L]) {
      ld_res<L>(d, xp + i * L);
#pragma unroll
      for (int q = 0; q < L; ++q) d[q] ^= rr;
    };
    ring_mul<MM, L, ResS<L>, decltype(xl), ResS<L>, T>(ResS<L>{sy + el * ES}, xl, ResS<L>{sy + el * ES}, k0, mc, w);
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < L; ++q) chk ^= w[t][q] + r;
  }
  out[blockIdx.x * NT + threadIdx.x] = chk;
}

template <int MM, int L, int T, int NT, int MINB>
void run(const char* name, const uint32_t* seed, uint32_t* out, ModCtx mc) {
  auto k = k_core<MM, L, T, NT, MINB>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  const int grid = 148 * occ, reps = 64;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<grid, NT>>>(seed, out, 2, mc);
  cudaEventRecord(e0);
  k<<<grid, NT>>>(seed, out, reps, mc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double rp = (double)grid * (NT / (MM / T)) * reps;  // ring products
  const double lp = rp * MM * MM * L * L;
  printf("{\"variant\": \"%s\", \"m\": %d, \"L\": %d, \"T\": %d, \"threads\": %d, \"regs\": %d, \"stack\": %zu, \"occ\": %d, "
         "\"ms\": %.3f, \"ring_products_per_s\": %.4e, \"limb_products_per_s\": %.4e, \"err\": \"%s\"}\n",
         name, MM, L, T, NT, fa.numRegs, fa.localSizeBytes, occ, ms, rp / (ms * 1e-3), lp / (ms * 1e-3),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint32_t* seed;
  uint32_t* out;
  cudaMalloc(&seed, 4096 * 4);
  cudaMalloc(&out, 148 * 32 * 1024 * 4);
  uint32_t h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = i * 2654435761u + 12345u;
  cudaMemcpy(seed, h, sizeof h, cudaMemcpyHostToDevice);
  ModCtx mc{};
  // p = 81*2^121 + 1
  mc.p[0] = 1; mc.p[1] = 0; mc.p[2] = 0; mc.p[3] = 81u << 25;
  mc.pinv = 0xFFFFFFFFu;
  mc.pf_inv = 1.0f / (float)(81.0 * 33554432.0);

  mc.proth = 1;
  run<16, 4, 2, 256, 2>("m16 T2 NT256 minb2", seed, out, mc);
  run<16, 4, 2, 256, 3>("m16 T2 NT256 minb3", seed, out, mc);
  run<16, 4, 2, 128, 5>("m16 T2 NT128 minb5", seed, out, mc);
  run<16, 4, 2, 384, 2>("m16 T2 NT384 minb2", seed, out, mc);
  run<32, 4, 2, 256, 2>("m32 T2 NT256 minb2", seed, out, mc);
  run<32, 4, 2, 256, 3>("m32 T2 NT256 minb3", seed, out, mc);
  return 0;
}
