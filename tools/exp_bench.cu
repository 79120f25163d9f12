// Microbenchmark: softmax-exponential throughput per SM (FFMA + ex2 + bf16
// pack + 16-byte smem store per 8 values), one to four warps per SMSP, with
// and without a share of the exponentials on the FMA pipe.  Development
// tool.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/exp_bench tools/exp_bench.cu -I paper_2512_16615_b200/csrc
#include <cstdint>
#include <cstdio>

#include "tc_common.cuh"

using namespace llsa_tc;

template <int kPoly>  // pairs out of every 4 on the FMA pipe
__global__ void exp_bench(int iters, float c2, float nb, unsigned long long* out, uint32_t* sink) {
  __shared__ __align__(16) uint8_t sm[32 * 1024];
  const uint32_t row = threadIdx.x & 127;
  float s[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) s[k] = (float)((threadIdx.x * 7 + k * 13) & 31) * 0.03f;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x >> 7) * 8192 % 16384;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      uint32_t pk[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x0 = fmaf(s[g * 8 + 2 * k], c2, nb);
        const float x1 = fmaf(s[g * 8 + 2 * k + 1], c2, nb);
        const bool poly = k < kPoly;
        pk[k] = pack_bf16(poly ? ex2_poly(x0) : ex2(x0), poly ? ex2_poly(x1) : ex2(x1));
      }
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(base + swz(row, g)),
                   "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]));
    }
    nb += 1e-7f;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
  if (threadIdx.x == 0) sink[blockIdx.x] = sm[threadIdx.x];
}

int main() {
  unsigned long long* d_out;
  uint32_t* sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&sink, 1024 * 4);
  const int iters = 1000;
  for (int poly = 0; poly < 3; ++poly)
    for (int warps : {4, 8, 16}) {
      if (poly == 0) exp_bench<0><<<148, warps * 32>>>(iters, 0.18f, -3.f, d_out, sink);
      if (poly == 1) exp_bench<1><<<148, warps * 32>>>(iters, 0.18f, -3.f, d_out, sink);
      if (poly == 2) exp_bench<2><<<148, warps * 32>>>(iters, 0.18f, -3.f, d_out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long cyc = 0;
      cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
      const double per_warp_iter = (double)cyc / iters;  // 64 values per thread per iter
      printf("poly %d/4 warps %2d: %7.1f cycles per 64 values/thread; %.2f exps/clk/SM %s\n", poly,
             warps, per_warp_iter, 64.0 * 32 * warps / per_warp_iter,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
