// Microbenchmark: TMEM → register read throughput per SM for the tcgen05.ld
// shapes the attention kernels use.  Development tool, not part of the
// library.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/tmem_bench tools/tmem_bench.cu -I paper_2512_16615_b200/csrc
#include <cstdio>
#include <cstdint>
#include "umma.cuh"

using namespace llsa_umma;

__device__ __forceinline__ void ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

// mode 0: 32x32b.x32 + wait each; 1: two x32 per wait; 2: 16x256b.x8 + wait;
// 3: 32x32b.x16 + wait
__global__ void tmem_bench(int mode, int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc((uint32_t)__cvta_generic_to_shared(&slot), 512);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  const uint32_t lane_off = (32u * (warp & 3)) << 16;
  // distinct column ranges per warp of the same sub-partition
  const uint32_t col0 = 64 * (warp >> 2);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t a = tmem + lane_off + ((col0 + 128 * (it & 1)) & 511);
    uint32_t r[32], s[32];
    if (mode == 0) {
      tmem_ld32(a, r);
      tmem_ld_wait();
      tmem_ld32(a + 32, s);
      tmem_ld_wait();
    } else if (mode == 1) {
      tmem_ld32(a, r);
      tmem_ld32(a + 32, s);
      tmem_ld_wait();
    } else if (mode == 2) {
      ld_16x256b_x8(a, r);
      ld_16x256b_x8(a + 32, s);
      tmem_ld_wait();
    } else {
      uint32_t h[16], g[16];
      tmem_ld16(a, h);
      tmem_ld16(a + 16, g);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 16; ++k) acc ^= h[k] + g[k];
      continue;
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) acc ^= r[k] + s[k];
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d_out;
  uint32_t* sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 2000;
  const char* names[] = {"32x32b.x32 wait each", "32x32b.x32 x2 one wait", "16x256b.x8 x2 one wait",
                         "32x32b.x16 x2 one wait"};
  for (int mode = 0; mode < 4; ++mode)
    for (int warps : {4, 8, 16})
      for (int blocks : {1, 148}) {
        tmem_bench<<<blocks, warps * 32>>>(mode, iters, d_out, sink);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long cyc = 0;
        cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
        const double bytes_per_iter = (mode == 3 ? 128.0 : 256.0) * 32 * warps;
        printf("%-26s warps %2d blocks %3d: %8.1f cycles/iter  %6.1f B/cycle/SM  %s\n",
               names[mode], warps, blocks, (double)cyc / iters, bytes_per_iter * iters / cyc,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
