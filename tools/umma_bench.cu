// Microbenchmark (development tool, not part of the library): issue cost and
// completion time of back-to-back tcgen05.mma kind::f16 (SS operands, SW128
// K-major) by one thread, for M = 128 and several N.  One CTA per SM (grid
// 148) so every SM's tensor core is measured under the same load.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_bench
//        tools/umma_bench.cu -I paper_2512_16615_b200/csrc
#include <cstdint>
#include <cstdio>

#include "umma.cuh"

using namespace llsa_umma;

__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// a_mn: 0 = A K-major in smem, 1 = A MN-major in smem, 2 = A in TMEM (TS mode)
// chains: MMA r accumulates into D number r % chains (independent accumulators
// at columns N * c): 1 = every MMA depends on the previous one's D
// b_mn: B MN-major (N spanning two 64-column atoms 16 KB apart when N > 64)
__global__ void __launch_bounds__(128) umma_bench(int M, int N, int reps, int a_mn, int chains,
                                                  unsigned long long* out, int b_mn = 0) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sbase = (base + 1023) & ~1023u;
  for (uint32_t i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem + (sbase - base))[i] = 0x3f803f80u;  // bf16 1.0
  if (warp == 0) tmem_alloc((uint32_t)__cvta_generic_to_shared(&slot), 512);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    mbar_init(mb, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(M, N, a_mn == 1, b_mn != 0);
    const uint32_t sa = sbase, sb = sbase + 32768;
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (a_mn == 2) {  // D in columns [0, 256), A in columns [256 + 8*(r&3), ...)
        mma_bf16_ts(tmem, tmem + 256 + 8 * (r & 3), desc_kmajor(sb + (r & 3) * kKStepKMajor),
                    idesc, r > 0);
      } else {
        const uint64_t ad = a_mn ? desc_mnmajor(sa + (r & 3) * kKStepMNMajor, 16384)
                                 : desc_kmajor(sa + (r & 3) * kKStepKMajor);
        const uint64_t bd = b_mn ? desc_mnmajor(sb + (r & 3) * kKStepMNMajor, 16384)
                                 : desc_kmajor(sb + (r & 3) * kKStepKMajor);
        mma_bf16(tmem + N * (r % chains), ad, bd, idesc, r >= chains);
      }
    }
    unsigned long long t1 = clock64();
    commit(mb);
    mbar_wait(mb, 0);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(umma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  // warm-up: ~0.5 s of back-to-back MMAs so the clocks leave their idle state
  for (int w = 0; w < 200; ++w) umma_bench<<<148, 128, 66 * 1024>>>(128, 256, 4096, 0, 1, d);
  cudaDeviceSynchronize();
  for (int a_mn = 0; a_mn < 3; ++a_mn)
    for (int N : {16, 32, 64, 128, 256}) {
      if (a_mn == 2 && N > 256 - 0) continue;
      const int reps = 256;
      unsigned long long h[2];
      for (int w = 0; w < 2; ++w) umma_bench<<<148, 128, 66 * 1024>>>(128, N, reps, a_mn, 1, d);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("M=128 N=%3d K=16 A=%s: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", N,
             a_mn == 2 ? "TMEM" : a_mn ? "MN" : "K ", (double)h[0] / reps, (double)h[1] / reps,
             cudaGetErrorString(cudaGetLastError()));
    }
  // operand majors: {A, B} in {K, MN} for the kvf accumulate shapes
  for (int M : {128, 64})
    for (int N : {32, 64, 128})
      for (int am = 0; am < 2; ++am)
        for (int bm = 0; bm < 2; ++bm) {
          const int reps = 256;
          unsigned long long h[2];
          for (int w = 0; w < 2; ++w)
            umma_bench<<<148, 128, 66 * 1024>>>(M, N, reps, am, 1, d, bm);
          cudaDeviceSynchronize();
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
          printf("M=%3d N=%3d K=16 A=%s B=%s: issue %.1f cyc/mma, complete %.1f  (%s)\n", M, N,
                 am ? "MN" : "K ", bm ? "MN" : "K ", (double)h[0] / reps, (double)h[1] / reps,
                 cudaGetErrorString(cudaGetLastError()));
        }
  // independent accumulators and M = 64 (SS, A K-major)
  for (int M : {128, 64})
    for (int N : {16, 32, 64, 128})
      for (int chains : {1, 2, 4}) {
        if (N * chains > 256) continue;
        const int reps = 256;
        unsigned long long h[2];
        for (int w = 0; w < 2; ++w) umma_bench<<<148, 128, 66 * 1024>>>(M, N, reps, 0, chains, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("M=%3d N=%3d K=16 chains=%d: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", M,
               N, chains, (double)h[0] / reps, (double)h[1] / reps,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
