// Self-test of the tcgen05 primitives in umma.cuh: one 128 x N x 64 bf16
// GEMM through shared-memory descriptors (K-major or MN-major A and B),
// accumulator in TMEM, read back with tcgen05.ld.  Checked against torch by
// tests/test_gpu_umma.py before any kernel relies on the encodings.
#include <cuda_bf16.h>

#include "../tc_common.cuh"
#include "../umma.cuh"

namespace {

using namespace llsa_umma;

__device__ __forceinline__ uint32_t tile_off(uint32_t row, uint32_t col) {
  // element (row, col) of a [rows][64] swizzled tile, col < 64
  return llsa_tc::swz(row, col >> 3) + (col & 7) * 2;
}

__global__ void __launch_bounds__(128) selftest_kernel(const __nv_bfloat16* a,
                                                       const __nv_bfloat16* b, float* d,
                                                       int N, int a_mn, int b_mn, int b_lbo) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                 // 16 KB
  uint8_t* sB = smem + 16384;         // MN-major: N blocks b_lbo bytes apart
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 16384 + 65536);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 16384 + 65536 + 8);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A: logical [128 m][64 k]; K-major: rows m; MN-major: rows k, 64-wide m blocks 8 KB apart
  for (int e = tid; e < 128 * 64; e += 128) {
    const int m = e / 64, k = e % 64;
    const __nv_bfloat16 v = a_mn ? a[k * 128 + m] : a[m * 64 + k];
    const uint32_t off = a_mn ? (m / 64) * 8192 + tile_off(k, m % 64) : tile_off(m, k);
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = v;
  }
  // B: logical [64 k][N n]; K-major: rows n; MN-major: rows k, 64-wide n blocks 8 KB apart
  for (int e = tid; e < N * 64; e += 128) {
    const int n = e / 64, k = e % 64;
    const __nv_bfloat16 v = b_mn ? b[k * N + n] : b[n * 64 + k];
    const uint32_t off = b_mn ? (n / 64) * b_lbo + tile_off(k, n % 64) : tile_off(n, k);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = v;
  }
  fence_proxy_async();
  const uint32_t ncols = N <= 64 ? 64 : N <= 128 ? 128 : 256;
  if (warp == 0) tmem_alloc(llsa_tc::smem_u32(tslot), ncols);
  if (tid == 0) {
    mbar_init(llsa_tc::smem_u32(mbar), 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(128, N, a_mn, b_mn);
    const uint32_t A = llsa_tc::smem_u32(sA), B = llsa_tc::smem_u32(sB);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t ad = a_mn ? desc_mnmajor(A + ks * kKStepMNMajor, 8192)
                               : desc_kmajor(A + ks * kKStepKMajor);
      const uint64_t bd = b_mn ? desc_mnmajor(B + ks * kKStepMNMajor, b_lbo)
                               : desc_kmajor(B + ks * kKStepKMajor);
      mma_bf16(tmem, ad, bd, idesc, ks > 0);
    }
    commit(llsa_tc::smem_u32(mbar));
  }
  mbar_wait(llsa_tc::smem_u32(mbar), 0);
  fence_after();
  for (int c = 0; c < (N + 31) / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32 && c * 32 + i < N; ++i)
      d[(32 * warp + lane) * N + c * 32 + i] = __uint_as_float(r[i]);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, ncols);
}

// tcgen05.st.16x256b from mma-fragment registers, read back with 32x32b:
// warp w writes lanes 32w + 16h (h = 0, 1) with value lane*100 + col.
__global__ void __launch_bounds__(128) frag_store_kernel(float* out) {
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc(llsa_tc::smem_u32(&tslot), 32);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tslot;
  for (int h = 0; h < 2; ++h) {
    const uint32_t base = 32 * warp + 16 * h;
    const int r = lane >> 2, c = 2 * (lane & 3);
    for (int t = 0; t < 4; ++t)  // columns 8t .. 8t+7
      tmem_st_frag(tmem + (base << 16) + 8 * t, (base + r) * 100.f + 8 * t + c,
                   (base + r) * 100.f + 8 * t + c + 1, (base + r + 8) * 100.f + 8 * t + c,
                   (base + r + 8) * 100.f + 8 * t + c + 1);
  }
  tmem_st_wait();
  fence_before();
  __syncthreads();
  fence_after();
  uint32_t v[32];
  tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), v);
  tmem_ld_wait();
  for (int i = 0; i < 32; ++i) out[(32 * warp + lane) * 32 + i] = __uint_as_float(v[i]);
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 32);
}

}  // namespace

extern "C" int llsa_umma_frag_selftest(float* out, void* stream) {
  frag_store_kernel<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(out);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int llsa_umma_selftest(const void* a, const void* b, float* d, int N, int a_mn,
                                  int b_mn, int b_lbo, void* stream) {
  if (N % 16 || N < 16 || N > 128 || b_lbo % 1024 || b_lbo < 8192 || b_lbo > 32768) return 1;
  const int smem = 16384 + 65536 + 64;
  cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  selftest_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(b), d, N, a_mn,
      b_mn, b_lbo);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
