// Shared device helpers for the LLSA sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace llsa_dev {

constexpr int kWarp = 32;

// Sticky device error bits (read by llsa_sync_status).
enum : uint32_t { kErrIndex = 1u, kErrNonFinite = 2u };

__device__ __forceinline__ void raise_flag(uint32_t* flag, uint32_t bit) {
  if (flag) atomicOr(flag, bit);
}

// Element loads widened to fp32 (bf16 → fp32 is exact).
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  return to_f(p[0]);
}

// detail::dot (P/include/llsa/detail/math.hpp:13-24) with the reference's
// association: lane j of four accumulators takes a[4i+j]*b[4i+j], tail into
// lane 0, result (s0+s1)+(s2+s3).  Explicit _rn intrinsics forbid FMA
// contraction, so the result is bit-identical to the f32 reference build.
__device__ __forceinline__ float dot4_exact(const float* __restrict__ a,
                                            const float* __restrict__ b, int n) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 = __fadd_rn(s0, __fmul_rn(a[i], b[i]));
    s1 = __fadd_rn(s1, __fmul_rn(a[i + 1], b[i + 1]));
    s2 = __fadd_rn(s2, __fmul_rn(a[i + 2], b[i + 2]));
    s3 = __fadd_rn(s3, __fmul_rn(a[i + 3], b[i + 3]));
  }
  for (; i < n; ++i) s0 = __fadd_rn(s0, __fmul_rn(a[i], b[i]));
  return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}

// Same, 128-bit smem/global vectorised for n % 4 == 0 with 16 B alignment.
__device__ __forceinline__ float dot4_exact_v4(const float4* __restrict__ a,
                                               const float4* __restrict__ b, int n4) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 4
  for (int i = 0; i < n4; ++i) {
    const float4 x = a[i], y = b[i];
    s0 = __fadd_rn(s0, __fmul_rn(x.x, y.x));
    s1 = __fadd_rn(s1, __fmul_rn(x.y, y.y));
    s2 = __fadd_rn(s2, __fmul_rn(x.z, y.z));
    s3 = __fadd_rn(s3, __fmul_rn(x.w, y.w));
  }
  return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// B^l as u64.
__host__ __device__ __forceinline__ uint64_t ipow_u64(uint32_t b, uint32_t e) {
  uint64_t p = 1;
  for (uint32_t i = 0; i < e; ++i) p *= b;
  return p;
}

}  // namespace llsa_dev
