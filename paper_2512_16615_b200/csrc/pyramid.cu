// K1 — hierarchical compression (mean pooling), P/src/pyramid.cpp:11-64.
//
// One launch per level: level l row t = (Σ_{b<B} level_{l-1}[tB+b]) · (1/B),
// the sum sequential from 0 in index order and rounded per add, then one
// multiply (pyramid.cpp:31-37) — bit-identical to the f32 reference.  Each
// thread owns VEC consecutive columns of one output row and streams the B
// input rows with 16-byte loads; a warp covers whole 128 B row segments, so
// every HBM sector fetched is used.  HBM-bound: bytes = rows_in·d·sizeof(in)
// + rows_out·d·4.
#include "common.cuh"
#include "internal.h"

namespace llsa_impl {
namespace {

using namespace llsa_dev;

template <typename T, int VEC>
struct Loader;

template <>
struct Loader<float, 4> {
  __device__ static void load(const float* p, float* v) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
};

template <>
struct Loader<__nv_bfloat16, 8> {
  __device__ static void load(const __nv_bfloat16* p, float* v) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};

template <typename T>
struct Loader1 {
  __device__ static void load(const T* p, float* v) { v[0] = to_f(p[0]); }
};

template <typename T, int VEC, bool VECTOR>
__global__ void __launch_bounds__(256) pool_level_kernel(
    const T* __restrict__ in, uint64_t in_unit_stride, float* __restrict__ out,
    uint64_t out_unit_stride, uint64_t rows_out, uint32_t d, uint32_t B,
    float inv_b, uint64_t total_threads) {
  const uint32_t groups = d / VEC;
  for (uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; tid < total_threads;
       tid += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t gcol = (uint32_t)(tid % groups);
    const uint64_t r = tid / groups;
    const uint64_t unit = r / rows_out;
    const uint64_t t = r - unit * rows_out;
    const T* src = in + unit * in_unit_stride + (t * B) * d + (uint64_t)gcol * VEC;
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
    for (uint32_t b = 0; b < B; ++b) {
      float x[VEC];
      if constexpr (VECTOR) {
        Loader<T, VEC>::load(src + (uint64_t)b * d, x);
      } else {
        Loader1<T>::load(src + (uint64_t)b * d, x);
      }
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] = __fadd_rn(acc[j], x[j]);
    }
    float* dst = out + unit * out_unit_stride + t * d + (uint64_t)gcol * VEC;
    if constexpr (VECTOR && VEC % 4 == 0) {
#pragma unroll
      for (int j = 0; j < VEC; j += 4) {
        float4 o = make_float4(__fmul_rn(acc[j], inv_b), __fmul_rn(acc[j + 1], inv_b),
                               __fmul_rn(acc[j + 2], inv_b), __fmul_rn(acc[j + 3], inv_b));
        *reinterpret_cast<float4*>(dst + j) = o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) dst[j] = __fmul_rn(acc[j], inv_b);
    }
  }
}

// pool_backward (P/src/pyramid.cpp:45-64): fine[t] = coarse[t/group]·(1/group)
__global__ void pool_backward_kernel(const float* __restrict__ g, uint64_t coarse_rows,
                                     uint32_t d, uint64_t group, float inv,
                                     float* __restrict__ out, uint64_t total) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t col = i % d;
    const uint64_t row = i / d;  // global fine row across units
    const uint64_t fine_rows = coarse_rows * group;
    const uint64_t unit = row / fine_rows;
    const uint64_t t = row - unit * fine_rows;
    out[i] = __fmul_rn(g[(unit * coarse_rows + t / group) * d + col], inv);
  }
}

unsigned grid_for(uint64_t threads, int block) {
  uint64_t blocks = (threads + block - 1) / block;
  const uint64_t cap = 148ull * 16;  // grid-stride beyond 16 CTAs/SM
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

}  // namespace

llsa_status launch_pool_level(const void* in, llsa_dtype in_dtype, uint64_t in_unit_stride,
                              float* out, uint64_t out_unit_stride, uint32_t units,
                              uint64_t rows_out, uint32_t d, uint32_t B, cudaStream_t s) {
  if (rows_out == 0 || units == 0) return LLSA_OK;
  const float inv_b = 1.0f / (float)B;
  const int blk = 256;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(in);
  if (in_dtype == LLSA_BF16) {
    const auto* x = static_cast<const __nv_bfloat16*>(in);
    if (d % 8 == 0 && addr % 16 == 0 && in_unit_stride % 8 == 0 &&
        reinterpret_cast<uintptr_t>(out) % 16 == 0 && out_unit_stride % 4 == 0) {
      const uint64_t total = (uint64_t)units * rows_out * (d / 8);
      pool_level_kernel<__nv_bfloat16, 8, true><<<grid_for(total, blk), blk, 0, s>>>(
          x, in_unit_stride, out, out_unit_stride, rows_out, d, B, inv_b, total);
    } else {
      const uint64_t total = (uint64_t)units * rows_out * d;
      pool_level_kernel<__nv_bfloat16, 1, false><<<grid_for(total, blk), blk, 0, s>>>(
          x, in_unit_stride, out, out_unit_stride, rows_out, d, B, inv_b, total);
    }
  } else {
    const auto* x = static_cast<const float*>(in);
    if (d % 4 == 0 && addr % 16 == 0 && in_unit_stride % 4 == 0 &&
        reinterpret_cast<uintptr_t>(out) % 16 == 0 && out_unit_stride % 4 == 0) {
      const uint64_t total = (uint64_t)units * rows_out * (d / 4);
      pool_level_kernel<float, 4, true><<<grid_for(total, blk), blk, 0, s>>>(
          x, in_unit_stride, out, out_unit_stride, rows_out, d, B, inv_b, total);
    } else {
      const uint64_t total = (uint64_t)units * rows_out * d;
      pool_level_kernel<float, 1, false><<<grid_for(total, blk), blk, 0, s>>>(
          x, in_unit_stride, out, out_unit_stride, rows_out, d, B, inv_b, total);
    }
  }
  count_launch();
  LLSA_LAUNCH_CHECK("pool_level_kernel");
  return LLSA_OK;
}

llsa_status launch_pool_backward(const float* g, uint32_t units, uint64_t coarse_rows,
                                 uint32_t d, uint64_t group, float* out, cudaStream_t s) {
  const uint64_t total = (uint64_t)units * coarse_rows * group * d;
  if (total == 0) return LLSA_OK;
  pool_backward_kernel<<<grid_for(total, 256), 256, 0, s>>>(g, coarse_rows, d, group,
                                                          1.0f / (float)group, out, total);
  count_launch();
  LLSA_LAUNCH_CHECK("pool_backward_kernel");
  return LLSA_OK;
}

}  // namespace llsa_impl
