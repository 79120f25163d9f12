// K1 — hierarchical compression (mean pooling), P/src/pyramid.cpp:11-64.
//
// One launch per level: level l row t = (Σ_{b<B} level_{l-1}[tB+b]) · (1/B),
// the sum sequential from 0 in index order and rounded per add, then one
// multiply (pyramid.cpp:31-37) — bit-identical to the f32 reference.  Each
// thread owns VEC consecutive columns of one output row and streams the B
// input rows with 16-byte loads; a warp covers whole 128 B row segments, so
// every HBM sector fetched is used.  HBM-bound: bytes = rows_in·d·sizeof(in)
// + rows_out·d·4.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "tc.h"

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

// ---------------------------------------------------------------------------
// Fused compression for the handle path (B = 16, d = 64): q, k and v in one
// launch (blockIdx.y), levels 1 and 2 in the same CTA (level 2 pooled from
// the CTA's own level-1 rows in shared memory, same sequential order, so
// bit-identical to per-level pooling), levels >= 3 in a second small launch.
// When `hilo` is given it also emits the tensor-core operand copies of the
// key/value pyramids: gain_l·x split into bf16 hi + lo (SURVEY.md hard
// part 3), which otherwise costs a separate pass over the pyramids.
// ---------------------------------------------------------------------------
namespace llsa_impl {
namespace {

struct PyrArgs {
  const void* in[3];
  float* out[3];
  __nv_bfloat16* hi[3];   // [k, v] hi (index 1, 2), null for q or when unused
  __nv_bfloat16* lo[3];
  uint64_t n, pyr_rows, off[kMaxLevels + 2];
  float gain[kMaxLevels + 2];
  uint32_t units, L, bf16_in;
  uint32_t zero_lo;  // bit t: tensor t's lo part is written as zeros (V': see tc.h)
};

__device__ __forceinline__ void emit(const PyrArgs& a, int t, uint64_t idx, float v0, float v1,
                                     float v2, float v3, float g) {
  float4* o = reinterpret_cast<float4*>(a.out[t] + idx);
  *o = make_float4(v0, v1, v2, v3);
  if (a.hi[t]) {
    const float x[4] = {v0 * g, v1 * g, v2 * g, v3 * g};
    __nv_bfloat16 h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[i] = __float2bfloat16_rn(x[i]);
      l[i] = (a.zero_lo >> t) & 1 ? __float2bfloat16_rn(0.f)
                                  : __float2bfloat16_rn(x[i] - __bfloat162float(h[i]));
    }
    *reinterpret_cast<uint2*>(a.hi[t] + idx) =
        make_uint2(*reinterpret_cast<uint32_t*>(&h[0]) | 0u, *reinterpret_cast<uint32_t*>(&h[2]));
    *reinterpret_cast<uint2*>(a.lo[t] + idx) =
        make_uint2(*reinterpret_cast<uint32_t*>(&l[0]), *reinterpret_cast<uint32_t*>(&l[2]));
  }
}

// CTA = 512 input rows of one unit and tensor (32 level-1 rows, 2 level-2
// rows); thread = (level-1 row, 4-column group).
__global__ void __launch_bounds__(512) pyr12_kernel(PyrArgs a) {
  __shared__ float l1[32][65];
  const int t = blockIdx.y;
  const uint64_t chunks = a.n / 512;
  const uint64_t unit = blockIdx.x / chunks, c = blockIdx.x % chunks;
  const uint32_t tid = threadIdx.x, r = tid >> 4, cg = tid & 15;
  const uint64_t row0 = c * 512 + (uint64_t)r * 16;  // first input row of level-1 row
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (a.bf16_in) {
    const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(a.in[t]) +
                               (unit * a.n + row0) * 64 + cg * 4;
#pragma unroll 4
    for (int b = 0; b < 16; ++b) {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(src + b * 64));
      acc[0] = __fadd_rn(acc[0], __uint_as_float(x.x << 16));
      acc[1] = __fadd_rn(acc[1], __uint_as_float(x.x & 0xffff0000u));
      acc[2] = __fadd_rn(acc[2], __uint_as_float(x.y << 16));
      acc[3] = __fadd_rn(acc[3], __uint_as_float(x.y & 0xffff0000u));
    }
  } else {
    const float* src = static_cast<const float*>(a.in[t]) + (unit * a.n + row0) * 64 + cg * 4;
#pragma unroll 4
    for (int b = 0; b < 16; ++b) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(src + b * 64));
      acc[0] = __fadd_rn(acc[0], x.x);
      acc[1] = __fadd_rn(acc[1], x.y);
      acc[2] = __fadd_rn(acc[2], x.z);
      acc[3] = __fadd_rn(acc[3], x.w);
    }
  }
  const float inv = 1.f / 16.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc[j] = __fmul_rn(acc[j], inv);
    l1[r][cg * 4 + j] = acc[j];
  }
  const uint64_t pu = unit * a.pyr_rows;
  emit(a, t, (pu + a.off[1] + c * 32 + r) * 64 + cg * 4, acc[0], acc[1], acc[2], acc[3],
       a.gain[1]);
  if (a.L < 2) return;
  __syncthreads();
  if (tid < 2 * 16) {  // level 2: rows 2c, 2c+1; thread = (row, column group)
    const uint32_t r2 = tid >> 4, g2 = tid & 15;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    for (int b = 0; b < 16; ++b)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[j] = __fadd_rn(s[j], l1[r2 * 16 + b][g2 * 4 + j]);
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = __fmul_rn(s[j], inv);
    emit(a, t, (pu + a.off[2] + c * 2 + r2) * 64 + g2 * 4, s[0], s[1], s[2], s[3], a.gain[2]);
  }
}

// levels >= 3 (tiny): thread = (unit, tensor, level row, 4-column group),
// one level after another inside the CTA (each CTA owns one unit).
__global__ void __launch_bounds__(256) pyr3_kernel(PyrArgs a) {
  const int t = blockIdx.y;
  const uint64_t unit = blockIdx.x;
  const uint64_t pu = unit * a.pyr_rows;
  const float inv = 1.f / 16.f;
  for (uint32_t l = 3; l <= a.L; ++l) {
    const uint64_t rows = a.n >> (4 * l);
    for (uint64_t i = threadIdx.x; i < rows * 16; i += blockDim.x) {
      const uint64_t r = i >> 4, g = i & 15;
      const float* src = a.out[t] + (pu + a.off[l - 1] + r * 16) * 64 + g * 4;
      float s[4] = {0.f, 0.f, 0.f, 0.f};
      for (int b = 0; b < 16; ++b) {
        const float4 x = *reinterpret_cast<const float4*>(src + b * 64);
        s[0] = __fadd_rn(s[0], x.x);
        s[1] = __fadd_rn(s[1], x.y);
        s[2] = __fadd_rn(s[2], x.z);
        s[3] = __fadd_rn(s[3], x.w);
      }
      emit(a, t, (pu + a.off[l] + r) * 64 + g * 4, __fmul_rn(s[0], inv), __fmul_rn(s[1], inv),
           __fmul_rn(s[2], inv), __fmul_rn(s[3], inv), a.gain[l]);
    }
    __syncthreads();  // level l is complete before level l+1 reads it
  }
}

}  // namespace

bool fused_pyramid_ok(const Geometry& g) {
  return g.B == 16 && g.d == 64 && g.n % 512 == 0 && g.L >= 1 && g.L <= kMaxLevels;
}

llsa_status fused_pyramids(const Geometry& g, uint32_t units, const void* q, const void* k,
                           const void* v, llsa_dtype dt, float* pq, float* pk, float* pv,
                           __nv_bfloat16* khi, __nv_bfloat16* klo, __nv_bfloat16* vhi,
                           __nv_bfloat16* vlo, cudaStream_t s) {
  PyrArgs a{};
  a.in[0] = q;
  a.in[1] = k;
  a.in[2] = v;
  a.out[0] = pq;
  a.out[1] = pk;
  a.out[2] = pv;
  a.hi[1] = khi;
  a.lo[1] = klo;
  a.hi[2] = vhi;
  a.lo[2] = vlo;
  a.n = g.n;
  a.pyr_rows = g.pyr_rows;
  for (uint32_t l = 0; l <= g.L && l < kMaxLevels + 2; ++l) {
    a.off[l] = g.pyr_off[l];
    a.gain[l] = g.mode == 0 ? (float)g.pow[l] : 1.f;  // ScaleKV gain B^l, LogitBias 1
  }
  a.units = units;
  a.L = g.L;
  a.bf16_in = dt == LLSA_BF16 ? 1u : 0u;
  a.zero_lo = 4u;  // V'_lo: the tensor cores multiply V'_hi only, forward and backward
  pyr12_kernel<<<dim3((unsigned)(units * (g.n / 512)), 3), 512, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("pyr12_kernel");
  if (g.L >= 3) {
    pyr3_kernel<<<dim3(units, 3), 256, 0, s>>>(a);
    count_launch();
    LLSA_LAUNCH_CHECK("pyr3_kernel");
  }
  return LLSA_OK;
}

}  // namespace llsa_impl
