// 2-D reordering, P/src/reorder2d.cpp:11-90.
//
// The hierarchical curve itself is host integer work (O(H·W), built once per
// network), restated from the header contract (reorder2d.hpp:21-33): every
// aligned s^i x s^i patch is a contiguous run of B^i positions, sub-patches
// visited row-major from coarse to fine, whole top-level patches row-major.
// The device side is the data movement: a row gather (apply_permutation)
// and the gather fused into compression, so the sequence-order pyramid of a
// raster-ordered image is built without materialising the reordered copy
// (level-1 row t = mean over b of x[map[tB + b]], same sequential order as
// pyramid.cpp:31-37, hence bit-identical to pooling the gathered sequence).
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace llsa_impl {
namespace {

// One thread per 16 bytes of a row: out[u][i] = x[u][map[i]].
template <typename T>
__global__ void permute_rows_kernel(const T* __restrict__ x, T* __restrict__ out,
                                    const uint32_t* __restrict__ map, uint64_t rows,
                                    uint32_t row_vecs, uint64_t total, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t vec = i % row_vecs, r = (i / row_vecs) % rows, u = i / (row_vecs * rows);
    uint32_t src = map[r];
    if (src >= rows) {
      llsa_dev::raise_flag(flag, llsa_dev::kErrIndex);
      continue;
    }
    reinterpret_cast<uint4*>(out)[(u * rows + r) * row_vecs + vec] =
        __ldg(reinterpret_cast<const uint4*>(x) + (u * rows + src) * row_vecs + vec);
  }
}

// Level 1 of the pyramid of the permuted sequence: thread = (unit, output
// row, 4-column group); the B gathered input rows are summed in index order.
template <typename T>
__global__ void pool_permuted_kernel(const T* __restrict__ x, const uint32_t* __restrict__ map,
                                     uint64_t rows, uint32_t d, uint32_t B, float inv_b,
                                     float* __restrict__ out, uint64_t out_unit_stride,
                                     uint64_t total, uint32_t* flag) {
  const uint32_t groups = d / 4;
  const uint64_t rows_out = rows / B;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = (uint32_t)(i % groups);
    const uint64_t t = (i / groups) % rows_out, u = i / ((uint64_t)groups * rows_out);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (uint32_t b = 0; b < B; ++b) {
      uint32_t src = map[t * B + b];
      if (src >= rows) {
        llsa_dev::raise_flag(flag, llsa_dev::kErrIndex);
        src = 0;
      }
      const T* p = x + (u * rows + src) * d + (uint64_t)g * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = __fadd_rn(acc[j], llsa_dev::to_f(p[j]));
    }
    float* o = out + u * out_unit_stride + t * d + (uint64_t)g * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = __fmul_rn(acc[j], inv_b);
  }
}

// Any row size: one thread per element (2 or 4 bytes).
template <typename W>
__global__ void permute_elems_kernel(const W* __restrict__ x, W* __restrict__ out,
                                     const uint32_t* __restrict__ map, uint64_t rows,
                                     uint32_t d, uint64_t total, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = i % d, r = (i / d) % rows, u = i / ((uint64_t)d * rows);
    const uint32_t src = map[r];
    if (src >= rows) {
      llsa_dev::raise_flag(flag, llsa_dev::kErrIndex);
      continue;
    }
    out[(u * rows + r) * d + c] = x[(u * rows + src) * d + c];
  }
}

unsigned grid_for(uint64_t threads, int block) {
  uint64_t blocks = (threads + block - 1) / block;
  const uint64_t cap = 148ull * 16;
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

}  // namespace
}  // namespace llsa_impl

using namespace llsa_impl;

namespace {
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
#define NONNULL(p)                                                       \
  do {                                                                   \
    if (!(p)) return fail(LLSA_ERR_ARGUMENT, "null pointer: %s", #p);   \
  } while (0)
llsa_status dtype_ok(llsa_dtype dt) {
  if (dt != LLSA_F32 && dt != LLSA_BF16) return fail(LLSA_ERR_ARGUMENT, "bad dtype %d", dt);
  return LLSA_OK;
}
}  // namespace

extern "C" {

llsa_status llsa_build_reorder(uint32_t height, uint32_t width, uint32_t block_size,
                               uint32_t* forward, uint32_t* inverse) {
  if (height == 0 || width == 0)
    return fail(LLSA_ERR_DIVISIBILITY, "image dimensions must be positive");
  uint32_t side = 0;
  while ((uint64_t)side * side < block_size) ++side;
  if (block_size == 0 || (uint64_t)side * side != block_size)
    return fail(LLSA_ERR_NOT_SQUARE_BLOCK, "block size %u is not a perfect square", block_size);
  uint32_t depth = 0;
  uint64_t patch = 1;
  while (height % (patch * side) == 0 && width % (patch * side) == 0) {
    patch *= side;
    ++depth;
  }
  if (depth == 0 && !(height == 1 && width == 1))
    return fail(LLSA_ERR_DIVISIBILITY, "side %u divides neither %u nor %u evenly", side, height,
                width);
  if (!forward || !inverse) return fail(LLSA_ERR_ARGUMENT, "null output");
  const uint64_t size = (uint64_t)height * width, cells = patch * patch;
  const uint64_t across = width / patch;
  for (uint64_t pos = 0; pos < size; ++pos) {
    const uint64_t top = pos / cells;
    uint64_t rest = pos % cells;
    uint64_t y = (top / across) * patch, x = (top % across) * patch;
    for (uint64_t edge = patch / side; edge >= 1 && rest > 0; edge /= side) {
      const uint64_t digit = rest / (edge * edge);  // which s x s sub-patch, row-major
      y += (digit / side) * edge;
      x += (digit % side) * edge;
      rest %= edge * edge;
      if (edge == 1) break;
    }
    forward[pos] = (uint32_t)(y * width + x);
  }
  for (uint64_t pos = 0; pos < size; ++pos) inverse[forward[pos]] = (uint32_t)pos;
  return LLSA_OK;
}

llsa_status llsa_apply_permutation(const void* x, llsa_dtype dt, uint32_t units, uint64_t rows,
                                   uint32_t d, const uint32_t* map, void* out, void* stream) {
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0 || rows == 0 || d == 0) return LLSA_OK;
  NONNULL(x);
  NONNULL(map);
  NONNULL(out);
  const uint64_t row_bytes = (uint64_t)d * (dt == LLSA_BF16 ? 2 : 4);
  if (row_bytes % 16 != 0 || reinterpret_cast<uintptr_t>(x) % 16 ||
      reinterpret_cast<uintptr_t>(out) % 16) {
    const uint64_t total = (uint64_t)units * rows * d;
    if (dt == LLSA_BF16)
      permute_elems_kernel<uint16_t><<<grid_for(total, 256), 256, 0, S(stream)>>>(
          static_cast<const uint16_t*>(x), static_cast<uint16_t*>(out), map, rows, d, total,
          device_flag());
    else
      permute_elems_kernel<uint32_t><<<grid_for(total, 256), 256, 0, S(stream)>>>(
          static_cast<const uint32_t*>(x), static_cast<uint32_t*>(out), map, rows, d, total,
          device_flag());
    count_launch();
    LLSA_LAUNCH_CHECK("permute_elems_kernel");
    return LLSA_OK;
  }
  const uint32_t vecs = (uint32_t)(row_bytes / 16);
  const uint64_t total = (uint64_t)units * rows * vecs;
  permute_rows_kernel<uint8_t><<<grid_for(total, 256), 256, 0, S(stream)>>>(
      static_cast<const uint8_t*>(x), static_cast<uint8_t*>(out), map, rows, vecs, total,
      device_flag());
  count_launch();
  LLSA_LAUNCH_CHECK("permute_rows_kernel");
  return LLSA_OK;
}

llsa_status llsa_build_pyramid_permuted(const void* x, llsa_dtype dt, uint32_t units,
                                        uint64_t rows, uint32_t d, uint32_t B, uint32_t levels,
                                        const uint32_t* map, float* out, void* stream) {
  if (llsa_status st = dtype_ok(dt)) return st;
  if (B < 2) return fail(LLSA_ERR_DIVISIBILITY, "block size must be at least 2");
  uint64_t r = rows;
  for (uint32_t l = 1; l <= levels; ++l) {
    if (r % B != 0)
      return fail(LLSA_ERR_DIVISIBILITY, "level %u has %llu rows, not a multiple of block size %u",
                  l - 1, (unsigned long long)r, B);
    r /= B;
  }
  if (levels == 0 || units == 0 || rows == 0) return LLSA_OK;
  if (d % 4) return fail(LLSA_ERR_UNSUPPORTED, "fused permuted pooling needs d % 4 == 0");
  NONNULL(x);
  NONNULL(map);
  NONNULL(out);
  const uint64_t pr = llsa_pyramid_rows(rows, B, levels);
  const uint64_t total = (uint64_t)units * (rows / B) * (d / 4);
  const float inv = 1.0f / (float)B;
  if (dt == LLSA_BF16)
    pool_permuted_kernel<__nv_bfloat16><<<grid_for(total, 256), 256, 0, S(stream)>>>(
        static_cast<const __nv_bfloat16*>(x), map, rows, d, B, inv, out, pr * d, total,
        device_flag());
  else
    pool_permuted_kernel<float><<<grid_for(total, 256), 256, 0, S(stream)>>>(
        static_cast<const float*>(x), map, rows, d, B, inv, out, pr * d, total, device_flag());
  count_launch();
  LLSA_LAUNCH_CHECK("pool_permuted_kernel");
  uint64_t off_prev = 0, rows_prev = rows / B;
  llsa_status st = LLSA_OK;
  for (uint32_t l = 2; l <= levels && st == LLSA_OK; ++l) {  // deeper levels: plain pooling
    const uint64_t off = off_prev + rows_prev;
    st = launch_pool_level(out + off_prev * d, LLSA_F32, pr * d, out + off * d, pr * d, units,
                           rows_prev / B, d, B, S(stream));
    off_prev = off;
    rows_prev /= B;
  }
  return st;
}

}  // extern "C"
