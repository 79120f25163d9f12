// Warp-level tensor-core primitives (sm_100a) for the d = 64, B = 16 path:
// cp.async staging, swizzled 64-column bf16 tiles, ldmatrix fragment loads
// and m16n8k16 bf16 MMAs with fp32 accumulation.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace llsa_tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gptr));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// A 64-column bf16 tile has 128 B rows of eight 16 B chunks; chunk c of row r
// lives at chunk (c ^ (r & 7)) so ldmatrix row groups hit distinct banks.
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

// Copies `rows` consecutive 128 B rows (global, contiguous) into a swizzled
// tile starting at tile row `row0`; `tid`/`nthr` spread the 16 B chunks.
__device__ __forceinline__ void load_rows_async(uint32_t tile, uint32_t row0,
                                                const __nv_bfloat16* g, uint32_t rows,
                                                uint32_t tid, uint32_t nthr) {
  const char* src = reinterpret_cast<const char*>(g);
  for (uint32_t i = tid; i < rows * 8; i += nthr) {
    const uint32_t r = i >> 3, c = i & 7;
    cp_async16(tile + swz(row0 + r, c), src + i * 16);
  }
}

// Per-lane constants for load_block16_async: the swizzled offsets of this
// lane's 16-byte chunk in rows (lane >> 3) + 4k, k even / odd.
struct Block16Lane {
  uint32_t even, odd;
};
__device__ __forceinline__ Block16Lane block16_lane(uint32_t lane) {
  const uint32_t r = lane >> 3, sw = (lane & 7) ^ r;
  return {r * 128u + (sw << 4), r * 128u + ((sw ^ 4u) << 4)};
}
// One warp copies a 16-row block (16 x 128 B, contiguous in global) into a
// swizzled tile at `dst` (the address of the block's first row, row index a
// multiple of 8): four 16-byte cp.async per lane at precomputed offsets.
__device__ __forceinline__ void load_block16_async(uint32_t dst, const void* g,
                                                   const Block16Lane& o, uint32_t lane) {
  const char* src = reinterpret_cast<const char*>(g) + lane * 16;
  cp_async16(dst + o.even, src);
  cp_async16(dst + 512 + o.odd, src + 512);
  cp_async16(dst + 1024 + o.even, src + 1024);
  cp_async16(dst + 1536 + o.odd, src + 1536);
}

// CTA-level variant: NTHR threads (a multiple of 64) copy ROWS contiguous
// 128-byte rows into a swizzled tile at `dst` (row index a multiple of 8).
// With NTHR/8 a multiple of 8, a thread's row phase (r & 7) is the same for
// every chunk it moves, so its swizzled offset is one add per copy.
template <int ROWS, int NTHR>
__device__ __forceinline__ void load_rows_fast(uint32_t dst, const void* g, uint32_t tid) {
  static_assert(NTHR % 64 == 0 && (ROWS * 8) % NTHR == 0, "shape");
  const uint32_t r = tid >> 3, c = tid & 7;
  const uint32_t off = r * 128u + ((c ^ (r & 7u)) << 4);
  const char* src = reinterpret_cast<const char*>(g) + tid * 16;
#pragma unroll
  for (int k = 0; k < ROWS * 8 / NTHR; ++k) cp_async16(dst + off + k * NTHR * 16, src + k * NTHR * 16);
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                        uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D += A(16x16 bf16, row) * B(16x8 bf16, col), fp32 accumulate.
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A fragment of the 16x16 block (rows r0..r0+15, k-step ks) of a swizzled tile.
__device__ __forceinline__ void lda(uint32_t tile, uint32_t r0, uint32_t ks, uint32_t lane,
                                    uint32_t (&a)[4]) {
  ldsm_x4(tile + swz(r0 + (lane & 15), 2 * ks + (lane >> 4)), a[0], a[1], a[2], a[3]);
}

// B fragments for two n8 tiles (rows n0..n0+15 of a [n][k] tile) at k-step ks:
// (b[0], b[1]) for rows n0..n0+7, (b[2], b[3]) for rows n0+8..n0+15.
__device__ __forceinline__ void ldb(uint32_t tile, uint32_t n0, uint32_t ks, uint32_t lane,
                                    uint32_t (&b)[4]) {
  ldsm_x4(tile + swz(n0 + (lane & 7) + ((lane >> 4) << 3), 2 * ks + ((lane >> 3) & 1)), b[0],
          b[1], b[2], b[3]);
}

// B fragments from a [k][n] tile (rows = k): k rows k0..k0+15, n columns
// n0..n0+15 (chunks n0/8, n0/8+1): (b[0], b[1]) for n0..n0+7, (b[2], b[3])
// for n0+8..n0+15.
__device__ __forceinline__ void ldb_t(uint32_t tile, uint32_t k0, uint32_t n0, uint32_t lane,
                                      uint32_t (&b)[4]) {
  ldsm_x4_t(tile + swz(k0 + (lane & 7) + (((lane >> 3) & 1) << 3), (n0 >> 3) + (lane >> 4)),
            b[0], b[1], b[2], b[3]);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe (relative error < 8e-5, far below a bf16 ulp): round
// x to n with the 1.5·2^23 trick, a degree-3 fit of 2^f on [-0.5, 0.5], and n
// added to the exponent.  Used for a share of the softmax exponentials so the
// MUFU unit (16 / clk / SM) is not the only pipe doing them.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float r = __fadd_rn(x, 12582912.f);
  const float f = x - __fsub_rn(r, 12582912.f);
  float q = fmaf(f, 0.05518098f, 0.24263459f);
  q = fmaf(q, f, 0.69326133f);
  q = fmaf(q, f, 0.99992621f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(r) << 23));
}

__device__ __forceinline__ float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

}  // namespace llsa_tc
