// Tensor-core attention path (d = 64, B = 16, bf16 inputs): interface used
// by the handle API in capi.cu.  Implementation: attn_tc.cu.
#pragma once

#include <cuda_bf16.h>

#include "internal.h"

namespace llsa_impl {

// Per-handle scratch of the tensor-core path.
struct TcBuffers {
  // Coarse levels 1..L, pre-scaled by the level's key/value gain and split
  // into bf16 hi + lo parts (SURVEY.md hard part 3): [units][pyr_rows][64].
  // K' uses both parts in every score (S forward and backward, so the
  // backward's P = exp(S - lse) matches the forward's).  V' is multiplied
  // by its hi part only, in P·V AND in dP = dO·V'^T: the backward is then
  // the exact gradient of the forward that ran, and D = rowsum(dO∘O) equals
  // Σ P·dP up to rounding.  (With dP on hi + lo, one-hot rows on a
  // gain-4096 coarse key gave D - dP ≈ 2^-9·|dO||V'| instead of 0, and dq
  // errors of ~200 where the reference has 0.)  v_lo is kept zero-filled
  // for the mma.sync fallback kernels that still read it.
  __nv_bfloat16* k_hi = nullptr;
  __nv_bfloat16* k_lo = nullptr;
  __nv_bfloat16* v_hi = nullptr;
  __nv_bfloat16* v_lo = nullptr;
};

bool tc_supported(const Geometry& g, llsa_dtype dt);

// Fused compression of q, k, v (pyramid.cu): B = 16, d = 64.  With non-null
// hi/lo buffers it also writes the tensor-core key/value operand copies, so
// tc_forward can skip its prep pass.
bool fused_pyramid_ok(const Geometry& g);
llsa_status fused_pyramids(const Geometry& g, uint32_t units, const void* q, const void* k,
                           const void* v, llsa_dtype dt, float* pq, float* pk, float* pv,
                           __nv_bfloat16* khi, __nv_bfloat16* klo, __nv_bfloat16* vhi,
                           __nv_bfloat16* vlo, cudaStream_t s);
size_t tc_buffer_bytes(const Geometry& g, uint32_t units);
void tc_carve(const Geometry& g, uint32_t units, char* base, TcBuffers* out);

// K'/V' = gain·pyramid as bf16 hi + lo from fp32 pyramids (the staged path;
// the handle gets them from fused_pyramids).
llsa_status tc_prep(const Geometry& g, uint32_t units, const float* pyr_k, const float* pyr_v,
                    const TcBuffers& tb, cudaStream_t s);
llsa_status tc_forward(const Geometry& g, uint32_t units, const void* q, const void* k,
                       const void* v, const float* pyr_k, const float* pyr_v,
                       const uint32_t* tables, float* out, float* row_max, float* row_denom,
                       const TcBuffers& tb, cudaStream_t s, StageMarker* mk = nullptr,
                       bool prepped = false, void* out16 = nullptr);
// whether tc_forward writes its `out16` (bf16 copy of O) itself (the tcgen05
// forward); otherwise the caller converts the fp32 output
bool tc_forward_writes_bf16(const Geometry& g);
size_t tc_backward_ws_bytes(const Geometry& g, uint32_t units);
llsa_status tc_backward(const Geometry& g, uint32_t units, const void* d_out,
                        const float* out, const float* row_max, const float* row_denom,
                        const void* q, const void* k, const void* v, const float* pyr_k,
                        const float* pyr_v, const uint32_t* tables,
                        const uint32_t* csc_offsets, const uint32_t* csc_flat, float* dq,
                        float* dk, float* dv, const TcBuffers& tb, void* ws, cudaStream_t s,
                        StageMarker* mk = nullptr, bool grad_bf16 = false);
// grad_bf16 = true (dq, dk, dv point to bf16 buffers) is valid when this holds
bool tc_bf16_grads_ok(const Geometry& g);

}  // namespace llsa_impl
