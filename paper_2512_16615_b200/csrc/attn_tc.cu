// Tensor-core attention (placeholder until the sm_100a kernels land).
#include "tc.h"

namespace llsa_impl {

bool tc_supported(const Geometry&, llsa_dtype) { return false; }
size_t tc_buffer_bytes(const Geometry&, uint32_t) { return 0; }
void tc_carve(const Geometry&, uint32_t, char*, TcBuffers*) {}
llsa_status tc_forward(const Geometry&, uint32_t, const void*, const void*, const void*,
                       const float*, const float*, const uint32_t*, float*, float*, float*,
                       const TcBuffers&, cudaStream_t, StageMarker*) {
  return fail(LLSA_ERR_UNSUPPORTED, "tensor-core path not built");
}
size_t tc_backward_ws_bytes(const Geometry&, uint32_t) { return 0; }
llsa_status tc_backward(const Geometry&, uint32_t, const void*, const float*, const float*,
                        const float*, const void*, const void*, const void*, const float*,
                        const float*, const uint32_t*, const uint32_t*, const uint32_t*,
                        float*, float*, float*, const TcBuffers&, void*, cudaStream_t,
                        StageMarker*) {
  return fail(LLSA_ERR_UNSUPPORTED, "tensor-core path not built");
}

}  // namespace llsa_impl
