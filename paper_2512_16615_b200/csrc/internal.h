// Host-side plumbing shared by the kernel files and the C ABI (capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "llsa_cuda.h"

namespace llsa_impl {

constexpr int kMaxLevels = 33;  // B >= 2 and n < 2^32 → L <= 31

// Every offset the kernels need, derived once on the host from a validated
// config (P/include/llsa/config.hpp:50-64 accessors).
struct Geometry {
  uint64_t n = 0;
  uint32_t d = 0, B = 0, K = 0, L = 0, Le = 0;
  float scale = 0.f;
  uint32_t mode = 0, safe = 1;
  uint32_t E = 0;                         // effective_block_count
  uint64_t pow[kMaxLevels + 2] = {};      // B^l, l = 0..L+1
  uint64_t pyr_rows = 0;                  // rows of levels 1..L per unit
  uint64_t pyr_off[kMaxLevels + 2] = {};  // row offset of level l (l >= 1)
  uint64_t table_entries = 0;             // u32 per unit, levels 0..L-1
  uint64_t table_off[kMaxLevels + 1] = {};
  uint64_t csc_off_entries = 0, csc_flat_entries = 0;
  uint64_t csc_off_off[kMaxLevels + 1] = {}, csc_flat_off[kMaxLevels + 1] = {};

  uint64_t level_tokens(uint32_t l) const { return n / pow[l]; }
  uint64_t level_blocks(uint32_t l) const { return n / pow[l + 1]; }
  uint32_t enrich_lim() const { return Le + 1 < L ? Le + 1 : L; }
  float weight(uint32_t l) const { return (float)pow[l]; }
};

// Validates (P/src/config.cpp:66-117 order) and fills a Geometry.
llsa_status make_geometry(const llsa_config* cfg, Geometry* g);

// Thread-local message for llsa_last_error.
llsa_status fail(llsa_status s, const char* fmt, ...);
llsa_status cuda_fail(cudaError_t e, const char* what);
#define LLSA_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::llsa_impl::cuda_fail(_e, #expr); \
  } while (0)
#define LLSA_LAUNCH_CHECK(what)                                       \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::llsa_impl::cuda_fail(_e, what);   \
  } while (0)

// Optional stage-boundary recorder (handle timing): records an event on the
// stream after a named group of launches.
struct StageMarker {
  virtual void mark(const char* name, cudaStream_t s) = 0;
  virtual ~StageMarker() = default;
};
#define LLSA_MARK(mk, name, s) \
  do {                         \
    if (mk) (mk)->mark(name, s); \
  } while (0)

// Per-device sticky error word (allocated lazily).
uint32_t* device_flag();

// Launch counter for the handle API (incremented by every launcher).
void count_launch(uint32_t n = 1);
uint32_t take_launch_count();

// ---- launchers (each returns LLSA_OK or an error; no synchronisation) ----
// Mask-based key→query lookup (transpose.cu): the kv-backward baseline
size_t mask_lookup_ws_bytes(const Geometry& g, uint32_t units);
llsa_status mask_lookup(const Geometry& g, uint32_t units, const uint32_t* tables,
                        uint32_t* offs, uint32_t* flat, void* ws, cudaStream_t s);
// CSR → CSC of every selection level in four launches (transpose.cu)
bool transpose_all_fused_ok(const Geometry& g);
size_t transpose_all_fused_ws(const Geometry& g, uint32_t units);
llsa_status transpose_all_fused(const Geometry& g, uint32_t units, const uint32_t* tables,
                                uint32_t* offs, uint32_t* flat, void* ws, cudaStream_t s);
llsa_status launch_pool_level(const void* in, llsa_dtype in_dtype, uint64_t in_unit_stride,
                              float* out, uint64_t out_unit_stride, uint32_t units,
                              uint64_t rows_out, uint32_t d, uint32_t B, cudaStream_t s);
llsa_status launch_pool_backward(const float* g, uint32_t units, uint64_t coarse_rows,
                                 uint32_t d, uint64_t group, float* out, cudaStream_t s);

llsa_status launch_select_coarsest(const float* q, uint64_t q_unit_stride, const float* k,
                                   uint64_t k_unit_stride, uint32_t units, uint32_t rows,
                                   uint32_t cands, uint32_t d, uint32_t K, float scale,
                                   uint32_t* out, uint64_t out_unit_stride, cudaStream_t s);
llsa_status launch_select_level(const float* q, uint64_t q_unit_stride, const float* k,
                                uint64_t k_unit_stride, const uint32_t* parent,
                                uint64_t parent_unit_stride, uint32_t units,
                                uint32_t parent_rows, uint32_t parent_k, uint64_t k_rows,
                                uint32_t d, uint32_t K, float scale, uint32_t B,
                                uint32_t* out, uint64_t out_unit_stride, cudaStream_t s);

size_t transpose_ws_bytes(uint32_t units, uint32_t rows, uint32_t k, uint32_t key_blocks);
llsa_status launch_transpose(const uint32_t* idx, uint64_t idx_unit_stride, uint32_t units,
                             uint32_t rows, uint32_t k, uint32_t key_blocks,
                             uint32_t* offsets, uint64_t off_unit_stride, uint32_t* flat,
                             uint64_t flat_unit_stride, void* ws, cudaStream_t s);

// CSC → per-level selection tables (sorted rows), for kv_backward's tensor-core path.
size_t tables_from_csc_ws(const Geometry& g, uint32_t units);
llsa_status tables_from_csc(const Geometry& g, uint32_t units, const uint32_t* csc_offsets,
                            const uint32_t* csc_flat, uint32_t* tables, void* ws,
                            cudaStream_t s);

llsa_status launch_build_plan(const Geometry& g, uint32_t units, const uint32_t* tables,
                              uint32_t* plan_level, uint32_t* plan_block,
                              float* plan_weight, cudaStream_t s);

// A materialised enriched plan ([units][n/B][epb] level, block, weight):
// hand-built plans are honoured exactly as the reference does.
struct PlanView {
  const uint32_t* level = nullptr;
  const uint32_t* block = nullptr;
  const float* weight = nullptr;
  uint32_t epb = 0;
};

// General (SIMT) attention, any d <= 256 and any B.
llsa_status simt_forward(const Geometry& g, uint32_t units, llsa_dtype dt, const void* q,
                         const void* k, const void* v, const float* pyr_k,
                         const float* pyr_v, const uint32_t* tables, float* out,
                         float* row_max, float* row_denom, cudaStream_t s,
                         const PlanView* plan = nullptr);
size_t simt_backward_ws_bytes(const Geometry& g, uint32_t units);
llsa_status simt_backward(const Geometry& g, uint32_t units, llsa_dtype dt,
                          const void* d_out, const float* out, const float* row_max,
                          const float* row_denom, const void* q, const void* k,
                          const void* v, const float* pyr_k, const float* pyr_v,
                          const uint32_t* tables, const uint32_t* csc_offsets,
                          const uint32_t* csc_flat, float* dq, float* dk, float* dv,
                          void* ws, cudaStream_t s, StageMarker* mk = nullptr,
                          const PlanView* plan = nullptr);

}  // namespace llsa_impl
