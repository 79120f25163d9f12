/*
 * llsa_cuda.h — C ABI of the B200-native LLSA hot path (arXiv 2512.16615).
 *
 * This is the drop-in boundary: every entry point replaces one function of
 * the reference CPU library's operator API (P/ = /root/reference/proj/), cited
 * beside it.  Plain pointers and sizes only; no C++ or torch types cross it.
 *
 * Conventions
 *   - Device pointers, caller-owned, for `units` independent (batch·head)
 *     slices laid out unit-major: a [n][d] matrix has unit stride n*d
 *     elements.  Pyramids are levels 1..L concatenated per unit
 *     (row stride d, unit stride llsa_pyramid_rows()*d).  Selection tables are
 *     per_level 0..L-1 concatenated per unit ([n/B^(l+1)][K] u32 each).  CSC
 *     per level l: offsets [T_l+1], flat [T_l*K] (T_l = n/B^(l+1)),
 *     concatenated per unit.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and never synchronise; device-detected errors
 *     (out-of-range indices, non-finite outputs) raise a sticky per-device flag
 *     that llsa_sync_status() reads.  Argument/config errors are returned
 *     immediately, before any work, exactly where the reference throws.
 *   - Status codes map 1:1 onto the reference's exception types
 *     (P/include/llsa/errors.hpp:10-79); llsa_last_error() gives the message
 *     (thread-local).
 *   - Work counters (mul_accs) are analytic host functions, as in the
 *     reference (selection.cpp:75-77, attention.cpp:163, attention_grad.cpp).
 */
#ifndef LLSA_CUDA_H
#define LLSA_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LLSA_CUDA_ABI_VERSION 1

typedef enum llsa_status {
  LLSA_OK = 0,
  LLSA_ERR_CONFIG = 1,          /* ConfigError       errors.hpp:17 */
  LLSA_ERR_DIVISIBILITY = 2,    /* DivisibilityError errors.hpp:23 */
  LLSA_ERR_LEVEL = 3,           /* LevelError        errors.hpp:28 */
  LLSA_ERR_TOPK = 4,            /* TopKError         errors.hpp:33 */
  LLSA_ERR_SHAPE = 5,           /* ShapeMismatch     errors.hpp:38 */
  LLSA_ERR_INDEX_RANGE = 6,     /* IndexOutOfRange   errors.hpp:43 */
  LLSA_ERR_NONFINITE = 7,       /* NonFiniteError    errors.hpp:48 */
  LLSA_ERR_STALE_STATE = 8,     /* StaleState        errors.hpp:53 */
  LLSA_ERR_FORMAT = 9,          /* FormatError       errors.hpp:58 */
  LLSA_ERR_IO = 10,             /* IoError           errors.hpp:63 */
  LLSA_ERR_PRECISION = 11,      /* PrecisionError    errors.hpp:68 */
  LLSA_ERR_NOT_SQUARE_BLOCK = 12, /* NotSquareBlock  errors.hpp:73 */
  LLSA_ERR_ORACLE_CAP = 13,     /* OracleCapExceeded errors.hpp:78 */
  LLSA_ERR_CUDA = 20,           /* CUDA runtime failure (no reference analogue) */
  LLSA_ERR_UNSUPPORTED = 21,    /* shape outside what the kernels implement */
  LLSA_ERR_ARGUMENT = 22        /* null pointer / bad enum */
} llsa_status;

typedef enum llsa_dtype { LLSA_F32 = 0, LLSA_BF16 = 1 } llsa_dtype;

/* Mirrors LLSAConfig, P/include/llsa/config.hpp:19-29. */
typedef struct llsa_config {
  uint64_t n;               /* sequence length */
  uint32_t d;               /* feature dimension */
  uint32_t block_size;      /* B */
  uint32_t top_k;           /* K */
  uint32_t levels;          /* L */
  uint32_t enrich_levels;   /* L_e */
  float softmax_scale;      /* 0 → 1/sqrt(d) */
  uint32_t reweight_mode;   /* 0 ScaleKV, 1 LogitBias (config.hpp:14) */
  uint32_t safe_softmax;    /* running-max rescaling */
} llsa_config;

/* ---- errors / metadata ------------------------------------------------ */
int llsa_abi_version(void);
const char* llsa_last_error(void);
const char* llsa_status_name(llsa_status s);
/* Synchronises `stream`, returns and clears the device-side sticky error
 * flag of the current device (IndexOutOfRange / NonFinite / CUDA). */
llsa_status llsa_sync_status(void* stream);

/* ---- config (host, no device work) -------------------------------------- */
/* max_levels, P/src/config.cpp:54-64 */
uint32_t llsa_max_levels(uint64_t n, uint32_t block_size);
/* validate_config + effective_block_count, P/src/config.cpp:66-125 */
llsa_status llsa_validate_config(const llsa_config* cfg, float* scale,
                                 uint32_t* effective_blocks);
/* rows of the levels-1..L pyramid concatenation for one unit */
uint64_t llsa_pyramid_rows(uint64_t n, uint32_t block_size, uint32_t levels);
/* u32 entries of the per-unit selection tables (all levels) */
uint64_t llsa_table_entries(const llsa_config* cfg);
/* u32 entries of the per-unit CSC offsets / flat arrays (all levels) */
uint64_t llsa_csc_offsets_entries(const llsa_config* cfg);
uint64_t llsa_csc_flat_entries(const llsa_config* cfg);
/* Analytic multiply-accumulate counters (selection.cpp:75-77,145-147;
 * attention.cpp:163; attention_grad.cpp:114,164,198,258-259). */
uint64_t llsa_select_mul_accs(const llsa_config* cfg);
uint64_t llsa_forward_mul_accs(const llsa_config* cfg);
uint64_t llsa_backward_mul_accs(const llsa_config* cfg);

/* ---- compression ---------------------------------------------------------- */
/* build_pyramid, P/include/llsa/pyramid.hpp:26-27 (P/src/pyramid.cpp:11-43).
 * x [units][rows][d] in `dtype` → levels 1..L fp32 (level 0 is x itself,
 * never copied).  Sequential fp32 sum then ×(1/B): bit-exact. */
llsa_status llsa_build_pyramid(const void* x, llsa_dtype dtype, uint32_t units,
                               uint64_t rows, uint32_t d, uint32_t block_size,
                               uint32_t levels, float* levels_out, void* stream);
/* pool_backward, P/include/llsa/pyramid.hpp:31-32 (P/src/pyramid.cpp:45-64) */
llsa_status llsa_pool_backward(const float* d_coarse, uint32_t units,
                               uint64_t coarse_rows, uint32_t d,
                               uint32_t block_size, uint32_t hops, float* d_fine,
                               void* stream);

/* ---- 2-D reordering (P/include/llsa/reorder2d.hpp) ------------------------- */
/* build_reorder, reorder2d.hpp:31-32 (P/src/reorder2d.cpp:11-69): host-side
 * hierarchical curve for an height x width image, block_size = s^2.  Writes
 * forward[pos] (raster index at sequence position pos) and inverse[raster]
 * (height*width entries each, host memory).  NotSquareBlock /
 * DivisibilityError exactly where the reference throws. */
llsa_status llsa_build_reorder(uint32_t height, uint32_t width, uint32_t block_size,
                               uint32_t* forward, uint32_t* inverse);
/* apply_permutation, reorder2d.hpp:38-39 (reorder2d.cpp:71-88): row gather
 * out[u][i] = x[u][map[i]] on device (map = forward or inverse, device
 * memory, `rows` entries); rows of d elements of `dtype`. */
llsa_status llsa_apply_permutation(const void* x, llsa_dtype dtype, uint32_t units,
                                   uint64_t rows, uint32_t d, const uint32_t* map, void* out,
                                   void* stream);
/* build_pyramid(apply_permutation(x, map)) without materialising the
 * permuted copy: the gather is fused into level-1 pooling (bit-identical). */
llsa_status llsa_build_pyramid_permuted(const void* x, llsa_dtype dtype, uint32_t units,
                                        uint64_t rows, uint32_t d, uint32_t block_size,
                                        uint32_t levels, const uint32_t* map, float* levels_out,
                                        void* stream);

/* ---- selection ------------------------------------------------------------ */
/* select_coarsest, P/include/llsa/selection.hpp:47-50 (selection.cpp:42-79).
 * q_top [units][rows][d], k_top [units][cands][d] → out [units][rows][K]. */
llsa_status llsa_select_coarsest(const float* q_top, const float* k_top,
                                 uint32_t units, uint32_t rows, uint32_t cands,
                                 uint32_t d, uint32_t top_k, float scale,
                                 uint32_t* out, void* stream);
/* select_level, P/include/llsa/selection.hpp:57-61 (selection.cpp:81-149).
 * q_l [units][parent_rows*B][d], k_l [units][k_rows][d], parent
 * [units][parent_rows][parent_k] → out [units][parent_rows*B][K]. */
llsa_status llsa_select_level(const float* q_l, const float* k_l,
                              const uint32_t* parent, uint32_t units,
                              uint32_t parent_level, uint32_t parent_rows,
                              uint32_t parent_k, uint64_t k_rows, uint32_t d,
                              uint32_t top_k, float scale, uint32_t block_size,
                              uint32_t* out, void* stream);
/* hierarchical_topk, P/include/llsa/selection.hpp:64-65 (selection.cpp:151-179)
 * on pyramids from llsa_build_pyramid → per-unit tables. */
llsa_status llsa_hierarchical_topk(const llsa_config* cfg, uint32_t units,
                                   const float* pyr_q, const float* pyr_k,
                                   uint32_t* tables, void* stream);

/* ---- CSR → CSC ------------------------------------------------------------ */
/* Scratch for llsa_transpose_indices / llsa_transpose_all (bytes). */
size_t llsa_transpose_workspace_bytes(uint32_t units, uint32_t rows, uint32_t k,
                                      uint32_t key_blocks);
/* transpose_indices, P/include/llsa/indexmap.hpp:32-33 (indexmap.cpp:14-72):
 * count → exclusive scan → scatter → canonical ascending segments.
 * idx [units][rows][k] → offsets [units][key_blocks+1], flat [units][rows*k]. */
llsa_status llsa_transpose_indices(const uint32_t* idx, uint32_t units,
                                   uint32_t rows, uint32_t k, uint32_t key_blocks,
                                   uint32_t* offsets, uint32_t* flat,
                                   void* workspace, size_t workspace_bytes,
                                   void* stream);
/* transpose_all, P/include/llsa/indexmap.hpp:36-37 (indexmap.cpp:74-88). */
size_t llsa_transpose_all_workspace_bytes(const llsa_config* cfg, uint32_t units);
llsa_status llsa_transpose_all(const llsa_config* cfg, uint32_t units,
                               const uint32_t* tables, uint32_t* csc_offsets,
                               uint32_t* csc_flat, void* workspace,
                               size_t workspace_bytes, void* stream);

/* ---- enriched plan + forward ----------------------------------------------- */
/* build_plan, P/include/llsa/attention.hpp:44-45 (attention.cpp:80-122).
 * → [units][n/B][E] (level, block, weight). */
llsa_status llsa_build_plan(const llsa_config* cfg, uint32_t units,
                            const uint32_t* tables, uint32_t* plan_level,
                            uint32_t* plan_block, float* plan_weight,
                            void* stream);
/* llsa_forward, P/include/llsa/attention.hpp:65-73 (attention.cpp:145-219).
 * Reads the selection tables directly (no materialised plan).  q, k, v in
 * `dtype`; pyr_k/pyr_v fp32 from llsa_build_pyramid.  Writes out [n][d]
 * fp32, row_max and row_denom [n] fp32 (ForwardState, attention.hpp:51-55). */
llsa_status llsa_forward(const llsa_config* cfg, uint32_t units, llsa_dtype dtype,
                         const void* q, const void* k, const void* v,
                         const float* pyr_k, const float* pyr_v,
                         const uint32_t* tables, float* out, float* row_max,
                         float* row_denom, void* stream);

/* llsa_forward over a materialised EnrichedKVPlan (attention.hpp:34-41):
 * plan_{level,block,weight} [units][n/B][entries_per_block], any entries
 * (hand-built plans included, weights honoured as attention.cpp:176-180).
 * The caller range-checks the plan (attention.cpp:74-76). */
llsa_status llsa_forward_plan(const llsa_config* cfg, uint32_t units, llsa_dtype dtype,
                              const void* q, const void* k, const void* v,
                              const float* pyr_k, const float* pyr_v,
                              const uint32_t* plan_level, const uint32_t* plan_block,
                              const float* plan_weight, uint32_t entries_per_block,
                              float* out, float* row_max, float* row_denom, void* stream);

/* ---- backward ---------------------------------------------------------------- */
size_t llsa_backward_workspace_bytes(const llsa_config* cfg, uint32_t units);
/* llsa_backward, P/include/llsa/attention_grad.hpp:45-52
 * (attention_grad.cpp:204-265): D pre-pass, query-major dq, key-major dk/dv
 * over the CSC lists plus the pooling adjoint for coarse levels.  Outputs
 * dq, dk, dv [n][d] fp32.  The reference's StaleState checksum is a host
 * concern (the C++ shim, include/llsa/attention.hpp). */
llsa_status llsa_backward(const llsa_config* cfg, uint32_t units, llsa_dtype dtype,
                          const void* d_out, const float* out,
                          const float* row_max, const float* row_denom,
                          const void* q, const void* k, const void* v,
                          const float* pyr_k, const float* pyr_v,
                          const uint32_t* tables, const uint32_t* csc_offsets,
                          const uint32_t* csc_flat, float* dq, float* dk,
                          float* dv, void* workspace, size_t workspace_bytes,
                          void* stream);
/* llsa_backward with dq taken over a materialised plan (as the reference's
 * query-major phase, attention_grad.cpp:229-257); dk/dv from the CSC lists. */
llsa_status llsa_backward_plan(const llsa_config* cfg, uint32_t units, llsa_dtype dtype,
                               const void* d_out, const float* out, const float* row_max,
                               const float* row_denom, const void* q, const void* k,
                               const void* v, const float* pyr_k, const float* pyr_v,
                               const uint32_t* plan_level, const uint32_t* plan_block,
                               const float* plan_weight, uint32_t entries_per_block,
                               const uint32_t* csc_offsets, const uint32_t* csc_flat,
                               float* dq, float* dk, float* dv, void* workspace,
                               size_t workspace_bytes, void* stream);
/* kv_backward, P/include/llsa/attention_grad.hpp:32-37 (attention_grad.cpp:90-202):
 * dk/dv only (dq not computed). */
llsa_status llsa_kv_backward(const llsa_config* cfg, uint32_t units,
                             llsa_dtype dtype, const void* d_out,
                             const float* out, const float* row_max,
                             const float* row_denom, const void* q,
                             const float* pyr_k, const float* pyr_v,
                             const void* k, const void* v,
                             const uint32_t* csc_offsets, const uint32_t* csc_flat,
                             float* dk, float* dv, void* workspace,
                             size_t workspace_bytes, void* stream);

/* mask_kv_backward, P/include/llsa/oracle.hpp:54-63 (P/src/oracle.cpp:365-501):
 * the measured baseline of the key/value backward.  The key→query lookup
 * goes through a dense query-block × key-block mask per level (O(T^2) build
 * and column scan) instead of the CSC; same math and kernels otherwise.
 * tables as produced by llsa_hierarchical_topk. */
size_t llsa_mask_kv_backward_workspace_bytes(const llsa_config* cfg, uint32_t units);
llsa_status llsa_mask_kv_backward(const llsa_config* cfg, uint32_t units,
                                  llsa_dtype dtype, const void* d_out,
                                  const float* out, const float* row_max,
                                  const float* row_denom, const void* q,
                                  const float* pyr_k, const float* pyr_v,
                                  const void* k, const void* v, const uint32_t* tables,
                                  float* dk, float* dv, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ---- fused path (the B200 fast path; one handle owns all scratch) ---------- */
/* A handle caches the per-unit pyramids, tables, CSC lists, softmax
 * statistics and every intermediate of the path for `units` units of one
 * config, so a training step is exactly two calls.  When d = 64, B = 16 and
 * dtype = BF16 the attention runs on the tensor-core kernels; every other
 * shape uses the general SIMT kernels.  Both paths are hand-written CUDA. */
typedef struct llsa_handle_s* llsa_handle;

typedef enum llsa_buffer {
  LLSA_BUF_PYR_Q = 0, LLSA_BUF_PYR_K = 1, LLSA_BUF_PYR_V = 2,
  LLSA_BUF_TABLES = 3, LLSA_BUF_CSC_OFFSETS = 4, LLSA_BUF_CSC_FLAT = 5,
  LLSA_BUF_ROW_MAX = 6, LLSA_BUF_ROW_DENOM = 7
} llsa_buffer;

llsa_status llsa_handle_create(const llsa_config* cfg, uint32_t units,
                               llsa_dtype dtype, llsa_handle* out);
llsa_status llsa_handle_destroy(llsa_handle h);
/* 1 when the handle runs the tensor-core attention kernels. */
int llsa_handle_uses_tensor_cores(llsa_handle h);
/* Forward: compress → select → attention.  out [units][n][d] fp32. */
llsa_status llsa_handle_forward(llsa_handle h, const void* q, const void* k,
                                const void* v, float* out, void* stream);
/* Backward: transpose → backward.  Requires the preceding forward on the
 * same handle and the same q/k/v/out buffers.  On the tensor-core path the
 * coarse-level dK'/dV' sums are unordered fp32 reductions by default (dk, dv
 * reproducible to fp32 rounding); LLSA_DETERMINISTIC=1 in the environment
 * selects the ordered form (bitwise reproducible, as the reference). */
llsa_status llsa_handle_backward(llsa_handle h, const void* d_out, const void* q,
                                 const void* k, const void* v, const float* out,
                                 float* dq, float* dk, float* dv, void* stream);
/* The same two calls with the outputs in `out_dtype`: LLSA_F32 is exactly
 * llsa_handle_forward / llsa_handle_backward; LLSA_BF16 writes out, dq, dk,
 * dv as bf16 (RNE of the fp32 results; half the bytes to move off the GPU).
 * In bf16 mode the handle keeps the fp32 output internally for the backward's
 * D = rowsum(dO∘O), so `out` given to the backward must be the bf16 output of
 * the handle's latest forward (else LLSA_ERR_STALE_STATE). */
llsa_status llsa_handle_forward_ex(llsa_handle h, const void* q, const void* k,
                                   const void* v, void* out, llsa_dtype out_dtype,
                                   void* stream);
llsa_status llsa_handle_backward_ex(llsa_handle h, const void* d_out, const void* q,
                                    const void* k, const void* v, const void* out,
                                    void* dq, void* dk, void* dv, llsa_dtype out_dtype,
                                    void* stream);
llsa_status llsa_handle_buffer(llsa_handle h, llsa_buffer which, void** ptr,
                               size_t* bytes);
/* Number of kernel launches the last forward / backward issued. */
uint32_t llsa_handle_last_launches(llsa_handle h);
/* Stage timing: when enabled, forward/backward record a CUDA event on the
 * call's stream between stages (no synchronisation).  llsa_handle_stage_times
 * synchronises on those events and returns up to `cap` (name, ms) pairs of
 * the most recent forward followed by the most recent backward; names are
 * static strings.  Returns the number of stages. */
llsa_status llsa_handle_enable_timing(llsa_handle h, int enable);
uint32_t llsa_handle_stage_times(llsa_handle h, const char** names, float* ms,
                                 uint32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* LLSA_CUDA_H */
