/*
 * TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * Plain-C restatement of the reference LLSA hot path (arXiv 2512.16615,
 * /root/reference/proj, f32 build) used as the oracle for the CUDA kernels.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  Every function cites the reference file:line it restates
 * (P/ = /root/reference/proj/).  Arithmetic is float with the reference's
 * exact operation order (4-lane dot, sequential pooling, no FMA), so outputs
 * are bit-identical to the reference f32 library; that equality is pinned by
 * tests/test_oracle.py against oracle/_ref and the golden fixtures.
 *
 * Layout conventions (all row-major, one (batch, head) unit):
 *   x, q, k, v, d_out : [n][d]
 *   pyramid levels    : levels 1..L concatenated, level l is [n/B^l][d]
 *   selection tables  : per_level 0..L-1 concatenated, level l is
 *                       [n/B^(l+1)][K] u32, rows ascending
 *   CSC               : per level l: offsets [T_l+1], flat [T_l*K]
 *                       (T_l = n/B^(l+1)), concatenated over levels
 * Status codes equal llsa_status in include/llsa_cuda.h.
 */
#ifndef LLSA_ORACLE_H
#define LLSA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
/* build_reorder, P/src/reorder2d.cpp:11-69: the hierarchical 2-D curve
 * (forward[pos] = raster index, inverse = its inverse).  Returns a status
 * code (2 DivisibilityError, 12 NotSquareBlock) like the reference throws. */
int oracle_build_reorder(uint32_t height, uint32_t width, uint32_t block_size,
                         uint32_t* forward, uint32_t* inverse);

#endif

typedef struct oracle_config {
  uint64_t n;
  uint32_t d, block_size, top_k, levels, enrich_levels;
  float softmax_scale;    /* 0 → 1/sqrt(d) */
  uint32_t reweight_mode; /* 0 ScaleKV, 1 LogitBias */
  uint32_t safe_softmax;
} oracle_config;

uint32_t oracle_max_levels(uint64_t n, uint32_t block_size);
int oracle_validate(const oracle_config* c, float* scale, uint32_t* eff);
void oracle_gen_random(float* out, size_t rows, size_t cols, uint64_t seed,
                       int uniform);

int oracle_build_pyramid(const float* x, size_t rows, size_t d, uint32_t B,
                         uint32_t levels, float* levels_out);
int oracle_pool_backward(const float* g, size_t rows, size_t d, uint32_t B,
                         uint32_t hops, float* out);
int oracle_select_coarsest(const float* q, size_t q_rows, const float* k,
                           size_t k_rows, size_t d, uint32_t top_k, float scale,
                           uint32_t* out);
int oracle_select_level(const float* q, size_t q_rows, const float* k,
                        size_t k_rows, size_t d, const uint32_t* parent,
                        uint32_t parent_level, uint32_t parent_rows,
                        uint32_t parent_k, uint32_t top_k, float scale,
                        uint32_t B, uint32_t* out);
int oracle_hierarchical_topk(const oracle_config* c, const float* pyr_q,
                             const float* pyr_k, uint32_t* tables,
                             uint64_t* mul_accs);
int oracle_transpose(const uint32_t* idx, uint32_t rows, uint32_t k,
                     uint32_t key_blocks, uint32_t* offsets, uint32_t* flat);
int oracle_build_plan(const oracle_config* c, const uint32_t* tables,
                      uint32_t* plan_level, uint32_t* plan_block,
                      float* plan_weight);
int oracle_forward(const oracle_config* c, const float* q, const float* k,
                   const float* v, const float* pyr_k, const float* pyr_v,
                   const uint32_t* tables, float* out, float* row_max,
                   float* row_denom);
int oracle_backward(const oracle_config* c, const float* d_out,
                    const float* out, const float* row_max,
                    const float* row_denom, const float* q, const float* k,
                    const float* v, const float* pyr_k, const float* pyr_v,
                    const uint32_t* tables, const uint32_t* csc_offsets,
                    const uint32_t* csc_flat, float* dq, float* dk, float* dv);
uint64_t oracle_input_checksum(const oracle_config* c, const float* q,
                               const float* k, const float* v);

#ifdef __cplusplus
}
/* build_reorder, P/src/reorder2d.cpp:11-69: the hierarchical 2-D curve
 * (forward[pos] = raster index, inverse = its inverse).  Returns a status
 * code (2 DivisibilityError, 12 NotSquareBlock) like the reference throws. */
int oracle_build_reorder(uint32_t height, uint32_t width, uint32_t block_size,
                         uint32_t* forward, uint32_t* inverse);

#endif
/* build_reorder, P/src/reorder2d.cpp:11-69: the hierarchical 2-D curve
 * (forward[pos] = raster index, inverse = its inverse).  Returns a status
 * code (2 DivisibilityError, 12 NotSquareBlock) like the reference throws. */
int oracle_build_reorder(uint32_t height, uint32_t width, uint32_t block_size,
                         uint32_t* forward, uint32_t* inverse);

#endif
