// The C ABI (include/llsa_cuda.h): argument/config validation in the
// reference's order and error kinds, then stream-ordered kernel launches.
// No entry point synchronises; device-detected errors land in a sticky
// per-device flag read by llsa_sync_status().
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include "internal.h"
#include "tc.h"
#include "common.cuh"

namespace llsa_impl {

namespace {
thread_local char g_msg[512] = "";
thread_local uint32_t g_launches = 0;
std::mutex g_flag_mu;
uint32_t* g_flags[64] = {};
}  // namespace

llsa_status fail(llsa_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return s;
}

llsa_status cuda_fail(cudaError_t e, const char* what) {
  return fail(LLSA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

void count_launch(uint32_t n) { g_launches += n; }
uint32_t take_launch_count() {
  const uint32_t n = g_launches;
  g_launches = 0;
  return n;
}

uint32_t* device_flag() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_flag_mu);
  if (!g_flags[dev]) {
    uint32_t* p = nullptr;
    if (cudaMalloc(&p, sizeof(uint32_t)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, sizeof(uint32_t));
    g_flags[dev] = p;
  }
  return g_flags[dev];
}

static uint32_t max_levels_impl(uint64_t n, uint32_t b) {
  if (b < 2 || n == 0) return 0;  // config.cpp:54-64
  uint32_t l = 0;
  uint64_t p = b;
  while (p <= n / b) {
    p *= b;
    ++l;
  }
  return l;
}

llsa_status make_geometry(const llsa_config* c, Geometry* g) {
  if (!c) return fail(LLSA_ERR_ARGUMENT, "null config");
  // validate_config, P/src/config.cpp:66-117 — same checks, same order.
  if (c->n == 0) return fail(LLSA_ERR_CONFIG, "sequence length must be positive");
  if (c->d == 0) return fail(LLSA_ERR_CONFIG, "feature dimension must be positive");
  if (c->block_size < 2) return fail(LLSA_ERR_CONFIG, "block size must be at least 2");
  if (c->n > 0xffffffffull)
    return fail(LLSA_ERR_CONFIG, "sequence length exceeds the 32-bit index range");
  if (!std::isfinite(c->softmax_scale) || c->softmax_scale < 0.f)
    return fail(LLSA_ERR_CONFIG, "softmax scale must be finite and non-negative");
  const uint32_t lmax = max_levels_impl(c->n, c->block_size);
  if (c->levels < 1 || c->levels > lmax)
    return fail(LLSA_ERR_LEVEL, "levels must lie in [1, %u] for n=%llu, block size %u", lmax,
                (unsigned long long)c->n, c->block_size);
  uint64_t pow_l = 1;
  for (uint32_t l = 0; l < c->levels; ++l) pow_l *= c->block_size;
  if (c->n % pow_l != 0)
    return fail(LLSA_ERR_DIVISIBILITY,
                "sequence length %llu is not divisible by block_size^levels = %llu",
                (unsigned long long)c->n, (unsigned long long)pow_l);
  if (c->enrich_levels > c->levels)
    return fail(LLSA_ERR_LEVEL, "enrich_levels %u exceeds levels %u", c->enrich_levels,
                c->levels);
  const uint64_t coarsest = c->n / pow_l;
  if (c->top_k < 1 || c->top_k > coarsest)
    return fail(LLSA_ERR_TOPK, "top_k must lie in [1, %llu] (coarsest-level candidate count)",
                (unsigned long long)coarsest);
  if (c->reweight_mode > 1) return fail(LLSA_ERR_ARGUMENT, "bad reweight mode");

  Geometry G;
  G.n = c->n;
  G.d = c->d;
  G.B = c->block_size;
  G.K = c->top_k;
  G.L = c->levels;
  G.Le = c->enrich_levels;
  G.scale = c->softmax_scale > 0.f ? c->softmax_scale : 1.0f / std::sqrt((float)c->d);
  G.mode = c->reweight_mode;
  G.safe = c->safe_softmax ? 1 : 0;
  G.pow[0] = 1;
  for (uint32_t l = 1; l <= G.L + 1; ++l) G.pow[l] = G.pow[l - 1] * G.B;
  G.pyr_rows = 0;
  for (uint32_t l = 1; l <= G.L; ++l) {
    G.pyr_off[l] = G.pyr_rows;
    G.pyr_rows += G.n / G.pow[l];
  }
  G.table_entries = 0;
  G.csc_off_entries = G.csc_flat_entries = 0;
  for (uint32_t l = 0; l < G.L; ++l) {
    G.table_off[l] = G.table_entries;
    G.csc_off_off[l] = G.csc_off_entries;
    G.csc_flat_off[l] = G.csc_flat_entries;
    G.table_entries += G.level_blocks(l) * G.K;
    G.csc_off_entries += G.level_blocks(l) + 1;
    G.csc_flat_entries += G.level_blocks(l) * G.K;
  }
  // effective_block_count, config.cpp:119-125
  G.E = G.K * G.enrich_lim() + (G.Le == G.L ? (uint32_t)G.level_blocks(G.L) : 0u);
  *g = G;
  return LLSA_OK;
}

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

llsa_status hier_topk(const Geometry& g, uint32_t units, const float* pyr_q,
                      const float* pyr_k, uint32_t* tables, cudaStream_t s) {
  const uint64_t ps = g.pyr_rows * g.d;
  const uint64_t top = g.level_tokens(g.L);
  // coarsest stage on level L → table level L-1 (selection.cpp:167-169)
  llsa_status st = launch_select_coarsest(
      pyr_q + g.pyr_off[g.L] * g.d, ps, pyr_k + g.pyr_off[g.L] * g.d, ps, units,
      (uint32_t)top, (uint32_t)top, g.d, g.K, g.scale, tables + g.table_off[g.L - 1],
      g.table_entries, s);
  if (st) return st;
  for (uint32_t l = g.L - 1; l >= 1; --l) {  // selection.cpp:170-175
    st = launch_select_level(pyr_q + g.pyr_off[l] * g.d, ps, pyr_k + g.pyr_off[l] * g.d, ps,
                             tables + g.table_off[l], g.table_entries, units,
                             (uint32_t)g.level_blocks(l), g.K, g.level_tokens(l), g.d, g.K,
                             g.scale, g.B, tables + g.table_off[l - 1], g.table_entries, s);
    if (st) return st;
  }
  return LLSA_OK;
}

llsa_status pyramid(const Geometry& g, uint32_t units, const void* x, llsa_dtype dt,
                    float* out, cudaStream_t s) {
  const uint64_t ps = g.pyr_rows * g.d;
  llsa_status st = launch_pool_level(x, dt, g.n * g.d, out, ps, units, g.level_tokens(1), g.d,
                                     g.B, s);
  for (uint32_t l = 2; l <= g.L && st == LLSA_OK; ++l)
    st = launch_pool_level(out + g.pyr_off[l - 1] * g.d, LLSA_F32, ps, out + g.pyr_off[l] * g.d,
                           ps, units, g.level_tokens(l), g.d, g.B, s);
  return st;
}

llsa_status transpose_all_impl(const Geometry& g, uint32_t units, const uint32_t* tables,
                               uint32_t* offs, uint32_t* flat, void* ws, cudaStream_t s) {
  for (uint32_t l = 0; l < g.L; ++l) {
    const uint32_t kb = (uint32_t)g.level_blocks(l);
    llsa_status st = launch_transpose(tables + g.table_off[l], g.table_entries, units, kb,
                                      g.K, kb, offs + g.csc_off_off[l], g.csc_off_entries,
                                      flat + g.csc_flat_off[l], g.csc_flat_entries, ws, s);
    if (st) return st;
  }
  return LLSA_OK;
}

size_t transpose_all_ws(const Geometry& g, uint32_t units) {
  size_t m = 256;
  for (uint32_t l = 0; l < g.L; ++l) {
    const uint32_t kb = (uint32_t)g.level_blocks(l);
    const size_t b = transpose_ws_bytes(units, kb, g.K, kb);
    if (b > m) m = b;
  }
  return m;
}

}  // namespace

extern "C" {

int llsa_abi_version(void) { return LLSA_CUDA_ABI_VERSION; }
const char* llsa_last_error(void) { return g_msg; }

const char* llsa_status_name(llsa_status s) {
  switch (s) {
    case LLSA_OK: return "ok";
    case LLSA_ERR_CONFIG: return "ConfigError";
    case LLSA_ERR_DIVISIBILITY: return "DivisibilityError";
    case LLSA_ERR_LEVEL: return "LevelError";
    case LLSA_ERR_TOPK: return "TopKError";
    case LLSA_ERR_SHAPE: return "ShapeMismatch";
    case LLSA_ERR_INDEX_RANGE: return "IndexOutOfRange";
    case LLSA_ERR_NONFINITE: return "NonFiniteError";
    case LLSA_ERR_STALE_STATE: return "StaleState";
    case LLSA_ERR_FORMAT: return "FormatError";
    case LLSA_ERR_IO: return "IoError";
    case LLSA_ERR_PRECISION: return "PrecisionError";
    case LLSA_ERR_NOT_SQUARE_BLOCK: return "NotSquareBlock";
    case LLSA_ERR_ORACLE_CAP: return "OracleCapExceeded";
    case LLSA_ERR_CUDA: return "CudaError";
    case LLSA_ERR_UNSUPPORTED: return "Unsupported";
    case LLSA_ERR_ARGUMENT: return "ArgumentError";
  }
  return "unknown";
}

llsa_status llsa_sync_status(void* stream) {
  LLSA_CUDA_TRY(cudaStreamSynchronize(S(stream)));
  uint32_t* f = device_flag();
  if (!f) return fail(LLSA_ERR_CUDA, "no device flag");
  uint32_t h = 0;
  LLSA_CUDA_TRY(cudaMemcpy(&h, f, sizeof(h), cudaMemcpyDeviceToHost));
  if (h) LLSA_CUDA_TRY(cudaMemset(f, 0, sizeof(uint32_t)));
  if (h & llsa_dev::kErrIndex)
    return fail(LLSA_ERR_INDEX_RANGE, "selection or plan entry outside its level");
  if (h & llsa_dev::kErrNonFinite)
    return fail(LLSA_ERR_NONFINITE, "attention output contains non-finite values");
  return LLSA_OK;
}

uint32_t llsa_max_levels(uint64_t n, uint32_t b) { return max_levels_impl(n, b); }

llsa_status llsa_validate_config(const llsa_config* cfg, float* scale, uint32_t* eff) {
  Geometry g;
  llsa_status st = make_geometry(cfg, &g);
  if (st) return st;
  if (scale) *scale = g.scale;
  if (eff) *eff = g.E;
  return LLSA_OK;
}

uint64_t llsa_pyramid_rows(uint64_t n, uint32_t b, uint32_t levels) {
  uint64_t r = 0, t = n;
  for (uint32_t l = 1; l <= levels && b; ++l) {
    t /= b;
    r += t;
  }
  return r;
}

uint64_t llsa_table_entries(const llsa_config* cfg) {
  Geometry g;
  return make_geometry(cfg, &g) ? 0 : g.table_entries;
}
uint64_t llsa_csc_offsets_entries(const llsa_config* cfg) {
  Geometry g;
  return make_geometry(cfg, &g) ? 0 : g.csc_off_entries;
}
uint64_t llsa_csc_flat_entries(const llsa_config* cfg) {
  Geometry g;
  return make_geometry(cfg, &g) ? 0 : g.csc_flat_entries;
}

uint64_t llsa_select_mul_accs(const llsa_config* cfg) {
  Geometry g;
  if (make_geometry(cfg, &g)) return 0;
  const uint64_t top = g.level_tokens(g.L);
  uint64_t m = top * top * g.d;  // selection.cpp:75-77
  for (uint32_t l = 1; l < g.L; ++l) m += g.level_tokens(l) * g.K * g.B * g.d;  // :145-147
  return m;
}

uint64_t llsa_forward_mul_accs(const llsa_config* cfg) {
  Geometry g;
  if (make_geometry(cfg, &g)) return 0;
  return g.n * g.E * g.B * g.d;  // attention.cpp:163
}

uint64_t llsa_backward_mul_accs(const llsa_config* cfg) {
  Geometry g;
  if (make_geometry(cfg, &g)) return 0;
  // attention_grad.cpp:258-259 (dq + D) and :114,164,198 (kv incl. its own D)
  uint64_t m = g.n * g.E * g.B * 3 * g.d + 2 * g.n * g.d;
  uint64_t kv = 2 * g.n * g.d;
  for (uint32_t l = 0; l < g.enrich_lim(); ++l)
    kv += g.level_blocks(l) * g.K * g.pow[l + 1] * g.B * 4 * g.d;
  if (g.Le == g.L) kv += g.n * g.level_tokens(g.L) * 4 * g.d;
  return m + kv;
}

llsa_status llsa_build_pyramid(const void* x, llsa_dtype dt, uint32_t units, uint64_t rows,
                               uint32_t d, uint32_t B, uint32_t levels, float* out,
                               void* stream) {
  if (llsa_status st = dtype_ok(dt)) return st;
  if (B < 2) return fail(LLSA_ERR_DIVISIBILITY, "block size must be at least 2");
  uint64_t r = rows;
  for (uint32_t l = 1; l <= levels; ++l) {  // pyramid.cpp:23-28
    if (r % B != 0)
      return fail(LLSA_ERR_DIVISIBILITY, "level %u has %llu rows, not a multiple of block size %u",
                  l - 1, (unsigned long long)r, B);
    r /= B;
  }
  if (levels == 0 || units == 0 || rows == 0) return LLSA_OK;
  NONNULL(x);
  NONNULL(out);
  const uint64_t pr = llsa_pyramid_rows(rows, B, levels);
  llsa_status st = launch_pool_level(x, dt, rows * d, out, pr * d, units, rows / B, d, B,
                                     S(stream));
  uint64_t off_prev = 0, rows_prev = rows / B;
  for (uint32_t l = 2; l <= levels && st == LLSA_OK; ++l) {
    const uint64_t off = off_prev + rows_prev;
    st = launch_pool_level(out + off_prev * d, LLSA_F32, pr * d, out + off * d, pr * d, units,
                           rows_prev / B, d, B, S(stream));
    off_prev = off;
    rows_prev /= B;
  }
  return st;
}

llsa_status llsa_pool_backward(const float* g, uint32_t units, uint64_t coarse_rows, uint32_t d,
                               uint32_t B, uint32_t hops, float* out, void* stream) {
  const uint64_t group = llsa_dev::ipow_u64(B, hops);
  if (hops == 0) {  // pyramid.cpp:47: identity
    if (units && coarse_rows && d) {
      NONNULL(g);
      NONNULL(out);
      LLSA_CUDA_TRY(cudaMemcpyAsync(out, g, (size_t)units * coarse_rows * d * 4,
                                    cudaMemcpyDeviceToDevice, S(stream)));
    }
    return LLSA_OK;
  }
  if (B < 2) return fail(LLSA_ERR_DIVISIBILITY, "block size must be at least 2");
  if (units == 0 || coarse_rows == 0 || d == 0) return LLSA_OK;
  NONNULL(g);
  NONNULL(out);
  return launch_pool_backward(g, units, coarse_rows, d, group, out, S(stream));
}

llsa_status llsa_select_coarsest(const float* q, const float* k, uint32_t units, uint32_t rows,
                                 uint32_t cands, uint32_t d, uint32_t top_k, float scale,
                                 uint32_t* out, void* stream) {
  if (top_k < 1 || top_k > cands)  // selection.cpp:48-51
    return fail(LLSA_ERR_TOPK, "top_k %u outside [1, %u]", top_k, cands);
  if (units == 0 || rows == 0) return LLSA_OK;
  NONNULL(q);
  NONNULL(k);
  NONNULL(out);
  return launch_select_coarsest(q, (uint64_t)rows * d, k, (uint64_t)cands * d, units, rows,
                                cands, d, top_k, scale, out, (uint64_t)rows * top_k, S(stream));
}

llsa_status llsa_select_level(const float* q, const float* k, const uint32_t* parent,
                              uint32_t units, uint32_t parent_level, uint32_t parent_rows,
                              uint32_t parent_k, uint64_t k_rows, uint32_t d, uint32_t top_k,
                              float scale, uint32_t B, uint32_t* out, void* stream) {
  // selection.cpp:84-105, same order
  if (parent_level == 0)
    return fail(LLSA_ERR_LEVEL, "select_level needs a parent table at level >= 1");
  if (B == 0 || k_rows % B != 0)
    return fail(LLSA_ERR_SHAPE, "level selection: key token count not a multiple of the "
                "block size");
  const uint64_t cand = (uint64_t)parent_k * B;
  if (top_k < 1 || top_k > cand)
    return fail(LLSA_ERR_TOPK, "top_k %u outside [1, %llu]", top_k, (unsigned long long)cand);
  if (units == 0 || parent_rows == 0) return LLSA_OK;
  NONNULL(q);
  NONNULL(k);
  NONNULL(parent);
  NONNULL(out);
  return launch_select_level(q, (uint64_t)parent_rows * B * d, k, k_rows * d, parent,
                             (uint64_t)parent_rows * parent_k, units, parent_rows, parent_k,
                             k_rows, d, top_k, scale, B, out,
                             (uint64_t)parent_rows * B * top_k, S(stream));
}

llsa_status llsa_hierarchical_topk(const llsa_config* cfg, uint32_t units, const float* pyr_q,
                                   const float* pyr_k, uint32_t* tables, void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(pyr_q);
  NONNULL(pyr_k);
  NONNULL(tables);
  return hier_topk(g, units, pyr_q, pyr_k, tables, S(stream));
}

size_t llsa_transpose_workspace_bytes(uint32_t units, uint32_t rows, uint32_t k,
                                      uint32_t key_blocks) {
  return transpose_ws_bytes(units, rows, k, key_blocks);
}

llsa_status llsa_transpose_indices(const uint32_t* idx, uint32_t units, uint32_t rows,
                                   uint32_t k, uint32_t key_blocks, uint32_t* offsets,
                                   uint32_t* flat, void* ws, size_t ws_bytes, void* stream) {
  if (units == 0) return LLSA_OK;
  NONNULL(offsets);
  if (rows != 0 && k != 0) {
    NONNULL(idx);
    NONNULL(flat);
  }
  if (!ws || ws_bytes < transpose_ws_bytes(units, rows, k, key_blocks))
    return fail(LLSA_ERR_ARGUMENT, "transpose workspace too small");
  return launch_transpose(idx, (uint64_t)rows * k, units, rows, k, key_blocks, offsets,
                          (uint64_t)key_blocks + 1, flat, (uint64_t)rows * k, ws, S(stream));
}

size_t llsa_transpose_all_workspace_bytes(const llsa_config* cfg, uint32_t units) {
  Geometry g;
  if (make_geometry(cfg, &g)) return 0;
  return transpose_all_ws(g, units);
}

llsa_status llsa_transpose_all(const llsa_config* cfg, uint32_t units, const uint32_t* tables,
                               uint32_t* offs, uint32_t* flat, void* ws, size_t ws_bytes,
                               void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(tables);
  NONNULL(offs);
  NONNULL(flat);
  if (!ws || ws_bytes < transpose_all_ws(g, units))
    return fail(LLSA_ERR_ARGUMENT, "transpose workspace too small");
  return transpose_all_impl(g, units, tables, offs, flat, ws, S(stream));
}

llsa_status llsa_build_plan(const llsa_config* cfg, uint32_t units, const uint32_t* tables,
                            uint32_t* pl, uint32_t* pb, float* pw, void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(tables);
  NONNULL(pl);
  NONNULL(pb);
  NONNULL(pw);
  return launch_build_plan(g, units, tables, pl, pb, pw, S(stream));
}

llsa_status llsa_forward(const llsa_config* cfg, uint32_t units, llsa_dtype dt, const void* q,
                         const void* k, const void* v, const float* pyr_k, const float* pyr_v,
                         const uint32_t* tables, float* out, float* rm, float* rd,
                         void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(tables);
  NONNULL(out);
  NONNULL(rm);
  NONNULL(rd);
  if (g.L >= 1 && (!pyr_k || !pyr_v)) return fail(LLSA_ERR_ARGUMENT, "null pyramid");
  if (tc_supported(g, dt)) {
    // the handle's tensor-core kernels; the K'/V' operand copies live in a
    // stream-ordered allocation for the duration of the call
    cudaStream_t s = S(stream);
    void* buf = nullptr;
    LLSA_CUDA_TRY(cudaMallocAsync(&buf, tc_buffer_bytes(g, units), s));
    TcBuffers tb;
    tc_carve(g, units, static_cast<char*>(buf), &tb);
    llsa_status st = tc_forward(g, units, q, k, v, pyr_k, pyr_v, tables, out, rm, rd, tb, s);
    cudaFreeAsync(buf, s);
    return st;
  }
  return simt_forward(g, units, dt, q, k, v, pyr_k, pyr_v, tables, out, rm, rd, S(stream));
}

llsa_status llsa_forward_plan(const llsa_config* cfg, uint32_t units, llsa_dtype dt,
                              const void* q, const void* k, const void* v, const float* pyr_k,
                              const float* pyr_v, const uint32_t* pl, const uint32_t* pb,
                              const float* pw, uint32_t epb, float* out, float* rm, float* rd,
                              void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(out);
  NONNULL(rm);
  NONNULL(rd);
  if (epb && (!pl || !pb || !pw)) return fail(LLSA_ERR_ARGUMENT, "null plan");
  PlanView plan{pl, pb, pw, epb};
  return simt_forward(g, units, dt, q, k, v, pyr_k, pyr_v, nullptr, out, rm, rd, S(stream),
                      &plan);
}

llsa_status llsa_backward_plan(const llsa_config* cfg, uint32_t units, llsa_dtype dt,
                               const void* d_out, const float* out, const float* rm,
                               const float* rd, const void* q, const void* k, const void* v,
                               const float* pyr_k, const float* pyr_v, const uint32_t* pl,
                               const uint32_t* pb, const float* pw, uint32_t epb,
                               const uint32_t* offs, const uint32_t* flat, float* dq,
                               float* dk, float* dv, void* ws, size_t ws_bytes, void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(d_out);
  NONNULL(out);
  NONNULL(rm);
  NONNULL(rd);
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(offs);
  NONNULL(flat);
  NONNULL(dq);
  NONNULL(dk);
  NONNULL(dv);
  if (g.L >= 1 && (!pyr_k || !pyr_v)) return fail(LLSA_ERR_ARGUMENT, "null pyramid");
  if (epb && (!pl || !pb || !pw)) return fail(LLSA_ERR_ARGUMENT, "null plan");
  if (!ws || ws_bytes < simt_backward_ws_bytes(g, units))
    return fail(LLSA_ERR_ARGUMENT, "backward workspace too small");
  PlanView plan{pl, pb, pw, epb};
  return simt_backward(g, units, dt, d_out, out, rm, rd, q, k, v, pyr_k, pyr_v, nullptr, offs,
                       flat, dq, dk, dv, ws, S(stream), nullptr, &plan);
}

namespace {
// Workspace of the staged tensor-core backward: K'/V' operand copies, the
// kernels' own scratch, and (kv_backward only) rebuilt tables + a scratch dq.
struct TcStagedWs {
  size_t tcb, bwd, tab, cur, dq, total;
  TcStagedWs(const Geometry& g, uint32_t units) {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    tcb = al(tc_buffer_bytes(g, units));
    bwd = al(tc_backward_ws_bytes(g, units));
    tab = al((size_t)units * g.table_entries * 4);
    cur = al(tables_from_csc_ws(g, units));
    dq = al((size_t)units * g.n * g.d * 4);
    total = tcb + bwd + tab + cur + dq;
  }
};
size_t backward_ws(const Geometry& g, uint32_t units) {
  const size_t simt = simt_backward_ws_bytes(g, units);
  if (!tc_supported(g, LLSA_BF16)) return simt;
  const size_t tc = TcStagedWs(g, units).total;
  return tc > simt ? tc : simt;
}
}  // namespace

size_t llsa_backward_workspace_bytes(const llsa_config* cfg, uint32_t units) {
  Geometry g;
  if (make_geometry(cfg, &g)) return 0;
  return backward_ws(g, units);
}

llsa_status llsa_backward(const llsa_config* cfg, uint32_t units, llsa_dtype dt,
                          const void* d_out, const float* out, const float* rm,
                          const float* rd, const void* q, const void* k, const void* v,
                          const float* pyr_k, const float* pyr_v, const uint32_t* tables,
                          const uint32_t* offs, const uint32_t* flat, float* dq, float* dk,
                          float* dv, void* ws, size_t ws_bytes, void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(d_out);
  NONNULL(out);
  NONNULL(rm);
  NONNULL(rd);
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(pyr_k);
  NONNULL(pyr_v);
  NONNULL(tables);
  NONNULL(offs);
  NONNULL(flat);
  NONNULL(dq);
  NONNULL(dk);
  NONNULL(dv);
  if (!ws || ws_bytes < backward_ws(g, units))
    return fail(LLSA_ERR_ARGUMENT, "backward workspace too small");
  if (tc_supported(g, dt)) {
    const TcStagedWs w(g, units);
    char* p = static_cast<char*>(ws);
    TcBuffers tb;
    tc_carve(g, units, p, &tb);
    cudaStream_t s = S(stream);
    if (llsa_status st = tc_prep(g, units, pyr_k, pyr_v, tb, s)) return st;
    return tc_backward(g, units, d_out, out, rm, rd, q, k, v, pyr_k, pyr_v, tables, offs, flat,
                       dq, dk, dv, tb, p + w.tcb, s);
  }
  return simt_backward(g, units, dt, d_out, out, rm, rd, q, k, v, pyr_k, pyr_v, tables, offs,
                       flat, dq, dk, dv, ws, S(stream));
}

llsa_status llsa_kv_backward(const llsa_config* cfg, uint32_t units, llsa_dtype dt,
                             const void* d_out, const float* out, const float* rm,
                             const float* rd, const void* q, const float* pyr_k,
                             const float* pyr_v, const void* k, const void* v,
                             const uint32_t* offs, const uint32_t* flat, float* dk, float* dv,
                             void* ws, size_t ws_bytes, void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(d_out);
  NONNULL(out);
  NONNULL(rm);
  NONNULL(rd);
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(pyr_k);
  NONNULL(pyr_v);
  NONNULL(offs);
  NONNULL(flat);
  NONNULL(dk);
  NONNULL(dv);
  if (!ws || ws_bytes < backward_ws(g, units))
    return fail(LLSA_ERR_ARGUMENT, "backward workspace too small");
  if (tc_supported(g, dt)) {
    // the tensor-core backward also walks the query-major tables (and
    // produces dq, here into scratch): rebuild the tables from the CSC lists
    const TcStagedWs w(g, units);
    char* p = static_cast<char*>(ws);
    TcBuffers tb;
    tc_carve(g, units, p, &tb);
    cudaStream_t s = S(stream);
    uint32_t* tables = reinterpret_cast<uint32_t*>(p + w.tcb + w.bwd);
    if (llsa_status st = tables_from_csc(g, units, offs, flat, tables,
                                         p + w.tcb + w.bwd + w.tab, s))
      return st;
    if (llsa_status st = tc_prep(g, units, pyr_k, pyr_v, tb, s)) return st;
    float* dq = reinterpret_cast<float*>(p + w.tcb + w.bwd + w.tab + w.cur);
    return tc_backward(g, units, d_out, out, rm, rd, q, k, v, pyr_k, pyr_v, tables, offs, flat,
                       dq, dk, dv, tb, p + w.tcb, s);
  }
  return simt_backward(g, units, dt, d_out, out, rm, rd, q, k, v, pyr_k, pyr_v, nullptr, offs,
                       flat, nullptr, dk, dv, ws, S(stream));
}

namespace {
size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
size_t mask_kv_ws(const Geometry& g, uint32_t units) {
  return al256((size_t)units * g.csc_off_entries * 4) +
         al256((size_t)units * g.csc_flat_entries * 4) + al256(mask_lookup_ws_bytes(g, units)) +
         al256(backward_ws(g, units));
}
}  // namespace

size_t llsa_mask_kv_backward_workspace_bytes(const llsa_config* cfg, uint32_t units) {
  Geometry g;
  if (make_geometry(cfg, &g)) return 0;
  return mask_kv_ws(g, units);
}

llsa_status llsa_mask_kv_backward(const llsa_config* cfg, uint32_t units, llsa_dtype dt,
                                  const void* d_out, const float* out, const float* rm,
                                  const float* rd, const void* q, const float* pyr_k,
                                  const float* pyr_v, const void* k, const void* v,
                                  const uint32_t* tables, float* dk, float* dv, void* ws,
                                  size_t ws_bytes, void* stream) {
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0) return LLSA_OK;
  NONNULL(d_out);
  NONNULL(out);
  NONNULL(rm);
  NONNULL(rd);
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(pyr_k);
  NONNULL(pyr_v);
  NONNULL(tables);
  NONNULL(dk);
  NONNULL(dv);
  if (!ws || ws_bytes < mask_kv_ws(g, units))
    return fail(LLSA_ERR_ARGUMENT, "mask kv-backward workspace too small");
  char* p = static_cast<char*>(ws);
  uint32_t* offs = reinterpret_cast<uint32_t*>(p);
  p += al256((size_t)units * g.csc_off_entries * 4);
  uint32_t* flat = reinterpret_cast<uint32_t*>(p);
  p += al256((size_t)units * g.csc_flat_entries * 4);
  void* mws = p;
  p += al256(mask_lookup_ws_bytes(g, units));
  if (llsa_status st = mask_lookup(g, units, tables, offs, flat, mws, S(stream))) return st;
  if (tc_supported(g, dt)) {  // the same tensor-core kernels as llsa_kv_backward
    const TcStagedWs w(g, units);
    TcBuffers tb;
    tc_carve(g, units, p, &tb);
    cudaStream_t s = S(stream);
    if (llsa_status st = tc_prep(g, units, pyr_k, pyr_v, tb, s)) return st;
    float* dq = reinterpret_cast<float*>(p + w.tcb + w.bwd + w.tab + w.cur);
    return tc_backward(g, units, d_out, out, rm, rd, q, k, v, pyr_k, pyr_v, tables, offs, flat,
                       dq, dk, dv, tb, p + w.tcb, s);
  }
  return simt_backward(g, units, dt, d_out, out, rm, rd, q, k, v, pyr_k, pyr_v, nullptr, offs,
                       flat, nullptr, dk, dv, p, S(stream));
}

// ---------------------------------------------------------------------------
// Handle (fused) API
// ---------------------------------------------------------------------------
// Records named CUDA events between stages of one phase (forward or
// backward) of a handle call; read back by llsa_handle_stage_times.
// A ring of kRounds calls is kept so the stage times can be averaged over a
// whole timed region without any synchronisation inside it.
struct EventMarker final : StageMarker {
  static constexpr int kMax = 24, kRounds = 64;
  cudaEvent_t ev[kRounds][kMax] = {};
  int cnt[kRounds] = {};
  const char* name[kMax] = {};
  int round = -1, rounds = 0;
  bool ready = false;
  bool init() {
    for (int r = 0; r < kRounds; ++r)
      for (int i = 0; i < kMax; ++i)
        if (cudaEventCreate(&ev[r][i]) != cudaSuccess) return false;
    ready = true;
    return true;
  }
  ~EventMarker() override {
    if (ready)
      for (int r = 0; r < kRounds; ++r)
        for (int i = 0; i < kMax; ++i) cudaEventDestroy(ev[r][i]);
  }
  void start(cudaStream_t s) {
    round = (round + 1) % kRounds;
    if (rounds < kRounds) ++rounds;
    cnt[round] = 0;
    mark("start", s);
  }
  void mark(const char* n, cudaStream_t s) override {
    int& c = cnt[round];
    if (c < kMax) {
      name[c] = n;
      cudaEventRecord(ev[round][c++], s);
    }
  }
};

struct llsa_handle_s {
  Geometry g;
  EventMarker* timers[2] = {nullptr, nullptr};  // forward, backward
  uint32_t units = 0;
  llsa_dtype dt = LLSA_BF16;
  bool tc = false;
  int device = 0;
  char* arena = nullptr;
  size_t arena_bytes = 0;
  float *pyr_q = nullptr, *pyr_k = nullptr, *pyr_v = nullptr;
  uint32_t *tables = nullptr, *csc_off = nullptr, *csc_flat = nullptr;
  float *row_max = nullptr, *row_denom = nullptr;
  void* tr_ws = nullptr;
  size_t tr_ws_bytes = 0;
  void* bwd_ws = nullptr;
  size_t bwd_ws_bytes = 0;
  // bf16-output mode (llsa_handle_*_ex): fp32 results land here first; the
  // backward reads O from out32 (D = rowsum(dO∘O) needs the fp32 output).
  float* out32 = nullptr;      // [units][n][d]
  float* grad32 = nullptr;     // dq | dk | dv, [3][units][n][d]
  const void* last_out16 = nullptr;
  TcBuffers tcb;
  uint32_t last_launches = 0;
  size_t sizes[8] = {};
};

// The handle's kernels run on the device it was created on, whatever device
// is current in the calling thread; the caller's current device is restored.
struct DeviceGuard {
  int prev = -1, want;
  explicit DeviceGuard(int dev) : want(dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != want) cudaSetDevice(want);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

llsa_status llsa_handle_create(const llsa_config* cfg, uint32_t units, llsa_dtype dt,
                               llsa_handle* out) {
  NONNULL(out);
  *out = nullptr;
  Geometry g;
  if (llsa_status st = make_geometry(cfg, &g)) return st;
  if (llsa_status st = dtype_ok(dt)) return st;
  if (units == 0) return fail(LLSA_ERR_ARGUMENT, "units must be positive");
  auto* h = new (std::nothrow) llsa_handle_s();
  if (!h) return fail(LLSA_ERR_CUDA, "out of host memory");
  h->g = g;
  h->units = units;
  h->dt = dt;
  h->tc = tc_supported(g, dt);
  cudaGetDevice(&h->device);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t pyr = al((size_t)units * g.pyr_rows * g.d * 4);
  const size_t tab = al((size_t)units * g.table_entries * 4);
  const size_t coff = al((size_t)units * g.csc_off_entries * 4);
  const size_t cflat = al((size_t)units * g.csc_flat_entries * 4);
  const size_t rows = al((size_t)units * g.n * 4);
  h->tr_ws_bytes = al(transpose_all_fused_ok(g) ? transpose_all_fused_ws(g, units)
                                                : transpose_all_ws(g, units));
  h->bwd_ws_bytes = al(h->tc ? tc_backward_ws_bytes(g, units) : simt_backward_ws_bytes(g, units));
  const size_t tcb = h->tc ? al(tc_buffer_bytes(g, units)) : 0;
  h->arena_bytes = 3 * pyr + tab + coff + cflat + 2 * rows + h->tr_ws_bytes + h->bwd_ws_bytes +
                   tcb + 256;
  if (cudaMalloc(&h->arena, h->arena_bytes) != cudaSuccess) {
    delete h;
    return fail(LLSA_ERR_CUDA, "cudaMalloc of %zu bytes failed", (size_t)0);
  }
  char* p = h->arena;
  auto take = [&](size_t b) {
    char* r = p;
    p += b;
    return r;
  };
  h->pyr_q = reinterpret_cast<float*>(take(pyr));
  h->pyr_k = reinterpret_cast<float*>(take(pyr));
  h->pyr_v = reinterpret_cast<float*>(take(pyr));
  h->tables = reinterpret_cast<uint32_t*>(take(tab));
  h->csc_off = reinterpret_cast<uint32_t*>(take(coff));
  h->csc_flat = reinterpret_cast<uint32_t*>(take(cflat));
  h->row_max = reinterpret_cast<float*>(take(rows));
  h->row_denom = reinterpret_cast<float*>(take(rows));
  h->tr_ws = take(h->tr_ws_bytes);
  h->bwd_ws = take(h->bwd_ws_bytes);
  if (h->tc) tc_carve(g, units, take(tcb), &h->tcb);
  const size_t sz[8] = {pyr, pyr, pyr, tab, coff, cflat, rows, rows};
  memcpy(h->sizes, sz, sizeof(sz));
  *out = h;
  return LLSA_OK;
}

llsa_status llsa_handle_destroy(llsa_handle h) {
  if (!h) return LLSA_OK;
  delete h->timers[0];
  delete h->timers[1];
  if (h->arena) cudaFree(h->arena);
  if (h->out32) cudaFree(h->out32);
  if (h->grad32) cudaFree(h->grad32);
  delete h;
  return LLSA_OK;
}

int llsa_handle_uses_tensor_cores(llsa_handle h) { return h && h->tc ? 1 : 0; }

}  // extern "C"

static llsa_status handle_forward_f32(llsa_handle h, const void* q, const void* k,
                                      const void* v, float* out, void* stream,
                                      void* out16 = nullptr);
static llsa_status handle_backward_f32(llsa_handle h, const void* d_out, const void* q,
                                       const void* k, const void* v, const float* out,
                                       float* dq, float* dk, float* dv, void* stream,
                                       bool grad_bf16 = false);

namespace llsa_impl {
namespace cvt {
// fp32 → bf16 (RNE) of up to three equally sized tensors in one launch
struct CvtArgs {
  const float* src[3];
  __nv_bfloat16* dst[3];
  uint32_t count;
  uint64_t n4;  // elements / 4 per tensor
};
__global__ void __launch_bounds__(256) to_bf16_kernel(CvtArgs a) {
  const uint64_t total = a.n4 * a.count;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(i / a.n4);
    const uint64_t j = i - t * a.n4;
    const float4 x = __ldcs(reinterpret_cast<const float4*>(a.src[t]) + j);
    __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&lo);
    o.y = *reinterpret_cast<uint32_t*>(&hi);
    __stcs(reinterpret_cast<uint2*>(a.dst[t]) + j, o);
  }
}
}  // namespace cvt
}  // namespace llsa_impl

static llsa_status to_bf16(const float* const* src, void* const* dst, uint32_t count,
                           size_t elems, cudaStream_t s) {
  llsa_impl::cvt::CvtArgs a{};
  for (uint32_t t = 0; t < count; ++t) {
    a.src[t] = src[t];
    a.dst[t] = static_cast<__nv_bfloat16*>(dst[t]);
  }
  a.count = count;
  a.n4 = elems / 4;  // n·d is a multiple of 4 on every tensor-core shape (d = 64)
  if (elems % 4) return fail(LLSA_ERR_UNSUPPORTED, "bf16 outputs need n*d %% 4 == 0");
  llsa_impl::cvt::to_bf16_kernel<<<148 * 8, 256, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("to_bf16_kernel");
  return LLSA_OK;
}

extern "C" {

llsa_status llsa_handle_forward(llsa_handle h, const void* q, const void* k, const void* v,
                                float* out, void* stream) {
  return llsa_handle_forward_ex(h, q, k, v, out, LLSA_F32, stream);
}

llsa_status llsa_handle_backward(llsa_handle h, const void* d_out, const void* q,
                                 const void* k, const void* v, const float* out, float* dq,
                                 float* dk, float* dv, void* stream) {
  return llsa_handle_backward_ex(h, d_out, q, k, v, out, dq, dk, dv, LLSA_F32, stream);
}

static llsa_status ensure(float** p, size_t bytes) {
  if (*p) return LLSA_OK;
  if (cudaMalloc(reinterpret_cast<void**>(p), bytes) != cudaSuccess) {
    *p = nullptr;
    return fail(LLSA_ERR_CUDA, "cudaMalloc of %zu bytes failed", bytes);
  }
  return LLSA_OK;
}

llsa_status llsa_handle_forward_ex(llsa_handle h, const void* q, const void* k, const void* v,
                                   void* out_user, llsa_dtype out_dtype, void* stream) {
  NONNULL(h);
  NONNULL(out_user);
  if (llsa_status st = dtype_ok(out_dtype)) return st;
  const size_t elems = (size_t)h->units * h->g.n * h->g.d;
  float* out = static_cast<float*>(out_user);
  if (out_dtype == LLSA_BF16) {
    DeviceGuard dg(h->device);
    if (llsa_status st = ensure(&h->out32, elems * 4)) return st;
    out = h->out32;
  }
  // the tcgen05 forward writes the bf16 copy in its epilogue; other paths
  // convert the fp32 output afterwards
  const bool fused16 = out_dtype == LLSA_BF16 && h->tc && tc_forward_writes_bf16(h->g);
  llsa_status st = handle_forward_f32(h, q, k, v, out, stream, fused16 ? out_user : nullptr);
  if (!st && out_dtype == LLSA_BF16) {
    if (!fused16) {
      DeviceGuard dg(h->device);
      const float* src[3] = {h->out32, nullptr, nullptr};
      void* dst[3] = {out_user, nullptr, nullptr};
      st = to_bf16(src, dst, 1, elems, S(stream));
      h->last_launches += 1;
    }
    h->last_out16 = out_user;
  }
  return st;
}

llsa_status llsa_handle_backward_ex(llsa_handle h, const void* d_out, const void* q,
                                    const void* k, const void* v, const void* out_user,
                                    void* dq, void* dk, void* dv, llsa_dtype out_dtype,
                                    void* stream) {
  NONNULL(h);
  NONNULL(out_user);
  NONNULL(dq);
  NONNULL(dk);
  NONNULL(dv);
  if (llsa_status st = dtype_ok(out_dtype)) return st;
  if (out_dtype == LLSA_F32)
    return handle_backward_f32(h, d_out, q, k, v, static_cast<const float*>(out_user),
                               static_cast<float*>(dq), static_cast<float*>(dk),
                               static_cast<float*>(dv), stream);
  if (!h->out32 || out_user != h->last_out16)
    return fail(LLSA_ERR_STALE_STATE,
                "bf16-output backward needs the bf16 output of this handle's latest forward");
  if (h->tc && tc_bf16_grads_ok(h->g))  // the kernels write bf16 gradients directly
    return handle_backward_f32(h, d_out, q, k, v, h->out32, static_cast<float*>(dq),
                               static_cast<float*>(dk), static_cast<float*>(dv), stream, true);
  const size_t elems = (size_t)h->units * h->g.n * h->g.d;
  {
    DeviceGuard dg(h->device);
    if (llsa_status st = ensure(&h->grad32, 3 * elems * 4)) return st;
  }
  float* g = h->grad32;
  llsa_status st = handle_backward_f32(h, d_out, q, k, v, h->out32, g, g + elems, g + 2 * elems,
                                       stream);
  if (!st) {
    DeviceGuard dg(h->device);
    const float* src[3] = {g, g + elems, g + 2 * elems};
    void* dst[3] = {dq, dk, dv};
    st = to_bf16(src, dst, 3, elems, S(stream));
    h->last_launches += 1;
  }
  return st;
}

}  // extern "C"

static llsa_status handle_forward_f32(llsa_handle h, const void* q, const void* k,
                                      const void* v, float* out, void* stream, void* out16) {
  NONNULL(h);
  DeviceGuard dg(h->device);
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(out);
  const Geometry& g = h->g;
  cudaStream_t s = S(stream);
  take_launch_count();
  EventMarker* mk = h->timers[0];
  if (mk) mk->start(s);
  llsa_status st = LLSA_OK;
  const bool fused = fused_pyramid_ok(g);
  if (fused) {  // one pass over q, k, v; emits the tensor-core hi/lo copies too
    st = fused_pyramids(g, h->units, q, k, v, h->dt, h->pyr_q, h->pyr_k, h->pyr_v,
                        h->tc ? h->tcb.k_hi : nullptr, h->tc ? h->tcb.k_lo : nullptr,
                        h->tc ? h->tcb.v_hi : nullptr, h->tc ? h->tcb.v_lo : nullptr, s);
  } else {
    st = pyramid(g, h->units, q, h->dt, h->pyr_q, s);
    if (!st) st = pyramid(g, h->units, k, h->dt, h->pyr_k, s);
    if (!st) st = pyramid(g, h->units, v, h->dt, h->pyr_v, s);
  }
  LLSA_MARK(mk, "compress", s);
  if (!st) st = hier_topk(g, h->units, h->pyr_q, h->pyr_k, h->tables, s);
  LLSA_MARK(mk, "select", s);
  if (!st) {
    if (h->tc) {
      st = tc_forward(g, h->units, q, k, v, h->pyr_k, h->pyr_v, h->tables, out, h->row_max,
                      h->row_denom, h->tcb, s, mk, fused, out16);
    } else {
      st = simt_forward(g, h->units, h->dt, q, k, v, h->pyr_k, h->pyr_v, h->tables, out,
                        h->row_max, h->row_denom, s);
      LLSA_MARK(mk, "fwd_attention", s);
    }
  }
  h->last_launches = take_launch_count();
  return st;
}

static llsa_status handle_backward_f32(llsa_handle h, const void* d_out, const void* q,
                                       const void* k, const void* v, const float* out,
                                       float* dq, float* dk, float* dv, void* stream,
                                       bool grad_bf16) {
  NONNULL(h);
  DeviceGuard dg(h->device);
  NONNULL(d_out);
  NONNULL(q);
  NONNULL(k);
  NONNULL(v);
  NONNULL(out);
  NONNULL(dq);
  NONNULL(dk);
  NONNULL(dv);
  const Geometry& g = h->g;
  cudaStream_t s = S(stream);
  take_launch_count();
  EventMarker* mk = h->timers[1];
  if (mk) mk->start(s);
  llsa_status st = transpose_all_fused_ok(g)
                        ? transpose_all_fused(g, h->units, h->tables, h->csc_off, h->csc_flat,
                                              h->tr_ws, s)
                        : transpose_all_impl(g, h->units, h->tables, h->csc_off, h->csc_flat,
                                             h->tr_ws, s);
  LLSA_MARK(mk, "transpose", s);
  if (!st) {
    if (h->tc)
      st = tc_backward(g, h->units, d_out, out, h->row_max, h->row_denom, q, k, v, h->pyr_k,
                       h->pyr_v, h->tables, h->csc_off, h->csc_flat, dq, dk, dv, h->tcb,
                       h->bwd_ws, s, mk, grad_bf16);
    else
      st = simt_backward(g, h->units, h->dt, d_out, out, h->row_max, h->row_denom, q, k, v,
                         h->pyr_k, h->pyr_v, h->tables, h->csc_off, h->csc_flat, dq, dk, dv,
                         h->bwd_ws, s, mk);
  }
  h->last_launches = take_launch_count();
  return st;
}

extern "C" {

llsa_status llsa_handle_buffer(llsa_handle h, llsa_buffer which, void** ptr, size_t* bytes) {
  NONNULL(h);
  NONNULL(ptr);
  void* p[8] = {h->pyr_q, h->pyr_k, h->pyr_v, h->tables, h->csc_off, h->csc_flat, h->row_max,
                h->row_denom};
  if ((int)which < 0 || (int)which > 7) return fail(LLSA_ERR_ARGUMENT, "bad buffer id");
  *ptr = p[which];
  if (bytes) *bytes = h->sizes[which];
  return LLSA_OK;
}

uint32_t llsa_handle_last_launches(llsa_handle h) { return h ? h->last_launches : 0; }

llsa_status llsa_handle_enable_timing(llsa_handle h, int enable) {
  NONNULL(h);
  for (int i = 0; i < 2; ++i) {
    delete h->timers[i];
    h->timers[i] = nullptr;
    if (enable) {
      h->timers[i] = new EventMarker();
      if (!h->timers[i]->init()) return fail(LLSA_ERR_CUDA, "cudaEventCreate failed");
    }
  }
  return LLSA_OK;
}

uint32_t llsa_handle_stage_times(llsa_handle h, const char** names, float* ms, uint32_t cap) {
  if (!h) return 0;
  uint32_t k = 0;
  for (int i = 0; i < 2; ++i) {
    EventMarker* m = h->timers[i];
    if (!m || m->rounds == 0) continue;
    const int n = m->cnt[m->round];
    for (int j = 1; j < n; ++j) {
      if (k >= cap) return k;
      double sum = 0.0;
      int used = 0;
      for (int r = 0; r < m->rounds; ++r) {
        if (m->cnt[r] != n) continue;
        float t = 0.f;
        if (cudaEventSynchronize(m->ev[r][j]) != cudaSuccess ||
            cudaEventElapsedTime(&t, m->ev[r][j - 1], m->ev[r][j]) != cudaSuccess)
          continue;
        sum += t;
        ++used;
      }
      if (names) names[k] = m->name[j];
      if (ms) ms[k] = used ? (float)(sum / used) : -1.f;
      ++k;
    }
  }
  return k;
}

}  // extern "C"
