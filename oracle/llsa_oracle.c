/*
 * TEST INFRASTRUCTURE ONLY — see llsa_oracle.h.  Plain-C restatement of the
 * reference LLSA hot path in float (the reference's f32 build), citing the
 * reference file:line for every step (P/ = /root/reference/proj/).
 *
 * Compile with -ffp-contract=off: every multiply and add must round on its
 * own, exactly as the reference's x86-64 build does (no vfmadd emitted).
 */
#include "llsa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum {
  ST_OK = 0, ST_CONFIG = 1, ST_DIVISIBILITY = 2, ST_LEVEL = 3, ST_TOPK = 4,
  ST_SHAPE = 5, ST_INDEX = 6, ST_NONFINITE = 7, ST_STALE = 8, ST_ALLOC = 98
};

/* ---- config (P/src/config.cpp:54-125) ----------------------------------- */

/* P/src/config.cpp:54-64: largest L with B^(L+1) <= n. */
uint32_t oracle_max_levels(uint64_t n, uint32_t b) {
  if (b < 2 || n == 0) return 0;
  uint32_t l = 0;
  uint64_t p = b;
  while (p <= n / b) {
    p *= b;
    ++l;
  }
  return l;
}

static uint64_t ipow(uint64_t b, uint32_t e) {
  uint64_t p = 1;
  for (uint32_t i = 0; i < e; ++i) p *= b;
  return p;
}

/* P/src/config.cpp:66-117 (same check order, same error kinds);
 * effective_block_count P/src/config.cpp:119-125. */
int oracle_validate(const oracle_config* c, float* scale, uint32_t* eff) {
  if (c->n == 0) return ST_CONFIG;
  if (c->d == 0) return ST_CONFIG;
  if (c->block_size < 2) return ST_CONFIG;
  if (c->n > 0xffffffffull) return ST_CONFIG;
  if (!isfinite(c->softmax_scale) || c->softmax_scale < 0.0f) return ST_CONFIG;
  const uint32_t lmax = oracle_max_levels(c->n, c->block_size);
  if (c->levels < 1 || c->levels > lmax) return ST_LEVEL;
  const uint64_t pow_l = ipow(c->block_size, c->levels);
  if (c->n % pow_l != 0) return ST_DIVISIBILITY;
  if (c->enrich_levels > c->levels) return ST_LEVEL;
  const uint64_t coarsest = c->n / pow_l;
  if (c->top_k < 1 || c->top_k > coarsest) return ST_TOPK;
  if (scale) {
    *scale = c->softmax_scale > 0.0f ? c->softmax_scale
                                     : 1.0f / sqrtf((float)c->d);
  }
  if (eff) {
    const uint32_t le = c->enrich_levels, L = c->levels;
    uint32_t count = c->top_k * (le + 1 < L ? le + 1 : L);
    if (le == L) count += (uint32_t)(c->n / pow_l / c->block_size);
    *eff = count;
  }
  return ST_OK;
}

/* ---- deterministic random stream (P/src/tensorio.cpp:64-100,163-186) --- */

static uint64_t splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t xoshiro_next(uint64_t s[4]) {
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

void oracle_gen_random(float* out, size_t rows, size_t cols, uint64_t seed,
                       int uniform) {
  uint64_t sm = seed, s[4];
  for (int i = 0; i < 4; ++i) s[i] = splitmix_next(&sm);
  const size_t count = rows * cols;
  if (uniform) {
    for (size_t i = 0; i < count; ++i)
      out[i] = (float)((double)(xoshiro_next(s) >> 11) * 0x1.0p-53);
    return;
  }
  const double pi = 3.141592653589793; /* std::numbers::pi */
  for (size_t i = 0; i < count; i += 2) {
    const double u1 = (double)((xoshiro_next(s) >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(xoshiro_next(s) >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * pi * u2;
    out[i] = (float)(radius * cos(angle));
    if (i + 1 < count) out[i + 1] = (float)(radius * sin(angle));
  }
}

/* ---- inner product (P/include/llsa/detail/math.hpp:13-24) ---------------- */

static float dot4(const float* a, const float* b, size_t n) {
  float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  size_t i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 += a[i] * b[i];
    s1 += a[i + 1] * b[i + 1];
    s2 += a[i + 2] * b[i + 2];
    s3 += a[i + 3] * b[i + 3];
  }
  for (; i < n; ++i) s0 += a[i] * b[i];
  return (s0 + s1) + (s2 + s3);
}

/* P/include/llsa/detail/math.hpp:27-29 */
static void axpy(float* out, const float* v, float scale, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] += scale * v[i];
}

/* ---- pyramid (P/src/pyramid.cpp:11-64) ----------------------------------- */

/* Level l row t = (sum_{b<B} level_{l-1}[tB+b]) * (1/B): sequential sum from
 * 0 in index order, then one multiply (P/src/pyramid.cpp:28-39). */
int oracle_build_pyramid(const float* x, size_t rows, size_t d, uint32_t B,
                         uint32_t levels, float* levels_out) {
  if (B < 2) return ST_DIVISIBILITY;
  const float* prev = x;
  size_t prev_rows = rows;
  float* out = levels_out;
  const float inv_b = 1.0f / (float)B;
  for (uint32_t l = 1; l <= levels; ++l) {
    if (prev_rows % B != 0) return ST_DIVISIBILITY;
    const size_t cr = prev_rows / B;
    for (size_t t = 0; t < cr; ++t) {
      float* o = out + t * d;
      for (size_t j = 0; j < d; ++j) o[j] = 0.0f;
      for (uint32_t b = 0; b < B; ++b) {
        const float* in = prev + (t * B + b) * d;
        for (size_t j = 0; j < d; ++j) o[j] += in[j];
      }
      for (size_t j = 0; j < d; ++j) o[j] *= inv_b;
    }
    prev = out;
    prev_rows = cr;
    out += cr * d;
  }
  return ST_OK;
}

/* P/src/pyramid.cpp:45-64: fine[t] = coarse[t/B^h] * (1/B^h). */
int oracle_pool_backward(const float* g, size_t rows, size_t d, uint32_t B,
                         uint32_t hops, float* out) {
  if (hops == 0) {
    memcpy(out, g, rows * d * sizeof(float));
    return ST_OK;
  }
  if (B < 2) return ST_DIVISIBILITY;
  const size_t group = (size_t)ipow(B, hops);
  const float inv = 1.0f / (float)group;
  for (size_t t = 0; t < rows * group; ++t)
    for (size_t j = 0; j < d; ++j) out[t * d + j] = g[(t / group) * d + j] * inv;
  return ST_OK;
}

/* ---- selection (P/src/selection.cpp:21-189) ------------------------------ */

/* topk_row, P/src/selection.cpp:21-38: keep the top_k positions by
 * (score desc, position asc) — a float comparison, so -0.0 ties +0.0 — map
 * them through ids, emit ascending.  Restated as K rounds of "best remaining"
 * (the ranked set is unique because the order is total). */
static void topk_row(const float* scores, uint32_t count, uint32_t top_k,
                     const uint32_t* ids, unsigned char* taken, uint32_t* out) {
  memset(taken, 0, count);
  for (uint32_t j = 0; j < top_k; ++j) {
    uint32_t best = UINT32_MAX;
    for (uint32_t c = 0; c < count; ++c) {
      if (taken[c]) continue;
      if (best == UINT32_MAX || scores[c] > scores[best]) best = c;
      /* equal scores: the earlier position (already in best) wins */
    }
    taken[best] = 1;
    out[j] = ids ? ids[best] : best;
  }
  for (uint32_t a = 1; a < top_k; ++a) { /* insertion sort ascending */
    const uint32_t v = out[a];
    uint32_t b = a;
    while (b > 0 && out[b - 1] > v) {
      out[b] = out[b - 1];
      --b;
    }
    out[b] = v;
  }
}

/* P/src/selection.cpp:42-79: score[c] = scale * dot(q[r], k[c]) (:68-70). */
int oracle_select_coarsest(const float* q, size_t q_rows, const float* k,
                           size_t k_rows, size_t d, uint32_t top_k, float scale,
                           uint32_t* out) {
  const uint32_t cand = (uint32_t)k_rows;
  if (top_k < 1 || top_k > cand) return ST_TOPK;
  float* scores = (float*)malloc(sizeof(float) * (cand ? cand : 1));
  unsigned char* taken = (unsigned char*)malloc(cand ? cand : 1);
  if (!scores || !taken) return ST_ALLOC;
  for (size_t r = 0; r < q_rows; ++r) {
    for (uint32_t c = 0; c < cand; ++c)
      scores[c] = scale * dot4(q + r * d, k + (size_t)c * d, d);
    topk_row(scores, cand, top_k, NULL, taken, out + r * top_k);
  }
  free(scores);
  free(taken);
  return ST_OK;
}

/* P/src/selection.cpp:81-149: level-l query block i gathers the K·B
 * candidate tokens parent[i][j]*B + b (:124-134), each of its B rows scores
 * them and keeps top_k (:135-142).  Errors in the reference's order. */
int oracle_select_level(const float* q, size_t q_rows, const float* k,
                        size_t k_rows, size_t d, const uint32_t* parent,
                        uint32_t parent_level, uint32_t parent_rows,
                        uint32_t parent_k, uint32_t top_k, float scale,
                        uint32_t B, uint32_t* out) {
  if (parent_level == 0) return ST_LEVEL;
  if (q_rows != (size_t)parent_rows * B) return ST_SHAPE;
  if (k_rows % B != 0) return ST_SHAPE;
  const uint32_t cand = parent_k * B;
  if (top_k < 1 || top_k > cand) return ST_TOPK;
  const uint32_t key_blocks = (uint32_t)(k_rows / B);
  uint32_t* ids = (uint32_t*)malloc(sizeof(uint32_t) * cand);
  float* scores = (float*)malloc(sizeof(float) * cand);
  unsigned char* taken = (unsigned char*)malloc(cand);
  if (!ids || !scores || !taken) return ST_ALLOC;
  int st = ST_OK;
  for (uint32_t i = 0; i < parent_rows && st == ST_OK; ++i) {
    const uint32_t* prow = parent + (size_t)i * parent_k;
    for (uint32_t j = 0; j < parent_k; ++j) {
      if (prow[j] >= key_blocks) {
        st = ST_INDEX;
        break;
      }
      for (uint32_t b = 0; b < B; ++b) ids[j * B + b] = prow[j] * B + b;
    }
    if (st != ST_OK) break;
    for (uint32_t r = 0; r < B; ++r) {
      const float* qr = q + ((size_t)i * B + r) * d;
      for (uint32_t c = 0; c < cand; ++c)
        scores[c] = scale * dot4(qr, k + (size_t)ids[c] * d, d);
      topk_row(scores, cand, top_k, ids, taken, out + ((size_t)i * B + r) * top_k);
    }
  }
  free(ids);
  free(scores);
  free(taken);
  return st;
}

static size_t level_offset_rows(uint64_t n, uint32_t B, uint32_t l) {
  /* rows before level l in the levels-1..L concatenation */
  size_t off = 0;
  uint64_t t = n;
  for (uint32_t j = 1; j < l; ++j) {
    t /= B;
    off += (size_t)t;
  }
  return off;
}

static const float* level_ptr(const float* base_level0, const float* levels,
                              uint64_t n, uint32_t d, uint32_t B, uint32_t l) {
  if (l == 0) return base_level0;
  return levels + level_offset_rows(n, B, l) * d;
}

static size_t table_offset(uint64_t n, uint32_t B, uint32_t K, uint32_t l) {
  size_t off = 0;
  uint64_t t = n / B;
  for (uint32_t j = 0; j < l; ++j) {
    off += (size_t)t * K;
    t /= B;
  }
  return off;
}

/* P/src/selection.cpp:151-179: coarsest table first, then refine L-1..1. */
int oracle_hierarchical_topk(const oracle_config* c, const float* pyr_q,
                             const float* pyr_k, uint32_t* tables,
                             uint64_t* mul_accs) {
  float scale;
  int st = oracle_validate(c, &scale, NULL);
  if (st) return st;
  const uint64_t n = c->n;
  const uint32_t B = c->block_size, K = c->top_k, L = c->levels, d = c->d;
  const uint64_t top_rows = n / ipow(B, L);
  const float* qL = level_ptr(NULL, pyr_q, n, d, B, L);
  const float* kL = level_ptr(NULL, pyr_k, n, d, B, L);
  st = oracle_select_coarsest(qL, top_rows, kL, top_rows, d, K, scale,
                              tables + table_offset(n, B, K, L - 1));
  if (st) return st;
  uint64_t macs = top_rows * top_rows * d;
  for (uint32_t l = L - 1; l >= 1; --l) {
    const uint64_t rows_l = n / ipow(B, l);
    st = oracle_select_level(level_ptr(NULL, pyr_q, n, d, B, l), rows_l,
                             level_ptr(NULL, pyr_k, n, d, B, l), rows_l, d,
                             tables + table_offset(n, B, K, l), l,
                             (uint32_t)(rows_l / B), K, K, scale, B,
                             tables + table_offset(n, B, K, l - 1));
    if (st) return st;
    macs += rows_l * (uint64_t)K * B * d;
  }
  if (mul_accs) *mul_accs += macs;
  return ST_OK;
}

/* ---- CSR → CSC (P/src/indexmap.cpp:14-72) -------------------------------- */

/* Count (:18-38), exclusive prefix (:40-47), scatter (:49-62) and the
 * canonical ascending order per segment (:64-70).  Scattering rows in
 * ascending order is a stable counting sort, which yields that canonical
 * order directly. */
int oracle_transpose(const uint32_t* idx, uint32_t rows, uint32_t k,
                     uint32_t key_blocks, uint32_t* offsets, uint32_t* flat) {
  const size_t total = (size_t)rows * k;
  uint32_t* cursor = (uint32_t*)calloc((size_t)key_blocks + 1, sizeof(uint32_t));
  if (!cursor) return ST_ALLOC;
  for (size_t e = 0; e < total; ++e) {
    if (idx[e] >= key_blocks) {
      free(cursor);
      return ST_INDEX;
    }
    cursor[idx[e]]++;
  }
  offsets[0] = 0;
  for (uint32_t b = 0; b < key_blocks; ++b) offsets[b + 1] = offsets[b] + cursor[b];
  for (uint32_t b = 0; b < key_blocks; ++b) cursor[b] = offsets[b];
  for (uint32_t i = 0; i < rows; ++i)
    for (uint32_t j = 0; j < k; ++j) flat[cursor[idx[(size_t)i * k + j]]++] = i;
  free(cursor);
  return ST_OK;
}

/* ---- enriched plan (P/src/attention.cpp:80-122) -------------------------- */

int oracle_build_plan(const oracle_config* c, const uint32_t* tables,
                      uint32_t* plan_level, uint32_t* plan_block,
                      float* plan_weight) {
  uint32_t eff;
  int st = oracle_validate(c, NULL, &eff);
  if (st) return st;
  const uint64_t n = c->n;
  const uint32_t B = c->block_size, K = c->top_k, L = c->levels,
                 Le = c->enrich_levels;
  const uint32_t fine = (uint32_t)(n / B);
  const uint32_t lim = Le + 1 < L ? Le + 1 : L;
  for (uint32_t i = 0; i < fine; ++i) {
    size_t e = (size_t)i * eff;
    for (uint32_t l = 0; l < lim; ++l) {
      const uint32_t row = (uint32_t)(i / ipow(B, l));
      const uint32_t* tr = tables + table_offset(n, B, K, l) + (size_t)row * K;
      for (uint32_t j = 0; j < K; ++j, ++e) {
        plan_level[e] = l;
        plan_block[e] = tr[j];
        plan_weight[e] = (float)ipow(B, l);
      }
    }
    if (Le == L) {
      const uint32_t top_blocks = (uint32_t)(n / ipow(B, L + 1));
      for (uint32_t b = 0; b < top_blocks; ++b, ++e) {
        plan_level[e] = L;
        plan_block[e] = b;
        plan_weight[e] = (float)ipow(B, L);
      }
    }
  }
  return ST_OK;
}

/* ---- forward (P/src/attention.cpp:145-219) ------------------------------- */

int oracle_forward(const oracle_config* c, const float* q, const float* k,
                   const float* v, const float* pyr_k, const float* pyr_v,
                   const uint32_t* tables, float* out, float* row_max,
                   float* row_denom) {
  float scale;
  uint32_t E;
  int st = oracle_validate(c, &scale, &E);
  if (st) return st;
  const uint64_t n = c->n;
  const uint32_t d = c->d, B = c->block_size;
  const int safe = c->safe_softmax != 0;
  const int scale_kv = c->reweight_mode == 0;
  const uint32_t fine = (uint32_t)(n / B);
  uint32_t* pl = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)fine * E);
  uint32_t* pb = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)fine * E);
  float* pw = (float*)malloc(sizeof(float) * (size_t)fine * E);
  float* acc = (float*)malloc(sizeof(float) * d);
  float* kg = (float*)malloc(sizeof(float) * E);
  float* lb = (float*)malloc(sizeof(float) * E);
  if (!pl || !pb || !pw || !acc || !kg || !lb) return ST_ALLOC;
  oracle_build_plan(c, tables, pl, pb, pw);
  int bad = 0;
  for (uint32_t i = 0; i < fine; ++i) {
    const size_t e0 = (size_t)i * E;
    /* gains per entry, :176-180 */
    for (uint32_t e = 0; e < E; ++e) {
      kg[e] = scale_kv ? pw[e0 + e] : 1.0f;
      lb[e] = scale_kv ? 0.0f : logf(pw[e0 + e]);
    }
    for (uint32_t r = 0; r < B; ++r) {
      const size_t t = (size_t)i * B + r;
      const float* qt = q + t * d;
      float m = safe ? -INFINITY : 0.0f;
      float denom = 0.0f;
      for (uint32_t j = 0; j < d; ++j) acc[j] = 0.0f;
      for (uint32_t e = 0; e < E; ++e) {
        const uint32_t lvl = pl[e0 + e];
        const float* keys = level_ptr(k, pyr_k, n, d, B, lvl);
        const float* vals = level_ptr(v, pyr_v, n, d, B, lvl);
        const size_t base = (size_t)pb[e0 + e] * B;
        for (uint32_t b = 0; b < B; ++b) {
          /* :188-190 */
          const float s = scale * kg[e] * dot4(qt, keys + (base + b) * d, d) + lb[e];
          if (safe && s > m) { /* :191-196 */
            const float rescale = expf(m - s);
            denom *= rescale;
            for (uint32_t j = 0; j < d; ++j) acc[j] *= rescale;
            m = s;
          }
          const float p = expf(s - m); /* :197-200 */
          denom += p;
          axpy(acc, vals + (base + b) * d, p * kg[e], d);
        }
      }
      float* o = out + t * d; /* :203-211 */
      const float inv = 1.0f / denom;
      for (uint32_t j = 0; j < d; ++j) {
        o[j] = acc[j] * inv;
        if (!isfinite(o[j])) bad = 1;
      }
      row_max[t] = safe ? m : 0.0f;
      row_denom[t] = denom;
      if (!isfinite(denom) || denom <= 0.0f) bad = 1;
    }
  }
  free(pl);
  free(pb);
  free(pw);
  free(acc);
  free(kg);
  free(lb);
  return bad ? ST_NONFINITE : ST_OK;
}

/* ---- backward (P/src/attention_grad.cpp:16-265) -------------------------- */

/* accumulate_key_block, P/src/attention_grad.cpp:43-73 */
static void accumulate_key_block(const float* d_out, const float* row_max,
                                 const float* row_denom, const float* q,
                                 const float* keys, const float* values,
                                 const float* d_row, const uint32_t* seg,
                                 uint32_t seg_len, uint32_t key_block,
                                 size_t span, float key_gain, float value_gain,
                                 float bias, float scale, uint32_t B, uint32_t d,
                                 float* grad_k, float* grad_v) {
  const size_t key_base = (size_t)key_block * B;
  for (uint32_t s_i = 0; s_i < seg_len; ++s_i) {
    const size_t t_begin = (size_t)seg[s_i] * span;
    for (size_t t = t_begin; t < t_begin + span; ++t) {
      const float* qt = q + t * d;
      const float* dout = d_out + t * d;
      const float m = row_max[t];
      const float inv_denom = 1.0f / row_denom[t];
      for (uint32_t b = 0; b < B; ++b) {
        const size_t kt = key_base + b;
        const float s = scale * key_gain * dot4(qt, keys + kt * d, d) + bias;
        const float p = expf(s - m) * inv_denom;
        const float dp = value_gain * dot4(dout, values + kt * d, d);
        const float ds = p * (dp - d_row[t]);
        axpy(grad_k + kt * d, qt, scale * key_gain * ds, d);
        axpy(grad_v + kt * d, dout, p * value_gain, d);
      }
    }
  }
}

static size_t csc_offsets_offset(uint64_t n, uint32_t B, uint32_t l) {
  size_t off = 0;
  uint64_t t = n / B;
  for (uint32_t j = 0; j < l; ++j) {
    off += (size_t)t + 1;
    t /= B;
  }
  return off;
}

int oracle_backward(const oracle_config* c, const float* d_out,
                    const float* out, const float* row_max,
                    const float* row_denom, const float* q, const float* k,
                    const float* v, const float* pyr_k, const float* pyr_v,
                    const uint32_t* tables, const uint32_t* csc_offsets,
                    const uint32_t* csc_flat, float* dq, float* dk, float* dv) {
  float scale;
  uint32_t E;
  int st = oracle_validate(c, &scale, &E);
  if (st) return st;
  const uint64_t n = c->n;
  const uint32_t d = c->d, B = c->block_size, K = c->top_k, L = c->levels,
                 Le = c->enrich_levels;
  const int scale_kv = c->reweight_mode == 0;
  const uint32_t fine = (uint32_t)(n / B);

  /* D_t = dot(d_out_t, out_t), :16-25 */
  float* d_row = (float*)malloc(sizeof(float) * n);
  uint32_t* pl = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)fine * E);
  uint32_t* pb = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)fine * E);
  float* pw = (float*)malloc(sizeof(float) * (size_t)fine * E);
  if (!d_row || !pl || !pb || !pw) return ST_ALLOC;
  for (uint64_t t = 0; t < n; ++t) d_row[t] = dot4(d_out + t * d, out + t * d, d);
  oracle_build_plan(c, tables, pl, pb, pw);

  /* query-major dq over the plan, :229-257 */
  memset(dq, 0, sizeof(float) * n * d);
  for (uint32_t i = 0; i < fine; ++i) {
    const size_t e0 = (size_t)i * E;
    for (uint32_t r = 0; r < B; ++r) {
      const size_t t = (size_t)i * B + r;
      const float* qt = q + t * d;
      const float* dout = d_out + t * d;
      float* dqt = dq + t * d;
      const float m = row_max[t];
      const float inv_denom = 1.0f / row_denom[t];
      for (uint32_t e = 0; e < E; ++e) {
        const float w = pw[e0 + e]; /* gains_for, :41-46 */
        const float kg = scale_kv ? w : 1.0f;
        const float bias = scale_kv ? 0.0f : logf(w);
        const uint32_t lvl = pl[e0 + e];
        const float* keys = level_ptr(k, pyr_k, n, d, B, lvl);
        const float* vals = level_ptr(v, pyr_v, n, d, B, lvl);
        const size_t base = (size_t)pb[e0 + e] * B;
        for (uint32_t b = 0; b < B; ++b) {
          const float* kt = keys + (base + b) * d;
          const float s = scale * kg * dot4(qt, kt, d) + bias;
          const float p = expf(s - m) * inv_denom;
          const float dp = kg * dot4(dout, vals + (base + b) * d, d);
          const float ds = p * (dp - d_row[t]);
          axpy(dqt, kt, scale * kg * ds, d);
        }
      }
    }
  }
  free(pl);
  free(pb);
  free(pw);

  /* kv_backward, :90-202 */
  memset(dk, 0, sizeof(float) * n * d);
  memset(dv, 0, sizeof(float) * n * d);
  const uint32_t lim = Le + 1 < L ? Le + 1 : L;
  size_t flat_off = 0;
  for (uint32_t l = 0; l < L; ++l) {
    const uint32_t key_blocks = (uint32_t)(n / ipow(B, l + 1));
    if (l < lim) {
      const float w = (float)ipow(B, l);
      const float kg = scale_kv ? w : 1.0f;
      const float bias = scale_kv ? 0.0f : logf(w);
      const size_t span = (size_t)ipow(B, l + 1);
      const float* keys = level_ptr(k, pyr_k, n, d, B, l);
      const float* vals = level_ptr(v, pyr_v, n, d, B, l);
      const uint32_t* offs = csc_offsets + csc_offsets_offset(n, B, l);
      const uint32_t* flat = csc_flat + flat_off;
      if (l == 0) { /* :127-135 */
        for (uint32_t b = 0; b < key_blocks; ++b)
          accumulate_key_block(d_out, row_max, row_denom, q, keys, vals, d_row,
                               flat + offs[b], offs[b + 1] - offs[b], b, span,
                               kg, kg, bias, scale, B, d, dk, dv);
      } else { /* :136-162 */
        const size_t tok = (size_t)(n / ipow(B, l));
        float* gk = (float*)calloc(tok * d, sizeof(float));
        float* gv = (float*)calloc(tok * d, sizeof(float));
        if (!gk || !gv) return ST_ALLOC;
        for (uint32_t b = 0; b < key_blocks; ++b)
          accumulate_key_block(d_out, row_max, row_denom, q, keys, vals, d_row,
                               flat + offs[b], offs[b + 1] - offs[b], b, span,
                               kg, kg, bias, scale, B, d, gk, gv);
        const float inv = 1.0f / (float)ipow(B, l);
        const size_t group = (size_t)ipow(B, l);
        for (uint64_t t = 0; t < n; ++t)
          for (uint32_t j = 0; j < d; ++j) {
            dk[t * d + j] += gk[(t / group) * d + j] * inv;
            dv[t * d + j] += gv[(t / group) * d + j] * inv;
          }
        free(gk);
        free(gv);
      }
    }
    flat_off += (size_t)key_blocks * K;
  }
  if (Le == L) { /* coarsest level, every query attends: :167-199 */
    const float w = (float)ipow(B, L);
    const float kg = scale_kv ? w : 1.0f;
    const float bias = scale_kv ? 0.0f : logf(w);
    const float* keys = level_ptr(k, pyr_k, n, d, B, L);
    const float* vals = level_ptr(v, pyr_v, n, d, B, L);
    const uint32_t key_blocks = (uint32_t)(n / ipow(B, L + 1));
    const size_t tok = (size_t)(n / ipow(B, L));
    float* gk = (float*)calloc(tok * d, sizeof(float));
    float* gv = (float*)calloc(tok * d, sizeof(float));
    if (!gk || !gv) return ST_ALLOC;
    const uint32_t all_queries = 0;
    for (uint32_t b = 0; b < key_blocks; ++b)
      accumulate_key_block(d_out, row_max, row_denom, q, keys, vals, d_row,
                           &all_queries, 1, b, (size_t)n, kg, kg, bias, scale, B,
                           d, gk, gv);
    const float inv = 1.0f / (float)ipow(B, L);
    const size_t group = (size_t)ipow(B, L);
    for (uint64_t t = 0; t < n; ++t)
      for (uint32_t j = 0; j < d; ++j) {
        dk[t * d + j] += gk[(t / group) * d + j] * inv;
        dv[t * d + j] += gv[(t / group) * d + j] * inv;
      }
    free(gk);
    free(gv);
  }
  free(d_row);
  return ST_OK;
}

/* ---- staleness token (P/src/attention.cpp:18-34,124-143) ----------------- */

static void fnv_word(uint64_t* h, uint64_t w) {
  *h ^= w;
  *h *= 0x100000001b3ull;
}

static void fnv_matrix(uint64_t* h, const float* m, uint64_t rows, uint64_t cols) {
  fnv_word(h, rows);
  fnv_word(h, cols);
  for (uint64_t i = 0; i < rows * cols; ++i) {
    uint32_t bits;
    memcpy(&bits, m + i, 4);
    fnv_word(h, bits);
  }
}

uint64_t oracle_input_checksum(const oracle_config* c, const float* q,
                               const float* k, const float* v) {
  float scale = 0;
  uint32_t E = 0;
  if (oracle_validate(c, &scale, &E)) return 0;
  uint64_t h = 0xcbf29ce484222325ull;
  fnv_word(&h, c->n);
  fnv_word(&h, c->d);
  fnv_word(&h, c->block_size);
  fnv_word(&h, c->top_k);
  fnv_word(&h, c->levels);
  fnv_word(&h, c->enrich_levels);
  fnv_word(&h, c->reweight_mode);
  fnv_word(&h, c->safe_softmax ? 1 : 0);
  const double sd = (double)scale;
  uint64_t sbits;
  memcpy(&sbits, &sd, 8);
  fnv_word(&h, sbits);
  fnv_word(&h, c->n / c->block_size);
  fnv_word(&h, E);
  fnv_matrix(&h, q, c->n, c->d);
  fnv_matrix(&h, k, c->n, c->d);
  fnv_matrix(&h, v, c->n, c->d);
  return h;
}

/* build_reorder, P/src/reorder2d.cpp:11-69.  Checks in the reference's order
 * (:13-30): empty image, non-square block, no patch level (1x1 excepted).
 * Positions are decoded top-down: the top-level patch row-major across the
 * image (:46-50), then one base-B digit per sub-patch level (:51-59). */
int oracle_build_reorder(uint32_t height, uint32_t width, uint32_t block_size,
                         uint32_t* forward, uint32_t* inverse) {
  if (height == 0 || width == 0) return 2;
  uint32_t side = 0;
  while ((uint64_t)side * side < block_size) ++side;
  if ((uint64_t)side * side != block_size || block_size == 0) return 12;
  uint32_t depth = 0;
  uint64_t patch = 1;
  while (height % (patch * side) == 0 && width % (patch * side) == 0) {
    patch *= side;
    ++depth;
  }
  if (depth == 0 && !(height == 1 && width == 1)) return 2;
  const uint64_t size = (uint64_t)height * width, per_patch = patch * patch;
  const uint64_t grid_w = width / patch;
  for (uint64_t pos = 0; pos < size; ++pos) {
    const uint64_t patch_id = pos / per_patch;
    uint64_t within = pos % per_patch;
    uint64_t y = (patch_id / grid_w) * patch, x = (patch_id % grid_w) * patch;
    uint64_t sub = patch / side;
    while (sub >= 1 && within > 0) {
      const uint64_t digit = within / (sub * sub);
      y += (digit / side) * sub;
      x += (digit % side) * sub;
      within %= sub * sub;
      if (sub == 1) break;
      sub /= side;
    }
    forward[pos] = (uint32_t)(y * width + x);
  }
  for (uint64_t pos = 0; pos < size; ++pos) inverse[forward[pos]] = (uint32_t)pos;
  return 0;
}
