// General-shape attention kernels (any d <= 256, any block size B):
//   K10 build_plan        P/src/attention.cpp:80-122
//   K5' forward           P/src/attention.cpp:145-219
//   K6-K9' backward       P/src/attention_grad.cpp:16-265
//
// One warp per query token (forward, dq) or per key token (dk/dv); lanes own
// columns j = lane + 32c of the d-vector.  The enriched KV set is read
// straight from the selection tables — fine block i uses per_level[l] row
// i/B^l for l < min(L_e+1, L), plus every coarsest block when L_e = L — so no
// plan is materialised and no dense mask exists.  fp32 throughout (dots are
// warp-reduced, so results match the reference to rounding, not bitwise).
// These kernels carry the fp32 configs (BASELINE C1) and every shape the
// tensor-core path (attn_tc.cu: d = 64, B = 16, bf16) does not cover.
#include "common.cuh"
#include "internal.h"

namespace llsa_impl {
namespace {

using namespace llsa_dev;

// Pointers + strides of one operand pyramid (level 0 = the input tensor).
template <typename T>
struct Levels {
  const T* lvl0;          // [units][n][d]
  const float* pyr;       // [units][pyr_rows][d]
  uint64_t lvl0_stride;   // n*d
  uint64_t pyr_stride;    // pyr_rows*d
  uint64_t off[kMaxLevels + 2];  // element offset of level l (>=1) within a unit
};

struct Dims {
  uint64_t n;
  uint32_t d, B, K, L, Le, lim, mode, safe;
  float scale;
  uint64_t pow[kMaxLevels + 2];
  uint64_t table_off[kMaxLevels + 1];
  uint64_t table_stride;
  // Optional materialised plan (llsa_forward_plan / llsa_backward_plan):
  // [units][n/B][epb] (level, block, weight); when set it replaces the tables.
  const uint32_t* plan_level;
  const uint32_t* plan_block;
  const float* plan_weight;
  uint32_t epb;
};

template <int COLS, typename T>
__device__ __forceinline__ void load_row(const T* row, uint32_t d, uint32_t lane,
                                         float (&x)[COLS]) {
#pragma unroll
  for (int c = 0; c < COLS; ++c) {
    const uint32_t j = lane + 32u * c;
    x[c] = j < d ? to_f(row[j]) : 0.f;
  }
}

template <int COLS>
__device__ __forceinline__ float row_dot(const float (&a)[COLS], const float (&b)[COLS]) {
  float p = 0.f;
#pragma unroll
  for (int c = 0; c < COLS; ++c) p = fmaf(a[c], b[c], p);
  p = warp_sum(p);
  return __shfl_sync(0xffffffffu, p, 0);  // one value for every lane
}

// Key (or value) row kt at level l of unit u.
template <typename T, int COLS>
__device__ __forceinline__ void level_row(const Levels<T>& P, uint32_t u, uint32_t l,
                                          uint64_t row, uint32_t d, uint32_t lane,
                                          float (&x)[COLS]) {
  if (l == 0) {
    load_row<COLS>(P.lvl0 + u * P.lvl0_stride + row * d, d, lane, x);
  } else {
    load_row<COLS>(P.pyr + u * P.pyr_stride + P.off[l] + row * d, d, lane, x);
  }
}

// Iterates the enriched KV entries of fine block i of unit u in canonical
// plan order (attention.cpp:107-118), calling f(level, block, weight); with a
// materialised plan the entries (and their weights) come from the plan.
template <typename F>
__device__ __forceinline__ void for_each_entry(const Dims& D, const uint32_t* tables,
                                               uint64_t u, uint64_t i, F&& f) {
  if (D.plan_level) {
    const uint64_t base = (u * (D.n / D.B) + i) * D.epb;
    for (uint32_t e = 0; e < D.epb; ++e)
      f(D.plan_level[base + e], D.plan_block[base + e], D.plan_weight[base + e]);
    return;
  }
  const uint32_t* tables_u = tables + u * D.table_stride;
  for (uint32_t l = 0; l < D.lim; ++l) {
    const uint64_t row = i / D.pow[l];
    const uint32_t* tr = tables_u + D.table_off[l] + row * D.K;
    for (uint32_t j = 0; j < D.K; ++j) f(l, tr[j], (float)D.pow[l]);
  }
  if (D.Le == D.L) {
    const uint64_t top = D.n / D.pow[D.L + 1];
    for (uint64_t b = 0; b < top; ++b) f(D.L, (uint32_t)b, (float)D.pow[D.L]);
  }
}

__global__ void plan_kernel(Dims D, uint32_t E, uint32_t units, const uint32_t* tables,
                            uint32_t* pl, uint32_t* pb, float* pw) {
  const uint64_t fine = D.n / D.B;
  const uint64_t total = fine * units;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = x / fine, i = x - u * fine;
    uint64_t e = x * E;
    for_each_entry(D, tables, u, i, [&](uint32_t l, uint32_t b, float w) {
      pl[e] = l;
      pb[e] = b;
      pw[e] = w;
      ++e;
    });
  }
}

template <typename T, int COLS>
__global__ void __launch_bounds__(256) fwd_kernel(Dims D, uint32_t units, const T* q,
                                                  Levels<T> Kp, Levels<T> Vp,
                                                  const uint32_t* tables, float* out,
                                                  float* row_max, float* row_denom,
                                                  uint32_t* flag) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp >= D.n * units) return;
  const uint32_t u = (uint32_t)(warp / D.n);
  const uint64_t t = warp - (uint64_t)u * D.n;
  const uint32_t d = D.d, B = D.B;
  const bool scale_kv = D.mode == 0;
  float qv[COLS], acc[COLS];
  load_row<COLS>(q + (uint64_t)u * D.n * d + t * d, d, lane, qv);
#pragma unroll
  for (int c = 0; c < COLS; ++c) acc[c] = 0.f;
  float m = D.safe ? -INFINITY : 0.f, denom = 0.f;
  for_each_entry(D, tables, u, t / B, [&](uint32_t l, uint32_t blk, float w) {
    const float kg = scale_kv ? w : 1.f;          // attention.cpp:176-180
    const float bias = scale_kv ? 0.f : logf(w);
    for (uint32_t b = 0; b < B; ++b) {
      const uint64_t row = (uint64_t)blk * B + b;
      float kv[COLS];
      level_row<T, COLS>(Kp, u, l, row, d, lane, kv);
      const float s = D.scale * kg * row_dot<COLS>(qv, kv) + bias;
      if (D.safe && s > m) {  // attention.cpp:191-196
        const float rs = expf(m - s);
        denom *= rs;
#pragma unroll
        for (int c = 0; c < COLS; ++c) acc[c] *= rs;
        m = s;
      }
      const float p = expf(s - m);
      denom += p;
      level_row<T, COLS>(Vp, u, l, row, d, lane, kv);
      const float pg = p * kg;
#pragma unroll
      for (int c = 0; c < COLS; ++c) acc[c] = fmaf(pg, kv[c], acc[c]);
    }
  });
  const float inv = 1.f / denom;
  float* o = out + (uint64_t)u * D.n * d + t * d;
  bool bad = !isfinite(denom) || denom <= 0.f;
#pragma unroll
  for (int c = 0; c < COLS; ++c) {
    const uint32_t j = lane + 32u * c;
    if (j < d) {
      const float y = acc[c] * inv;
      o[j] = y;
      bad |= !isfinite(y);
    }
  }
  if (lane == 0) {
    row_max[(uint64_t)u * D.n + t] = D.safe ? m : 0.f;
    row_denom[(uint64_t)u * D.n + t] = denom;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_flag(flag, kErrNonFinite);
}

// D_t = dot(dO_t, O_t), attention_grad.cpp:16-25 (computed once, not twice).
template <typename T, int COLS>
__global__ void __launch_bounds__(256) drow_kernel(uint64_t rows, uint32_t d, const T* dout,
                                                   const float* out, float* drow) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp >= rows) return;
  float a[COLS], b[COLS];
  load_row<COLS>(dout + warp * d, d, lane, a);
  load_row<COLS>(out + warp * d, d, lane, b);
  const float v = row_dot<COLS>(a, b);
  if (lane == 0) drow[warp] = v;
}

// Query-major dq over the enriched set, attention_grad.cpp:229-257.
template <typename T, int COLS>
__global__ void __launch_bounds__(256) dq_kernel(Dims D, uint32_t units, const T* q,
                                                 const T* dout, Levels<T> Kp, Levels<T> Vp,
                                                 const uint32_t* tables,
                                                 const float* row_max,
                                                 const float* row_denom,
                                                 const float* drow, float* dq) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp >= D.n * units) return;
  const uint32_t u = (uint32_t)(warp / D.n);
  const uint64_t t = warp - (uint64_t)u * D.n;
  const uint32_t d = D.d, B = D.B;
  const bool scale_kv = D.mode == 0;
  const uint64_t tok = (uint64_t)u * D.n + t;
  float qv[COLS], gv[COLS], acc[COLS];
  load_row<COLS>(q + tok * d, d, lane, qv);
  load_row<COLS>(dout + tok * d, d, lane, gv);
#pragma unroll
  for (int c = 0; c < COLS; ++c) acc[c] = 0.f;
  const float m = row_max[tok], inv_den = 1.f / row_denom[tok], Dt = drow[tok];
  for_each_entry(D, tables, u, t / B, [&](uint32_t l, uint32_t blk, float w) {
    const float kg = scale_kv ? w : 1.f;
    const float bias = scale_kv ? 0.f : logf(w);
    for (uint32_t b = 0; b < B; ++b) {
      const uint64_t row = (uint64_t)blk * B + b;
      float kv[COLS], vv[COLS];
      level_row<T, COLS>(Kp, u, l, row, d, lane, kv);
      level_row<T, COLS>(Vp, u, l, row, d, lane, vv);
      const float s = D.scale * kg * row_dot<COLS>(qv, kv) + bias;
      const float p = expf(s - m) * inv_den;
      const float dp = kg * row_dot<COLS>(gv, vv);
      const float ds = p * (dp - Dt);
      const float coef = D.scale * kg * ds;
#pragma unroll
      for (int c = 0; c < COLS; ++c) acc[c] = fmaf(coef, kv[c], acc[c]);
    }
  });
#pragma unroll
  for (int c = 0; c < COLS; ++c) {
    const uint32_t j = lane + 32u * c;
    if (j < d) dq[tok * d + j] = acc[c];
  }
}

// Key-major dk/dv for one key token over a range of its query list
// (accumulate_key_block, attention_grad.cpp:43-73).  The query list of key
// block b at level l is the CSC segment (rows ascending) expanded to `span`
// fine tokens per row; the coarsest level uses the single row 0 with
// span = n.  Level 0 writes dk/dv directly (nsplit = 1); coarse levels write
// per-split partials reduced later in a fixed order.
template <typename T, int COLS>
__global__ void __launch_bounds__(256) kv_kernel(
    Dims D, uint32_t units, uint32_t level, uint64_t tokens, uint64_t span,
    uint32_t nsplit, const uint32_t* csc_offsets, const uint32_t* csc_flat,
    uint64_t off_stride, uint64_t flat_stride, bool coarsest, const T* q, const T* dout,
    Levels<T> Kp, Levels<T> Vp, const float* row_max, const float* row_denom,
    const float* drow, float* gk, float* gv, uint64_t g_unit_stride,
    uint64_t g_split_stride) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp >= tokens * nsplit * units) return;
  const uint32_t u = (uint32_t)(warp / (tokens * nsplit));
  const uint64_t rem = warp - (uint64_t)u * tokens * nsplit;
  const uint32_t split = (uint32_t)(rem / tokens);
  const uint64_t kt = rem - (uint64_t)split * tokens;
  const uint32_t d = D.d, B = D.B;
  const uint64_t blk = kt / B;
  const bool scale_kv = D.mode == 0;
  const float w = (float)D.pow[level];
  const float kg = scale_kv ? w : 1.f;
  const float bias = scale_kv ? 0.f : logf(w);

  const uint32_t* seg;
  uint64_t seg_len;
  uint32_t zero_row = 0;
  if (coarsest) {
    seg = &zero_row;
    seg_len = 1;
  } else {
    const uint32_t* off = csc_offsets + (uint64_t)u * off_stride;
    seg = csc_flat + (uint64_t)u * flat_stride + off[blk];
    seg_len = off[blk + 1] - off[blk];
  }
  const uint64_t total = seg_len * span;
  const uint64_t lo = total * split / nsplit, hi = total * (split + 1) / nsplit;

  float kv[COLS], vv[COLS], ak[COLS], av[COLS];
  level_row<T, COLS>(Kp, u, level, kt, d, lane, kv);
  level_row<T, COLS>(Vp, u, level, kt, d, lane, vv);
#pragma unroll
  for (int c = 0; c < COLS; ++c) ak[c] = av[c] = 0.f;
  for (uint64_t f = lo; f < hi; ++f) {
    const uint64_t t = (uint64_t)seg[f / span] * span + f % span;
    const uint64_t tok = (uint64_t)u * D.n + t;
    float qv[COLS], gvv[COLS];
    load_row<COLS>(q + tok * d, d, lane, qv);
    load_row<COLS>(dout + tok * d, d, lane, gvv);
    const float s = D.scale * kg * row_dot<COLS>(qv, kv) + bias;
    const float p = expf(s - row_max[tok]) * (1.f / row_denom[tok]);
    const float dp = kg * row_dot<COLS>(gvv, vv);
    const float ds = p * (dp - drow[tok]);
    const float ck = D.scale * kg * ds, cv = p * kg;
#pragma unroll
    for (int c = 0; c < COLS; ++c) {
      ak[c] = fmaf(ck, qv[c], ak[c]);
      av[c] = fmaf(cv, gvv[c], av[c]);
    }
  }
  float* ok = gk + (uint64_t)u * g_unit_stride + (uint64_t)split * g_split_stride + kt * d;
  float* ov = gv + (uint64_t)u * g_unit_stride + (uint64_t)split * g_split_stride + kt * d;
#pragma unroll
  for (int c = 0; c < COLS; ++c) {
    const uint32_t j = lane + 32u * c;
    if (j < d) {
      ok[j] = ak[c];
      ov[j] = av[c];
    }
  }
}

// partial[0] = Σ_s partial[s] (fixed order) for one coarse level.
__global__ void reduce_splits_kernel(float* gk, float* gv, uint32_t units, uint64_t elems,
                                     uint32_t nsplit, uint64_t unit_stride,
                                     uint64_t split_stride) {
  const uint64_t total = elems * units;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = x / elems, e = x - u * elems;
    float* a = gk + u * unit_stride + e;
    float* b = gv + u * unit_stride + e;
    float sk = a[0], sv = b[0];
    for (uint32_t s = 1; s < nsplit; ++s) {
      sk += a[s * split_stride];
      sv += b[s * split_stride];
    }
    a[0] = sk;
    b[0] = sv;
  }
}

// Pooling adjoint (attention_grad.cpp:149-161, 184-196): every fine row t
// adds g_l[t / B^l] · (1/B^l), levels in ascending order.
struct AdjointLevels {
  const float* gk[kMaxLevels + 2];
  const float* gv[kMaxLevels + 2];
  uint64_t unit_stride[kMaxLevels + 2];
  uint64_t group[kMaxLevels + 2];
  float inv[kMaxLevels + 2];
  uint32_t count;
};

__global__ void adjoint_kernel(AdjointLevels A, uint64_t n, uint32_t d, uint32_t units,
                               float* dk, float* dv) {
  const uint64_t total = n * d * units;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = x / (n * d), r = x - u * n * d;
    const uint64_t t = r / d, j = r - t * d;
    float k = dk[x], v = dv[x];
    for (uint32_t i = 0; i < A.count; ++i) {
      const uint64_t src = u * A.unit_stride[i] + (t / A.group[i]) * d + j;
      k += A.gk[i][src] * A.inv[i];
      v += A.gv[i][src] * A.inv[i];
    }
    dk[x] = k;
    dv[x] = v;
  }
}

unsigned grid_for(uint64_t threads, int block) {
  uint64_t blocks = (threads + block - 1) / block;
  const uint64_t cap = 148ull * 32;
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

unsigned warps_grid(uint64_t warps) { return (unsigned)((warps * 32 + 255) / 256); }

Dims make_dims(const Geometry& g, const PlanView* plan = nullptr) {
  Dims D{};
  if (plan && plan->level) {
    D.plan_level = plan->level;
    D.plan_block = plan->block;
    D.plan_weight = plan->weight;
    D.epb = plan->epb;
  }
  D.n = g.n;
  D.d = g.d;
  D.B = g.B;
  D.K = g.K;
  D.L = g.L;
  D.Le = g.Le;
  D.lim = g.enrich_lim();
  D.mode = g.mode;
  D.safe = g.safe;
  D.scale = g.scale;
  for (int l = 0; l < kMaxLevels + 2; ++l) D.pow[l] = g.pow[l];
  for (int l = 0; l < kMaxLevels + 1; ++l) D.table_off[l] = g.table_off[l];
  D.table_stride = g.table_entries;
  return D;
}

template <typename T>
Levels<T> make_levels(const Geometry& g, const void* lvl0, const float* pyr) {
  Levels<T> P{};
  P.lvl0 = static_cast<const T*>(lvl0);
  P.pyr = pyr;
  P.lvl0_stride = g.n * g.d;
  P.pyr_stride = g.pyr_rows * g.d;
  for (int l = 1; l <= (int)g.L; ++l) P.off[l] = g.pyr_off[l] * g.d;
  return P;
}

int cols_for(uint32_t d) { return d <= 32 ? 1 : d <= 64 ? 2 : d <= 128 ? 4 : 8; }

// Coarse levels handled by the split kv kernel: l = 1..lim-1 and, when
// L_e = L, the coarsest level L.
struct CoarsePlan {
  uint32_t count = 0;
  uint32_t level[kMaxLevels + 2];
  uint32_t nsplit[kMaxLevels + 2];
  uint64_t tokens[kMaxLevels + 2];
  uint64_t bytes_off[kMaxLevels + 2];  // offset of the level's gk buffer in ws
  uint64_t unit_stride[kMaxLevels + 2];
  uint64_t split_stride[kMaxLevels + 2];
  uint64_t total = 0;
};

CoarsePlan coarse_plan(const Geometry& g, uint32_t units, uint64_t base) {
  CoarsePlan P;
  uint64_t off = base;
  auto add = [&](uint32_t l, uint64_t avg_queries) {
    const uint32_t i = P.count++;
    P.level[i] = l;
    uint64_t s = (avg_queries + 1023) / 1024;
    P.nsplit[i] = (uint32_t)(s < 1 ? 1 : s > 64 ? 64 : s);
    P.tokens[i] = g.level_tokens(l);
    P.split_stride[i] = P.tokens[i] * g.d;
    P.unit_stride[i] = P.split_stride[i] * P.nsplit[i];
    P.bytes_off[i] = off;
    off += 2 * ((units * P.unit_stride[i] * 4 + 255) & ~255ull);
  };
  for (uint32_t l = 1; l < g.enrich_lim(); ++l) add(l, (uint64_t)g.K * g.pow[l + 1]);
  if (g.Le == g.L) add(g.L, g.n);
  P.total = off;
  return P;
}

}  // namespace

llsa_status launch_build_plan(const Geometry& g, uint32_t units, const uint32_t* tables,
                              uint32_t* pl, uint32_t* pb, float* pw, cudaStream_t s) {
  const uint64_t total = (g.n / g.B) * units;
  if (total == 0) return LLSA_OK;
  plan_kernel<<<grid_for(total, 256), 256, 0, s>>>(make_dims(g), g.E, units, tables, pl, pb,
                                                   pw);
  count_launch();
  LLSA_LAUNCH_CHECK("plan_kernel");
  return LLSA_OK;
}

template <typename T, int COLS>
static void fwd_dispatch(const Geometry& g, uint32_t units, const void* q, const void* k,
                         const void* v, const float* pyr_k, const float* pyr_v,
                         const uint32_t* tables, float* out, float* rm, float* rd,
                         cudaStream_t s, const PlanView* plan) {
  fwd_kernel<T, COLS><<<warps_grid(g.n * units), 256, 0, s>>>(
      make_dims(g, plan), units, static_cast<const T*>(q), make_levels<T>(g, k, pyr_k),
      make_levels<T>(g, v, pyr_v), tables, out, rm, rd, device_flag());
}

llsa_status simt_forward(const Geometry& g, uint32_t units, llsa_dtype dt, const void* q,
                         const void* k, const void* v, const float* pyr_k,
                         const float* pyr_v, const uint32_t* tables, float* out,
                         float* row_max, float* row_denom, cudaStream_t s,
                         const PlanView* plan) {
  if (g.d > 256) return fail(LLSA_ERR_UNSUPPORTED, "d = %u > 256", g.d);
  if (units == 0) return LLSA_OK;
  const int cols = cols_for(g.d);
#define FWD(T)                                                                             \
  switch (cols) {                                                                          \
    case 1: fwd_dispatch<T, 1>(g, units, q, k, v, pyr_k, pyr_v, tables, out, row_max,      \
                               row_denom, s, plan); break;                                 \
    case 2: fwd_dispatch<T, 2>(g, units, q, k, v, pyr_k, pyr_v, tables, out, row_max,      \
                               row_denom, s, plan); break;                                 \
    case 4: fwd_dispatch<T, 4>(g, units, q, k, v, pyr_k, pyr_v, tables, out, row_max,      \
                               row_denom, s, plan); break;                                 \
    default: fwd_dispatch<T, 8>(g, units, q, k, v, pyr_k, pyr_v, tables, out, row_max,     \
                                row_denom, s, plan); break;                                \
  }
  if (dt == LLSA_BF16) {
    FWD(__nv_bfloat16)
  } else {
    FWD(float)
  }
#undef FWD
  count_launch();
  LLSA_LAUNCH_CHECK("fwd_kernel");
  return LLSA_OK;
}

size_t simt_backward_ws_bytes(const Geometry& g, uint32_t units) {
  const uint64_t drow = (units * g.n * 4 + 255) & ~255ull;
  return coarse_plan(g, units, drow).total + 256;
}

template <typename T, int COLS>
static llsa_status bwd_impl(const Geometry& g, uint32_t units, const void* d_out_,
                            const float* out, const float* row_max, const float* row_denom,
                            const void* q_, const void* k, const void* v,
                            const float* pyr_k, const float* pyr_v, const uint32_t* tables,
                            const uint32_t* csc_offsets, const uint32_t* csc_flat,
                            float* dq, float* dk, float* dv, void* ws, cudaStream_t s,
                            StageMarker* mk, const PlanView* plan) {
  const T* q = static_cast<const T*>(q_);
  const T* dout = static_cast<const T*>(d_out_);
  char* base = static_cast<char*>(ws);
  float* drow = reinterpret_cast<float*>(base);
  const uint64_t drow_bytes = (units * g.n * 4 + 255) & ~255ull;
  const Dims D = make_dims(g, plan);
  const Levels<T> Kp = make_levels<T>(g, k, pyr_k), Vp = make_levels<T>(g, v, pyr_v);

  drow_kernel<T, COLS><<<warps_grid(g.n * units), 256, 0, s>>>(g.n * units, g.d, dout, out,
                                                               drow);
  count_launch();
  LLSA_LAUNCH_CHECK("drow_kernel");
  LLSA_MARK(mk, "bwd_drow", s);
  if (dq) {
    dq_kernel<T, COLS><<<warps_grid(g.n * units), 256, 0, s>>>(
        D, units, q, dout, Kp, Vp, tables, row_max, row_denom, drow, dq);
    count_launch();
    LLSA_LAUNCH_CHECK("dq_kernel");
    LLSA_MARK(mk, "bwd_dq", s);
  }
  // level 0: straight into dk/dv (attention_grad.cpp:127-135)
  kv_kernel<T, COLS><<<warps_grid(g.n * units), 256, 0, s>>>(
      D, units, 0, g.n, g.pow[1], 1, csc_offsets + g.csc_off_off[0],
      csc_flat + g.csc_flat_off[0], g.csc_off_entries, g.csc_flat_entries, false, q, dout,
      Kp, Vp, row_max, row_denom, drow, dk, dv, g.n * g.d, 0);
  count_launch();
  LLSA_LAUNCH_CHECK("kv_kernel level 0");
  LLSA_MARK(mk, "bwd_kv_fine", s);

  const CoarsePlan P = coarse_plan(g, units, drow_bytes);
  AdjointLevels A{};
  for (uint32_t i = 0; i < P.count; ++i) {
    const uint32_t l = P.level[i];
    const bool top = (l == g.L);  // only reached when L_e = L
    float* gk = reinterpret_cast<float*>(base + P.bytes_off[i]);
    float* gv = reinterpret_cast<float*>(base + P.bytes_off[i] +
                                         ((units * P.unit_stride[i] * 4 + 255) & ~255ull));
    const uint64_t warps = P.tokens[i] * P.nsplit[i] * units;
    kv_kernel<T, COLS><<<warps_grid(warps), 256, 0, s>>>(
        D, units, l, P.tokens[i], top ? g.n : g.pow[l + 1], P.nsplit[i],
        top ? nullptr : csc_offsets + g.csc_off_off[l],
        top ? nullptr : csc_flat + g.csc_flat_off[l], g.csc_off_entries,
        g.csc_flat_entries, top, q, dout, Kp, Vp, row_max, row_denom, drow, gk, gv,
        P.unit_stride[i], P.split_stride[i]);
    count_launch();
    LLSA_LAUNCH_CHECK("kv_kernel coarse");
    if (P.nsplit[i] > 1) {
      const uint64_t elems = P.tokens[i] * g.d;
      reduce_splits_kernel<<<grid_for(elems * units, 256), 256, 0, s>>>(
          gk, gv, units, elems, P.nsplit[i], P.unit_stride[i], P.split_stride[i]);
      count_launch();
      LLSA_LAUNCH_CHECK("reduce_splits_kernel");
    }
    A.gk[A.count] = gk;
    A.gv[A.count] = gv;
    A.unit_stride[A.count] = P.unit_stride[i];
    A.group[A.count] = g.pow[l];
    A.inv[A.count] = 1.0f / (float)g.pow[l];
    ++A.count;
  }
  if (A.count) {
    adjoint_kernel<<<grid_for(g.n * g.d * units, 256), 256, 0, s>>>(A, g.n, g.d, units, dk,
                                                                    dv);
    count_launch();
    LLSA_LAUNCH_CHECK("adjoint_kernel");
  }
  LLSA_MARK(mk, "bwd_kv_coarse", s);
  return LLSA_OK;
}

llsa_status simt_backward(const Geometry& g, uint32_t units, llsa_dtype dt,
                          const void* d_out, const float* out, const float* row_max,
                          const float* row_denom, const void* q, const void* k,
                          const void* v, const float* pyr_k, const float* pyr_v,
                          const uint32_t* tables, const uint32_t* csc_offsets,
                          const uint32_t* csc_flat, float* dq, float* dk, float* dv,
                          void* ws, cudaStream_t s, StageMarker* mk, const PlanView* plan) {
  if (g.d > 256) return fail(LLSA_ERR_UNSUPPORTED, "d = %u > 256", g.d);
  if (units == 0) return LLSA_OK;
  const int cols = cols_for(g.d);
#define BWD(T, C)                                                                           \
  return bwd_impl<T, C>(g, units, d_out, out, row_max, row_denom, q, k, v, pyr_k, pyr_v,   \
                        tables, csc_offsets, csc_flat, dq, dk, dv, ws, s, mk, plan)
  if (dt == LLSA_BF16) {
    switch (cols) {
      case 1: BWD(__nv_bfloat16, 1);
      case 2: BWD(__nv_bfloat16, 2);
      case 4: BWD(__nv_bfloat16, 4);
      default: BWD(__nv_bfloat16, 8);
    }
  }
  switch (cols) {
    case 1: BWD(float, 1);
    case 2: BWD(float, 2);
    case 4: BWD(float, 4);
    default: BWD(float, 8);
  }
#undef BWD
}

}  // namespace llsa_impl
