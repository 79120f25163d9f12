// Tensor-core LLSA attention for d = 64, B = 16, bf16 inputs (the BASELINE
// shapes).  Replaces P/src/attention.cpp:145-219 (forward) and
// P/src/attention_grad.cpp:16-265 (backward).
//
// Tiling follows the structure of the enriched KV set:
//   * A CTA owns 128 consecutive queries = 8 fine query blocks, one per warp.
//     All 8 share the same coarse entries (levels 1..L: per_level[l] row
//     i/B^l and the full coarsest level), so the coarse keys are staged once
//     per CTA in shared memory (double-buffered chunks, cp.async) and consumed
//     by every warp as dense m16n8k16 tiles.
//   * Each warp's own fine part (its K gathered level-0 blocks, each a
//     contiguous 2 KB run of K and of V) streams through a per-warp double
//     buffer.  The 16-query fine block is exactly one m16 MMA tile.
//   * Online softmax in fp32 (exp2 domain), P rounded to bf16 for PV.
//   * Coarse keys/values are the fp32 pyramid pre-scaled by the level gain
//     (ScaleKV: B^l) and split into bf16 hi + lo (SURVEY.md hard part 3):
//     S and dP use hi + lo (two MMAs), PV and dQ use hi.
//   * <= 112.5 KB smem and <= 128 registers per thread: 2 CTAs (16 warps) per
//     SM, so HMMA latency is hidden across warps.
// Backward (mask-free, Alg. 2 of the paper):
//   * dq kernel: query-major, same tiling; recomputes P from the saved
//     (row_max, row_denom), dP = dO V'^T, dS = P∘(dP − D) with D = rowsum(dO∘O)
//     from the fp32 forward output; writes dq, D and log2-LSE.
//   * kv kernels: key-major; one warp owns one 16-key block (the m16 tile)
//     and streams the queries that selected it (CSC segment × span, or all
//     queries for the coarsest level) in 16-query chunks; dK', dV' stay in
//     registers — no atomics.  Coarse levels split long query lists into
//     fixed slices reduced in a fixed order; the fine kernel then adds the
//     pooling adjoint of every coarse level and writes dk, dv once.
#include <cuda.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "tc.h"
#include "tc_common.cuh"
#include "umma.cuh"

namespace llsa_impl {
static int num_sms();  // SM count of the current device (below)

namespace {

using namespace llsa_tc;
using bf16 = __nv_bfloat16;

constexpr int kD = 64;
constexpr int kBS = 16;
constexpr int kTileQ = 128;
constexpr int kMaxCoarse = 64;  // coarse entries per tile (64 × 16 = 1024 keys)
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kTile16 = kBS * 128;  // one 16-row swizzled 64-column bf16 tile

struct TcParams {
  const bf16 *q, *k, *v, *dout;
  const bf16 *khi, *klo, *vhi, *vlo;  // [units][pyr_rows][64] (coarse levels)
  const uint32_t* tables;
  const uint32_t *csc_off, *csc_flat;
  const float* out_in;               // forward output (backward input)
  float *out, *row_max, *row_denom;  // forward outputs
  const float *rm_in, *rd_in;        // saved statistics (backward)
  float *lse2, *drow;                // [units][n] backward scratch
  float *dq, *dk, *dv;
  uint32_t grad_bf16;  // dq/dk/dv are bf16 buffers (tc5_dqf + tc5_kvf write them directly)
  float* part;  // coarse dK'/dV' partials
  uint32_t* flag;
  uint64_t n, pyr_rows, table_entries, csc_off_entries, csc_flat_entries;
  uint32_t K, L, Le, lim, nce;
  float scale;
  uint64_t pow[kMaxLevels + 2];
  uint64_t pyr_off[kMaxLevels + 2];
  uint64_t table_off[kMaxLevels + 1];
  uint64_t csc_off_off[kMaxLevels + 1], csc_flat_off[kMaxLevels + 1];
  float bias2[kMaxLevels + 2];  // per-level logit bias × log2e (LogitBias)
  // Coarse levels >= hilo_level use the bf16 hi + lo split in S and dP;
  // shallower ones (gain B^l small) use hi only.
  uint32_t hilo_level;
  // Coarse-entry split (coarse sets past the 24-entry TMEM budget of the
  // tcgen05 forward / dQ kernels run in two passes): this pass covers plan
  // entries [ce_base, ce_base + nce); fine_mode 1 = no fine blocks in this
  // pass — the forward's fine warps contribute the previous pass's (O,
  // row_max, row_denom) as their partition instead, the dQ fine warps only
  // D and the LSE, and dq is added to (TMA reduce-add) instead of stored.
  uint32_t ce_base, fine_mode;
  uint32_t dbg;    // LLSA_DBG: timing probes, see probe()
  uint32_t trace;  // 1: record pipeline timestamps of CTA 0 (LLSA_TRACE=1; debugging)
  uint32_t trace_rows2;  // LLSA_TRACE_ONLY=rows2: trace only the level-1 rows2 launch
  // coarse-level partial layout (kv kernels)
  uint32_t ncl;  // number of coarse level slots
  uint32_t cl_level[kMaxLevels + 2];
  uint32_t cl_split[kMaxLevels + 2];
  uint64_t cl_tasks[kMaxLevels + 2];     // task prefix (coarse launch)
  uint64_t cl_part_off[kMaxLevels + 2];  // float offset of slot (per unit)
  float cl_ck[kMaxLevels + 2], cl_cv[kMaxLevels + 2];
  uint64_t part_unit_stride;  // floats per unit (dk + dv)
  // tcgen05 row-major coarse dK/dV (levels 1..lim-1): one task per
  // (level, selection row, query slice, 8-block key group)
  float* rpart;                           // row partials
  uint32_t rows_on, groups;               // path enabled; key groups per row (ceil(K/8))
  uint32_t rows_atomic;                   // rows2 reduces into the level slots (TMA add)
  uint32_t kv_atomic;                     // tc_kv coarse splits add into split 0 (red.add)
  void* out16;                            // forward: also write O as bf16 here (or null)
  uint32_t rl_count;                      // levels handled (1..lim-1)
  uint32_t rl_level[kMaxLevels + 2];
  uint32_t rl_slices[kMaxLevels + 2];     // query slices per row
  uint64_t rl_qs[kMaxLevels + 2];         // queries per slice
  uint64_t rl_tasks[kMaxLevels + 3];      // task prefix (per unit)
  uint64_t rl_part_off[kMaxLevels + 2];   // float offset per unit
  uint32_t rl_groups[kMaxLevels + 2];     // 8-block key groups per row
  uint32_t rl_top[kMaxLevels + 2];        // 1: the coarsest level (one row = all n queries,
                                          //    its blocks 0 .. n/B^(L+1)-1, no table)
  uint64_t rpart_unit_stride;
};

// Pipeline trace (debug only): CTA 0 records (role, tile, event, clock) so the
// hand-offs of the warp-specialised kernels can be inspected offline.
__device__ unsigned long long g_trace[8192];  // [role 0..7][tile 0..31][event 0..31]
// Timing probes, compiled in only with -DLLSA_PROBES (LLSA_NVCC_EXTRA): with
// them LLSA_DBG bit 8 skips the fine attention and bit 16 the fine gathers of
// the forward and dQ kernels (results are then wrong).  A runtime check in
// the fine loops costs ~10 us of forward time, hence the macro.
__device__ __forceinline__ bool probe(const TcParams& p, uint32_t bit) {
#ifdef LLSA_PROBES
  return p.dbg & bit;
#else
  (void)p;
  (void)bit;
  return false;
#endif
}

// Pipeline timestamps of CTA 0 (tools/trace_fwd.py), compiled in only with
// -DLLSA_TRACE_EVENTS so the hot loops carry no runtime check.
__device__ __forceinline__ void trace_ev(const TcParams& p, uint32_t role, uint32_t tile,
                                         uint32_t ev) {
#ifdef LLSA_TRACE_EVENTS
  if (p.trace && blockIdx.x == 0 && tile < 32 && ev < 32)
    g_trace[role * 1024 + tile * 32 + ev] = clock64() | (1ull << 63);
#else
  (void)p;
  (void)role;
  (void)tile;
  (void)ev;
#endif
}

// Coarse entry e of the tile whose first fine block is fb0 → (level, first
// pyramid row), canonical plan order (attention.cpp:107-118).
__device__ __forceinline__ void coarse_entry(const TcParams& p, const uint32_t* tab,
                                             uint64_t fb0, uint32_t e, uint32_t& lvl,
                                             uint32_t& row) {
  e += p.ce_base;
  const uint32_t ksel = p.K * (p.lim - 1);
  uint32_t b;
  if (e < ksel) {
    lvl = 1 + e / p.K;
    const uint64_t r = fb0 / p.pow[lvl];
    b = tab[p.table_off[lvl] + r * p.K + e % p.K];
  } else {
    lvl = p.L;
    b = e - ksel;
  }
  const uint64_t blocks = p.n / p.pow[lvl + 1];
  if (b >= blocks) {
    raise_flag(p.flag, llsa_dev::kErrIndex);
    b = 0;
  }
  row = (uint32_t)(p.pyr_off[lvl] + (uint64_t)b * kBS);
}

// Copies entries e0..e0+ne-1 (16 rows each, contiguous in global) of `narr`
// arrays into a stage whose array a starts at stage + a*arr_stride.
__device__ __forceinline__ void load_coarse_chunk(uint32_t stage, uint32_t arr_stride,
                                                  const uint32_t* ce_row, uint32_t e0,
                                                  uint32_t ne, const bf16* const* arrays,
                                                  int narr, uint64_t unit_off, uint32_t tid,
                                                  uint32_t nthr) {
  const uint32_t per_arr = ne * 128;  // 16 B chunks per array
  for (uint32_t i = tid; i < per_arr * narr; i += nthr) {
    const uint32_t a = i / per_arr, r = i % per_arr;
    const uint32_t e = r >> 7, w = r & 127;
    const char* src =
        reinterpret_cast<const char*>(arrays[a] + unit_off + (uint64_t)ce_row[e0 + e] * kD) +
        w * 16;
    cp_async16(stage + a * arr_stride + swz(e * 16 + (w >> 3), w & 7), src);
  }
}

// ---------------------------------------------------------------------------
// prep: coarse K'/V' = gain_l · pyramid, split into bf16 hi + lo
// ---------------------------------------------------------------------------
__global__ void prep_kernel(const float* __restrict__ pk, const float* __restrict__ pv,
                            bf16* khi, bf16* klo, bf16* vhi, bf16* vlo, uint64_t pyr_rows,
                            uint32_t units, float g1, float g2, float g3, float g4, uint64_t o2,
                            uint64_t o3, uint64_t o4) {
  const uint64_t total = (uint64_t)units * pyr_rows * kD;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = (i / kD) % pyr_rows;  // level of the row from its offset
    const float g = row >= o4 ? g4 : row >= o3 ? g3 : row >= o2 ? g2 : g1;
    const float a = pk[i] * g, b = pv[i] * g;
    const bf16 ah = __float2bfloat16_rn(a), bh = __float2bfloat16_rn(b);
    khi[i] = ah;
    klo[i] = __float2bfloat16_rn(a - __bfloat162float(ah));
    vhi[i] = bh;
    vlo[i] = __float2bfloat16_rn(0.f);  // see tc.h: dP uses V'_hi, the forward's value
  }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
struct SoftmaxState {
  float o[8][4];
  float m[2], l[2];
};

// Attends the warp's 16 queries (qf) to `ne` (<= 2) 16-key entries at rows
// row0 + 16e of the K'/V' tiles.  Online softmax in log2 units.
template <bool HILO>
__device__ __forceinline__ void attend_fwd(uint32_t kHi, uint32_t kLo, uint32_t vHi,
                                           uint32_t row0, int ne, float bias_a, float bias_b,
                                           float c, const uint32_t (&qf)[4][4], uint32_t lane,
                                           SoftmaxState& st) {
  float s[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[j][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (e < ne) {
        uint32_t b[4];
        ldb(kHi, row0 + e * 16, ks, lane, b);
        mma16816(s[2 * e], qf[ks], b[0], b[1]);
        mma16816(s[2 * e + 1], qf[ks], b[2], b[3]);
        if (HILO) {
          ldb(kLo, row0 + e * 16, ks, lane, b);
          mma16816(s[2 * e], qf[ks], b[0], b[1]);
          mma16816(s[2 * e + 1], qf[ks], b[2], b[3]);
        }
      }
    }
  }
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    if (e < ne) {
      const float bias = e ? bias_b : bias_a;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float* x = s[2 * e + h];
        x[0] = fmaf(x[0], c, bias);
        x[1] = fmaf(x[1], c, bias);
        x[2] = fmaf(x[2], c, bias);
        x[3] = fmaf(x[3], c, bias);
        mx0 = fmaxf(mx0, fmaxf(x[0], x[1]));
        mx1 = fmaxf(mx1, fmaxf(x[2], x[3]));
      }
    }
  }
  mx0 = quad_max(mx0);
  mx1 = quad_max(mx1);
  const float mn0 = fmaxf(st.m[0], mx0), mn1 = fmaxf(st.m[1], mx1);
  const float a0 = ex2(st.m[0] - mn0), a1 = ex2(st.m[1] - mn1);
  st.m[0] = mn0;
  st.m[1] = mn1;
  st.l[0] *= a0;
  st.l[1] *= a1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    st.o[j][0] *= a0;
    st.o[j][1] *= a0;
    st.o[j][2] *= a1;
    st.o[j][3] *= a1;
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    if (e < ne) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float* x = s[2 * e + h];
        x[0] = ex2(x[0] - mn0);
        x[1] = ex2(x[1] - mn0);
        x[2] = ex2(x[2] - mn1);
        x[3] = ex2(x[3] - mn1);
        st.l[0] += x[0] + x[1];
        st.l[1] += x[2] + x[3];
      }
      const uint32_t a[4] = {pack_bf16(s[2 * e][0], s[2 * e][1]),
                             pack_bf16(s[2 * e][2], s[2 * e][3]),
                             pack_bf16(s[2 * e + 1][0], s[2 * e + 1][1]),
                             pack_bf16(s[2 * e + 1][2], s[2 * e + 1][3])};
#pragma unroll
      for (int dn = 0; dn < 4; ++dn) {
        uint32_t b[4];
        ldb_t(vHi, row0 + e * 16, dn * 16, lane, b);
        mma16816(st.o[2 * dn], a, b[0], b[1]);
        mma16816(st.o[2 * dn + 1], a, b[2], b[3]);
      }
    }
  }
}

// smem (bytes): 2 coarse stages of 64 keys × {Khi, Klo, V} + per-warp double
// buffer of one fine block {K, V} (its second stage first holds the warp's Q)
constexpr int kFwdArr = 64 * 128;              // 8 KB per array per stage
constexpr int kFwdCStage = 3 * kFwdArr;        // 24 KB
constexpr int kFStage = 2 * kTile16;           // 4 KB
constexpr int kFwdSmem = 2 * kFwdCStage + 8 * 2 * kFStage + 2 * kMaxCoarse * 4;  // 112.5 KB

__global__ void __launch_bounds__(256, 2) tc_fwd_kernel(TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t unit = blockIdx.y;
  const uint64_t q0 = (uint64_t)blockIdx.x * kTileQ;
  const uint64_t fb0 = q0 / kBS;
  const uint64_t fb = fb0 + warp;
  const uint32_t sC = smem_u32(smem);
  const uint32_t sF = sC + 2 * kFwdCStage + warp * 2 * kFStage;
  uint32_t* ce_row = reinterpret_cast<uint32_t*>(smem + 2 * kFwdCStage + 16 * kFStage);
  uint32_t* ce_lvl = ce_row + kMaxCoarse;

  const uint64_t in_off = (uint64_t)unit * p.n * kD;
  const uint64_t pyr_off = (uint64_t)unit * p.pyr_rows * kD;
  const uint32_t* tab = p.tables + (uint64_t)unit * p.table_entries;
  const bf16* coarse[3] = {p.khi, p.klo, p.vhi};

  for (uint32_t e = tid; e < p.nce; e += blockDim.x) {
    uint32_t l, r;
    coarse_entry(p, tab, fb0, e, l, r);
    ce_row[e] = r;
    ce_lvl[e] = l;
  }
  const uint32_t* frow = tab + p.table_off[0] + fb * p.K;
  const uint64_t nfb = p.n / kBS;
  auto load_fine = [&](uint32_t j, uint32_t stage) {
    uint32_t b = frow[j];
    if (b >= nfb) {
      raise_flag(p.flag, llsa_dev::kErrIndex);
      b = 0;
    }
    const uint32_t base = sF + stage * kFStage;
    load_rows_async(base, 0, p.k + in_off + (uint64_t)b * kBS * kD, kBS, lane, 32);
    load_rows_async(base + kTile16, 0, p.v + in_off + (uint64_t)b * kBS * kD, kBS, lane, 32);
  };
  __syncthreads();  // entry list visible

  // group 0: this warp's Q rows (into fine stage 1), fine block 0, coarse chunk 0
  load_rows_async(sF + kFStage, 0, p.q + in_off + (q0 + warp * 16) * kD, kBS, lane, 32);
  load_fine(0, 0);
  const uint32_t nchunks = (p.nce + 3) / 4;
  if (nchunks)
    load_coarse_chunk(sC, kFwdArr, ce_row, 0, min(4u, p.nce), coarse, 3, pyr_off, tid, 256);
  cp_async_commit();

  SoftmaxState st;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) st.o[j][i] = 0.f;
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = 0.f;
  const float c = p.scale * kLog2e;

  uint32_t qf[4][4];
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) lda(sF + kFStage, 0, ks, lane, qf[ks]);
  __syncwarp();

  // ---- coarse part: CTA-shared chunks of up to 4 entries (64 keys) ----
  for (uint32_t ch = 0; ch < nchunks; ++ch) {
    const uint32_t stage = sC + (ch & 1) * kFwdCStage;
    if (ch + 1 < nchunks) {
      const uint32_t e0 = (ch + 1) * 4;
      load_coarse_chunk(sC + ((ch + 1) & 1) * kFwdCStage, kFwdArr, ce_row, e0,
                        min(4u, p.nce - e0), coarse, 3, pyr_off, tid, 256);
    }
    cp_async_commit();
    if (ch > 0) {
      cp_async_wait<1>();
      __syncthreads();
    }
    const uint32_t e0 = ch * 4;
    const int ne = (int)min(4u, p.nce - e0);
    for (int h = 0; h < ne; h += 2) {
      const int n2 = min(2, ne - h);
      const float ba = p.bias2[ce_lvl[e0 + h]];
      const float bb = n2 > 1 ? p.bias2[ce_lvl[e0 + h + 1]] : 0.f;
      const uint32_t lv = max(ce_lvl[e0 + h], n2 > 1 ? ce_lvl[e0 + h + 1] : 0u);
      if (lv >= p.hilo_level)
        attend_fwd<true>(stage, stage + kFwdArr, stage + 2 * kFwdArr, h * 16, n2, ba, bb, c, qf,
                         lane, st);
      else
        attend_fwd<false>(stage, stage + kFwdArr, stage + 2 * kFwdArr, h * 16, n2, ba, bb, c,
                          qf, lane, st);
    }
    __syncthreads();  // stage may be overwritten by the next prefetch
  }
  cp_async_wait<0>();
  __syncwarp();

  // ---- fine part: this warp's K gathered level-0 blocks ----
  const float bf = p.bias2[0];
  for (uint32_t j = 0; j < p.K; ++j) {
    if (j + 1 < p.K) load_fine(j + 1, (j + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const uint32_t base = sF + (j & 1) * kFStage;
    attend_fwd<false>(base, base, base + kTile16, 0, 1, bf, bf, c, qf, lane, st);
    __syncwarp();
  }

  // ---- epilogue: O = acc / l; (row_max, row_denom) in natural-log units ----
  const float l0 = quad_sum(st.l[0]), l1 = quad_sum(st.l[1]);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  const uint32_t r = lane >> 2, cc = (lane & 3) * 2;
  const uint64_t t0 = q0 + warp * 16 + r, t1 = t0 + 8;
  float* o0 = p.out + in_off + t0 * kD;
  float* o1 = p.out + in_off + t1 * kD;
  bool bad = !(l0 > 0.f) || !(l1 > 0.f) || !isfinite(l0) || !isfinite(l1);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 v0 = make_float2(st.o[j][0] * i0, st.o[j][1] * i0);
    const float2 v1 = make_float2(st.o[j][2] * i1, st.o[j][3] * i1);
    bad |= !isfinite(v0.x) || !isfinite(v0.y) || !isfinite(v1.x) || !isfinite(v1.y);
    *reinterpret_cast<float2*>(o0 + j * 8 + cc) = v0;
    *reinterpret_cast<float2*>(o1 + j * 8 + cc) = v1;
  }
  if ((lane & 3) == 0) {
    const uint64_t ro = (uint64_t)unit * p.n;
    p.row_max[ro + t0] = st.m[0] / kLog2e;
    p.row_max[ro + t1] = st.m[1] / kLog2e;
    p.row_denom[ro + t0] = l0;
    p.row_denom[ro + t1] = l1;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_flag(p.flag, llsa_dev::kErrNonFinite);
}

// ---------------------------------------------------------------------------
// backward: dq (query-major)
// ---------------------------------------------------------------------------
// One 16-key entry at row0 of the K'/V' tiles: P, dP, dS, dQ += dS·K'.
template <bool HILO>
__device__ __forceinline__ void attend_dq(uint32_t kHi, uint32_t kLo, uint32_t vHi,
                                          uint32_t vLo, uint32_t row0, float bias, float c,
                                          const uint32_t (&qf)[4][4],
                                          const uint32_t (&gf)[4][4], float lse0, float lse1,
                                          float D0, float D1, uint32_t lane,
                                          float (&dq)[8][4]) {
  float s[2][4], sl[2][4], g[2][4], gl[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[j][i] = sl[j][i] = g[j][i] = gl[j][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t b[4];
    ldb(kHi, row0, ks, lane, b);
    mma16816(s[0], qf[ks], b[0], b[1]);
    mma16816(s[1], qf[ks], b[2], b[3]);
    ldb(vHi, row0, ks, lane, b);
    mma16816(g[0], gf[ks], b[0], b[1]);
    mma16816(g[1], gf[ks], b[2], b[3]);
    if (HILO) {
      ldb(kLo, row0, ks, lane, b);
      mma16816(sl[0], qf[ks], b[0], b[1]);
      mma16816(sl[1], qf[ks], b[2], b[3]);
      ldb(vLo, row0, ks, lane, b);
      mma16816(gl[0], gf[ks], b[0], b[1]);
      mma16816(gl[1], gf[ks], b[2], b[3]);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float* x = s[h];
    const float* y = g[h];
    if (HILO) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[i] += sl[h][i];
        g[h][i] += gl[h][i];
      }
    }
    // packed fp32x2 (rows r: elements 0, 1; row r+8: 2, 3), same rounding
    const float2 c22 = make_float2(c, c), b22 = make_float2(bias, bias);
    const float2 t01 = __fadd2_rn(__ffma2_rn(make_float2(x[0], x[1]), c22, b22),
                                  make_float2(-lse0, -lse0));
    const float2 t23 = __fadd2_rn(__ffma2_rn(make_float2(x[2], x[3]), c22, b22),
                                  make_float2(-lse1, -lse1));
    const float2 g01 = __fadd2_rn(make_float2(y[0], y[1]), make_float2(-D0, -D0));
    const float2 g23 = __fadd2_rn(make_float2(y[2], y[3]), make_float2(-D1, -D1));
    const float2 r01 = __fmul2_rn(make_float2(ex2(t01.x), ex2(t01.y)), g01);
    const float2 r23 = __fmul2_rn(make_float2(ex2(t23.x), ex2(t23.y)), g23);
    x[0] = r01.x;
    x[1] = r01.y;
    x[2] = r23.x;
    x[3] = r23.y;
  }
  const uint32_t a[4] = {pack_bf16(s[0][0], s[0][1]), pack_bf16(s[0][2], s[0][3]),
                         pack_bf16(s[1][0], s[1][1]), pack_bf16(s[1][2], s[1][3])};
#pragma unroll
  for (int dn = 0; dn < 4; ++dn) {
    uint32_t b[4];
    ldb_t(kHi, row0, dn * 16, lane, b);
    mma16816(dq[2 * dn], a, b[0], b[1]);
    mma16816(dq[2 * dn + 1], a, b[2], b[3]);
  }
}

// smem: 2 coarse stages of 32 keys × {Khi, Klo, Vhi, Vlo} + per-warp fine
// double buffer (stage 1 first holds the warp's Q and dO)
constexpr int kDqArr = 32 * 128;              // 4 KB
constexpr int kDqCStage = 4 * kDqArr;         // 16 KB
constexpr int kDqSmem = 2 * kDqCStage + 8 * 2 * kFStage + 2 * kMaxCoarse * 4;  // 96.5 KB

__global__ void __launch_bounds__(256, 2) tc_dq_kernel(TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t unit = blockIdx.y;
  const uint64_t q0 = (uint64_t)blockIdx.x * kTileQ;
  const uint64_t fb0 = q0 / kBS;
  const uint64_t fb = fb0 + warp;
  const uint32_t sC = smem_u32(smem);
  const uint32_t sF = sC + 2 * kDqCStage + warp * 2 * kFStage;
  uint32_t* ce_row = reinterpret_cast<uint32_t*>(smem + 2 * kDqCStage + 16 * kFStage);
  uint32_t* ce_lvl = ce_row + kMaxCoarse;

  const uint64_t in_off = (uint64_t)unit * p.n * kD;
  const uint64_t pyr_off = (uint64_t)unit * p.pyr_rows * kD;
  const uint32_t* tab = p.tables + (uint64_t)unit * p.table_entries;
  const bf16* coarse[4] = {p.khi, p.klo, p.vhi, p.vlo};

  for (uint32_t e = tid; e < p.nce; e += blockDim.x) {
    uint32_t l, r;
    coarse_entry(p, tab, fb0, e, l, r);
    ce_row[e] = r;
    ce_lvl[e] = l;
  }
  const uint32_t* frow = tab + p.table_off[0] + fb * p.K;
  const uint64_t nfb = p.n / kBS;
  const Block16Lane bl = block16_lane(lane);
  auto load_fine = [&](uint32_t j, uint32_t stage) {
    uint32_t b = frow[j];
    if (b >= nfb) b = 0;
    const uint32_t base = sF + stage * kFStage;
    load_block16_async(base, p.k + in_off + (uint64_t)b * kBS * kD, bl, lane);
    load_block16_async(base + kTile16, p.v + in_off + (uint64_t)b * kBS * kD, bl, lane);
  };
  __syncthreads();

  const uint64_t qrow0 = q0 + warp * 16;
  load_block16_async(sF + kFStage, p.q + in_off + qrow0 * kD, bl, lane);
  load_block16_async(sF + kFStage + kTile16, p.dout + in_off + qrow0 * kD, bl, lane);
  load_fine(0, 0);
  const uint32_t nchunks = (p.nce + 1) / 2;
  if (nchunks)
    load_coarse_chunk(sC, kDqArr, ce_row, 0, min(2u, p.nce), coarse, 4, pyr_off, tid, 256);
  cp_async_commit();

  // D_t = rowsum(dO ∘ O) from the fp32 output (attention_grad.cpp:16-25) and
  // the log2 LSE, for this warp's 16 rows; lane pair (2ρ, 2ρ+1) owns row ρ.
  const uint32_t rr = lane >> 1, half = lane & 1;
  const uint64_t trow = qrow0 + rr;
  float dsum = 0.f;
  {
    const float4* o4 = reinterpret_cast<const float4*>(p.out_in + in_off + trow * kD + half * 32);
    const uint4* g4 = reinterpret_cast<const uint4*>(p.dout + in_off + trow * kD + half * 32);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 gv = g4[i];
      const float4 oa = o4[2 * i], ob = o4[2 * i + 1];
      const uint32_t w[4] = {gv.x, gv.y, gv.z, gv.w};
      const float of[8] = {oa.x, oa.y, oa.z, oa.w, ob.x, ob.y, ob.z, ob.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        dsum = fmaf(__uint_as_float(w[k] << 16), of[2 * k], dsum);
        dsum = fmaf(__uint_as_float(w[k] & 0xffff0000u), of[2 * k + 1], dsum);
      }
    }
  }
  dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
  const uint64_t ro = (uint64_t)unit * p.n;
  const float lse_r = p.rm_in[ro + trow] * kLog2e + __log2f(p.rd_in[ro + trow]);
  if (half == 0) {
    p.drow[ro + trow] = dsum;
    p.lse2[ro + trow] = lse_r;
  }
  const uint32_t r = lane >> 2;
  const float D0 = __shfl_sync(0xffffffffu, dsum, 2 * r);
  const float D1 = __shfl_sync(0xffffffffu, dsum, 2 * (r + 8));
  const float lse0 = __shfl_sync(0xffffffffu, lse_r, 2 * r);
  const float lse1 = __shfl_sync(0xffffffffu, lse_r, 2 * (r + 8));

  float dq[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) dq[j][i] = 0.f;
  const float c = p.scale * kLog2e;

  uint32_t qf[4][4], gf[4][4];
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    lda(sF + kFStage, 0, ks, lane, qf[ks]);
    lda(sF + kFStage + kTile16, 0, ks, lane, gf[ks]);
  }
  __syncwarp();

  for (uint32_t ch = 0; ch < nchunks; ++ch) {
    const uint32_t stage = sC + (ch & 1) * kDqCStage;
    if (ch + 1 < nchunks) {
      const uint32_t e0 = (ch + 1) * 2;
      load_coarse_chunk(sC + ((ch + 1) & 1) * kDqCStage, kDqArr, ce_row, e0,
                        min(2u, p.nce - e0), coarse, 4, pyr_off, tid, 256);
    }
    cp_async_commit();
    if (ch > 0) {
      cp_async_wait<1>();
      __syncthreads();
    }
    const uint32_t e0 = ch * 2;
    const int ne = (int)min(2u, p.nce - e0);
    for (int e = 0; e < ne; ++e) {
      if (ce_lvl[e0 + e] >= p.hilo_level)
        attend_dq<true>(stage, stage + kDqArr, stage + 2 * kDqArr, stage + 3 * kDqArr, e * 16,
                        p.bias2[ce_lvl[e0 + e]], c, qf, gf, lse0, lse1, D0, D1, lane, dq);
      else
        attend_dq<false>(stage, stage + kDqArr, stage + 2 * kDqArr, stage + 3 * kDqArr, e * 16,
                         p.bias2[ce_lvl[e0 + e]], c, qf, gf, lse0, lse1, D0, D1, lane, dq);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncwarp();

  const float bf = p.bias2[0];
  for (uint32_t j = 0; j < p.K; ++j) {
    if (j + 1 < p.K) load_fine(j + 1, (j + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const uint32_t base = sF + (j & 1) * kFStage;
    attend_dq<false>(base, base, base + kTile16, base + kTile16, 0, bf, c, qf, gf, lse0, lse1,
                     D0, D1, lane, dq);
    __syncwarp();
  }

  const uint32_t cc = (lane & 3) * 2;
  const uint64_t t0 = qrow0 + r, t1 = t0 + 8;
  float* d0 = p.dq + in_off + t0 * kD;
  float* d1 = p.dq + in_off + t1 * kD;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    *reinterpret_cast<float2*>(d0 + j * 8 + cc) =
        make_float2(dq[j][0] * p.scale, dq[j][1] * p.scale);
    *reinterpret_cast<float2*>(d1 + j * 8 + cc) =
        make_float2(dq[j][2] * p.scale, dq[j][3] * p.scale);
  }
}

// ---------------------------------------------------------------------------
// backward: dK/dV (key-major, one 16-key block per warp)
// ---------------------------------------------------------------------------
// Coarse levels stream 32-query chunks (rows span >= 256 queries), the fine
// level 16-query chunks (one fine query block); 3-stage cp.async pipeline.
constexpr int kKvWarps = 4;
constexpr int kKvKeyTiles = 4 * kTile16;  // Khi, Klo, Vhi, Vlo: 8 KB
constexpr int kKvStages = 3;
template <bool COARSE>
struct KvCfg {
  static constexpr int QC = COARSE ? 32 : 16;                 // queries per chunk
  static constexpr int QTile = QC * 128;                      // bf16 Q (or dO) tile
  static constexpr int Stage = 2 * QTile + 2 * QC * 4;        // Q, dO, lse2[QC], D[QC]
  static constexpr int WarpSmem = kKvKeyTiles + kKvStages * Stage;
  static constexpr int Smem = kKvWarps * WarpSmem;            // fine 60 KB, coarse 107 KB
  static constexpr int MinBlocks = COARSE ? 2 : 3;
};

// MODE 0: fine level; 1: coarse levels with hi-only K'/V'; 2: coarse levels
// with hi + lo.  A launch covers the coarse slots [slot_begin, slot_end).
template <int MODE>
__global__ void __launch_bounds__(kKvWarps * 32, KvCfg<(MODE > 0)>::MinBlocks)
    tc_kv_kernel(TcParams p, uint64_t tasks_per_unit, uint32_t units, uint32_t slot_begin) {
  constexpr bool COARSE = MODE > 0;
  constexpr bool use_lo = MODE == 2;
  using Cfg = KvCfg<COARSE>;
  constexpr int QC = Cfg::QC, NT = QC / 8;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * kKvWarps + warp;
  const uint32_t unit = (uint32_t)(gw / tasks_per_unit);
  uint64_t task = gw % tasks_per_unit;
  if (unit >= units) return;  // tail warps of the last CTA
  uint8_t* wbase = smem + warp * Cfg::WarpSmem;
  const uint32_t sK = smem_u32(wbase);
  const uint32_t sQs = sK + kKvKeyTiles;

  // decode (level, key block, split)
  uint32_t level = 0, slot = slot_begin, split = 0, nsplit = 1;
  uint64_t blk = task;
  if (COARSE) {
    task += p.cl_tasks[slot_begin];
    while (slot + 1 < p.ncl && task >= p.cl_tasks[slot + 1]) ++slot;
    task -= p.cl_tasks[slot];
    level = p.cl_level[slot];
    nsplit = p.cl_split[slot];
    blk = task / nsplit;
    split = (uint32_t)(task % nsplit);
  }

  const uint64_t in_off = (uint64_t)unit * p.n * kD;
  const uint64_t pyr_off = (uint64_t)unit * p.pyr_rows * kD;
  const bool top = COARSE && level == p.L && p.Le == p.L;
  const uint64_t span = top ? p.n : p.pow[level + 1];

  // query list: CSC segment rows × span, or all queries for the coarsest level
  const uint32_t* seg = nullptr;
  uint64_t seg_len = 1;
  if (!top) {
    const uint32_t* off = p.csc_off + (uint64_t)unit * p.csc_off_entries + p.csc_off_off[level];
    seg = p.csc_flat + (uint64_t)unit * p.csc_flat_entries + p.csc_flat_off[level] + off[blk];
    seg_len = off[blk + 1] - off[blk];
  }
  const uint64_t cpr = span / QC;  // chunks per row
  const uint64_t total = seg_len * cpr;
  const uint64_t c_lo = total * split / nsplit, c_hi = total * (split + 1) / nsplit;

  // key block tiles (A operands): level 0 → inputs; coarse → K'/V' hi, lo
  if (COARSE) {
    const uint64_t row0 = p.pyr_off[level] + blk * kBS;
    load_rows_async(sK, 0, p.khi + pyr_off + row0 * kD, kBS, lane, 32);
    load_rows_async(sK + 2 * kTile16, 0, p.vhi + pyr_off + row0 * kD, kBS, lane, 32);
    if (use_lo) load_rows_async(sK + kTile16, 0, p.klo + pyr_off + row0 * kD, kBS, lane, 32);
  } else {
    load_rows_async(sK, 0, p.k + in_off + blk * kBS * kD, kBS, lane, 32);
    load_rows_async(sK + 2 * kTile16, 0, p.v + in_off + blk * kBS * kD, kBS, lane, 32);
  }
  const uint64_t ro = (uint64_t)unit * p.n;
  const Block16Lane bl = block16_lane(lane);
  auto load_chunk = [&](uint64_t cidx, uint32_t stage) {
    const uint64_t row = top ? 0 : seg[cidx / cpr];
    const uint64_t t0 = row * span + (cidx % cpr) * QC;
    const uint32_t base = sQs + stage * Cfg::Stage;
#pragma unroll
    for (int h = 0; h < QC / 16; ++h) {
      load_block16_async(base + h * kTile16, p.q + in_off + (t0 + 16 * h) * kD, bl, lane);
      load_block16_async(base + Cfg::QTile + h * kTile16, p.dout + in_off + (t0 + 16 * h) * kD,
                         bl, lane);
    }
    constexpr uint32_t nv = QC / 4;  // 16 B vectors of lse2 (then of D)
    if (lane < nv)
      cp_async16(base + 2 * Cfg::QTile + lane * 16, p.lse2 + ro + t0 + lane * 4);
    else if (lane < 2 * nv)
      cp_async16(base + 2 * Cfg::QTile + QC * 4 + (lane - nv) * 16,
                 p.drow + ro + t0 + (lane - nv) * 4);
  };
  const uint64_t nchunk = c_hi - c_lo;
  if (nchunk > 0) load_chunk(c_lo, 0);
  cp_async_commit();
  if (nchunk > 1) load_chunk(c_lo + 1, 1);
  cp_async_commit();
  cp_async_wait<1>();
  __syncwarp();

  uint32_t kf[4][4], kl[4][4], vf[4][4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    lda(sK, 0, ks, lane, kf[ks]);
    lda(sK + 2 * kTile16, 0, ks, lane, vf[ks]);
    if (use_lo) lda(sK + kTile16, 0, ks, lane, kl[ks]);
  }
  float dk[8][4], dv[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) dk[j][i] = dv[j][i] = 0.f;
  const float c = p.scale * kLog2e;
  const float bias = p.bias2[level];
  const uint32_t cc = (lane & 3) * 2;

  for (uint64_t i = 0; i < nchunk; ++i) {
    const uint32_t st = (uint32_t)(i % kKvStages);
    if (i + 2 < nchunk) load_chunk(c_lo + i + 2, (uint32_t)((i + 2) % kKvStages));
    cp_async_commit();
    cp_async_wait<2>();
    __syncwarp();
    const uint32_t sq = sQs + st * Cfg::Stage;
    const uint32_t sg = sq + Cfg::QTile;
    const float* lse =
        reinterpret_cast<const float*>(wbase + kKvKeyTiles + st * Cfg::Stage + 2 * Cfg::QTile);
    const float* Dq = lse + QC;
    // S^T = K' Q^T and dP^T = V' dO^T over QC queries (NT n-tiles of 8)
    float s[NT][4], g[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = g[j][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int h = 0; h < NT / 2; ++h) {
        uint32_t b[4];
        ldb(sq, h * 16, ks, lane, b);  // Q rows as B (k = d, n = query)
        mma16816(s[2 * h], kf[ks], b[0], b[1]);
        mma16816(s[2 * h + 1], kf[ks], b[2], b[3]);
        if (use_lo) {
          mma16816(s[2 * h], kl[ks], b[0], b[1]);
          mma16816(s[2 * h + 1], kl[ks], b[2], b[3]);
        }
        ldb(sg, h * 16, ks, lane, b);  // dO rows as B
        mma16816(g[2 * h], vf[ks], b[0], b[1]);
        mma16816(g[2 * h + 1], vf[ks], b[2], b[3]);
      }
    }
    // P^T, dS^T: element (key row, query col = nt*8 + cc + e%2)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float la = lse[nt * 8 + cc], lb = lse[nt * 8 + cc + 1];
      const float da = Dq[nt * 8 + cc], db = Dq[nt * 8 + cc + 1];
      const float p0 = ex2(fmaf(s[nt][0], c, bias) - la), p1 = ex2(fmaf(s[nt][1], c, bias) - lb);
      const float p2 = ex2(fmaf(s[nt][2], c, bias) - la), p3 = ex2(fmaf(s[nt][3], c, bias) - lb);
      s[nt][0] = p0;
      s[nt][1] = p1;
      s[nt][2] = p2;
      s[nt][3] = p3;
      g[nt][0] = p0 * (g[nt][0] - da);
      g[nt][1] = p1 * (g[nt][1] - db);
      g[nt][2] = p2 * (g[nt][2] - da);
      g[nt][3] = p3 * (g[nt][3] - db);
    }
    // dV' += P^T dO, dK' += dS^T Q: k-steps of 16 queries
#pragma unroll
    for (int kk = 0; kk < NT / 2; ++kk) {
      const uint32_t ap[4] = {pack_bf16(s[2 * kk][0], s[2 * kk][1]),
                              pack_bf16(s[2 * kk][2], s[2 * kk][3]),
                              pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                              pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
      const uint32_t as[4] = {pack_bf16(g[2 * kk][0], g[2 * kk][1]),
                              pack_bf16(g[2 * kk][2], g[2 * kk][3]),
                              pack_bf16(g[2 * kk + 1][0], g[2 * kk + 1][1]),
                              pack_bf16(g[2 * kk + 1][2], g[2 * kk + 1][3])};
#pragma unroll
      for (int dn = 0; dn < 4; ++dn) {
        uint32_t b[4];
        ldb_t(sg, kk * 16, dn * 16, lane, b);  // dO as [k = query][n = d]
        mma16816(dv[2 * dn], ap, b[0], b[1]);
        mma16816(dv[2 * dn + 1], ap, b[2], b[3]);
        ldb_t(sq, kk * 16, dn * 16, lane, b);  // Q as [k = query][n = d]
        mma16816(dk[2 * dn], as, b[0], b[1]);
        mma16816(dk[2 * dn + 1], as, b[2], b[3]);
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();

  const uint32_t r = lane >> 2;
  if (COARSE && p.kv_atomic) {
    // scaled partial sums added into split 0 of the slot (zeroed by the host;
    // unordered fp32 adds: LLSA_DETERMINISTIC=1 keeps the split partials)
    const uint64_t tok_l = p.n / p.pow[level];
    float* pk = p.part + (uint64_t)unit * p.part_unit_stride + p.cl_part_off[slot];
    float* pv = pk + (uint64_t)nsplit * tok_l * kD;
    const float ck = p.cl_ck[slot], cv = p.cl_cv[slot];
    const uint64_t k0 = blk * kBS + r;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      atomicAdd(reinterpret_cast<float2*>(pk + k0 * kD + j * 8 + cc),
                make_float2(dk[j][0] * ck, dk[j][1] * ck));
      atomicAdd(reinterpret_cast<float2*>(pk + (k0 + 8) * kD + j * 8 + cc),
                make_float2(dk[j][2] * ck, dk[j][3] * ck));
      atomicAdd(reinterpret_cast<float2*>(pv + k0 * kD + j * 8 + cc),
                make_float2(dv[j][0] * cv, dv[j][1] * cv));
      atomicAdd(reinterpret_cast<float2*>(pv + (k0 + 8) * kD + j * 8 + cc),
                make_float2(dv[j][2] * cv, dv[j][3] * cv));
    }
  } else if (COARSE) {
    // raw partial sums for (slot, split): [split][token][64]
    const uint64_t tok_l = p.n / p.pow[level];
    float* pk = p.part + (uint64_t)unit * p.part_unit_stride + p.cl_part_off[slot] +
                (uint64_t)split * tok_l * kD;
    float* pv = pk + (uint64_t)nsplit * tok_l * kD;
    const uint64_t k0 = blk * kBS + r;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      *reinterpret_cast<float2*>(pk + k0 * kD + j * 8 + cc) = make_float2(dk[j][0], dk[j][1]);
      *reinterpret_cast<float2*>(pk + (k0 + 8) * kD + j * 8 + cc) =
          make_float2(dk[j][2], dk[j][3]);
      *reinterpret_cast<float2*>(pv + k0 * kD + j * 8 + cc) = make_float2(dv[j][0], dv[j][1]);
      *reinterpret_cast<float2*>(pv + (k0 + 8) * kD + j * 8 + cc) =
          make_float2(dv[j][2], dv[j][3]);
    }
  } else {
    // level 0: scale, add every coarse level's pooled-adjoint contribution
    // (already reduced and scaled into split 0 of its slot), write once.
    const uint64_t t0 = blk * kBS + r, t1 = t0 + 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dk[j][0] *= p.scale;
      dk[j][1] *= p.scale;
      dk[j][2] *= p.scale;
      dk[j][3] *= p.scale;
    }
    for (uint32_t sl = 0; sl < p.ncl; ++sl) {
      const uint32_t l = p.cl_level[sl];
      const uint64_t tok_l = p.n / p.pow[l];
      const float* gk = p.part + (uint64_t)unit * p.part_unit_stride + p.cl_part_off[sl];
      const float* gv = gk + (uint64_t)p.cl_split[sl] * tok_l * kD;
      const uint64_t u0 = t0 / p.pow[l], u1 = t1 / p.pow[l];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 k0 = *reinterpret_cast<const float2*>(gk + u0 * kD + j * 8 + cc);
        const float2 k1 = *reinterpret_cast<const float2*>(gk + u1 * kD + j * 8 + cc);
        const float2 v0 = *reinterpret_cast<const float2*>(gv + u0 * kD + j * 8 + cc);
        const float2 v1 = *reinterpret_cast<const float2*>(gv + u1 * kD + j * 8 + cc);
        dk[j][0] += k0.x;
        dk[j][1] += k0.y;
        dk[j][2] += k1.x;
        dk[j][3] += k1.y;
        dv[j][0] += v0.x;
        dv[j][1] += v0.y;
        dv[j][2] += v1.x;
        dv[j][3] += v1.y;
      }
    }
    float* dk0 = p.dk + in_off + t0 * kD;
    float* dk1 = p.dk + in_off + t1 * kD;
    float* dv0 = p.dv + in_off + t0 * kD;
    float* dv1 = p.dv + in_off + t1 * kD;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      *reinterpret_cast<float2*>(dk0 + j * 8 + cc) = make_float2(dk[j][0], dk[j][1]);
      *reinterpret_cast<float2*>(dk1 + j * 8 + cc) = make_float2(dk[j][2], dk[j][3]);
      *reinterpret_cast<float2*>(dv0 + j * 8 + cc) = make_float2(dv[j][0], dv[j][1]);
      *reinterpret_cast<float2*>(dv1 + j * 8 + cc) = make_float2(dv[j][2], dv[j][3]);
    }
  }
}

// ---------------------------------------------------------------------------
// backward: coarse dK'/dV' on the 5th-gen tensor cores (tcgen05 + TMEM)
// ---------------------------------------------------------------------------
// Task = (level l, selection row r, query slice, key group of 8 blocks).  The
// 128 keys of the group (A operands, K-major, M = 128 = one TMEM lane each)
// are attended by every query of row r (span B^(l+1)), which streams through
// a double-buffered 64-query ring (B operands).  Per tile:
//   S^T  = K' Q^T   and dP^T = V' dO^T   (hi [+ lo]), N = 64 → TMEM
//   thread = key: P^T = exp2(S^T c + b − lse2_q), dS^T = P^T∘(dP^T − D_q)
//   → bf16 smem tiles [key][q] (K-major A)
//   dV' += P^T dO,  dK' += dS^T Q   (B = dO, Q as MN-major [q][d]) → TMEM
// One elected thread issues every tcgen05.mma; completion is tracked with
// tcgen05.commit → mbarrier.  The 128×64 dK', dV' partial of the task is
// written once; rows_reduce_kernel sums them per key block over its CSC
// segment in ascending row order (deterministic, no atomics).
namespace rows {
constexpr int kKeys = 128, kQT = 64;
constexpr int kKeyTile = kKeys * 128;                // 16 KB
constexpr int kQTile = kQT * 128;                     // 8 KB
constexpr int kStage = 2 * kQTile + 2 * kQT * 4;      // Q, dO, lse2, D
constexpr int kStageAl = (kStage + 1023) & ~1023;     // 17 KB
// smem: key tiles Khi, Vhi (, Klo, Vlo) | 2 query stages | P^T | dS^T | barriers
template <bool LO>
struct Layout {
  static constexpr int kOffStage = (LO ? 4 : 2) * kKeyTile;
  static constexpr int kOffPT = kOffStage + 2 * kStageAl;      // P^T  [key][q]
  static constexpr int kOffDST = kOffPT + kKeys * kQT * 2;     // dS^T [key][q]
  static constexpr int kOffBar = kOffDST + kKeys * kQT * 2;
  static constexpr int kSmem = kOffBar + 64 + 1024;            // 131 KB / 99 KB
  static constexpr int kMinBlocks = LO ? 1 : 2;
};
constexpr uint32_t kTmemCols = 256;                   // S^T | dP^T | dK' | dV'
}  // namespace rows

template <bool LO>
__global__ void __launch_bounds__(256, rows::Layout<LO>::kMinBlocks)
    tc5_kv_rows_kernel(TcParams p, uint32_t li, uint32_t units) {
  using namespace llsa_umma;
  using namespace rows;
  using L = Layout<LO>;
  constexpr int kOffStage = L::kOffStage, kOffPT = L::kOffPT, kOffDST = L::kOffDST,
                kOffBar = L::kOffBar;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t tasks_per_unit = p.rl_tasks[li + 1] - p.rl_tasks[li];
  const uint64_t task_g = blockIdx.x;
  const uint32_t unit = (uint32_t)(task_g / tasks_per_unit);
  if (unit >= units) return;
  uint64_t task = task_g % tasks_per_unit;
  const uint32_t level = p.rl_level[li];
  const uint32_t slices = p.rl_slices[li];
  const uint32_t group = (uint32_t)(task % p.groups);
  const uint64_t rs = task / p.groups;
  const uint32_t slice = (uint32_t)(rs % slices);
  const uint64_t row = rs / slices;
  const uint64_t span = p.pow[level + 1];
  const uint64_t q_begin = row * span + (uint64_t)slice * p.rl_qs[li];
  const uint32_t ntiles = (uint32_t)(p.rl_qs[li] / kQT);

  const uint32_t sbase = smem_u32(smem);
  const uint32_t sKhi = sbase, sVhi = sKhi + kKeyTile, sKlo = sVhi + kKeyTile,
                 sVlo = sKlo + kKeyTile;
  const uint32_t sPT = sbase + kOffPT, sDST = sbase + kOffDST;
  const uint32_t mbar_s = sbase + kOffBar, mbar_kv = mbar_s + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kOffBar + 16);

  const uint64_t in_off = (uint64_t)unit * p.n * kD;
  const uint64_t pyr_off = (uint64_t)unit * p.pyr_rows * kD;
  const uint64_t ro = (uint64_t)unit * p.n;
  const uint32_t* trow = p.tables + (uint64_t)unit * p.table_entries + p.table_off[level] +
                         row * p.K + group * 8;
  const uint64_t nblk = p.n / p.pow[level + 1];

  // key group: 8 selected blocks × 16 rows of K', V' (hi [, lo])
  for (uint32_t i = tid; i < 8 * 16 * 8; i += blockDim.x) {
    const uint32_t key = i >> 3, ch = i & 7;
    uint32_t b = group * 8 + (key >> 4) < p.K ? trow[key >> 4] : 0u;  // dummy tail keys
    if (b >= nblk) b = 0;
    const uint64_t grow = p.pyr_off[level] + (uint64_t)b * kBS + (key & 15);
    const uint64_t src = pyr_off + grow * kD + ch * 8;
    cp_async16(sKhi + swz(key, ch), p.khi + src);
    cp_async16(sVhi + swz(key, ch), p.vhi + src);
    if (LO) {
      cp_async16(sKlo + swz(key, ch), p.klo + src);
      cp_async16(sVlo + swz(key, ch), p.vlo + src);
    }
  }
  auto load_tile = [&](uint32_t j, uint32_t stage) {
    const uint64_t t0 = q_begin + (uint64_t)j * kQT;
    const uint32_t base = sbase + kOffStage + stage * kStageAl;
    load_rows_fast<kQT, 256>(base, p.q + in_off + t0 * kD, tid);
    load_rows_fast<kQT, 256>(base + kQTile, p.dout + in_off + t0 * kD, tid);
    if (tid < 16) cp_async16(base + 2 * kQTile + tid * 16, p.lse2 + ro + t0 + tid * 4);
    else if (tid < 32)
      cp_async16(base + 2 * kQTile + kQT * 4 + (tid - 16) * 16, p.drow + ro + t0 + (tid - 16) * 4);
  };
  load_tile(0, 0);
  cp_async_commit();

  if (warp == 0) tmem_alloc(smem_u32(tslot), kTmemCols);
  if (tid == 0) {
    mbar_init(mbar_s, 1);
    mbar_init(mbar_kv, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tP = tmem + 64, tDK = tmem + 128, tDV = tmem + 192;
  const uint32_t idesc_s = idesc_bf16(128, kQT, false, false);  // A, B K-major
  const uint32_t idesc_kv = idesc_bf16(128, kD, false, true);   // B MN-major
  const float c = p.scale * kLog2e;
  const float bias = p.bias2[level];
  const uint32_t krow = 32 * (warp & 3) + lane;   // this thread's key (TMEM lane)
  const uint32_t qhalf = warp >> 2;               // query columns [32 qhalf, +32)
  const uint32_t lane_off = (32u * (warp & 3)) << 16;
  uint32_t kv_done = 0;
  auto ensure_kv = [&](uint32_t n) {
    while (kv_done < n) {
      mbar_wait(mbar_kv, kv_done & 1);
      ++kv_done;
    }
  };

  for (uint32_t j = 0; j < ntiles; ++j) {
    const uint32_t st = j & 1;
    if (j + 1 < ntiles) {
      ensure_kv(j);  // tile j-1's MMAs read stage (j+1)&1
      load_tile(j + 1, st ^ 1);
    }
    cp_async_commit();
    cp_async_wait<1>();
    fence_proxy_async();
    __syncthreads();
    const uint32_t sQ = sbase + kOffStage + st * kStageAl, sG = sQ + kQTile;
    if (tid == 0) {
      fence_after();
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t bq = desc_kmajor(sQ + ks * kKStepKMajor);
        const uint64_t bg = desc_kmajor(sG + ks * kKStepKMajor);
        mma_bf16(tS, desc_kmajor(sKhi + ks * kKStepKMajor), bq, idesc_s, ks > 0);
        if (LO) mma_bf16(tS, desc_kmajor(sKlo + ks * kKStepKMajor), bq, idesc_s, 1);
        mma_bf16(tP, desc_kmajor(sVhi + ks * kKStepKMajor), bg, idesc_s, ks > 0);
        if (LO) mma_bf16(tP, desc_kmajor(sVlo + ks * kKStepKMajor), bg, idesc_s, 1);
      }
      commit(mbar_s);
    }
    mbar_wait(mbar_s, j & 1);
    fence_after();
    ensure_kv(j);  // P^T / dS^T tiles free (tile j-1's dV/dK done)
    uint32_t sv[32], pv[32];
    tmem_ld32(tS + lane_off + qhalf * 32, sv);
    tmem_ld32(tP + lane_off + qhalf * 32, pv);
    tmem_ld_wait();
    const float* lse = reinterpret_cast<const float*>(smem + kOffStage + st * kStageAl + 2 * kQTile);
    const float* Dq = lse + kQT;
#pragma unroll
    for (int c8 = 0; c8 < 4; ++c8) {
      uint32_t pk[4], dk4[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float pe[2], de[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = c8 * 8 + h * 2 + e;
          const int q = qhalf * 32 + i;
          const float pr = ex2(fmaf(__uint_as_float(sv[i]), c, bias) - lse[q]);
          pe[e] = pr;
          de[e] = pr * (__uint_as_float(pv[i]) - Dq[q]);
        }
        pk[h] = pack_bf16(pe[0], pe[1]);
        dk4[h] = pack_bf16(de[0], de[1]);
      }
      const uint32_t chunk = qhalf * 4 + c8;
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sPT + swz(krow, chunk)),
                   "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]));
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sDST + swz(krow, chunk)),
                   "r"(dk4[0]), "r"(dk4[1]), "r"(dk4[2]), "r"(dk4[3]));
    }
    fence_proxy_async();
    fence_before();
    __syncthreads();
    if (tid == 0) {
      fence_after();
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {  // K = 64 queries
        mma_bf16(tDV, desc_kmajor(sPT + ks * kKStepKMajor),
                 desc_mnmajor(sG + ks * kKStepMNMajor, 8192), idesc_kv, (j | ks) > 0);
        mma_bf16(tDK, desc_kmajor(sDST + ks * kKStepKMajor),
                 desc_mnmajor(sQ + ks * kKStepMNMajor, 8192), idesc_kv, (j | ks) > 0);
      }
      commit(mbar_kv);
    }
  }
  cp_async_wait<0>();
  ensure_kv(ntiles);
  fence_after();
  // raw partial sums of this task, transposed: [64 d][128 keys] dK', then
  // dV' (a warp's 32 keys of one d column are one 128-byte store)
  const uint64_t pidx = (row * slices + slice) * p.groups + group;
  float* dst = p.rpart + (uint64_t)unit * p.rpart_unit_stride + p.rl_part_off[li] +
               pidx * (2 * kKeys * kD) + (qhalf ? kKeys * kD : 0) + krow;
  const uint32_t tsrc = (qhalf ? tDV : tDK) + lane_off;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t r[32];
    tmem_ld32(tsrc + half * 32, r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) dst[(uint64_t)(half * 32 + i) * kKeys] = __uint_as_float(r[i]);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// Per level-l key block b: Σ over the rows r of its CSC segment (ascending)
// and over query slices of the partial rows of b's position in row r, scaled
// by the pooling-adjoint coefficient, into split 0 of the level's slot (the
// layout tc_kv_kernel<fine> consumes).  One CTA per (unit, level, block);
// thread = (token, 4 columns), so every partial row is read with full
// 128-bit coalescing and ~2·len·slices independent loads in flight.
__global__ void __launch_bounds__(256) rows_reduce_kernel(TcParams p, uint32_t units,
                                                          uint64_t blocks_per_unit) {
  const uint64_t cta = blockIdx.x;
  const uint32_t unit = (uint32_t)(cta / blocks_per_unit);
  if (unit >= units) return;
  uint64_t w = cta % blocks_per_unit;
  uint32_t li = 0;
  uint64_t base_w = 0;
  for (; li < p.rl_count; ++li) {
    const uint64_t nb = p.n / p.pow[p.rl_level[li] + 1];
    if (w < base_w + nb) break;
    base_w += nb;
  }
  if (li >= p.rl_count) return;
  const uint32_t level = p.rl_level[li];
  const uint64_t b = w - base_w;
  const uint32_t slices = p.rl_slices[li], groups = p.rl_groups[li];
  // the coarsest level (rl_top) is one row that holds every block at its
  // own position; the selected levels find their rows through the CSC
  const bool top = p.rl_top[li] != 0;
  const uint32_t* off =
      top ? nullptr : p.csc_off + (uint64_t)unit * p.csc_off_entries + p.csc_off_off[level];
  const uint32_t* seg =
      top ? nullptr
          : p.csc_flat + (uint64_t)unit * p.csc_flat_entries + p.csc_flat_off[level] + off[b];
  const uint32_t len = top ? 1u : off[b + 1] - off[b];
  const uint32_t* tab = p.tables + (uint64_t)unit * p.table_entries +
                        (top ? 0 : p.table_off[level]);
  const float* part = p.rpart + (uint64_t)unit * p.rpart_unit_stride + p.rl_part_off[li];
  // thread = (token, 4 d columns) with the token fastest: the partials are
  // [d][key], so 16 neighbouring lanes read 64 contiguous bytes per column
  const uint32_t tok = threadIdx.x & 15, c4 = (threadIdx.x >> 4) * 4;
  // the segment's (row, position of b in the row) pairs are resolved by one
  // thread each into smem first, so the summation below issues independent
  // loads instead of a seg → table → partial chain per row
  __shared__ uint32_t s_row[256], s_pos[256];
  float4 ak = make_float4(0.f, 0.f, 0.f, 0.f), av = ak;
  for (uint32_t base = 0; base < len; base += 256) {
    const uint32_t nrow = min(256u, len - base);
    if (threadIdx.x < nrow) {
      uint32_t r = 0, pos = (uint32_t)b;
      if (!top) {
        r = seg[base + threadIdx.x];
        pos = 0;
        for (uint32_t j = 0; j < p.K; ++j)
          if (tab[(uint64_t)r * p.K + j] == b) pos = j;
      }
      s_row[threadIdx.x] = r;
      s_pos[threadIdx.x] = pos;
    }
    __syncthreads();
    for (uint32_t si = 0; si < nrow; ++si) {
      const uint32_t r = s_row[si], pos = s_pos[si];
      const uint32_t g = pos / 8, key = (pos % 8) * kBS + tok;
      const float* src0 = part + ((uint64_t)r * slices * groups + g) * (2 * rows::kKeys * kD) +
                          (uint64_t)c4 * rows::kKeys + key;
#pragma unroll 4
      for (uint32_t s = 0; s < slices; ++s) {
        const float* src = src0 + (uint64_t)s * groups * (2 * rows::kKeys * kD);
        const float* srv = src + rows::kKeys * kD;
        const float4 x = make_float4(__ldg(src), __ldg(src + rows::kKeys),
                                     __ldg(src + 2 * rows::kKeys), __ldg(src + 3 * rows::kKeys));
        const float4 y = make_float4(__ldg(srv), __ldg(srv + rows::kKeys),
                                     __ldg(srv + 2 * rows::kKeys), __ldg(srv + 3 * rows::kKeys));
        ak.x += x.x;
        ak.y += x.y;
        ak.z += x.z;
        ak.w += x.w;
        av.x += y.x;
        av.y += y.y;
        av.z += y.z;
        av.w += y.w;
      }
    }
    __syncthreads();
  }
  // slot of this level in the coarse-slot table (levels 1..lim-1 come first)
  uint32_t sl = 0;
  while (sl < p.ncl && p.cl_level[sl] != level) ++sl;
  const uint64_t tok_l = p.n / p.pow[level];
  float* gk = p.part + (uint64_t)unit * p.part_unit_stride + p.cl_part_off[sl];
  float* gv = gk + (uint64_t)p.cl_split[sl] * tok_l * kD;
  // through smem, so the block's 16 output rows are written row-contiguous
  __shared__ float4 s_out[2][16][17];
  const float ck = p.cl_ck[sl], cv = p.cl_cv[sl];
  s_out[0][tok][c4 / 4] = make_float4(ak.x * ck, ak.y * ck, ak.z * ck, ak.w * ck);
  s_out[1][tok][c4 / 4] = make_float4(av.x * cv, av.y * cv, av.z * cv, av.w * cv);
  __syncthreads();
  const uint32_t orow = threadIdx.x >> 4, ocol = threadIdx.x & 15;
  const uint64_t t = b * kBS + orow;
  reinterpret_cast<float4*>(gk + t * kD)[ocol] = s_out[0][orow][ocol];
  reinterpret_cast<float4*>(gv + t * kD)[ocol] = s_out[1][orow][ocol];
}

// ---------------------------------------------------------------------------
// backward: dq over the coarse keys on tcgen05 (query-major, M = 128 queries)
// ---------------------------------------------------------------------------
// The CTA's 128 queries share their coarse set (levels 1..L), streamed in
// chunks of up to 4 entries (64 keys, double-buffered cp.async):
//   S = Q K'^T, dP = dO V'^T (hi [+ lo]) → TMEM (N = 16·entries)
//   thread = query row: dS = P∘(dP − D), P = exp2(S c + b − lse2) → bf16 tile
//   dQ += dS K'_hi (A = dS K-major, B = K' MN-major) → TMEM, whole tile
// and finally dq[t] += scale · dQ (the fine part was written by tc_dq_kernel
// with the coarse set skipped, which also produced D and lse2).
namespace dqc {
constexpr int kArr = 64 * 128;                 // one 64-key array tile: 8 KB
constexpr int kStage = 4 * kArr;               // Khi, Vhi, Klo, Vlo
constexpr int kOffQ = 0, kOffG = 16384, kOffStage = 32768;
constexpr int kOffDS = kOffStage + 2 * kStage;  // 96 KB
constexpr int kOffEnt = kOffDS + 16384;         // ce_row[64], ce_lvl[64]
constexpr int kOffBar = kOffEnt + 2 * kMaxCoarse * 4;
constexpr int kSmem = kOffBar + 64;             // 112.6 KB: 2 CTAs / SM
constexpr uint32_t kTmemCols = 256;             // S | dP | dQ
}  // namespace dqc

__global__ void __launch_bounds__(256, 2) tc5_dq_coarse_kernel(TcParams p) {
  using namespace llsa_umma;
  using namespace dqc;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t unit = blockIdx.y;
  const uint64_t q0 = (uint64_t)blockIdx.x * kTileQ;
  const uint64_t fb0 = q0 / kBS;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sQ = sbase + kOffQ, sG = sbase + kOffG, sDS = sbase + kOffDS;
  uint32_t* ce_row = reinterpret_cast<uint32_t*>(smem + kOffEnt);
  uint32_t* ce_lvl = ce_row + kMaxCoarse;
  const uint32_t mbar_s = sbase + kOffBar, mbar_q = mbar_s + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kOffBar + 16);
  const uint64_t in_off = (uint64_t)unit * p.n * kD;
  const uint64_t pyr_off = (uint64_t)unit * p.pyr_rows * kD;
  const uint32_t* tab = p.tables + (uint64_t)unit * p.table_entries;
  const bf16* arrays[4] = {p.khi, p.vhi, p.klo, p.vlo};

  for (uint32_t e = tid; e < p.nce; e += blockDim.x) {
    uint32_t l, r;
    coarse_entry(p, tab, fb0, e, l, r);
    ce_row[e] = r;
    ce_lvl[e] = l;
  }
  __syncthreads();
  const uint32_t nchunks = (p.nce + 3) / 4;
  auto chunk_lo = [&](uint32_t ch) {
    const uint32_t e0 = ch * 4, ne = min(4u, p.nce - e0);
    bool lo = false;
    for (uint32_t e = 0; e < ne; ++e) lo |= ce_lvl[e0 + e] >= p.hilo_level;
    return lo;
  };
  auto load_chunk = [&](uint32_t ch, uint32_t stage) {
    const uint32_t e0 = ch * 4, ne = min(4u, p.nce - e0);
    load_coarse_chunk(sbase + kOffStage + stage * kStage, kArr, ce_row, e0, ne, arrays,
                      chunk_lo(ch) ? 4 : 2, pyr_off, tid, blockDim.x);
  };
  load_rows_async(sQ, 0, p.q + in_off + q0 * kD, kTileQ, tid, blockDim.x);
  load_rows_async(sG, 0, p.dout + in_off + q0 * kD, kTileQ, tid, blockDim.x);
  load_chunk(0, 0);
  cp_async_commit();

  if (warp == 0) tmem_alloc(smem_u32(tslot), kTmemCols);
  if (tid == 0) {
    mbar_init(mbar_s, 1);
    mbar_init(mbar_q, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tP = tmem + 64, tQ = tmem + 128;
  const uint32_t row = 32 * (warp & 3) + lane;  // this thread's query (TMEM lane)
  const uint32_t chalf = warp >> 2;             // key columns [32 chalf, +32)
  const uint32_t lane_off = (32u * (warp & 3)) << 16;
  const uint64_t ro = (uint64_t)unit * p.n + q0 + row;
  const float lse = p.lse2[ro], Drow = p.drow[ro];
  const float c = p.scale * kLog2e;
  uint32_t q_done = 0;
  auto ensure_q = [&](uint32_t n) {
    while (q_done < n) {
      mbar_wait(mbar_q, q_done & 1);
      ++q_done;
    }
  };

  for (uint32_t ch = 0; ch < nchunks; ++ch) {
    const uint32_t st = ch & 1;
    if (ch + 1 < nchunks) {
      ensure_q(ch);  // dQ MMA of chunk ch-1 read stage (ch+1)&1
      load_chunk(ch + 1, st ^ 1);
    }
    cp_async_commit();
    cp_async_wait<1>();
    fence_proxy_async();
    __syncthreads();
    const uint32_t e0 = ch * 4, ne = min(4u, p.nce - e0);
    const uint32_t stage = sbase + kOffStage + st * kStage;
    const uint32_t sKhi = stage, sVhi = stage + kArr, sKlo = stage + 2 * kArr,
                   sVlo = stage + 3 * kArr;
    const bool lo = chunk_lo(ch);
    if (tid == 0) {
      fence_after();
      const uint32_t idesc = idesc_bf16(128, 16 * ne, false, false);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t aq = desc_kmajor(sQ + ks * kKStepKMajor);
        const uint64_t ag = desc_kmajor(sG + ks * kKStepKMajor);
        mma_bf16(tS, aq, desc_kmajor(sKhi + ks * kKStepKMajor), idesc, ks > 0);
        mma_bf16(tP, ag, desc_kmajor(sVhi + ks * kKStepKMajor), idesc, ks > 0);
        if (lo) {
          mma_bf16(tS, aq, desc_kmajor(sKlo + ks * kKStepKMajor), idesc, 1);
          mma_bf16(tP, ag, desc_kmajor(sVlo + ks * kKStepKMajor), idesc, 1);
        }
      }
      commit(mbar_s);
    }
    mbar_wait(mbar_s, ch & 1);
    fence_after();
    ensure_q(ch);  // previous dQ MMA finished reading the dS tile
    if (chalf * 32 < 16 * ne) {
      uint32_t sv[32], pv[32];
      tmem_ld32(tS + lane_off + chalf * 32, sv);
      tmem_ld32(tP + lane_off + chalf * 32, pv);
      tmem_ld_wait();
      const float b0 = p.bias2[ce_lvl[e0 + 2 * chalf]];
      const float b1 = 2 * chalf + 1 < ne ? p.bias2[ce_lvl[e0 + 2 * chalf + 1]] : 0.f;
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint32_t pk[4];
        const float bias = c8 < 2 ? b0 : b1;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float de[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = c8 * 8 + h * 2 + e;
            const float pr = ex2(fmaf(__uint_as_float(sv[i]), c, bias) - lse);
            de[e] = pr * (__uint_as_float(pv[i]) - Drow);
          }
          pk[h] = pack_bf16(de[0], de[1]);
        }
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sDS + swz(row, chalf * 4 + c8)),
                     "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]));
      }
    }
    fence_proxy_async();
    fence_before();
    __syncthreads();
    if (tid == 0) {
      fence_after();
      const uint32_t idesc_q = idesc_bf16(128, kD, false, true);
      for (uint32_t ks = 0; ks < ne; ++ks)
        mma_bf16(tQ, desc_kmajor(sDS + ks * kKStepKMajor),
                 desc_mnmajor(sKhi + ks * kKStepMNMajor, 8192), idesc_q, (ch | ks) > 0);
      commit(mbar_q);
    }
  }
  cp_async_wait<0>();
  ensure_q(nchunks);
  fence_after();
  {
    uint32_t r[32];
    tmem_ld32(tQ + lane_off + chalf * 32, r);
    tmem_ld_wait();
    float* d = p.dq + in_off + (q0 + row) * kD + chalf * 32;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 v = *reinterpret_cast<float4*>(d + i);
      v.x += __uint_as_float(r[i]) * p.scale;
      v.y += __uint_as_float(r[i + 1]) * p.scale;
      v.z += __uint_as_float(r[i + 2]) * p.scale;
      v.w += __uint_as_float(r[i + 3]) * p.scale;
      *reinterpret_cast<float4*>(d + i) = v;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// backward: coarse dq — persistent, warp-specialised tcgen05 pipeline
// ---------------------------------------------------------------------------
// One CTA per SM walks query tiles (128 queries, all units).  Roles:
//   warp 4 (1 lane)  TMA producer: Q/dO tile → 2-stage ring; the coarse
//                    entries' K'/V' (16-row boxes, hi [+ lo]) → 3-stage ring
//   warp 5 (1 lane)  MMA issuer: S, dP of chunk c into TMEM buffer c&1, then
//                    dQ += dS·K' of chunk c-1 into the tile's TMEM dQ buffer
//   warps 0-3        thread = query row: dS from S, dP (TMEM) → bf16 smem,
//                    then the tile epilogue dq[t] += scale·dQ
// Every hand-off is an mbarrier (TMA complete_tx, tcgen05.commit or 128
// thread arrivals), so loads, MMAs and the elementwise work of consecutive
// chunks and tiles overlap.
struct TmaMaps {
  CUtensorMap q, g, khi, vhi, klo, vlo, o;
};

namespace dqp {
constexpr int kQStage = 2 * kTileQ * 128;  // Q + dO: 32 KB
constexpr int kArr = 64 * 128;             // 64 keys × 64 d bf16
constexpr int kCStage = 4 * kArr;          // Khi, Vhi, Klo, Vlo: 32 KB
constexpr int kOffQ = 0;
constexpr int kOffC = 2 * kQStage;         // 64 KB
constexpr int kOffDS = kOffC + 3 * kCStage;  // 160 KB
constexpr int kOffBar = kOffDS + 2 * 16384;  // 192 KB
enum { CFULL = 0, CEMPTY = 3, QFULL = 6, QEMPTY = 8, SREADY = 10, TFREE = 12, DSREADY = 14,
       DSFREE = 16, DQREADY = 18, DQFREE = 20, NBAR = 22 };
constexpr int kSmem = kOffBar + NBAR * 8 + 16;
constexpr uint32_t kTmemCols = 512;  // S/dP x2 (256) + dQ x2 (128)
}  // namespace dqp

__device__ __forceinline__ uint32_t entry_level(const TcParams& p, uint32_t e) {
  e += p.ce_base;
  const uint32_t ksel = p.K * (p.lim - 1);
  return e < ksel ? 1 + e / p.K : p.L;
}

__global__ void __launch_bounds__(320, 1)
    tc5_dq_pipe_kernel(const __grid_constant__ TcParams p, const __grid_constant__ TmaMaps m,
                       uint32_t units) {
  using namespace llsa_umma;
  using namespace dqp;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  auto bar = [&](int i) { return sbase + kOffBar + 8u * i; };
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kOffBar + NBAR * 8);
  const uint64_t tpu = p.n / kTileQ;
  const uint64_t total = tpu * units;
  const uint32_t nce = p.nce, nch = (nce + 3) / 4;
  auto chunk_ne = [&](uint32_t ch) { return min(4u, nce - ch * 4); };
  auto chunk_lo = [&](uint32_t ch) {
    bool lo = false;
    for (uint32_t e = ch * 4; e < ch * 4 + chunk_ne(ch); ++e)
      lo |= entry_level(p, e) >= p.hilo_level;
    return lo;
  };

  if (warp == 0) tmem_alloc(smem_u32(tslot), kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(bar(CFULL + i), 1);
      mbar_init(bar(CEMPTY + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(QFULL + i), 1);
      mbar_init(bar(QEMPTY + i), 1);
      mbar_init(bar(SREADY + i), 1);
      mbar_init(bar(TFREE + i), 256);
      mbar_init(bar(DSREADY + i), 256);
      mbar_init(bar(DSFREE + i), 1);
      mbar_init(bar(DQREADY + i), 1);
      mbar_init(bar(DQFREE + i), 256);
    }
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    // The whole warp resolves the tile's coarse rows in parallel (one table
    // latency per tile, lanes hold entries lane and lane+32); lane 0 issues
    // the TMA copies.
    if (lane == 0) {
      prefetch_map(&m.q);
      prefetch_map(&m.g);
      prefetch_map(&m.khi);
      prefetch_map(&m.vhi);
      prefetch_map(&m.klo);
      prefetch_map(&m.vlo);
    }
    uint32_t c = 0, i = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint64_t q0 = (id % tpu) * kTileQ;
      const uint32_t* tab = p.tables + (uint64_t)unit * p.table_entries;
      const uint64_t fb0 = q0 / kBS;
      uint32_t myrow[2] = {0, 0};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const uint32_t e = lane + 32 * k;
        if (e < nce) {
          uint32_t l;
          coarse_entry(p, tab, fb0, e, l, myrow[k]);
        }
      }
      const uint32_t qs = i & 1;
      if (lane == 0) {
        if (i >= 2) mbar_wait(bar(QEMPTY + qs), ((i >> 1) - 1) & 1);
        const uint32_t qdst = sbase + kOffQ + qs * kQStage;
        mbar_expect_tx(bar(QFULL + qs), kQStage);
        tma_load_2d(qdst, &m.q, 0, (int)(unit * p.n + q0), bar(QFULL + qs));
        tma_load_2d(qdst + kTileQ * 128, &m.g, 0, (int)(unit * p.n + q0), bar(QFULL + qs));
      }
      for (uint32_t ch = 0; ch < nch; ++ch, ++c) {
        const uint32_t s = c % 3;
        const uint32_t ne = chunk_ne(ch);
        const bool lo = chunk_lo(ch);
        uint32_t rows4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t ei = ch * 4 + e;
          const uint32_t v0 = __shfl_sync(0xffffffffu, myrow[0], ei & 31);
          const uint32_t v1 = __shfl_sync(0xffffffffu, myrow[1], ei & 31);
          rows4[e] = ei < 32 ? v0 : v1;
        }
        if (lane == 0) {
          if (c >= 3) mbar_wait(bar(CEMPTY + s), ((c / 3) - 1) & 1);
          const uint32_t dst = sbase + kOffC + s * kCStage;
          mbar_expect_tx(bar(CFULL + s), ne * (lo ? 4 : 2) * kBS * 128);
          for (uint32_t e = 0; e < ne; ++e) {
            const int y = (int)((uint64_t)unit * p.pyr_rows + rows4[e]);
            tma_load_2d(dst + e * 2048, &m.khi, 0, y, bar(CFULL + s));
            tma_load_2d(dst + kArr + e * 2048, &m.vhi, 0, y, bar(CFULL + s));
            if (lo) {
              tma_load_2d(dst + 2 * kArr + e * 2048, &m.klo, 0, y, bar(CFULL + s));
              tma_load_2d(dst + 3 * kArr + e * 2048, &m.vlo, 0, y, bar(CFULL + s));
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc_q = idesc_bf16(128, kD, false, true);
      struct Prev {
        uint32_t c, s, ne, tp, first, last, ti;
      } pv{};
      bool have = false;
      auto do_dq = [&](const Prev& x) {
        const uint32_t b = x.c & 1;
        mbar_wait(bar(DSREADY + b), (x.c >> 1) & 1);
        if (x.first && x.ti >= 2) mbar_wait(bar(DQFREE + x.tp), ((x.ti >> 1) - 1) & 1);
        fence_after();
        const uint32_t sds = sbase + kOffDS + b * 16384;
        const uint32_t khi = sbase + kOffC + x.s * kCStage;
        const uint32_t tq = tmem + 256 + x.tp * 64;
        for (uint32_t ks = 0; ks < x.ne; ++ks)
          mma_bf16(tq, desc_kmajor(sds + ks * kKStepKMajor),
                   desc_mnmajor(khi + ks * kKStepMNMajor, 8192), idesc_q,
                   (x.first && ks == 0) ? 0u : 1u);
        commit(bar(CEMPTY + x.s));
        commit(bar(DSFREE + b));
        if (x.last) commit(bar(DQREADY + x.tp));
      };
      uint32_t c = 0, i = 0;
      for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
        const uint32_t qs = i & 1;
        mbar_wait(bar(QFULL + qs), (i >> 1) & 1);
        const uint32_t sq = sbase + kOffQ + qs * kQStage, sg = sq + kTileQ * 128;
        for (uint32_t ch = 0; ch < nch; ++ch, ++c) {
          const uint32_t s = c % 3, b = c & 1;
          mbar_wait(bar(CFULL + s), (c / 3) & 1);
          if (c >= 2) mbar_wait(bar(TFREE + b), ((c >> 1) - 1) & 1);
          fence_after();
          const uint32_t ne = chunk_ne(ch);
          const bool lo = chunk_lo(ch);
          const uint32_t idesc = idesc_bf16(128, 16 * ne, false, false);
          const uint32_t st = sbase + kOffC + s * kCStage;
          const uint32_t tS = tmem + b * 128, tP = tS + 64;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t aq = desc_kmajor(sq + ks * kKStepKMajor);
            const uint64_t ag = desc_kmajor(sg + ks * kKStepKMajor);
            mma_bf16(tS, aq, desc_kmajor(st + ks * kKStepKMajor), idesc, ks > 0);
            mma_bf16(tP, ag, desc_kmajor(st + kArr + ks * kKStepKMajor), idesc, ks > 0);
            if (lo) {
              mma_bf16(tS, aq, desc_kmajor(st + 2 * kArr + ks * kKStepKMajor), idesc, 1);
              mma_bf16(tP, ag, desc_kmajor(st + 3 * kArr + ks * kKStepKMajor), idesc, 1);
            }
          }
          commit(bar(SREADY + b));
          if (ch + 1 == nch) commit(bar(QEMPTY + qs));
          if (have) do_dq(pv);
          pv = Prev{c, s, ne, qs, ch == 0 ? 1u : 0u, ch + 1 == nch ? 1u : 0u, i};
          have = true;
        }
      }
      if (have) do_dq(pv);
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    // warp w: TMEM lanes (queries) 32(w&3).., key columns [32(w>>2), +32)
    const uint32_t row = 32 * (warp & 3) + lane, h = warp >> 2;
    const uint32_t lane_off = (32u * (warp & 3)) << 16;
    const float c2 = p.scale * kLog2e;
    uint32_t c = 0, i = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint64_t q0 = (id % tpu) * kTileQ;
      const uint64_t ro = (uint64_t)unit * p.n + q0 + row;
      const float lse = p.lse2[ro], Drow = p.drow[ro];
      float* d = p.dq + ro * kD + h * 32;
      float4 acc[8];  // this row's dq columns, prefetched for the epilogue
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = reinterpret_cast<const float4*>(d)[k];
      for (uint32_t ch = 0; ch < nch; ++ch, ++c) {
        const uint32_t b = c & 1;
        mbar_wait(bar(SREADY + b), (c >> 1) & 1);
        fence_after();
        uint32_t sv[32], gv[32];
        tmem_ld32(tmem + lane_off + b * 128 + h * 32, sv);
        tmem_ld32(tmem + lane_off + b * 128 + 64 + h * 32, gv);
        tmem_ld_wait();
        fence_before();
        mbar_arrive(bar(TFREE + b));
        if (c >= 2) mbar_wait(bar(DSFREE + b), ((c >> 1) - 1) & 1);
        const uint32_t ne = chunk_ne(ch);
        const uint32_t sds = sbase + kOffDS + b * 16384;
#pragma unroll
        for (int ee = 0; ee < 2; ++ee) {
          const uint32_t e = 2 * h + ee;
          if (e < ne) {
            const float bias = p.bias2[entry_level(p, ch * 4 + e)];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t pk[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int i0 = ee * 16 + half * 8 + k * 2;
                const float p0 = ex2(fmaf(__uint_as_float(sv[i0]), c2, bias) - lse);
                const float p1 = ex2(fmaf(__uint_as_float(sv[i0 + 1]), c2, bias) - lse);
                pk[k] = pack_bf16(p0 * (__uint_as_float(gv[i0]) - Drow),
                                  p1 * (__uint_as_float(gv[i0 + 1]) - Drow));
              }
              asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(
                               sds + swz(row, e * 2 + half)),
                           "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]));
            }
          }
        }
        fence_proxy_async();
        mbar_arrive(bar(DSREADY + b));
      }
      // tile epilogue: dq[t] += scale · dQ
      const uint32_t tp = i & 1;
      mbar_wait(bar(DQREADY + tp), (i >> 1) & 1);
      fence_after();
      uint32_t r0[32];
      tmem_ld32(tmem + lane_off + 256 + tp * 64 + h * 32, r0);
      tmem_ld_wait();
      fence_before();
      mbar_arrive(bar(DQFREE + tp));
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float4 v = acc[k];
        v.x += __uint_as_float(r0[4 * k]) * p.scale;
        v.y += __uint_as_float(r0[4 * k + 1]) * p.scale;
        v.z += __uint_as_float(r0[4 * k + 2]) * p.scale;
        v.w += __uint_as_float(r0[4 * k + 3]) * p.scale;
        reinterpret_cast<float4*>(d)[k] = v;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// forward — persistent, warp-specialised: coarse keys on tcgen05 / TMEM,
// fine blocks on mma.sync, running concurrently on separate warps
// ---------------------------------------------------------------------------
// One CTA per SM walks 128-query tiles.  The tile's coarse set (levels 1..L,
// shared by its 8 fine query blocks; <= 24 entries = 384 keys) is a dense
// M = 128 problem: its whole score block S = Q K'^T lives in TMEM and its
// softmax is exact (two passes over TMEM: row max, then P), so no TMEM
// accumulator is ever rescaled.  The fine part (each fine query block's own
// K gathered level-0 blocks) is block-diagonal and runs on mma.sync.  The
// two halves are independent softmax partitions merged at the end
// (m = max(m_f, m_c), O = (O_f 2^(m_f-m) + O_c 2^(m_c-m)) / l).  Roles:
//   warp 0 (1 lane)  TMA producer: Q tile; coarse K' chunks (hi [+ lo],
//                    64 keys) → 3-stage ring
//   warp 2 (1 lane)  TMA producer: coarse V' chunks → 2-stage ring
//   warp 1 (1 lane)  MMA issuer: S chunks into TMEM; O_c += P·V'_hi chunk by
//                    chunk as the coarse warps publish P
//   warps 3-6        coarse softmax, thread = query row (its TMEM lane):
//                    row max over S, P = exp2(.) → bf16 smem ring (K-major
//                    A operand of the PV MMA), then O_c (raw) → out, and
//                    (m_c, l_c) → smem
//   warps 7-14       fine part, warp 7+w = fine query block w: its K blocks
//                    streamed by a 3-stage cp.async ring, online softmax in
//                    registers; then merges with the coarse partial in `out`
// The producer and MMA warps take the lowest warp ids: the scheduler favours
// older warps, and starving the single-thread roles stalls the whole tile.
// Replaces P/src/attention.cpp:166-214 for the tensor-core shapes.
// Fine part of the forward (one 16-query fine block x one 16-key block) with
// a lazily rescaled online softmax: the running reference max m only moves
// when a block's max exceeds it by more than kLazy (log2 units), so P stays
// <= 2^kLazy and the O rescale (32 FMUL) is skipped for most blocks; the
// true row max is tracked separately for ForwardState.  l accumulates on the
// tensor core (P times a ones column).
struct FineState {
  float o[8][4];
  float lo[4];           // l: this lane's partial row sums of rows r, r + 8 in [0], [2]
                         // (quad-reduced once per tile)
  float m[2], mt[2];     // reference max, true max (log2 units)
};
constexpr float kLazy = 8.f;
__device__ __forceinline__ void attend_fine(uint32_t kT, uint32_t vT, float bias, float c,
                                            const uint32_t (&qf)[4][4], uint32_t lane,
                                            FineState& st) {
  float s[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[j][i] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t b[4];
    ldb(kT, 0, ks, lane, b);
    mma16816(s[0], qf[ks], b[0], b[1]);
    mma16816(s[1], qf[ks], b[2], b[3]);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[h][i] = fmaf(s[h][i], c, bias);
  float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
  float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
  mx0 = quad_max(mx0);
  mx1 = quad_max(mx1);
  st.mt[0] = fmaxf(st.mt[0], mx0);
  st.mt[1] = fmaxf(st.mt[1], mx1);
  if (__any_sync(0xffffffffu, mx0 > st.m[0] + kLazy || mx1 > st.m[1] + kLazy)) {
    const float mn0 = fmaxf(st.m[0], mx0), mn1 = fmaxf(st.m[1], mx1);
    const float a0 = ex2(st.m[0] - mn0), a1 = ex2(st.m[1] - mn1);
    st.m[0] = mn0;
    st.m[1] = mn1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      st.o[j][0] *= a0;
      st.o[j][1] *= a0;
      st.o[j][2] *= a1;
      st.o[j][3] *= a1;
    }
    st.lo[0] *= a0;
    st.lo[1] *= a0;
    st.lo[2] *= a1;
    st.lo[3] *= a1;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    s[h][0] = ex2(s[h][0] - st.m[0]);
    s[h][1] = ex2(s[h][1] - st.m[0]);
    s[h][2] = ex2(s[h][2] - st.m[1]);
    s[h][3] = ex2(s[h][3] - st.m[1]);
  }
  const uint32_t a[4] = {pack_bf16(s[0][0], s[0][1]), pack_bf16(s[0][2], s[0][3]),
                         pack_bf16(s[1][0], s[1][1]), pack_bf16(s[1][2], s[1][3])};
#pragma unroll
  for (int dn = 0; dn < 4; ++dn) {
    uint32_t b[4];
    ldb_t(vT, 0, dn * 16, lane, b);
    mma16816(st.o[2 * dn], a, b[0], b[1]);
    mma16816(st.o[2 * dn + 1], a, b[2], b[3]);
  }
  // row sums of the bf16-rounded P (what P·V multiplies), per lane in fp32
  // (FADD instead of a 17th HMMA per block: the fine loop is HMMA-bound)
  auto lo_f = [](uint32_t x) { return __uint_as_float(x << 16); };
  auto hi_f = [](uint32_t x) { return __uint_as_float(x & 0xffff0000u); };
  st.lo[0] += (lo_f(a[0]) + hi_f(a[0])) + (lo_f(a[2]) + hi_f(a[2]));
  st.lo[2] += (lo_f(a[1]) + hi_f(a[1])) + (lo_f(a[3]) + hi_f(a[3]));
}

namespace fw5 {
constexpr int kQBytes = kTileQ * 128;           // 16 KB
constexpr int kKRing = 3;                       // K' ring: hi + lo of 64 keys
constexpr int kKStage = 16384;
constexpr int kVRing = 2;                       // V' ring: hi of 64 keys
constexpr int kVStage = 8192;
constexpr int kPBytes = kTileQ * 128;           // 128 rows x 64 keys bf16
constexpr int kFineStages = 2;
constexpr int kQStages = 1;
constexpr int kFineWarp = kFineStages * 4096;   // per fine warp: {K, V} blocks
constexpr int kMaxChunks = 6;
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kQStages * kQBytes;      // 16 KB
constexpr int kOffV = kOffK + kKRing * kKStage;        // 64 KB
constexpr int kOffP = kOffV + kVRing * kVStage;        // 80 KB
constexpr int kOffFine = kOffP + 2 * kPBytes;          // 112 KB
// 176 KB: fine partial O_f, then the merged output tile, fp32 as two SW128
// halves [128 rows][32 cols] — the TMA store box layout
constexpr int kOffOf = kOffFine + 8 * kFineWarp;
constexpr int kOfHalf = kTileQ * 128;
constexpr int kOffStat = kOffOf + 2 * kOfHalf;
constexpr int kOffEnt = kOffStat + 5 * kTileQ * 4;  // m_f, l_f, true max, pair max [2]
// ones tile (1024-aligned: a SW128 atom): B operand column 64 of the PV MMA (l_c)
constexpr int kOffOnes = (kOffEnt + 1024 + 1023) & ~1023;  // after bias[32], chunk info, unit table
constexpr int kOffBar = kOffOnes + 8192;
enum { QFULL = 0, QEMPTY = 2, KFULL = 4, KEMPTY = 8, VFULL = 12, VEMPTY = 15, SREADY = 18,
       SFREE = 24, PFULL = 30, PEMPTY = 32, OREADY = 34, OFREE = 36, FDONE = 38, FFREE = 39,
       NBAR = 40 };
constexpr int kSmem = kOffBar + NBAR * 8 + 16;
// warps: 0 K' gather, 1 S MMA, 2 V' gather, 3-10 coarse (two per TMEM lane
// quadrant), 11-18 fine, 19 Q TMA + PV MMA
constexpr int kCoarse0 = 3, kFine0 = 11, kQPV = 19;
constexpr int kThreads = 20 * 32;
constexpr uint32_t kTmemCols = 512;  // S [0, 64·nch), O_c | l_c buffers of 96
constexpr uint32_t kMaxEntries = 4 * kMaxChunks;
}  // namespace fw5

__global__ void __launch_bounds__(fw5::kThreads, 1)
    tc5_fwd_kernel(const __grid_constant__ TcParams p, const __grid_constant__ TmaMaps m,
                   uint32_t units) {
  using namespace llsa_umma;
  using namespace fw5;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  auto bar = [&](int i) { return sbase + kOffBar + 8u * i; };
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kOffBar + NBAR * 8);
  float* fstat = reinterpret_cast<float*>(smem + kOffStat);  // [m_f | l_f][128]
  // byte offset of float4 column group c4 (0..15) of row r in the O_f tile
  auto of_off = [](uint32_t r, uint32_t c4) {
    return (c4 >> 3) * kOfHalf + r * 128 + (((c4 & 7) ^ (r & 7)) << 4);
  };
  const uint64_t tpu = p.n / kTileQ;
  const uint64_t total = tpu * units;
  const uint32_t nce = p.nce, nch = (nce + 3) / 4;
  auto chunk_ne = [&](uint32_t ch) { return min(4u, nce - ch * 4); };
  auto chunk_lo = [&](uint32_t ch) {
    bool lo = false;
    for (uint32_t e = ch * 4; e < ch * 4 + chunk_ne(ch); ++e)
      lo |= entry_level(p, e) >= p.hilo_level;
    return lo;
  };

  // tile-invariant entry facts, computed once: bias (log2 units) per coarse
  // entry, and per 64-key chunk its entry count and whether it needs K'_lo
  float* ent_bias = reinterpret_cast<float*>(smem + kOffEnt);
  uint32_t* ch_info = reinterpret_cast<uint32_t*>(smem + kOffEnt + 128);
  if (tid < nce) ent_bias[tid] = p.bias2[entry_level(p, tid)];
  if (tid < nch) ch_info[tid] = chunk_ne(tid) | (chunk_lo(tid) ? 0x100u : 0u);
  // coarse-warp work units: 32 TMEM columns (two entries) each, as
  // chunk | half << 5 | last-of-chunk << 6
  uint32_t* utab = reinterpret_cast<uint32_t*>(smem + kOffEnt + 192);
  uint32_t nu = 0;
  for (uint32_t ch = 0; ch < nch; ++ch) {
    const bool two = chunk_ne(ch) > 2;
    if (tid == 0) utab[nu] = ch | (two ? 0u : 64u);
    ++nu;
    if (two) {
      if (tid == 0) utab[nu] = ch | 32u | 64u;
      ++nu;
    }
  }
  // a [64 keys][64] MN-major SW128 tile whose column 0 is 1.0: the second N
  // block of the PV MMA's B operand, so TMEM column 64 of O_c accumulates l_c
  for (uint32_t x = tid; x < 64 * 8; x += blockDim.x) {
    const uint32_t kr = x >> 3, c = x & 7;
    const uint32_t v = c == (kr & 7) ? 0x3F80u : 0u;  // logical chunk 0 of row kr
    *reinterpret_cast<uint4*>(smem + kOffOnes + kr * 128 + c * 16) = make_uint4(v, 0, 0, 0);
  }
  fence_proxy_async();
  // TMEM: S chunks at [0, 64·nch); O_c buffers (80 columns: O and l_c) after
  const uint32_t o_base = 64 * nch;
  const uint32_t nob = o_base + 2 * 96 <= kTmemCols ? 2u : 1u;
  const uint32_t o_stride = 96;
  if (warp == 0) tmem_alloc(smem_u32(tslot), kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(QFULL + i), 1);
      mbar_init(bar(QEMPTY + i), 1 + 256);  // S MMAs done + fine warps hold Q
      mbar_init(bar(PFULL + i), 256);
      mbar_init(bar(PEMPTY + i), 1);
      mbar_init(bar(OREADY + i), 1);
      mbar_init(bar(OFREE + i), 256);
    }
    for (int i = 0; i < kKRing; ++i) {
      mbar_init(bar(KFULL + i), 32);  // one cp.async arrival per producer lane
      mbar_init(bar(KEMPTY + i), 1);
    }
    for (int i = 0; i < kVRing; ++i) {
      mbar_init(bar(VFULL + i), 32);
      mbar_init(bar(VEMPTY + i), 1);
    }
    for (int i = 0; i < kMaxChunks; ++i) {
      mbar_init(bar(SREADY + i), 1);
      mbar_init(bar(SFREE + i), 256);
    }
    mbar_init(bar(FDONE), 256);
    mbar_init(bar(FFREE), 256);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0 || warp == 2) {
    // ------------------------------------------------------------ producers
    // warp 0: coarse K' chunks; warp 2: coarse V' chunks.  Each resolves the
    // tiles' coarse rows itself (one tile ahead), so the K' side runs ahead
    // of the PV side by as many tiles as its ring allows.
    const bool kside = warp == 0;
    // The coarse rows are gathered with cp.async by all 32 lanes (16 B per
    // lane per instruction; a 2 KB entry is 4 per lane) into the 128-byte
    // swizzled layout the UMMA descriptors expect; each lane's copies of a
    // chunk arrive on the chunk's FULL barrier as they land (count 32), and
    // the consuming MMA thread fences the async proxy.  Per-entry TMA boxes
    // were issue-bound here (~150 cycles per 2 KB box).
    const uint32_t ring = kside ? kKRing : kVRing;
    const Block16Lane bl = block16_lane(lane);
    const bf16* arr0 = kside ? p.khi : p.vhi;
    const bf16* arr1 = p.klo;
    auto entry_row = [&](uint64_t id) -> uint32_t {
      if (id >= total || lane >= nce) return 0u;
      const uint32_t unit = (uint32_t)(id / tpu);
      uint32_t l, r;
      coarse_entry(p, p.tables + (uint64_t)unit * p.table_entries, (id % tpu) * kTileQ / kBS,
                   lane, l, r);
      return (uint32_t)(unit * p.pyr_rows) + r;
    };
    uint32_t rows_next = entry_row(blockIdx.x);
    uint32_t rc = 0, i = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t myrow = rows_next;
      rows_next = entry_row(id + gridDim.x);
      if (lane == 0) trace_ev(p, kside ? 1 : 2, i, 0);
      for (uint32_t ch = 0; ch < nch; ++ch, ++rc) {
        const uint32_t s = rc % ring;
        const uint32_t info = ch_info[ch], ne = info & 0xFF;
        const bool lo = kside && (info & 0x100u);
        if (rc >= ring) mbar_wait(bar((kside ? KEMPTY : VEMPTY) + s), ((rc / ring) - 1) & 1);
        const uint32_t dst = sbase + (kside ? kOffK + s * kKStage : kOffV + s * kVStage);
        for (uint32_t e = 0; e < ne; ++e) {
          const uint64_t row = __shfl_sync(0xffffffffu, myrow, ch * 4 + e);
          load_block16_async(dst + e * 2048, arr0 + row * kD, bl, lane);
          if (lo) load_block16_async(dst + 8192 + e * 2048, arr1 + row * kD, bl, lane);
        }
        cp_async_mbar_arrive(bar((kside ? KFULL : VFULL) + s));
        if (lane == 0) trace_ev(p, kside ? 1 : 2, i, 1 + ch);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // S chunk c of tile i reuses TMEM columns [64c, 64c+64) as soon as the
    // coarse warps have read chunk c of tile i-1 (per-chunk SREADY / SFREE).
    if (lane == 0) {
      uint32_t kc = 0, i = 0;
      for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
        const uint32_t qs = i % kQStages;
        mbar_wait(bar(QFULL + qs), (i / kQStages) & 1);
        const uint32_t sq = sbase + kOffQ + qs * kQBytes;
        for (uint32_t ch = 0; ch < nch; ++ch, ++kc) {
          const uint32_t s = kc % kKRing;
          mbar_wait(bar(KFULL + s), (kc / kKRing) & 1);
          if (i >= 1) mbar_wait(bar(SFREE + ch), (i - 1) & 1);
          fence_proxy_async();  // the K' chunk was written by cp.async
          fence_after();
          const uint32_t ne = ch_info[ch] & 0xFF;
          const bool lo = ch_info[ch] & 0x100u;
          const uint32_t idesc = idesc_bf16(128, 16 * ne, false, false);
          const uint32_t st = sbase + kOffK + s * kKStage;
          const uint32_t tS = tmem + 64 * ch;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t aq = desc_kmajor(sq + ks * kKStepKMajor);
            mma_bf16(tS, aq, desc_kmajor(st + ks * kKStepKMajor), idesc, ks > 0);
            if (lo) mma_bf16(tS, aq, desc_kmajor(st + 8192 + ks * kKStepKMajor), idesc, 1);
          }
          commit(bar(KEMPTY + s));
          commit(bar(SREADY + ch));
          trace_ev(p, 3, i, ch);
        }
        commit(bar(QEMPTY + qs));
      }
    }
  } else if (warp == kQPV) {
    // ------------------------------------------------------------ Q TMA + PV issuer
    // A second MMA-issuing thread, so the S chunks of tile i+1 do not wait
    // behind tile i's PV chunks.  It also streams the Q tiles: Q(i+1) goes
    // into the (single) Q buffer once tile i's S MMAs are done, which tile
    // i's PV needs anyway.
    if (lane == 0) {
      static_assert(kQStages == 1, "the Q schedule below assumes one Q buffer");
      prefetch_map(&m.q);
      auto load_q = [&](uint64_t id) {
        mbar_expect_tx(bar(QFULL), kQBytes);
        tma_load_2d(sbase + kOffQ, &m.q, 0, (int)((id / tpu) * p.n + (id % tpu) * kTileQ),
                    bar(QFULL));
      };
      if (blockIdx.x < total) load_q(blockIdx.x);
      const uint32_t idesc_o = idesc_bf16(128, kD + 16, false, true);  // O | l_c
      uint32_t vc = 0, pc = 0, i = 0;
      for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
        // Q(i+1) may load once tile i's S MMAs are done and the fine warps
        // hold their Q fragments (QEMPTY); the P·V MMAs of tile i do not read
        // Q, so that is polled between chunks instead of waited for here
        bool q_pending = id + gridDim.x < total;
        auto try_q = [&]() {
          if (q_pending && mbar_test(bar(QEMPTY), i & 1)) {
            load_q(id + gridDim.x);
            q_pending = false;
          }
        };
        try_q();
        const uint32_t ob = i % nob;
        if (i >= nob) mbar_wait(bar(OFREE + ob), ((i / nob) - 1) & 1);
        const uint32_t tO = tmem + o_base + o_stride * ob;
        for (uint32_t ch = 0; ch < nch; ++ch, ++vc, ++pc) {
          const uint32_t s = vc % kVRing, ps = pc & 1;
          mbar_wait(bar(VFULL + s), (vc / kVRing) & 1);
          mbar_wait(bar(PFULL + ps), (pc >> 1) & 1);
          fence_proxy_async();  // the V' chunk was written by cp.async
          fence_after();
          const uint32_t ne = chunk_ne(ch);
          const uint32_t sp = sbase + kOffP + ps * kPBytes;
          const uint32_t sv = sbase + kOffV + s * kVStage;
          const uint32_t ones_lbo = sbase + kOffOnes - sv;
          for (uint32_t ks = 0; ks < ne; ++ks)
            mma_bf16(tO, desc_kmajor(sp + ks * kKStepKMajor),
                     desc_mnmajor(sv + ks * kKStepMNMajor, ones_lbo), idesc_o, (ch | ks) > 0);
          commit(bar(VEMPTY + s));
          commit(bar(PEMPTY + ps));
          trace_ev(p, 3, i, 16 + ch);
          try_q();
        }
        commit(bar(OREADY + ob));
        if (q_pending) {
          mbar_wait(bar(QEMPTY), i & 1);
          load_q(id + gridDim.x);
        }
      }
    }
  } else if (warp >= kCoarse0 && warp < kCoarse0 + 8) {
    // ------------------------------------------------------------ coarse warps
    // Two warps per TMEM lane quadrant (= per SM sub-partition) split every
    // 64-column chunk: half h = 0 takes entries 0, 1 (columns 0-31), h = 1
    // entries 2, 3.  The row max is exchanged through smem once per tile
    // (named barrier per pair), so P, O_c and l_c share one exact reference.
    const uint32_t quad = warp & 3, h = (warp - kCoarse0) >> 2;
    const uint32_t row = 32 * quad + lane;
    const uint32_t lane_off = (32u * quad) << 16;
    const uint32_t pair_bar = 1 + quad;
    const float c2 = p.scale * kLog2e;
    const uint32_t crole = warp == kCoarse0 ? 4 : warp == kCoarse0 + 4 ? 6 : 7;  // trace
    float* pmax = reinterpret_cast<float*>(smem + kOffStat + 3 * kTileQ * 4);  // [2][128]
    uint32_t pc = 0, i = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint64_t q0 = (id % tpu) * kTileQ;
      // pass 1: row max of s·c + b over this half of the coarse set
      float mx = -INFINITY;
      for (uint32_t ch = 0; ch < nch; ++ch) {
        const uint32_t ne = chunk_ne(ch);
        mbar_wait(bar(SREADY + ch), i & 1);
        fence_after();
        if (2 * h < ne) {
          uint32_t sv[32];
          tmem_ld32(tmem + lane_off + 64 * ch + 32 * h, sv);
          tmem_ld_wait();
          const uint32_t ne_u = min(2u, ne - 2 * h);
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            if (e2 < (int)ne_u) {
              const uint32_t* se = sv + e2 * 16;
              float t[8];
#pragma unroll
              for (int k = 0; k < 8; ++k)
                t[k] = fmaxf(__uint_as_float(se[k]), __uint_as_float(se[k + 8]));
#pragma unroll
              for (int k = 0; k < 4; ++k) t[k] = fmaxf(t[k], t[k + 4]);
              const float x = fmaxf(fmaxf(t[0], t[2]), fmaxf(t[1], t[3]));
              mx = fmaxf(mx, fmaf(x, c2, ent_bias[ch * 4 + 2 * h + e2]));  // c > 0
            }
          }
        }
      }
      pmax[h * kTileQ + row] = mx;
      named_bar_sync(pair_bar, 64);
      mx = fmaxf(mx, pmax[(h ^ 1) * kTileQ + row]);
      if (lane == 0) trace_ev(p, crole, i, 0);
      // pass 2: P = exp2(s·c + b − m_c) → bf16 ring (this half's columns)
      for (uint32_t ch = 0; ch < nch; ++ch, ++pc) {
        const uint32_t ps = pc & 1;
        const bool has = 2 * h < chunk_ne(ch);
        uint32_t sv[32];
        if (has) tmem_ld32(tmem + lane_off + 64 * ch + 32 * h, sv);
        if (pc >= 2) mbar_wait(bar(PEMPTY + ps), ((pc >> 1) - 1) & 1);
        const uint32_t sp = sbase + kOffP + ps * kPBytes;
        tmem_ld_wait();
        if (has) {
          const uint32_t ne_u = min(2u, chunk_ne(ch) - 2 * h);
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            if (e2 < (int)ne_u) {
              const uint32_t e = 2 * h + e2;
              const float nb = ent_bias[ch * 4 + e] - mx;
#pragma unroll
              for (int half = 0; half < 2; ++half) {
                uint32_t pk[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int i0 = e2 * 16 + half * 8 + k * 2;
                  const float2 x = __ffma2_rn(
                      make_float2(__uint_as_float(sv[i0]), __uint_as_float(sv[i0 + 1])),
                      make_float2(c2, c2), make_float2(nb, nb));
                  pk[k] = pack_bf16(ex2(x.x), ex2(x.y));
                }
                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(
                                 sp + swz(row, e * 2 + half)),
                             "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]));
              }
            }
          }
        }
        fence_before();
        mbar_arrive(bar(SFREE + ch));
        fence_proxy_async();
        mbar_arrive(bar(PFULL + ps));
        if (lane == 0) trace_ev(p, crole, i, 24 + ch);
      }
      // epilogue: merge this half of the columns with the fine partition of
      // the same rows (staged in smem by the fine warps),
      // O = (O_c 2^(m_c-m) + O_f 2^(m_f-m)) / l, then a TMA store of the box
      const uint32_t ob = i % nob;
      if (lane == 0) trace_ev(p, crole, i, 1);
      mbar_wait(bar(OREADY + ob), (i / nob) & 1);
      mbar_wait(bar(FDONE), i & 1);
      if (lane == 0) trace_ev(p, crole, i, 2);
      fence_after();
      const uint32_t tO = tmem + lane_off + o_base + o_stride * ob;
      uint32_t lraw, ov[32];
      tmem_ld1(tO + kD, lraw);
      tmem_ld32(tO + 32 * h, ov);
      tmem_ld_wait();
      const float lsum = __uint_as_float(lraw);
      const float mf = fstat[row], lf = fstat[kTileQ + row];
      const float mrow = fmaxf(mx, fstat[2 * kTileQ + row]);  // the true row max
      const float ac = ex2(mx - mrow), af = ex2(mf - mrow);
      const float lt = lsum * ac + lf * af;
      const float inv = 1.f / lt;
      const float sc = ac * inv, sf = af * inv;
      const uint64_t ro = (uint64_t)unit * p.n + q0 + row;
      bool bad = !(lt > 0.f) || !isfinite(lt);
      // the merged half row overwrites its O_f half row in place; the warp
      // then stores its 32 rows with one TMA box (coalesced, asynchronous)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float4* a = reinterpret_cast<float4*>(smem + kOffOf + of_off(row, 8 * h + k));
        const float4 f = *a;
        float4 v;
        v.x = __uint_as_float(ov[4 * k]) * sc + f.x * sf;
        v.y = __uint_as_float(ov[4 * k + 1]) * sc + f.y * sf;
        v.z = __uint_as_float(ov[4 * k + 2]) * sc + f.z * sf;
        v.w = __uint_as_float(ov[4 * k + 3]) * sc + f.w * sf;
        bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
        *a = v;
      }
      if (p.out16) {  // bf16 copy (RNE of the fp32 result) of this thread's half
        // row, re-read from the staging: 32 bf16, 64 contiguous bytes
        uint4* d = reinterpret_cast<uint4*>(static_cast<bf16*>(p.out16) +
                                            ((uint64_t)unit * p.n + q0 + row) * kD + 32 * h);
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          const float4 x = *reinterpret_cast<const float4*>(smem + kOffOf +
                                                            of_off(row, 8 * h + 2 * k));
          const float4 y = *reinterpret_cast<const float4*>(smem + kOffOf +
                                                            of_off(row, 8 * h + 2 * k + 1));
          d[k] = make_uint4(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w), pack_bf16(y.x, y.y),
                            pack_bf16(y.z, y.w));
        }
      }
      fence_before();
      mbar_arrive(bar(OFREE + ob));
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        const int y = (int)((uint64_t)unit * p.n + q0 + 32 * quad);
        tma_store_2d(&m.o, sbase + kOffOf + h * kOfHalf + 32 * quad * 128, 32 * h, y);
        bulk_commit();
        bulk_wait_read();
      }
      __syncwarp();
      mbar_arrive(bar(FFREE));
      if (h == 0) {
        p.row_max[ro] = mrow / kLog2e;
        p.row_denom[ro] = lt;
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) raise_flag(p.flag, llsa_dev::kErrNonFinite);
      if (lane == 0) trace_ev(p, crole, i, 3);
    }
    if (lane == 0) bulk_wait_all();  // output stores complete before exit
  } else if (p.fine_mode == 1) {
    // ------------------------------------------------------------ previous pass
    // (second pass of a split coarse set) the fine warps' partition is the
    // first pass's result for their 16 rows: raw O = O·l, max m, sum l
    const uint32_t fw = warp - kFine0;
    uint32_t i = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint32_t qs = i % kQStages;
      const uint64_t row0 = (uint64_t)unit * p.n + (id % tpu) * kTileQ + fw * 16;
      mbar_wait(bar(QFULL + qs), (i / kQStages) & 1);
      mbar_arrive(bar(QEMPTY + qs));
      if (i >= 1) mbar_wait(bar(FFREE), (i - 1) & 1);
      // lane: row r = lane >> 1, 8 float4 groups (half = lane & 1)
      const uint32_t r = lane >> 1, half = lane & 1;
      const float l = p.row_denom[row0 + r];
      const float4* src = reinterpret_cast<const float4*>(p.out + (row0 + r) * kD) + half * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float4 v = src[k];
        v.x *= l;
        v.y *= l;
        v.z *= l;
        v.w *= l;
        *reinterpret_cast<float4*>(smem + kOffOf + of_off(fw * 16 + r, half * 8 + k)) = v;
      }
      if (half == 0) {
        const float m2 = p.row_max[row0 + r] * kLog2e;
        fstat[fw * 16 + r] = m2;
        fstat[kTileQ + fw * 16 + r] = l;
        fstat[2 * kTileQ + fw * 16 + r] = m2;
      }
      mbar_arrive(bar(FDONE));
    }
  } else {
    // ------------------------------------------------------------ fine warps
    const float c2 = p.scale * kLog2e;
    const uint32_t fw = warp - kFine0;  // fine query block of the tile
    const uint32_t sF = sbase + kOffFine + fw * kFineWarp;
    const uint64_t nfb = p.n / kBS;
    const uint32_t r = lane >> 2, cc = (lane & 3) * 2;
    const Block16Lane bl = block16_lane(lane);
    // the warp's K fine block ids of a tile, one per lane (K <= 32 on this
    // path); the next tile's are fetched while this one computes
    auto fine_ids = [&](uint64_t id) -> uint32_t {
      if (id >= total || lane >= p.K) return 0u;
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint64_t fb = (id % tpu) * (kTileQ / kBS) + fw;
      return p.tables[(uint64_t)unit * p.table_entries + p.table_off[0] + fb * p.K + lane];
    };
    uint32_t next_ids = fine_ids(blockIdx.x);
    uint32_t i = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint32_t qs = i % kQStages;
      const uint64_t in_off = (uint64_t)unit * p.n * kD;
      uint32_t myb = next_ids;  // the tile's block ids, range-checked once per tile
      if (myb >= nfb) {
        raise_flag(p.flag, llsa_dev::kErrIndex);
        myb = 0;
      }
      auto load_fine = [&](uint32_t j) {
        const uint32_t b = __shfl_sync(0xffffffffu, myb, j & 31);
        const uint32_t base = sF + (j % kFineStages) * 4096;
        if (!probe(p, 16)) {
          load_block16_async(base, p.k + in_off + (uint64_t)b * kBS * kD, bl, lane);
          load_block16_async(base + kTile16, p.v + in_off + (uint64_t)b * kBS * kD, bl, lane);
        }
      };
#pragma unroll
      for (uint32_t j = 0; j + 1 < (uint32_t)kFineStages; ++j) {
        if (j < p.K) load_fine(j);
        cp_async_commit();
      }
      next_ids = fine_ids(id + gridDim.x);
      FineState st;
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) st.o[j][e] = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) st.lo[e] = 0.f;
      st.m[0] = st.m[1] = st.mt[0] = st.mt[1] = -INFINITY;
      uint32_t qf[4][4];
      if (tid == kFine0 * 32) trace_ev(p, 5, i, 0);
      mbar_wait(bar(QFULL + qs), (i / kQStages) & 1);
      if (tid == kFine0 * 32) trace_ev(p, 5, i, 3);
      const uint32_t sq = sbase + kOffQ + qs * kQBytes;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) lda(sq, fw * 16, ks, lane, qf[ks]);
      mbar_arrive(bar(QEMPTY + qs));
      const float bf = p.bias2[0];
      for (uint32_t j = 0; j < p.K; ++j) {
        if (j + kFineStages - 1 < p.K) load_fine(j + kFineStages - 1);
        cp_async_commit();
        cp_async_wait<kFineStages - 1>();
        __syncwarp();
        const uint32_t base = sF + (j % kFineStages) * 4096;
        if (!probe(p, 8)) attend_fine(base, base + kTile16, bf, c2, qf, lane, st);
        __syncwarp();
      }
      // publish the fine partition (raw O_f, m_f, l_f) for the coarse warps
      if (tid == kFine0 * 32) trace_ev(p, 5, i, 1);
      if (i >= 1) mbar_wait(bar(FFREE), (i - 1) & 1);
      if (tid == kFine0 * 32) trace_ev(p, 5, i, 2);
      {
        // l of rows r, r + 8: the quad's partial sums
        float lf0 = st.lo[0], lf1 = st.lo[2];
        lf0 += __shfl_xor_sync(0xffffffffu, lf0, 1);
        lf1 += __shfl_xor_sync(0xffffffffu, lf1, 1);
        lf0 += __shfl_xor_sync(0xffffffffu, lf0, 2);
        lf1 += __shfl_xor_sync(0xffffffffu, lf1, 2);
        const uint32_t r0 = fw * 16 + r, r1 = r0 + 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t c4 = 2 * j + (cc >> 2), w = (cc & 3) * 4;
          *reinterpret_cast<float2*>(smem + kOffOf + of_off(r0, c4) + w) =
              make_float2(st.o[j][0], st.o[j][1]);
          *reinterpret_cast<float2*>(smem + kOffOf + of_off(r1, c4) + w) =
              make_float2(st.o[j][2], st.o[j][3]);
        }
        if ((lane & 3) == 0) {
          fstat[r0] = st.m[0];
          fstat[r1] = st.m[1];
          fstat[kTileQ + r0] = lf0;
          fstat[kTileQ + r1] = lf1;
          fstat[2 * kTileQ + r0] = st.mt[0];
          fstat[2 * kTileQ + r1] = st.mt[1];
        }
      }
      mbar_arrive(bar(FDONE));
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// backward dQ — persistent, warp-specialised, fine + coarse in one pass
// ---------------------------------------------------------------------------
// The query-major half of the mask-free backward (attention_grad.cpp:16-25,
// 229-257) for 128-query tiles, structured like tc5_fwd_kernel:
//   warp 15 (1 lane)  TMA: Q and dO tiles (single buffer)
//   warp 0            cp.async gather of the coarse K'/V' chunks (hi [+ lo],
//                     64 keys) → 2-stage ring
//   warp 1 (1 lane)   MMA: S = Q K'^T, dP = dO V'^T per chunk → TMEM (double
//                     buffer); dQ_c += dS K'_hi → TMEM (double buffer / tile)
//   warps 3-6         coarse, thread = query row: dS = P∘(dP − D) with
//                     P = exp2(S c + b − lse) → bf16 smem ring; at the end of a
//                     tile dq = scale (dQ_c + dQ_f), written once
//   warps 7-14        fine, warp 7+w = fine block w on mma.sync; they also
//                     produce D = rowsum(dO∘O) and the log2 LSE of their rows
//                     (smem for the coarse warps, global for the kv kernels)
namespace dqf {
constexpr int kTileBytes = kTileQ * 128;        // 16 KB
constexpr int kCStage = 3 * 8192;               // Khi, Klo, Vhi of 64 keys (V' hi only)
constexpr int kCRing = 2;
constexpr int kQS = 1;                          // Q/dO stages
constexpr int kDSBytes = kTileQ * 128;          // dS chunk: 128 rows x 64 keys bf16
constexpr int kFS = 3;                          // fine ring stages per warp
constexpr int kFineWarp = kFS * 4096;           // {K, V} block per stage
constexpr int kQStage = 2 * kTileBytes;                   // Q | dO of one tile
constexpr int kOffQ = 0;
constexpr int kOffC = kQS * kQStage;
constexpr int kOffDS = kOffC + kCRing * kCStage;
constexpr int kOffFine = kOffDS + 2 * kDSBytes;
// lse, D of three tiles: the fine warps (up to two tiles ahead of the coarse
// warps' read, bounded by FFREE) never refill a slot that is still unread
constexpr int kStatSlots = 3;
constexpr int kOffStat = kOffFine + 8 * kFineWarp;
constexpr int kOffEnt = kOffStat + kStatSlots * 2 * kTileQ * 4;  // bias[32], chunk info[8], rows[32]
constexpr int kOffBar = kOffEnt + 256;
enum { QFULL = 0, QEMPTY = 2, KFULL = 4, KEMPTY = 7, SREADY = 10, TFREE = 12, DSREADY = 14,
       DSFREE = 16, DQREADY = 18, DQFREE = 20, FDONE = 22, FFREE = 24, DREADY = 26,
       NBAR = 29 };
constexpr int kSmem = kOffBar + NBAR * 8 + 16;
static_assert(kSmem <= 232448, "dqf shared memory over the 227 KB opt-in limit");
constexpr int kThreads = 16 * 32;
constexpr uint32_t kTmemCols = 512;  // S/dP x 2 [0, 256), dQ_c x 2 [256, 384), dQ_f x 2 [384, 512)
constexpr uint32_t kMaxEntries = 24;  // ent_rows[24]
}  // namespace dqf

__global__ void __launch_bounds__(dqf::kThreads, 1)
    tc5_dqf_kernel(const __grid_constant__ TcParams p, const __grid_constant__ TmaMaps m,
                   uint32_t units) {
  using namespace llsa_umma;
  using namespace dqf;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  auto bar = [&](int i) { return sbase + kOffBar + 8u * i; };
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kOffBar + NBAR * 8);
  float* stat = reinterpret_cast<float*>(smem + kOffStat);  // [3 tiles][lse | D][128]
  float* ent_bias = reinterpret_cast<float*>(smem + kOffEnt);
  uint32_t* ch_info = reinterpret_cast<uint32_t*>(smem + kOffEnt + 128);
  const uint64_t tpu = p.n / kTileQ;
  const uint64_t total = tpu * units;
  const uint32_t nce = p.nce, nch = (nce + 3) / 4;
  if (tid < nce) ent_bias[tid] = p.bias2[entry_level(p, tid)];
  if (tid < nch) {
    bool lo = false;
    const uint32_t ne = min(4u, nce - tid * 4);
    for (uint32_t e = tid * 4; e < tid * 4 + ne; ++e) lo |= entry_level(p, e) >= p.hilo_level;
    ch_info[tid] = ne | (lo ? 0x100u : 0u);
  }
  if (warp == 0) tmem_alloc(smem_u32(tslot), kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < kCRing; ++i) {
      mbar_init(bar(KFULL + i), 32);  // every gather lane, via its copies
      mbar_init(bar(KEMPTY + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(QFULL + i), 1);
      mbar_init(bar(QEMPTY + i), 1);  // S/dP MMAs of the tile done
      mbar_init(bar(FDONE + i), 256);
      mbar_init(bar(FFREE + i), 128);
      mbar_init(bar(SREADY + i), 1);
      mbar_init(bar(TFREE + i), 128);
      mbar_init(bar(DSREADY + i), 128);
      mbar_init(bar(DSFREE + i), 1);
      mbar_init(bar(DQREADY + i), 1);
      mbar_init(bar(DQFREE + i), 128);

    }
    for (int i = 0; i < kStatSlots; ++i) mbar_init(bar(DREADY + i), 256);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const float c2 = p.scale * kLog2e;

  if (warp == 15) {
    // ------------------------------------------------------------ Q / dO TMA
    if (lane == 0) {
      prefetch_map(&m.q);
      prefetch_map(&m.g);
      uint32_t i = 0;
      for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
        const uint32_t unit = (uint32_t)(id / tpu);
        const uint64_t q0 = (id % tpu) * kTileQ;
        const uint32_t qs = i % kQS;
        if (i >= (uint32_t)kQS) mbar_wait(bar(QEMPTY + qs), ((i / kQS) - 1) & 1);
        mbar_expect_tx(bar(QFULL + qs), kQStage);
        tma_load_2d(sbase + kOffQ + qs * kQStage, &m.q, 0, (int)(unit * p.n + q0),
                    bar(QFULL + qs));
        tma_load_2d(sbase + kOffQ + qs * kQStage + kTileBytes, &m.g, 0, (int)(unit * p.n + q0),
                    bar(QFULL + qs));
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ K'/V' gather
    // Lane e holds coarse entry e's pyramid row, resolved one tile ahead.
    // Copies complete on KFULL asynchronously (cp.async.mbarrier.arrive, one
    // arrival per lane); the S/dP issuer fences the proxy after its wait.
    const Block16Lane bl = block16_lane(lane);
    auto entry_row = [&](uint64_t id) -> uint32_t {
      if (id >= total || lane >= nce) return 0u;
      const uint32_t unit = (uint32_t)(id / tpu);
      uint32_t l, r;
      coarse_entry(p, p.tables + (uint64_t)unit * p.table_entries, (id % tpu) * kTileQ / kBS,
                   lane, l, r);
      return (uint32_t)(unit * p.pyr_rows) + r;
    };
    uint32_t rows_next = entry_row(blockIdx.x);
    uint32_t rc = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x) {
      const uint32_t myrow = rows_next;
      rows_next = entry_row(id + gridDim.x);
      for (uint32_t ch = 0; ch < nch; ++ch, ++rc) {
        const uint32_t s = rc % kCRing;
        const uint32_t info = ch_info[ch], ne = info & 0xFF;
        const bool lo = info & 0x100u;
        if (lane == 0) trace_ev(p, 1, rc, 0);
        if (rc >= (uint32_t)kCRing) mbar_wait(bar(KEMPTY + s), ((rc / kCRing) - 1) & 1);
        if (lane == 0) trace_ev(p, 1, rc, 1);
        const uint32_t dst = sbase + kOffC + s * kCStage;
        for (uint32_t e = 0; e < ne; ++e) {
          const uint64_t o = (uint64_t)__shfl_sync(0xffffffffu, myrow, ch * 4 + e) * kD;
          load_block16_async(dst + e * 2048, p.khi + o, bl, lane);
          load_block16_async(dst + 16384 + e * 2048, p.vhi + o, bl, lane);
          if (lo) load_block16_async(dst + 8192 + e * 2048, p.klo + o, bl, lane);
        }
        cp_async_mbar_arrive(bar(KFULL + s));
        if (lane == 0) trace_ev(p, 1, rc, 2);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ S / dP issuer
    if (lane == 0) {
      uint32_t c = 0, i = 0;
      for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
        const uint32_t qs = i % kQS;
        mbar_wait(bar(QFULL + qs), (i / kQS) & 1);
        const uint32_t sq = sbase + kOffQ + qs * kQStage, sg = sq + kTileBytes;
        for (uint32_t ch = 0; ch < nch; ++ch, ++c) {
          const uint32_t s = c % kCRing, b = c & 1;
          mbar_wait(bar(KFULL + s), (c / kCRing) & 1);
          trace_ev(p, 3, c, 1);
          if (c >= 2) mbar_wait(bar(TFREE + b), ((c >> 1) - 1) & 1);
          trace_ev(p, 3, c, 2);
          fence_proxy_async();  // gathered cp.async data → async proxy
          fence_after();
          const uint32_t info = ch_info[ch], ne = info & 0xFF;
          const bool lo = info & 0x100u;
          const uint32_t idesc = idesc_bf16(128, 16 * ne, false, false);
          const uint32_t st = sbase + kOffC + s * kCStage;
          const uint32_t tS = tmem + b * 128, tP = tS + 64;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t aq = desc_kmajor(sq + ks * kKStepKMajor);
            const uint64_t ag = desc_kmajor(sg + ks * kKStepKMajor);
            mma_bf16(tS, aq, desc_kmajor(st + ks * kKStepKMajor), idesc, ks > 0);
            mma_bf16(tP, ag, desc_kmajor(st + 16384 + ks * kKStepKMajor), idesc, ks > 0);
            if (lo) mma_bf16(tS, aq, desc_kmajor(st + 8192 + ks * kKStepKMajor), idesc, 1);
          }
          commit(bar(SREADY + b));
          trace_ev(p, 3, c, 0);
          if (ch + 1 == nch) commit(bar(QEMPTY + qs));
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ dQ issuer
    // (a second MMA-issuing thread: dQ of chunk c overlaps S/dP of chunk c+1)
    if (lane == 0) {
      const uint32_t idesc_q = idesc_bf16(128, kD, false, true);
      uint32_t c = 0, i = 0;
      for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
        const uint32_t tb = i & 1;
        for (uint32_t ch = 0; ch < nch; ++ch, ++c) {
          const uint32_t s = c % kCRing, b = c & 1, ne = ch_info[ch] & 0xFF;
          mbar_wait(bar(DSREADY + b), (c >> 1) & 1);
          trace_ev(p, 6, c, 1);
          if (ch == 0 && i >= 2) mbar_wait(bar(DQFREE + tb), ((i >> 1) - 1) & 1);
          trace_ev(p, 6, c, 2);
          fence_proxy_async();
          fence_after();
          const uint32_t sds = sbase + kOffDS + b * kDSBytes;
          const uint32_t khi = sbase + kOffC + s * kCStage;
          const uint32_t tq = tmem + 256 + tb * 64;
          for (uint32_t ks = 0; ks < ne; ++ks)
            mma_bf16(tq, desc_kmajor(sds + ks * kKStepKMajor),
                     desc_mnmajor(khi + ks * kKStepMNMajor, 8192), idesc_q,
                     (ch == 0 && ks == 0) ? 0u : 1u);
          commit(bar(KEMPTY + s));
          commit(bar(DSFREE + b));
          trace_ev(p, 6, c, 0);
          if (ch + 1 == nch) commit(bar(DQREADY + tb));
        }
      }
    }
  } else if (warp >= 3 && warp < 7) {
    // ------------------------------------------------------------ coarse warps
    const uint32_t row = 32 * (warp & 3) + lane;
    const uint32_t lane_off = (32u * (warp & 3)) << 16;
    uint32_t c = 0, i = 0;
    // this warp's dq TMA store of the previous tile may still be reading its
    // rows of the dS ring: waited for only before the next dS store
    bool st_pending = false;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint64_t q0 = (id % tpu) * kTileQ;
      const uint32_t tb = i & 1;
      if (tid == 96) trace_ev(p, 7, i, 5);
      const uint32_t ts = i % kStatSlots;
      mbar_wait(bar(DREADY + ts), (i / kStatSlots) & 1);
      if (tid == 96) trace_ev(p, 7, i, 6);
      const float lse = stat[ts * 256 + row], Drow = stat[ts * 256 + 128 + row];
      for (uint32_t ch = 0; ch < nch; ++ch, ++c) {
        const uint32_t b = c & 1, ne = ch_info[ch] & 0xFF;
        if (tid == 96) trace_ev(p, 4, c, 1);
        mbar_wait(bar(SREADY + b), (c >> 1) & 1);
        if (tid == 96) trace_ev(p, 4, c, 2);
        fence_after();
        const uint32_t sds = sbase + kOffDS + b * kDSBytes;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (2 * hh < (int)ne) {
            uint32_t sv[32], gv[32];
            tmem_ld32(tmem + lane_off + b * 128 + 32 * hh, sv);
            tmem_ld32(tmem + lane_off + b * 128 + 64 + 32 * hh, gv);
            // the dS slot is needed only from the first store on: wait for
            // it while the TMEM loads are in flight
            if (hh == 0 && c >= 2) mbar_wait(bar(DSFREE + b), ((c >> 1) - 1) & 1);
            if (hh == 0 && st_pending) {
              if (lane == 0) bulk_wait_read();
              __syncwarp();
              st_pending = false;
            }
            tmem_ld_wait();
            if (2 * hh + 2 >= (int)ne) {  // S / dP all in registers: release the buffer
              fence_before();
              mbar_arrive(bar(TFREE + b));
            }
#pragma unroll
            for (int ee = 0; ee < 2; ++ee) {
              const uint32_t e = 2 * hh + ee;
              if (e < ne) {
                const float nb = ent_bias[ch * 4 + e] - lse;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                  uint32_t pk[4];
#pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    const int i0 = ee * 16 + half * 8 + k * 2;
                    // packed fp32x2: same per-element operations and rounding
                    const float2 x = __ffma2_rn(
                        make_float2(__uint_as_float(sv[i0]), __uint_as_float(sv[i0 + 1])),
                        make_float2(c2, c2), make_float2(nb, nb));
                    const float2 g = __fadd2_rn(
                        make_float2(__uint_as_float(gv[i0]), __uint_as_float(gv[i0 + 1])),
                        make_float2(-Drow, -Drow));
                    const float2 ds = __fmul2_rn(make_float2(ex2(x.x), ex2(x.y)), g);
                    pk[k] = pack_bf16(ds.x, ds.y);
                  }
                  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(
                                   sds + swz(row, e * 2 + half)),
                               "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]));
                }
              }
            }
          }
        }
        fence_proxy_async();
        mbar_arrive(bar(DSREADY + b));
        if (tid == 96) trace_ev(p, 4, c, 0);
      }
      // tile epilogue: dq = scale (dQ_c + dQ_f), written once
      if (tid == 96) trace_ev(p, 7, i, 0);
      mbar_wait(bar(DQREADY + tb), (i >> 1) & 1);
      if (tid == 96) trace_ev(p, 7, i, 1);
      mbar_wait(bar(FDONE + tb), (i >> 1) & 1);
      if (tid == 96) trace_ev(p, 7, i, 2);
      fence_after();
      // the dq row goes through the (idle: every dQ MMA of the tile is done)
      // dS ring as two SW128 fp32 boxes per warp and leaves by TMA store,
      // instead of 16 scattered 16-byte stores per thread; each warp only
      // touches its own 32 rows of the staging, and the store has read them
      // before this warp writes the next tile's dS there
      const uint32_t stg = sbase + kOffDS;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t r0[32], f[32];
        tmem_ld32(tmem + lane_off + 256 + tb * 64 + 32 * hh, r0);   // dQ_c
        tmem_ld32(tmem + lane_off + 384 + tb * 64 + 32 * hh, f);    // dQ_f (fine warps)
        tmem_ld_wait();
        if (hh == 1) {  // both accumulators are in registers: release them first
          fence_before();
          mbar_arrive(bar(DQFREE + tb));
          mbar_arrive(bar(FFREE + tb));
        }
        if (p.grad_bf16) {  // bf16 dq: one SW128 [32 rows][64] box per warp
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = 8 * k + 2 * e;
              w[e] = pack_bf16((__uint_as_float(r0[c]) + __uint_as_float(f[c])) * p.scale,
                               (__uint_as_float(r0[c + 1]) + __uint_as_float(f[c + 1])) * p.scale);
            }
            const uint32_t ch = 4 * hh + k;
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(
                             stg + row * 128 + ((ch ^ (row & 7)) << 4)),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]));
          }
          continue;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float v0 = (__uint_as_float(r0[4 * k]) + __uint_as_float(f[4 * k])) * p.scale;
          const float v1 = (__uint_as_float(r0[4 * k + 1]) + __uint_as_float(f[4 * k + 1])) * p.scale;
          const float v2 = (__uint_as_float(r0[4 * k + 2]) + __uint_as_float(f[4 * k + 2])) * p.scale;
          const float v3 = (__uint_as_float(r0[4 * k + 3]) + __uint_as_float(f[4 * k + 3])) * p.scale;
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(
                           stg + hh * kDSBytes + row * 128 + ((k ^ (row & 7)) << 4)),
                       "f"(v0), "f"(v1), "f"(v2), "f"(v3));
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (tid == 96) trace_ev(p, 7, i, 3);
      if (lane == 0) {
        const int y = (int)((uint64_t)unit * p.n + q0 + 32 * (warp & 3));
        if (p.fine_mode) {  // a later pass of a split coarse set: dq += this pass
          tma_reduce_add_2d(&m.o, stg + 32 * (warp & 3) * 128, 0, y);
          tma_reduce_add_2d(&m.o, stg + kDSBytes + 32 * (warp & 3) * 128, 32, y);
        } else {
          tma_store_2d(&m.o, stg + 32 * (warp & 3) * 128, 0, y);
          if (!p.grad_bf16) tma_store_2d(&m.o, stg + kDSBytes + 32 * (warp & 3) * 128, 32, y);
        }
        bulk_commit();
      }
      st_pending = true;
      __syncwarp();
      if (tid == 96) trace_ev(p, 7, i, 4);
    }
    if (lane == 0) bulk_wait_all();  // dq stores complete before exit
  } else if (warp >= 7) {
    // ------------------------------------------------------------ fine warps
    // fine block of this warp: its 16 rows must be TMEM lanes of the warp's
    // sub-partition (warp % 4), where it stages its dQ part
    const uint32_t fw = 2 * (warp & 3) + (warp >= 11 ? 1u : 0u);
    const uint32_t sF = sbase + kOffFine + fw * kFineWarp;
    const uint64_t nfb = p.n / kBS;
    const uint32_t r = lane >> 2;
    const Block16Lane bl = block16_lane(lane);
    auto fine_ids = [&](uint64_t id) -> uint32_t {
      if (id >= total || lane >= p.K) return 0u;
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint64_t fb = (id % tpu) * (kTileQ / kBS) + fw;
      return p.tables[(uint64_t)unit * p.table_entries + p.table_off[0] + fb * p.K + lane];
    };
    uint32_t next_ids = fine_ids(blockIdx.x);
    const float bf = p.bias2[0];
    uint32_t i = 0;
    for (uint64_t id = blockIdx.x; id < total; id += gridDim.x, ++i) {
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint64_t q0 = (id % tpu) * kTileQ;
      const uint64_t in_off = (uint64_t)unit * p.n * kD;
      uint32_t myb = next_ids;  // the tile's block ids, range-checked once per tile
      if (myb >= nfb) {
        raise_flag(p.flag, llsa_dev::kErrIndex);
        myb = 0;
      }
      auto load_fine = [&](uint32_t j) {
        const uint32_t b = __shfl_sync(0xffffffffu, myb, j & 31);
        const uint32_t base = sF + (j % kFS) * 4096;
        if (!probe(p, 16)) {
          load_block16_async(base, p.k + in_off + (uint64_t)b * kBS * kD, bl, lane);
          load_block16_async(base + kTile16, p.v + in_off + (uint64_t)b * kBS * kD, bl, lane);
        }
      };
      // blocks 0 .. kFS-2 prefetched; this warp's own 16 Q and dO rows go to
      // the last ring stage (free until block kFS-1 is loaded)
      constexpr uint32_t sQD = (kFS - 1) * 4096;
#pragma unroll
      for (uint32_t j = 0; j + 1 < (uint32_t)kFS; ++j)
        if (j < p.K && !p.fine_mode) load_fine(j);
      load_block16_async(sF + sQD, p.q + in_off + (q0 + fw * 16) * kD, bl, lane);
      if (tid == 224) trace_ev(p, 5, i, 4);
      load_block16_async(sF + sQD + kTile16, p.dout + in_off + (q0 + fw * 16) * kD, bl, lane);
      cp_async_commit();
      next_ids = fine_ids(id + gridDim.x);
      // D = rowsum(dO∘O) (fp32 O) and the log2 LSE of this warp's 16 rows;
      // lane pair (2ρ, 2ρ+1) owns row ρ (columns [32·half, +32))
      const uint32_t rr = lane >> 1, half = lane & 1;
      const uint64_t trow = q0 + fw * 16 + rr;
      const uint64_t ro = (uint64_t)unit * p.n;
      float4 ov[8];
      {
        const float4* o4 = reinterpret_cast<const float4*>(p.out_in + in_off + trow * kD + half * 32);
#pragma unroll
        for (int k = 0; k < 8; ++k) ov[k] = o4[k];
      }
      const float lse_r = p.rm_in[ro + trow] * kLog2e + __log2f(p.rd_in[ro + trow]);
      cp_async_wait<0>();
      __syncwarp();
      uint32_t qf[4][4], gf[4][4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        lda(sF + sQD, 0, ks, lane, qf[ks]);
        lda(sF + sQD + kTile16, 0, ks, lane, gf[ks]);
      }
      float dsum = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // dO row rr, 16-byte chunks 4·half + k
        uint4 gv;
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(gv.x), "=r"(gv.y), "=r"(gv.z), "=r"(gv.w)
                     : "r"(sF + sQD + kTile16 + swz(rr, half * 4 + k)));
        const uint32_t w[4] = {gv.x, gv.y, gv.z, gv.w};
        const float of[8] = {ov[2 * k].x, ov[2 * k].y, ov[2 * k].z, ov[2 * k].w,
                             ov[2 * k + 1].x, ov[2 * k + 1].y, ov[2 * k + 1].z, ov[2 * k + 1].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          dsum = fmaf(__uint_as_float(w[t] << 16), of[2 * t], dsum);
          dsum = fmaf(__uint_as_float(w[t] & 0xffff0000u), of[2 * t + 1], dsum);
        }
      }
      __syncwarp();  // the Q/dO stage is overwritten by fine block kFS-1
      dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
      const uint32_t tb = i & 1, ts = i % kStatSlots;
      if (half == 0) {
        p.drow[ro + trow] = dsum;
        p.lse2[ro + trow] = lse_r;
        stat[ts * 256 + fw * 16 + rr] = lse_r;
        stat[ts * 256 + 128 + fw * 16 + rr] = dsum;
      }
      mbar_arrive(bar(DREADY + ts));
      if (tid == 224) trace_ev(p, 5, i, 3);
      const float D0 = __shfl_sync(0xffffffffu, dsum, 2 * r);
      const float D1 = __shfl_sync(0xffffffffu, dsum, 2 * (r + 8));
      const float lse0 = __shfl_sync(0xffffffffu, lse_r, 2 * r);
      const float lse1 = __shfl_sync(0xffffffffu, lse_r, 2 * (r + 8));
      float dq[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) dq[j][e] = 0.f;
      const uint32_t nfine = p.fine_mode ? 0u : p.K;  // later passes: coarse entries only
      for (uint32_t j = 0; j < nfine; ++j) {
        if (j + kFS - 1 < nfine) load_fine(j + kFS - 1);
        cp_async_commit();
        cp_async_wait<kFS - 1>();
        __syncwarp();
        const uint32_t base = sF + (j % kFS) * 4096;
        if (!probe(p, 8)) attend_dq<false>(base, base, base + kTile16, base + kTile16, 0, bf, c2, qf, gf, lse0,
                         lse1, D0, D1, lane, dq);
        __syncwarp();
      }
      // publish the fine part of dQ (unscaled) in TMEM (lanes 16 fw.., the
      // mma fragment layout via tcgen05.st.16x256b) for the coarse epilogue
      if (tid == 224) trace_ev(p, 5, i, 1);
      if (i >= 2) mbar_wait(bar(FFREE + tb), ((i >> 1) - 1) & 1);
      if (tid == 224) trace_ev(p, 5, i, 2);
      fence_after();
      const uint32_t tq = tmem + ((16u * fw) << 16) + 384 + 64 * tb;
#pragma unroll
      for (int j = 0; j < 8; ++j) tmem_st_frag(tq + 8 * j, dq[j][0], dq[j][1], dq[j][2], dq[j][3]);
      tmem_st_wait();
      fence_before();
      mbar_arrive(bar(FDONE + tb));
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// backward: fine dK/dV on tcgen05 — persistent, key-major, warp-specialised
// ---------------------------------------------------------------------------
// Work item = one fine key block kb (16 keys) of one unit; its queries are the
// CSC segment of kb (query blocks that selected it), gathered 8 blocks (128
// queries) per chunk.  Per chunk:
//   S  = Q_g K_kb^T, dP = dO_g V_kb^T      M = 128 gathered queries, N = 16
//   thread = query: dS = P∘(dP − D), P = exp2(S c + b − lse)
//   B' = [dS | P | 0] (bf16, MN-major [query][64]) → smem
//   Acc += [Q_g^T ; dO_g^T] · B'           M = 128 (d of Q, d of dO), N = 64,
//                                          K = the chunk's valid queries
// so Acc[0:64, 0:16] = dK^T and Acc[64:128, 16:32] = dV^T accumulate in TMEM
// over the item's chunks (no atomics).  The epilogue adds every coarse level's
// pooled adjoint (already reduced) and writes dk, dv once.
// Replaces P/src/attention_grad.cpp:43-73,127-135 (+ :149-161,184-196).
//   warps 0,2,11,12  cp.async gather (Q, dO rows of the segment; K, V of kb;
//                    lse, D) → 5-stage ring, completion via
//                    cp.async.mbarrier.arrive; chunk facts in smem
//   warp 1 (1 ln)    S / dP issuer;  warp 13 (1 ln)  accumulate issuer
//   warps 3-6        softmax, thread = gathered query (TMEM lane)
//   warps 7-10       epilogue, thread = head-dim row of Acc (TMEM lane)
// Item facts (CSC offsets, query-block ids, coarse adjoint rows) are fetched
// two items ahead so no dependent global load sits on a role's critical path.
namespace kvf {
constexpr int kQOff = 0, kGOff = 16384, kKOff = 32768, kVOff = 34816, kLseOff = 36864,
              kDOff = 37376;
constexpr int kStage = 38912;                  // 38 KB, 1024-aligned
constexpr int kRing = 5;
constexpr int kOffB = kRing * kStage;          // 190 KB: B' x 2 (16 KB each)
constexpr int kOffInfo = kOffB + 2 * 16384;    // per-stage chunk facts
constexpr int kFactSlots = 16, kFactWords = 36;  // item facts ring: lo, hi, unit, kb, ids[32]
constexpr int kOffFacts = kOffInfo + 64;
constexpr int kOffBar = kOffFacts + kFactSlots * kFactWords * 4;
constexpr int kAB = 4;  // Acc buffers (items in flight between MMA and epilogue)
enum { FULL = 0, EMPTY = kRing, SREADY = 2 * kRing, SFREE = SREADY + 2, BREADY = SFREE + 2,
       BFREE = BREADY + 2, AREADY = BFREE + 2, AFREE = AREADY + kAB, FACTF = AFREE + kAB,
       FACTE = FACTF + kFactSlots, NBAR = FACTE + kFactSlots };
constexpr int kSmem = kOffBar + NBAR * 8 + 16;
// gather 0, 2, 11, 12; MMA 1, 13; softmax 3-6; epilogue 7-10; item facts 14
constexpr int kThreads = 15 * 32;
constexpr uint32_t kTmemCols = 512;  // S|dP x 2 at [0, 64), Acc x kAB at 64 + 64·i
}  // namespace kvf

__global__ void __launch_bounds__(kvf::kThreads, 1)
    tc5_kvf_kernel(const __grid_constant__ TcParams p, uint32_t units) {
  using namespace llsa_umma;
  using namespace kvf;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  auto bar = [&](int i) { return sbase + kOffBar + 8u * i; };
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kOffBar + NBAR * 8);
  uint32_t* info = reinterpret_cast<uint32_t*>(smem + kOffInfo);  // [stage]: mc | first | last
  const uint64_t nkb = p.n / kBS;
  const uint64_t total = nkb * units;
  // B' columns 32-63 stay zero for the whole kernel
  for (uint32_t x = tid; x < 2 * 128 * 4; x += blockDim.x) {
    const uint32_t b = x >> 9, r = (x >> 2) & 127, c = 4 + (x & 3);
    *reinterpret_cast<uint4*>(smem + kOffB + b * 16384 + swz(r, c)) = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc(smem_u32(tslot), kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(bar(FULL + i), 128);  // every gather lane, via its copies
      mbar_init(bar(EMPTY + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(SREADY + i), 1);
      mbar_init(bar(SFREE + i), 128);
      mbar_init(bar(BREADY + i), 128);
      mbar_init(bar(BFREE + i), 1);
    }
    for (int i = 0; i < kAB; ++i) {
      mbar_init(bar(AREADY + i), 1);
      mbar_init(bar(AFREE + i), 128);
    }
    for (int i = 0; i < kFactSlots; ++i) {
      mbar_init(bar(FACTF + i), 1);
      mbar_init(bar(FACTE + i), 8);  // the four gather warps + the four epilogue warps
    }
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0 || warp == 2 || warp == 11 || warp == 12) {
    // ------------------------------------------------------------ gather
    // Four warps share every chunk (warp gi: query blocks gi and gi + 4;
    // warp 0 also K_kb, V_kb, lse, D and the chunk facts).  Every lane's
    // copies arrive on the chunk's FULL barrier asynchronously
    // (cp.async.mbarrier.arrive.noinc, 128 arrivals), so the gather never
    // blocks on its own copies; the MMA issuer fences the generic→async
    // proxy after the wait.
    const uint32_t gi = warp == 0 ? 0u : warp == 2 ? 1u : warp - 9;
    const Block16Lane bl = block16_lane(lane);
    // Item facts (CSC segment bounds, first 32 query-block ids) come from the
    // facts warp through a smem ring filled up to 8 items ahead, so no
    // dependent global load sits on the issue path.
    const uint32_t* flat0 = p.csc_flat + p.csc_flat_off[0];
    const uint32_t* fact = reinterpret_cast<const uint32_t*>(smem + kOffFacts);
    const uint64_t G = gridDim.x;
    uint32_t rc = 0, it = 0;
    for (uint64_t id = blockIdx.x; id < total; id += G, ++it) {
      const uint32_t fs = it % kFactSlots;
      mbar_wait(bar(FACTF + fs), (it / kFactSlots) & 1);
      const uint32_t lo0 = fact[fs * kFactWords], hi0 = fact[fs * kFactWords + 1];
      const uint32_t unit = fact[fs * kFactWords + 2];
      const uint64_t kb = fact[fs * kFactWords + 3];
      const uint32_t ids0 = fact[fs * kFactWords + 4 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(FACTE + fs));
      const uint32_t m = hi0 - lo0;
      const uint32_t* seg = flat0 + (uint64_t)unit * p.csc_flat_entries + lo0;
      const uint64_t in_off = (uint64_t)unit * p.n * kD, ro = (uint64_t)unit * p.n;
      const uint32_t nch = (m + 7) / 8;
      for (uint32_t ch = 0; ch < nch; ++ch, ++rc) {
        const uint32_t s = rc % kRing;
        const uint32_t mc = min(8u, m - ch * 8);
        if (gi == 0 && lane == 0) trace_ev(p, 1, rc, 0);
        if (rc >= (uint32_t)kRing) mbar_wait(bar(EMPTY + s), ((rc / kRing) - 1) & 1);
        if (gi == 0 && lane == 0) trace_ev(p, 1, rc, 1);
        const uint32_t st = sbase + s * kStage;
        const uint32_t jj = ch * 8 + lane;
        const uint32_t pre = __shfl_sync(0xffffffffu, ids0, jj & 31);
        uint32_t qb = lane >= mc ? 0u : jj < 32 ? pre : seg[jj];
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
          const uint32_t b = gi + 4 * h;
          const uint64_t t0 = (uint64_t)__shfl_sync(0xffffffffu, qb, b) * kBS;
          if (b < mc) {
            load_block16_async(st + kQOff + b * 2048, p.q + in_off + t0 * kD, bl, lane);
            load_block16_async(st + kGOff + b * 2048, p.dout + in_off + t0 * kD, bl, lane);
          }
        }
        const uint64_t tl = (uint64_t)__shfl_sync(0xffffffffu, qb, lane >> 2) * kBS + (lane & 3) * 4;
        if (gi == 0) {
          load_block16_async(st + kKOff, p.k + in_off + kb * kBS * kD, bl, lane);
          load_block16_async(st + kVOff, p.v + in_off + kb * kBS * kD, bl, lane);
          if ((lane >> 2) < mc) {
            cp_async16(st + kLseOff + lane * 16, p.lse2 + ro + tl);
            cp_async16(st + kDOff + lane * 16, p.drow + ro + tl);
          }
          if (lane == 0)
            info[s] = mc | (ch == 0 ? 0x100u : 0u) | (ch + 1 == nch ? 0x200u : 0u);
        }
        cp_async_mbar_arrive(bar(FULL + s));
        if (gi == 0 && lane == 0) trace_ev(p, 1, rc, 2);
      }
    }
    // terminal marker
    {
      const uint32_t s = rc % kRing;
      if (rc >= (uint32_t)kRing) mbar_wait(bar(EMPTY + s), ((rc / kRing) - 1) & 1);
      if (gi == 0 && lane == 0) info[s] = 0x400u;
      __syncwarp();
      mbar_arrive(bar(FULL + s));
    }
  } else if (warp == 14) {
    // ------------------------------------------------------------ item facts
    // batches of kFactSlots items: lane j loads the segment bounds of item
    // k + j, then item by item the first 32 query-block ids (a loop, not
    // unrolled: this warp runs up to 8 items ahead and its code shares the
    // instruction cache with the hot roles)
    const uint32_t* off0 = p.csc_off + p.csc_off_off[0];
    const uint32_t* flat0 = p.csc_flat + p.csc_flat_off[0];
    uint32_t* fact = reinterpret_cast<uint32_t*>(smem + kOffFacts);
    const uint64_t G = gridDim.x;
    for (uint32_t k0 = 0;; k0 += kFactSlots) {
      const uint64_t id0 = blockIdx.x + (uint64_t)k0 * G;
      if (id0 >= total) break;
      uint32_t lo = 0, hi = 0;
      {
        const uint64_t id = id0 + (uint64_t)lane * G;
        if (lane < (uint32_t)kFactSlots && id < total) {
          const uint32_t* o =
              off0 + (uint64_t)(id / nkb) * p.csc_off_entries + id % nkb;
          lo = o[0];
          hi = o[1];
        }
      }
#pragma unroll 1
      for (int j = 0; j < kFactSlots; ++j) {
        const uint64_t id = id0 + (uint64_t)j * G;
        if (id >= total) break;
        const uint32_t it = k0 + j;
        const uint32_t l = __shfl_sync(0xffffffffu, lo, j), h = __shfl_sync(0xffffffffu, hi, j);
        const uint32_t qb =
            l + lane < h ? flat0[(uint64_t)(id / nkb) * p.csc_flat_entries + l + lane] : 0u;
        if (it >= (uint32_t)kFactSlots) mbar_wait(bar(FACTE + j), ((it / kFactSlots) - 1) & 1);
        if (lane == 0) {
          fact[j * kFactWords] = l;
          fact[j * kFactWords + 1] = h;
          fact[j * kFactWords + 2] = (uint32_t)(id / nkb);  // unit
          fact[j * kFactWords + 3] = (uint32_t)(id % nkb);  // key block
        }
        fact[j * kFactWords + 4 + lane] = qb;
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(FACTF + j));
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ S / dP issuer
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16(128, 16, false, false);
      for (uint32_t c = 0;; ++c) {
        const uint32_t s = c % kRing, b = c & 1;
        mbar_wait(bar(FULL + s), (c / kRing) & 1);
        if (info[s] & 0x400u) break;
        trace_ev(p, 3, c, 0);
        if (c >= 2) mbar_wait(bar(SFREE + b), ((c >> 1) - 1) & 1);
        trace_ev(p, 3, c, 2);
        fence_proxy_async();  // the gather's cp.async writes → the MMA's async proxy
        fence_after();
        trace_ev(p, 3, c, 3);
        const uint32_t st = sbase + s * kStage;
        const uint32_t tS = tmem + 32 * b, tP = tS + 16;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          mma_bf16(tS, desc_kmajor(st + kQOff + ks * kKStepKMajor),
                   desc_kmajor(st + kKOff + ks * kKStepKMajor), idesc_s, ks > 0);
          mma_bf16(tP, desc_kmajor(st + kGOff + ks * kKStepKMajor),
                   desc_kmajor(st + kVOff + ks * kKStepKMajor), idesc_s, ks > 0);
        }
        commit(bar(SREADY + b));
        trace_ev(p, 3, c, 1);
      }
    }
  } else if (warp == 13) {
    // ------------------------------------------------------------ dK/dV issuer
    // (a second MMA-issuing thread: the S/dP of chunk c+1 and the accumulate
    // of chunk c are issued concurrently)
    if (lane == 0) {
      // N = 32: B' = [dS | P] (16 + 16 columns); dK^T and dV^T are the two
      // diagonal 64 x 16 blocks of the 128 x 32 accumulator
      const uint32_t idesc_a = idesc_bf16(128, 32, true, true);
      uint32_t ai = 0;
      for (uint32_t c = 0;; ++c) {
        const uint32_t s = c % kRing, b = c & 1;
        mbar_wait(bar(FULL + s), (c / kRing) & 1);
        const uint32_t inf = info[s];
        if (inf & 0x400u) break;
        const uint32_t mc = inf & 0xFF, first = (inf >> 8) & 1, last = (inf >> 9) & 1;
        const uint32_t ab = ai % kAB;
        trace_ev(p, 6, c, 0);
        mbar_wait(bar(BREADY + b), (c >> 1) & 1);
        trace_ev(p, 6, c, 1);
        if (first && ai >= (uint32_t)kAB) mbar_wait(bar(AFREE + ab), ((ai / kAB) - 1) & 1);
        trace_ev(p, 6, c, 3);
        fence_proxy_async();
        fence_after();
        trace_ev(p, 6, c, 4);
        const uint32_t st = sbase + s * kStage;
        const uint32_t sb = sbase + kOffB + b * 16384;
        const uint32_t ta = tmem + 64 + 64 * ab;
        for (uint32_t ks = 0; ks < mc; ++ks)  // 16 gathered queries per k-step
          mma_bf16(ta, desc_mnmajor(st + kQOff + ks * kKStepMNMajor, kGOff - kQOff),
                   desc_mnmajor(sb + ks * kKStepMNMajor, 8192), idesc_a,
                   (first && ks == 0) ? 0u : 1u);
        commit(bar(EMPTY + s));
        commit(bar(BFREE + b));
        if (last) {
          commit(bar(AREADY + ab));
          ++ai;
        }
        trace_ev(p, 6, c, 2);
      }
    }
  } else if (warp >= 3 && warp < 7) {
    // ------------------------------------------------------------ softmax warps
    const uint32_t row = 32 * (warp & 3) + lane;  // gathered query (TMEM lane)
    const uint32_t lane_off = (32u * (warp & 3)) << 16;
    const float c2 = p.scale * kLog2e, bias = p.bias2[0];
    for (uint32_t c = 0;; ++c) {
      {
        const uint32_t s = c % kRing, b = c & 1;
        mbar_wait(bar(FULL + s), (c / kRing) & 1);
        if (info[s] & 0x400u) break;
        if (tid == 96) trace_ev(p, 4, c, 0);
        mbar_wait(bar(SREADY + b), (c >> 1) & 1);
        fence_after();
        if (tid == 96) trace_ev(p, 4, c, 2);
        uint32_t sv[32];
        tmem_ld32(tmem + lane_off + 32 * b, sv);  // S (16) | dP (16)
        tmem_ld_wait();
        fence_before();
        mbar_arrive(bar(SFREE + b));
        const uint32_t mc = info[s] & 0xFF;
        const bool valid = row < 16 * mc;
        const float* lse = reinterpret_cast<const float*>(smem + s * kStage + kLseOff);
        const float* Dq = reinterpret_cast<const float*>(smem + s * kStage + kDOff);
        const float nb = bias - (valid ? lse[row] : 0.f), Dr = valid ? Dq[row] : 0.f;
        uint32_t ds[8], pp[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          // packed fp32x2: same per-element operations and rounding
          const float2 x = __ffma2_rn(
              make_float2(__uint_as_float(sv[2 * k]), __uint_as_float(sv[2 * k + 1])),
              make_float2(c2, c2), make_float2(nb, nb));
          float2 pe = make_float2(ex2(x.x), ex2(x.y));
          const float2 g = __fadd2_rn(
              make_float2(__uint_as_float(sv[16 + 2 * k]), __uint_as_float(sv[17 + 2 * k])),
              make_float2(-Dr, -Dr));
          float2 de = __fmul2_rn(pe, g);
          if (!valid) pe = de = make_float2(0.f, 0.f);
          pp[k] = pack_bf16(pe.x, pe.y);
          ds[k] = pack_bf16(de.x, de.y);
        }
        if (c >= 2) mbar_wait(bar(BFREE + b), ((c >> 1) - 1) & 1);
        const uint32_t sb = sbase + kOffB + b * 16384;
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sb + swz(row, 0)),
                     "r"(ds[0]), "r"(ds[1]), "r"(ds[2]), "r"(ds[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sb + swz(row, 1)),
                     "r"(ds[4]), "r"(ds[5]), "r"(ds[6]), "r"(ds[7]));
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sb + swz(row, 2)),
                     "r"(pp[0]), "r"(pp[1]), "r"(pp[2]), "r"(pp[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sb + swz(row, 3)),
                     "r"(pp[4]), "r"(pp[5]), "r"(pp[6]), "r"(pp[7]));
        fence_proxy_async();
        mbar_arrive(bar(BREADY + b));
        if (tid == 96) trace_ev(p, 4, c, 1);
      }
    }
  } else if (warp >= 7) {
    // ------------------------------------------------------------ epilogue warps
    const uint32_t qd = warp & 3;                  // TMEM lane quadrant
    const bool is_v = qd >= 2;                     // rows 64-127: dO^T → dV
    const uint32_t dcol = lane + 32 * (qd & 1);    // head-dim column
    const uint32_t lane_off = (32u * qd) << 16;
    // per item: segment length and the coarse pooled-adjoint rows for this
    // column (B = 16 here: level-l row of token t is t >> 4l), loaded one
    // item ahead into one of two register sets (the loop is unrolled by two
    // so no loaded value is moved or touched before its item; deeper
    // unrolling grew the kernel past what the instruction cache holds)
    constexpr int kEL = 4;  // coarse level slots on this path (L <= 4)
    struct EpiFacts {
      uint32_t o0, o1, unit, kb;
      float v[kEL];
    };
    // Item facts come from the facts warp's smem ring (segment bounds, unit,
    // key block: no dependent global load, no 64-bit division); only the
    // coarse adjoint values are global loads, issued two items ahead.
    const uint32_t* fact = reinterpret_cast<const uint32_t*>(smem + kOffFacts);
    auto issue = [&](uint32_t it, EpiFacts& f) {
      f.o0 = f.o1 = 0;
      f.unit = 0;
      f.kb = 0;
#pragma unroll
      for (int sl = 0; sl < kEL; ++sl) f.v[sl] = 0.f;
      if (blockIdx.x + (uint64_t)it * gridDim.x >= total) return;
      const uint32_t fs = it % kFactSlots;
      mbar_wait(bar(FACTF + fs), (it / kFactSlots) & 1);
      f.o0 = fact[fs * kFactWords];
      f.o1 = fact[fs * kFactWords + 1];
      f.unit = fact[fs * kFactWords + 2];
      f.kb = fact[fs * kFactWords + 3];
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(FACTE + fs));
      const uint32_t unit = f.unit;
      const uint64_t kb = f.kb;
#pragma unroll
      for (int sl = 0; sl < kEL; ++sl) {
        if (sl < (int)p.ncl) {
          const uint32_t l = p.cl_level[sl];
          const float* gk = p.part + (uint64_t)unit * p.part_unit_stride + p.cl_part_off[sl];
          const float* src = is_v ? gk + (uint64_t)p.cl_split[sl] * (p.n >> (4 * l)) * kD : gk;
          f.v[sl] = src[((kb * kBS) >> (4 * l)) * kD + dcol];
        }
      }
    };
    uint32_t ai = 0;
    auto body = [&](const EpiFacts& f) {
      const uint32_t m = f.o1 - f.o0;
      float add = 0.f;
#pragma unroll
      for (int sl = 0; sl < kEL; ++sl) add += f.v[sl];
      const uint32_t unit = f.unit;
      const uint64_t kb = f.kb;
      float acc[16];
      if (m) {
        const uint32_t ab = ai % kAB;
        if (tid == 224) trace_ev(p, 5, ai, 0);
        mbar_wait(bar(AREADY + ab), (ai / kAB) & 1);
        if (tid == 224) trace_ev(p, 5, ai, 1);
        fence_after();
        uint32_t r[16];
        tmem_ld16(tmem + lane_off + 64 + 64 * ab + (is_v ? 16 : 0), r);
        tmem_ld_wait();
        fence_before();
        mbar_arrive(bar(AFREE + ab));
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = __uint_as_float(r[j]) * (is_v ? 1.f : p.scale);
        ++ai;
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.f;
      }
      const uint64_t o = ((uint64_t)unit * p.n + kb * kBS) * kD + dcol;
      if (p.grad_bf16) {
        bf16* dst = reinterpret_cast<bf16*>(is_v ? p.dv : p.dk) + o;
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[(uint64_t)j * kD] = __float2bfloat16_rn(acc[j] + add);
      } else {
        float* dst = (is_v ? p.dv : p.dk) + o;
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[(uint64_t)j * kD] = acc[j] + add;
      }
    };
    const uint64_t G = gridDim.x;
    EpiFacts fa, fb, fc;  // items it, it+1, it+2 (unrolled by three: no register moves)
    issue(0, fa);
    issue(1, fb);
    for (uint32_t it = 0; blockIdx.x + (uint64_t)it * G < total; it += 3) {
      issue(it + 2, fc);
      body(fa);
      if (blockIdx.x + (uint64_t)(it + 1) * G >= total) break;
      issue(it + 3, fa);
      body(fb);
      if (blockIdx.x + (uint64_t)(it + 2) * G >= total) break;
      issue(it + 4, fb);
      body(fc);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// backward: coarse dK'/dV' — persistent, warp-specialised tcgen05 version
// ---------------------------------------------------------------------------
// Same work items and partial layout as tc5_kv_rows_kernel (one item = level
// l, selection row, query slice, group of 8 selected blocks = 128 keys as M),
// but one CTA per SM walks the items and every stage overlaps the next:
//   warp 15 (1 lane)   TMA: 64-query Q / dO tiles (2-D boxes) + lse, D (1-D
//                      bulk) → 4-stage ring
//   warp 0             cp.async gather of the item's key tiles (K', V' hi
//                      [+ lo]) → completes via cp.async.mbarrier.arrive
//   warp 1 (1 lane)    S^T = K' Q^T, dP^T = V' dO^T → TMEM (double buffer)
//   warps 4-11         thread = key (TMEM lane) × 32 queries: P^T, dS^T → bf16
//                      smem (double buffer)
//   warp 2 (1 lane)    dV' += P^T dO, dK' += dS^T Q → TMEM (double buffer per
//                      item)
//   warps 3, 12-14     epilogue: the item's raw 128×64 dK', dV' partial → HBM
// Replaces P/src/attention_grad.cpp:136-162 (levels 1..L-1).
namespace rows2 {
constexpr int kKeys = 128, kQT = 64;
constexpr int kArr = kKeys * 128;                 // one 128-key array: 16 KB
constexpr int kQStage = 17408;                    // Q 8 KB | dO 8 KB | lse | D, 1 KB aligned
template <bool LO>
struct L {
  static constexpr int kKeyBufs = LO ? 1 : 2;
  static constexpr int kQRing = LO ? 5 : 4;
  static constexpr int kKeyBuf = (LO ? 3 : 2) * kArr;  // Khi, Vhi (, Klo)
  static constexpr int kOffQ = kKeyBufs * kKeyBuf;
  static constexpr int kOffP = kOffQ + kQRing * kQStage;  // P^T, dS^T x 2
  // reduce-add staging per epilogue warp: kStgBufs x (2 blocks x one 16-row,
  // 32-column fp32 SW128 box of 2 KB)
  static constexpr int kStgBufs = 1;
  static constexpr int kOffStg = kOffP + 2 * 2 * 16384;
  static constexpr int kOffBar = kOffStg + 4 * kStgBufs * 4096;
  static constexpr int kSmem = kOffBar + 256;
  static_assert(kSmem <= 232448, "rows2 shared memory over the 227 KB opt-in limit");
};
enum { KFULL = 0, KEMPTY = 2, QFULL = 4, QEMPTY = 9, SREADY = 14, SFREE = 16, PREADY = 18,
       PFREE = 20, AREADY = 22, AFREE = 24, NBAR = 26 };  // Q ring up to 5 slots
constexpr int kThreads = 16 * 32;
constexpr uint32_t kTmemCols = 512;  // S^T|dP^T x 2 at [0, 256), dK'|dV' x 2 at [256, 512)
}  // namespace rows2

template <bool LO>
__global__ void __launch_bounds__(rows2::kThreads, 1)
    tc5_rows2_kernel(const __grid_constant__ TcParams p, const __grid_constant__ TmaMaps m,
                     uint32_t li, uint32_t units) {
  using namespace llsa_umma;
  using namespace rows2;
  using Lay = L<LO>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  auto bar = [&](int i) { return sbase + Lay::kOffBar + 8u * i; };
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + Lay::kOffBar + NBAR * 8);
  const uint64_t tpu = p.rl_tasks[li + 1] - p.rl_tasks[li];
  const uint64_t total = tpu * units;
  const uint32_t level = p.rl_level[li], slices = p.rl_slices[li];
  const bool top = p.rl_top[li] != 0;
  const uint32_t groups = p.rl_groups[li];
  const uint64_t span = top ? p.n : p.pow[level + 1], qs = p.rl_qs[li];
  const uint32_t ntiles = (uint32_t)(qs / kQT);
  const uint64_t G = gridDim.x;
  // item → (unit, row, slice, group)
  auto decode = [&](uint64_t id, uint32_t& unit, uint64_t& row, uint32_t& slice,
                    uint32_t& group) {
    unit = (uint32_t)(id / tpu);
    const uint64_t task = id % tpu;
    group = (uint32_t)(task % groups);
    const uint64_t rs = task / groups;
    slice = (uint32_t)(rs % slices);
    row = rs / slices;
  };
  if (warp == 0) tmem_alloc(smem_u32(tslot), kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(KFULL + i), 32);  // every gather lane, via its copies
      mbar_init(bar(KEMPTY + i), 1);
      mbar_init(bar(SREADY + i), 1);
      mbar_init(bar(SFREE + i), 256);
      mbar_init(bar(PREADY + i), 256);
      mbar_init(bar(PFREE + i), 1);
      mbar_init(bar(AREADY + i), 1);
      mbar_init(bar(AFREE + i), 128);
    }
    for (int i = 0; i < Lay::kQRing; ++i) {
      mbar_init(bar(QFULL + i), 1);
      mbar_init(bar(QEMPTY + i), 1);
    }
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 15) {
    // ------------------------------------------------------------ Q / dO TMA
    if (lane == 0) {
      prefetch_map(&m.q);
      prefetch_map(&m.g);
      uint32_t t = 0;
      for (uint64_t id = blockIdx.x; id < total; id += G) {
        uint32_t unit, slice, group;
        uint64_t row;
        decode(id, unit, row, slice, group);
        const uint64_t q_begin = row * span + (uint64_t)slice * qs;
        const uint64_t ro = (uint64_t)unit * p.n;
        for (uint32_t j = 0; j < ntiles; ++j, ++t) {
          const uint32_t s = t % Lay::kQRing;
          trace_ev(p, 2, t, 0);
          if (t >= (uint32_t)Lay::kQRing) mbar_wait(bar(QEMPTY + s), ((t / Lay::kQRing) - 1) & 1);
          trace_ev(p, 2, t, 1);
          const uint32_t dst = sbase + Lay::kOffQ + s * kQStage;
          const uint64_t t0 = q_begin + (uint64_t)j * kQT;
          mbar_expect_tx(bar(QFULL + s), 2 * kQT * 128 + 2 * kQT * 4);
          tma_load_2d(dst, &m.q, 0, (int)(ro + t0), bar(QFULL + s));
          tma_load_2d(dst + kQT * 128, &m.g, 0, (int)(ro + t0), bar(QFULL + s));
          bulk_load(dst + 2 * kQT * 128, p.lse2 + ro + t0, kQT * 4, bar(QFULL + s));
          bulk_load(dst + 2 * kQT * 128 + kQT * 4, p.drow + ro + t0, kQT * 4, bar(QFULL + s));
        }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ key gather
    const Block16Lane bl = block16_lane(lane);
    const uint64_t nblk = p.n / p.pow[level + 1];
    auto key_ids = [&](uint64_t id) -> uint32_t {  // lane < 8: the item's block id
      if (id >= total || lane >= 8) return 0u;
      uint32_t unit, slice, group;
      uint64_t row;
      decode(id, unit, row, slice, group);
      // K not a multiple of 8: the last group's tail lanes gather block 0 as
      // dummy keys; their dK'/dV' rows are never read by rows_reduce_kernel
      if (top) return group * 8 + lane < nblk ? group * 8 + lane : 0u;
      if (group * 8 + lane >= p.K) return 0u;
      return p.tables[(uint64_t)unit * p.table_entries + p.table_off[level] + row * p.K +
                      group * 8 + lane];
    };
    // ids of item i+1 load while item i is issued; range-checked at use so
    // the load is not waited for early
    uint32_t ids_next = key_ids(blockIdx.x);
    uint32_t it = 0;
    for (uint64_t id = blockIdx.x; id < total; id += G, ++it) {
      uint32_t ids = ids_next;
      ids_next = key_ids(id + G);
      if (ids >= nblk) {
        raise_flag(p.flag, llsa_dev::kErrIndex);
        ids = 0;
      }
      const uint32_t kb = it % Lay::kKeyBufs;
      if (lane == 0) trace_ev(p, 1, it, 0);
      if (it >= (uint32_t)Lay::kKeyBufs)
        mbar_wait(bar(KEMPTY + kb), ((it / Lay::kKeyBufs) - 1) & 1);
      if (lane == 0) trace_ev(p, 1, it, 1);
      const uint32_t unit = (uint32_t)(id / tpu);
      const uint32_t dst = sbase + kb * Lay::kKeyBuf;
      const uint64_t base = (uint64_t)unit * p.pyr_rows + p.pyr_off[level];
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const uint64_t o = (base + (uint64_t)__shfl_sync(0xffffffffu, ids, b) * kBS) * kD;
        load_block16_async(dst + b * 2048, p.khi + o, bl, lane);
        load_block16_async(dst + kArr + b * 2048, p.vhi + o, bl, lane);
        if (LO) load_block16_async(dst + 2 * kArr + b * 2048, p.klo + o, bl, lane);
      }
      cp_async_mbar_arrive(bar(KFULL + kb));
      if (lane == 0) trace_ev(p, 1, it, 2);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ S^T / dP^T issuer
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16(128, kQT, false, false);
      uint32_t t = 0, it = 0;
      for (uint64_t id = blockIdx.x; id < total; id += G, ++it) {
        const uint32_t kb = it % Lay::kKeyBufs;
        const uint32_t sK = sbase + kb * Lay::kKeyBuf;
        for (uint32_t j = 0; j < ntiles; ++j, ++t) {
          const uint32_t s = t % Lay::kQRing, b = t & 1;
          trace_ev(p, 3, t, 0);
          if (j == 0) mbar_wait(bar(KFULL + kb), (it / Lay::kKeyBufs) & 1);
          trace_ev(p, 3, t, 1);
          mbar_wait(bar(QFULL + s), (t / Lay::kQRing) & 1);
          trace_ev(p, 3, t, 2);
          if (t >= 2) mbar_wait(bar(SFREE + b), ((t >> 1) - 1) & 1);
          trace_ev(p, 3, t, 3);
          fence_proxy_async();  // gathered key tiles (cp.async) → async proxy
          fence_after();
          const uint32_t sQ = sbase + Lay::kOffQ + s * kQStage, sG = sQ + kQT * 128;
          const uint32_t tS = tmem + 128 * b, tP = tS + 64;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bq = desc_kmajor(sQ + ks * kKStepKMajor);
            const uint64_t bg = desc_kmajor(sG + ks * kKStepKMajor);
            mma_bf16(tS, desc_kmajor(sK + ks * kKStepKMajor), bq, idesc_s, ks > 0);
            mma_bf16(tP, desc_kmajor(sK + kArr + ks * kKStepKMajor), bg, idesc_s, ks > 0);
            if (LO) mma_bf16(tS, desc_kmajor(sK + 2 * kArr + ks * kKStepKMajor), bq, idesc_s, 1);
          }
          commit(bar(SREADY + b));
          trace_ev(p, 3, t, 4);
          // the key tiles are read only by these MMAs: the gather may refill
          // the buffer while the item's last softmax / accumulate run
          if (j + 1 == ntiles) commit(bar(KEMPTY + kb));
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ dK'/dV' issuer
    if (lane == 0) {
      const uint32_t idesc_kv = idesc_bf16(128, kD, false, true);
      uint32_t t = 0, it = 0;
      for (uint64_t id = blockIdx.x; id < total; id += G, ++it) {
        const uint32_t kb = it % Lay::kKeyBufs, ab = it & 1;
        const uint32_t tDK = tmem + 256 + 128 * ab, tDV = tDK + 64;
        for (uint32_t j = 0; j < ntiles; ++j, ++t) {
          const uint32_t s = t % Lay::kQRing, b = t & 1;
          trace_ev(p, 6, t, 0);
          mbar_wait(bar(PREADY + b), (t >> 1) & 1);
          trace_ev(p, 6, t, 1);
          if (j == 0 && it >= 2) mbar_wait(bar(AFREE + ab), ((it >> 1) - 1) & 1);
          trace_ev(p, 6, t, 2);
          fence_after();
          const uint32_t sQ = sbase + Lay::kOffQ + s * kQStage, sG = sQ + kQT * 128;
          const uint32_t sPT = sbase + Lay::kOffP + b * 32768, sDST = sPT + 16384;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {  // K = 64 queries
            mma_bf16(tDV, desc_kmajor(sPT + ks * kKStepKMajor),
                     desc_mnmajor(sG + ks * kKStepMNMajor, 8192), idesc_kv, (j | ks) > 0);
            mma_bf16(tDK, desc_kmajor(sDST + ks * kKStepKMajor),
                     desc_mnmajor(sQ + ks * kKStepMNMajor, 8192), idesc_kv, (j | ks) > 0);
          }
          commit(bar(QEMPTY + s));
          commit(bar(PFREE + b));
          trace_ev(p, 6, t, 3);
          if (j + 1 == ntiles) commit(bar(AREADY + ab));
        }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ softmax warps
    const uint32_t krow = 32 * (warp & 3) + lane;   // key (TMEM lane)
    const uint32_t qh = (warp - 4) >> 2;            // query columns [32 qh, +32)
    const uint32_t lane_off = (32u * (warp & 3)) << 16;
    const float c2 = p.scale * kLog2e, bias = p.bias2[level];
    const uint32_t ntot = (uint32_t)((total + G - 1 - blockIdx.x) / G) * ntiles;
    for (uint32_t t = 0; t < ntot; ++t) {
      const uint32_t s = t % Lay::kQRing, b = t & 1;
      if (tid == 128) trace_ev(p, 4, t, 0);
      mbar_wait(bar(QFULL + s), (t / Lay::kQRing) & 1);
      mbar_wait(bar(SREADY + b), (t >> 1) & 1);
      if (tid == 128) trace_ev(p, 4, t, 1);
      fence_after();
      uint32_t sv[32], pv[32];
      tmem_ld32(tmem + lane_off + 128 * b + 32 * qh, sv);
      tmem_ld32(tmem + lane_off + 128 * b + 64 + 32 * qh, pv);
      // the P^T / dS^T slot is needed only for the stores: wait for it while
      // the TMEM loads are in flight
      if (t >= 2) mbar_wait(bar(PFREE + b), ((t >> 1) - 1) & 1);
      if (tid == 128) trace_ev(p, 4, t, 2);
      tmem_ld_wait();
      fence_before();
      mbar_arrive(bar(SFREE + b));
      const float* lse = reinterpret_cast<const float*>(smem + Lay::kOffQ + s * kQStage +
                                                        2 * kQT * 128) + 32 * qh;
      const float* Dq = lse + kQT;
      const uint32_t sPT = sbase + Lay::kOffP + b * 32768, sDST = sPT + 16384;
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint32_t pk[4], dk4[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          // packed fp32x2 over queries i, i+1: same per-element rounding
          const int i = c8 * 8 + h * 2;
          const float2 l2 = *reinterpret_cast<const float2*>(lse + i);
          const float2 d2 = *reinterpret_cast<const float2*>(Dq + i);
          const float2 nb2 = __fadd2_rn(make_float2(bias, bias), make_float2(-l2.x, -l2.y));
          const float2 x = __ffma2_rn(
              make_float2(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])),
              make_float2(c2, c2), nb2);
          const float2 pe = make_float2(ex2(x.x), ex2(x.y));
          const float2 g = __fadd2_rn(
              make_float2(__uint_as_float(pv[i]), __uint_as_float(pv[i + 1])),
              make_float2(-d2.x, -d2.y));
          const float2 de = __fmul2_rn(pe, g);
          pk[h] = pack_bf16(pe.x, pe.y);
          dk4[h] = pack_bf16(de.x, de.y);
        }
        const uint32_t chunk = qh * 4 + c8;
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sPT + swz(krow, chunk)),
                     "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(sDST + swz(krow, chunk)),
                     "r"(dk4[0]), "r"(dk4[1]), "r"(dk4[2]), "r"(dk4[3]));
      }
      fence_proxy_async();
      mbar_arrive(bar(PREADY + b));
      if (tid == 128) trace_ev(p, 4, t, 3);
    }
  } else if ((warp == 3 || warp >= 12) && p.rows_atomic) {
    // ------------------------------------------------------------ epilogue warps
    // (reduce form) each warp's 32 keys = two 16-key blocks of the group:
    // scaled by the level's pooling coefficients, staged as SW128 fp32 boxes
    // and added into the level slot by TMA reductions (L2-resident; no raw
    // partials, no rows_reduce_kernel).  Summation order across rows is
    // unordered: LLSA_DETERMINISTIC=1 selects the partial + ordered-sum form.
    const uint32_t qd = warp & 3;
    const uint32_t lane_off = (32u * qd) << 16;
    const uint32_t rr = lane & 15, bb = lane >> 4;
    const uint32_t stg = sbase + Lay::kOffStg + qd * Lay::kStgBufs * 4096;
    uint32_t sl = 0;
    while (sl < p.ncl && p.cl_level[sl] != level) ++sl;
    const float ck = p.cl_ck[sl], cv = p.cl_cv[sl];
    const uint64_t tok_l = p.n / p.pow[level];
    const uint64_t nblk = p.n / p.pow[level + 1];
    uint32_t it = 0, nb = 0;  // nb: bulk groups committed by lane 0
    for (uint64_t id = blockIdx.x; id < total; id += G, ++it) {
      uint32_t unit, slice, group;
      uint64_t row;
      decode(id, unit, row, slice, group);
      // this warp's two block ids (lanes 0, 1); ~0u: dummy keys, not added
      uint32_t blk = ~0u;
      if (lane < 2) {
        const uint32_t j = group * 8 + 2 * qd + lane;
        if (top)
          blk = j < nblk ? j : ~0u;
        else if (j < p.K)
          blk = p.tables[(uint64_t)unit * p.table_entries + p.table_off[level] + row * p.K + j];
        if (blk >= nblk) blk = ~0u;  // out of range (flagged by the gather warp): not added
      }
      const uint32_t blk0 = __shfl_sync(0xffffffffu, blk, 0),
                     blk1 = __shfl_sync(0xffffffffu, blk, 1);
      const uint64_t y0 = ((uint64_t)unit * p.part_unit_stride + p.cl_part_off[sl]) / kD;
      const uint32_t ab = it & 1;
      mbar_wait(bar(AREADY + ab), (it >> 1) & 1);
      fence_after();
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {  // dK' cols 0-31, 32-63, then dV' (+64 in TMEM)
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + 256 + 128 * ab + 32 * q4, r);
        tmem_ld_wait();
        if (q4 == 3) {
          fence_before();
          mbar_arrive(bar(AFREE + ab));
        }
        // the staging buffer's previous reduction must have read it
        if (lane == 0 && nb >= (uint32_t)Lay::kStgBufs) bulk_wait_read_n<Lay::kStgBufs - 1>();
        __syncwarp();
        const uint32_t buf = stg + (q4 % Lay::kStgBufs) * 4096 + bb * 2048 + rr * 128;
        const float c = q4 < 2 ? ck : cv;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4)
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(
                           buf + ((c4 ^ (rr & 7)) << 4)),
                       "f"(__uint_as_float(r[4 * c4]) * c), "f"(__uint_as_float(r[4 * c4 + 1]) * c),
                       "f"(__uint_as_float(r[4 * c4 + 2]) * c),
                       "f"(__uint_as_float(r[4 * c4 + 3]) * c));
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          const uint32_t src = stg + (q4 % Lay::kStgBufs) * 4096;
          const uint64_t yb = y0 + (q4 >= 2 ? (uint64_t)p.cl_split[sl] * tok_l : 0);
          const int x = 32 * (q4 & 1);
          if (blk0 != ~0u) tma_reduce_add_2d(&m.o, src, x, (int)(yb + (uint64_t)blk0 * kBS));
          if (blk1 != ~0u)
            tma_reduce_add_2d(&m.o, src + 2048, x, (int)(yb + (uint64_t)blk1 * kBS));
          bulk_commit();
          ++nb;
        }
      }
    }
    if (lane == 0) bulk_wait_all();
  } else if (warp == 3 || warp >= 12) {
    // ------------------------------------------------------------ epilogue warps
    const uint32_t krow = 32 * (warp & 3) + lane;
    const uint32_t lane_off = (32u * (warp & 3)) << 16;
    uint32_t it = 0;
    for (uint64_t id = blockIdx.x; id < total; id += G, ++it) {
      uint32_t unit, slice, group;
      uint64_t row;
      decode(id, unit, row, slice, group);
      const uint32_t ab = it & 1;
      mbar_wait(bar(AREADY + ab), (it >> 1) & 1);
      fence_after();
      // transposed partial [64 d][128 keys] (dK', then dV'): for one d a
      // warp's 32 keys are one coalesced 128-byte store
      const uint64_t pidx = (row * slices + slice) * groups + group;
      float* dst = p.rpart + (uint64_t)unit * p.rpart_unit_stride + p.rl_part_off[li] +
                   pidx * (2 * kKeys * kD) + krow;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {  // dK' cols 0-63 then dV' (+64 in TMEM)
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + 256 + 128 * ab + 32 * q4, r);
        tmem_ld_wait();
        if (q4 == 3) {  // the accumulators are in registers: release them before storing
          fence_before();
          mbar_arrive(bar(AFREE + ab));
        }
        float* d = dst + (q4 >= 2 ? kKeys * kD : 0) + (uint64_t)(32 * (q4 & 1)) * kKeys;
#pragma unroll
        for (int i = 0; i < 32; ++i) d[(uint64_t)i * kKeys] = __uint_as_float(r[i]);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// split 0 of coarse slots [s0, s1) ← coefficient · Σ_splits (fixed order)
__global__ void reduce_parts_kernel(TcParams p, uint32_t units, uint32_t s0, uint32_t s1) {
  for (uint32_t sl = s0; sl < s1; ++sl) {
    const uint64_t tok = p.n / p.pow[p.cl_level[sl]];
    const uint64_t elems = tok * kD;
    const uint32_t ns = p.cl_split[sl];
    const uint64_t total = elems * units * 2;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
         x += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t u = x / (2 * elems), rem = x % (2 * elems);
      const uint32_t which = (uint32_t)(rem / elems);  // 0: dk, 1: dv
      const uint64_t e = rem % elems;
      float* base = p.part + u * p.part_unit_stride + p.cl_part_off[sl] +
                    (uint64_t)which * ns * elems + e;
      float s = 0.f;
      for (uint32_t i = 0; i < ns; ++i) s += base[(uint64_t)i * elems];
      base[0] = s * (which ? p.cl_cv[sl] : p.cl_ck[sl]);
    }
  }
}

unsigned grid_for(uint64_t threads, int block) {
  uint64_t blocks = (threads + block - 1) / block;
  const uint64_t cap = 148ull * 16;
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

constexpr uint32_t kMaxCoarsePasses = 3;

uint32_t coarse_entries(const Geometry& g) {
  return g.K * (g.enrich_lim() - 1) + (g.Le == g.L ? (uint32_t)g.level_blocks(g.L) : 0u);
}

// Coarse kv slots: levels 1..lim-1, then the coarsest when L_e = L.
// The tcgen05 row-major coarse dK/dV kernel handles levels 1..lim-1 when the
// selection width is a multiple of 8 blocks (one 128-key group = M).
// dev: LLSA_TRACE_ONLY=rows2 records the trace events of the level-1
// tc5_rows2 launch only (the other kernels run untraced)
bool trace_only_rows2() {
  const char* e = getenv("LLSA_TRACE_ONLY");
  return e && strcmp(e, "rows2") == 0;
}

bool rows_path(const Geometry& g) {
  const char* e = getenv("LLSA_NO_TCGEN05");
  return !(e && e[0] == '1') && g.enrich_lim() >= 2;
}

// tcgen05 forward: every coarse entry's scores fit the TMEM S block
bool fwd5_path(const Geometry& g) {
  const char* e = getenv("LLSA_NO_TCGEN05");
  const char* f = getenv("LLSA_FWD5");
  const uint32_t nce = coarse_entries(g);
  // coarse sets past the 24-entry TMEM budget run as several passes of at
  // most 24 entries (TcParams::ce_base / fine_mode)
  return !(e && e[0] == '1') && !(f && f[0] == '0') && nce >= 1 &&
         nce <= kMaxCoarsePasses * fw5::kMaxEntries && g.K <= 32;
}

// tcgen05 fine dK/dV (key-major, gathered queries as M)
bool kvf_path(const Geometry& g) {
  const char* e = getenv("LLSA_NO_TCGEN05");
  const char* f = getenv("LLSA_KVF");
  // the epilogue holds at most 4 coarse level slots per item (ncl <= L)
  return !(e && e[0] == '1') && !(f && f[0] == '0') && g.L <= 4;
}

// fused tcgen05 dq: coarse chunks of <= 4 entries, K <= 32 fine blocks per row
bool dqf_path(const Geometry& g) {
  const char* e = getenv("LLSA_NO_TCGEN05");
  const char* f = getenv("LLSA_DQF");
  const uint32_t nce = coarse_entries(g);
  return !(e && e[0] == '1') && !(f && f[0] == '0') && nce >= 1 &&
         nce <= kMaxCoarsePasses * dqf::kMaxEntries && g.K <= 32;
}

// Whether the coarsest level (L_e = L: every query attends its n/B^(L+1)
// blocks) also runs on the tcgen05 row kernel, as one row of all n queries
// whose key groups are the level's blocks (dummy-padded to 8).
// With fewer than 4 coarsest blocks (C3: one) the 128-key groups would be
// mostly dummy keys and the key-major tc_kv kernel is faster (measured: C3
// 0.465 → 0.551 ms for the coarse stages; C2, C5 with four blocks gain).
bool rows_top(const Geometry& g) {
  const char* r2 = getenv("LLSA_ROWS2");
  const char* t = getenv("LLSA_ROWS_TOP");
  return rows_path(g) && g.Le == g.L && g.level_blocks(g.L) >= 4 && !(r2 && r2[0] == '0') &&
         !(t && t[0] == '0');
}

void rows_layout(const Geometry& g, TcParams& P) {
  P.rows_on = rows_path(g) ? 1u : 0u;
  P.rl_count = 0;
  P.groups = (g.K + 7) / 8;  // a last partial group carries dummy keys (block 0)
  uint64_t tasks = 0, off = 0;
  auto add = [&](uint32_t l, uint64_t span, uint64_t rows, uint32_t groups, bool top) {
    const uint32_t i = P.rl_count++;
    const uint64_t qs = span < 1024 ? span : 1024;
    P.rl_level[i] = l;
    P.rl_qs[i] = qs;
    P.rl_slices[i] = (uint32_t)(span / qs);
    P.rl_groups[i] = groups;
    P.rl_top[i] = top ? 1u : 0u;
    P.rl_tasks[i] = tasks;
    const uint64_t parts = rows * P.rl_slices[i] * groups;
    tasks += parts;
    P.rl_part_off[i] = off;
    off += parts * 2 * rows::kKeys * kD;
  };
  if (P.rows_on) {
    for (uint32_t l = 1; l < g.enrich_lim(); ++l)
      add(l, g.pow[l + 1], g.level_blocks(l), P.groups, false);
    if (rows_top(g))
      add(g.L, g.n, 1, (uint32_t)((g.level_blocks(g.L) + 7) / 8), true);
  }
  P.rl_tasks[P.rl_count] = tasks;
  P.rpart_unit_stride = off;
}

// units > 0: the launch's batch is known, so a lone key-major coarse slot (C3:
// the coarsest level's one 16-key block) gets the split count that fills
// whole waves of 4-warp CTAs, one per SM (C3 × 16: 32 → 37 splits, 0.058 →
// 0.052 ms; an extra partial wave costs more than the smaller tasks gain).
// reserve: workspace sizing — the lone slot's layout at the largest split
// count, so a workspace sized on one device fits a launch on any other.
void coarse_slots(const Geometry& g, TcParams& P, uint32_t units = 0, bool reserve = false) {
  P.ncl = 0;
  uint64_t tasks = 0, off = 0;
  const bool rows = rows_path(g);
  uint32_t kv_slots = 0;
  for (uint32_t l = 1; l < g.enrich_lim(); ++l) kv_slots += rows ? 0u : 1u;
  if (g.Le == g.L && !(rows && rows_top(g))) ++kv_slots;
  auto add = [&](uint32_t l, uint64_t avg_queries, uint64_t blocks) {
    const uint32_t i = P.ncl++;
    static const uint64_t qpt = [] {  // queries per split task (dev knob)
      const char* e = getenv("LLSA_KV_SPLIT_Q");
      return e ? (uint64_t)atoll(e) : 2048ull;
    }();
    uint64_t s = avg_queries / qpt;
    s = s < 1 ? 1 : s > 256 ? 256 : s;
    const bool on_rows = rows && (l < g.enrich_lim() || rows_top(g));
    // (not in the ordered mode, whose per-unit results must not depend on the
    // batch: the fp32 split sums would change with the split count)
    const char* det = getenv("LLSA_DETERMINISTIC");
    const bool ordered = det && det[0] == '1';
    if (units && kv_slots == 1 && !on_rows && !getenv("LLSA_KV_SPLIT_Q") &&
        (!ordered || reserve)) {
      const uint64_t slots = (uint64_t)num_sms() * kKvWarps;  // warps of one wave
      const uint64_t per = (uint64_t)units * blocks;             // warps per split
      uint64_t waves = (per * s + slots / 2) / slots;
      waves = waves < 1 ? 1 : waves;
      uint64_t fit = waves * slots / per;
      if (fit >= 1 && fit <= 256) s = fit;
      if (reserve) s = 256;
    }
    if (on_rows) s = 1;  // reduced by rows_reduce_kernel
    P.cl_level[i] = l;
    P.cl_split[i] = (uint32_t)s;
    P.cl_tasks[i] = tasks;
    tasks += blocks * s;
    P.cl_part_off[i] = off;
    off += 2 * s * g.level_tokens(l) * kD;
    const float gain = g.mode == 0 ? (float)g.pow[l] : 1.f;
    P.cl_ck[i] = g.scale * gain / (float)g.pow[l];
    P.cl_cv[i] = gain / (float)g.pow[l];
  };
  for (uint32_t l = 1; l < g.enrich_lim(); ++l)
    add(l, (uint64_t)g.K * g.pow[l + 1], g.level_blocks(l));
  if (g.Le == g.L) add(g.L, g.n, g.level_blocks(g.L));
  P.cl_tasks[P.ncl] = tasks;
  P.part_unit_stride = off;
}

TcParams make_params(const Geometry& g, uint32_t units) {
  TcParams P{};
  P.n = g.n;
  P.pyr_rows = g.pyr_rows;
  P.table_entries = g.table_entries;
  P.csc_off_entries = g.csc_off_entries;
  P.csc_flat_entries = g.csc_flat_entries;
  P.K = g.K;
  P.L = g.L;
  P.Le = g.Le;
  P.lim = g.enrich_lim();
  P.nce = coarse_entries(g);
  P.scale = g.scale;
  for (int l = 0; l < kMaxLevels + 2; ++l) {
    P.pow[l] = g.pow[l];
    P.pyr_off[l] = g.pyr_off[l];
    P.bias2[l] = g.mode == 1 && g.pow[l] ? std::log((float)g.pow[l]) * kLog2e : 0.f;
  }
  for (int l = 0; l < kMaxLevels + 1; ++l) {
    P.table_off[l] = g.table_off[l];
    P.csc_off_off[l] = g.csc_off_off[l];
    P.csc_flat_off[l] = g.csc_flat_off[l];
  }
  P.flag = device_flag();
  const char* dg = getenv("LLSA_DBG");
  P.dbg = dg ? (uint32_t)atoi(dg) : 0u;
  const char* tr = getenv("LLSA_TRACE");
  P.trace = tr && tr[0] == '1' ? 1u : 0u;
  // (tc_backward gives the rows2 level-1 launch its own flag in that mode)
  if (trace_only_rows2()) {
    P.trace_rows2 = P.trace;
    P.trace = 0;
  }
  const char* hl = getenv("LLSA_HILO_LEVEL");  // default: hi + lo on every coarse level
  P.hilo_level = hl ? (uint32_t)atoi(hl) : 1u;
  coarse_slots(g, P, units);
  rows_layout(g, P);
  // rows2 adds its items into the level slots with TMA reductions (fp32,
  // unordered); LLSA_DETERMINISTIC=1 keeps the raw partials and sums them in
  // a fixed order (rows_reduce_kernel): bitwise run-to-run reproducible
  const char* det = getenv("LLSA_DETERMINISTIC");
  const bool unordered = !(det && det[0] == '1');
  P.rows_atomic = P.rows_on && unordered ? 1u : 0u;
  P.kv_atomic = unordered ? 1u : 0u;
  return P;
}

}  // namespace

// dq, dk, dv written once each, by tc5_dqf_kernel and tc5_kvf_kernel: they
// can be written as bf16 directly
bool tc_bf16_grads_ok(const Geometry& g) {
  return dqf_path(g) && kvf_path(g) && coarse_entries(g) <= dqf::kMaxEntries;  // one dq pass
}

bool tc_supported(const Geometry& g, llsa_dtype dt) {
  return dt == LLSA_BF16 && g.d == 64 && g.B == 16 && g.safe && g.n % kTileQ == 0 &&
         g.L >= 1 && g.L <= 4 && coarse_entries(g) <= (uint32_t)kMaxCoarse;
}

size_t tc_buffer_bytes(const Geometry& g, uint32_t units) {
  const size_t a = ((size_t)units * g.pyr_rows * kD * 2 + 255) & ~size_t(255);
  return 4 * a;
}

void tc_carve(const Geometry& g, uint32_t units, char* base, TcBuffers* out) {
  const size_t a = ((size_t)units * g.pyr_rows * kD * 2 + 255) & ~size_t(255);
  out->k_hi = reinterpret_cast<bf16*>(base);
  out->k_lo = reinterpret_cast<bf16*>(base + a);
  out->v_hi = reinterpret_cast<bf16*>(base + 2 * a);
  out->v_lo = reinterpret_cast<bf16*>(base + 3 * a);
}

// 2-D TMA map over a [rows][64] bf16 tensor, boxes of box_rows × 64,
// 128-byte swizzle (the K-major / MN-major SW128 operand layout).
// With f32 = true: a [rows][64] fp32 tensor, boxes of box_rows × 32 (the
// output tile store).
static llsa_status make_tma_map(CUtensorMap* map, const void* base, uint64_t rows,
                                uint32_t box_rows, bool f32 = false) {
  const cuuint64_t dims[2] = {(cuuint64_t)kD, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)kD * (f32 ? 4 : 2)};
  const cuuint32_t box[2] = {(cuuint32_t)(f32 ? 32 : kD), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  // resolved through the runtime so the library has no link-time libcuda
  // dependency (it must load on hosts without a driver)
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !fn)
      return fail(LLSA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const CUresult r = encode(
      map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
      const_cast<void*>(base), dims, strides, box,
      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LLSA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return LLSA_OK;
}

static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 ? 0 : dev;
}

// SM count of the current device (cached per device; a process may drive
// several GPUs, one handle each).
static int num_sms() {
  static std::atomic<int> cache[64];
  const int dev = current_device() & 63;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Kernel attributes (the >48 KB dynamic shared memory opt-ins) are per device
// context: one "done" bit per device.  Two threads racing on the same device
// both set the attributes, which is harmless.
static bool attrs_done(const std::atomic<uint64_t>& mask) {
  return (mask.load(std::memory_order_acquire) >> (current_device() & 63)) & 1;
}
static void mark_attrs_done(std::atomic<uint64_t>& mask) {
  mask.fetch_or(1ull << (current_device() & 63), std::memory_order_release);
}

static llsa_status launch_prep(const Geometry& g, uint32_t units, const float* pk,
                               const float* pv, const TcBuffers& tb, cudaStream_t s) {
  float gl[5] = {1, 1, 1, 1, 1};
  for (uint32_t l = 1; l <= g.L && l <= 4; ++l) gl[l] = g.mode == 0 ? (float)g.pow[l] : 1.f;
  const uint64_t total = (uint64_t)units * g.pyr_rows * kD;
  prep_kernel<<<grid_for(total, 256), 256, 0, s>>>(
      pk, pv, tb.k_hi, tb.k_lo, tb.v_hi, tb.v_lo, g.pyr_rows, units, gl[1], gl[2], gl[3],
      gl[4], g.L >= 2 ? g.pyr_off[2] : ~0ull, g.L >= 3 ? g.pyr_off[3] : ~0ull,
      g.L >= 4 ? g.pyr_off[4] : ~0ull);
  count_launch();
  LLSA_LAUNCH_CHECK("prep_kernel");
  return LLSA_OK;
}

llsa_status tc_prep(const Geometry& g, uint32_t units, const float* pyr_k, const float* pyr_v,
                    const TcBuffers& tb, cudaStream_t s) {
  return launch_prep(g, units, pyr_k, pyr_v, tb, s);
}

bool tc_forward_writes_bf16(const Geometry& g) { return fwd5_path(g); }

llsa_status tc_forward(const Geometry& g, uint32_t units, const void* q, const void* k,
                       const void* v, const float* pyr_k, const float* pyr_v,
                       const uint32_t* tables, float* out, float* row_max, float* row_denom,
                       const TcBuffers& tb, cudaStream_t s, StageMarker* mk, bool prepped,
                       void* out16) {
  if (!prepped) {
    if (llsa_status st = launch_prep(g, units, pyr_k, pyr_v, tb, s)) return st;
    LLSA_MARK(mk, "fwd_prep", s);
  }
  TcParams P = make_params(g, units);
  P.q = static_cast<const bf16*>(q);
  P.k = static_cast<const bf16*>(k);
  P.v = static_cast<const bf16*>(v);
  P.khi = tb.k_hi;
  P.klo = tb.k_lo;
  P.vhi = tb.v_hi;
  P.vlo = tb.v_lo;
  P.tables = tables;
  P.out = out;
  P.out16 = out16;
  P.row_max = row_max;
  P.row_denom = row_denom;
  static std::atomic<uint64_t> attr{0};
  if (!attrs_done(attr)) {
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kFwdSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_fwd_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, fw5::kSmem));
    mark_attrs_done(attr);
  }
  if (fwd5_path(g)) {
    TmaMaps maps{};
    const uint64_t in_rows = (uint64_t)units * g.n, pyr_rows = (uint64_t)units * g.pyr_rows;
    if (llsa_status st = make_tma_map(&maps.q, q, in_rows, kTileQ)) return st;
    if (llsa_status st = make_tma_map(&maps.khi, tb.k_hi, pyr_rows, kBS)) return st;
    if (llsa_status st = make_tma_map(&maps.klo, tb.k_lo, pyr_rows, kBS)) return st;
    if (llsa_status st = make_tma_map(&maps.vhi, tb.v_hi, pyr_rows, kBS)) return st;
    if (llsa_status st = make_tma_map(&maps.o, out, in_rows, 32, true)) return st;
    const uint64_t tiles = (g.n / kTileQ) * units;
    const unsigned grid = (unsigned)(tiles < (uint64_t)num_sms() ? tiles : num_sms());
    // one pass per 24 coarse entries; later passes merge into the output
    const uint32_t tot = P.nce;
    for (uint32_t base = 0; base < tot; base += fw5::kMaxEntries) {
      TcParams Pp = P;
      Pp.ce_base = base;
      Pp.nce = tot - base < fw5::kMaxEntries ? tot - base : fw5::kMaxEntries;
      Pp.fine_mode = base ? 1u : 0u;
      Pp.out16 = base + fw5::kMaxEntries >= tot ? out16 : nullptr;  // the final pass only
      tc5_fwd_kernel<<<grid, fw5::kThreads, fw5::kSmem, s>>>(Pp, maps, units);
      count_launch();
      LLSA_LAUNCH_CHECK("tc5_fwd_kernel");
    }
  } else {
    tc_fwd_kernel<<<dim3((unsigned)(g.n / kTileQ), units), 256, kFwdSmem, s>>>(P);
    count_launch();
    LLSA_LAUNCH_CHECK("tc_fwd_kernel");
  }
  LLSA_MARK(mk, "fwd_attention", s);
  return LLSA_OK;
}

size_t tc_backward_ws_bytes(const Geometry& g, uint32_t units) {
  TcParams P{};
  coarse_slots(g, P, units, true);
  rows_layout(g, P);
  const size_t rows = ((size_t)units * g.n * 4 + 255) & ~size_t(255);
  const size_t part = ((size_t)units * P.part_unit_stride * 4 + 255) & ~size_t(255);
  return 2 * rows + part + (size_t)units * P.rpart_unit_stride * 4 + 256;
}

llsa_status tc_backward(const Geometry& g, uint32_t units, const void* d_out,
                        const float* out, const float* row_max, const float* row_denom,
                        const void* q, const void* k, const void* v, const float* pyr_k,
                        const float* pyr_v, const uint32_t* tables,
                        const uint32_t* csc_offsets, const uint32_t* csc_flat, float* dq,
                        float* dk, float* dv, const TcBuffers& tb, void* ws, cudaStream_t s,
                        StageMarker* mk, bool grad_bf16) {
  (void)pyr_k;
  (void)pyr_v;
  if (grad_bf16 && !tc_bf16_grads_ok(g))
    return fail(LLSA_ERR_UNSUPPORTED, "bf16 gradients need the fused dQ and fine dK/dV kernels");
  TcParams P = make_params(g, units);
  P.q = static_cast<const bf16*>(q);
  P.k = static_cast<const bf16*>(k);
  P.v = static_cast<const bf16*>(v);
  P.dout = static_cast<const bf16*>(d_out);
  P.khi = tb.k_hi;
  P.klo = tb.k_lo;
  P.vhi = tb.v_hi;
  P.vlo = tb.v_lo;
  P.tables = tables;
  P.csc_off = csc_offsets;
  P.csc_flat = csc_flat;
  P.out_in = out;
  P.rm_in = row_max;
  P.rd_in = row_denom;
  const size_t rows = ((size_t)units * g.n * 4 + 255) & ~size_t(255);
  P.lse2 = static_cast<float*>(ws);
  P.drow = reinterpret_cast<float*>(static_cast<char*>(ws) + rows);
  P.part = reinterpret_cast<float*>(static_cast<char*>(ws) + 2 * rows);
  P.rpart = reinterpret_cast<float*>(
      static_cast<char*>(ws) + 2 * rows +
      (((size_t)units * P.part_unit_stride * 4 + 255) & ~size_t(255)));
  P.dq = dq;
  P.dk = dk;
  P.dv = dv;
  P.grad_bf16 = grad_bf16 ? 1u : 0u;
  static std::atomic<uint64_t> attr{0};
  if (!attrs_done(attr)) {
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kDqSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc_kv_kernel<2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       KvCfg<true>::Smem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc_kv_kernel<1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       KvCfg<true>::Smem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_rows2_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       rows2::L<true>::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_rows2_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       rows2::L<false>::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_kvf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kvf::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_dqf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       dqf::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_dq_pipe_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, dqp::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_dq_coarse_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, dqc::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_kv_rows_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       rows::Layout<true>::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc5_kv_rows_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       rows::Layout<false>::kSmem));
    LLSA_CUDA_TRY(cudaFuncSetAttribute(tc_kv_kernel<0>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       KvCfg<false>::Smem));
    mark_attrs_done(attr);
  }
  const bool dqf = dqf_path(g);
  if (dqf) {
    TmaMaps maps{};
    const uint64_t in_rows = (uint64_t)units * g.n;
    if (llsa_status st = make_tma_map(&maps.q, q, in_rows, kTileQ)) return st;
    if (llsa_status st = make_tma_map(&maps.g, d_out, in_rows, kTileQ)) return st;
    if (llsa_status st = make_tma_map(&maps.o, P.dq, in_rows, 32, !grad_bf16)) return st;
    const uint64_t tiles = (g.n / kTileQ) * units;
    const unsigned grid = (unsigned)(tiles < (uint64_t)num_sms() ? tiles : num_sms());
    // one pass per 24 coarse entries; later passes add their dq (TMA reduce)
    const uint32_t tot = P.nce;
    for (uint32_t base = 0; base < tot; base += dqf::kMaxEntries) {
      TcParams Pp = P;
      Pp.ce_base = base;
      Pp.nce = tot - base < dqf::kMaxEntries ? tot - base : dqf::kMaxEntries;
      Pp.fine_mode = base ? 1u : 0u;
      tc5_dqf_kernel<<<grid, dqf::kThreads, dqf::kSmem, s>>>(Pp, maps, units);
      count_launch();
      LLSA_LAUNCH_CHECK("tc5_dqf_kernel");
    }
    LLSA_MARK(mk, "bwd_dq", s);
  }
  // dq: fine part (+ D, lse2) on mma.sync; coarse part on tcgen05 when enabled
  const bool dq5 = !dqf && P.nce > 0 && rows_path(g);
  if (!dqf) {
    TcParams Pf = P;
    if (dq5) Pf.nce = 0;
    tc_dq_kernel<<<dim3((unsigned)(g.n / kTileQ), units), 256, kDqSmem, s>>>(Pf);
    count_launch();
    LLSA_LAUNCH_CHECK("tc_dq_kernel");
  }
  if (!dqf) LLSA_MARK(mk, "bwd_dq", s);
  if (dq5) {
    const char* old = getenv("LLSA_DQ5_SYNC");
    if (old && old[0] == '1') {
      tc5_dq_coarse_kernel<<<dim3((unsigned)(g.n / kTileQ), units), 256, dqc::kSmem, s>>>(P);
      count_launch();
      LLSA_LAUNCH_CHECK("tc5_dq_coarse_kernel");
    } else {
      TmaMaps maps;
      const uint64_t in_rows = (uint64_t)units * g.n, pyr_rows = (uint64_t)units * g.pyr_rows;
      if (llsa_status st = make_tma_map(&maps.q, q, in_rows, kTileQ)) return st;
      if (llsa_status st = make_tma_map(&maps.g, d_out, in_rows, kTileQ)) return st;
      if (llsa_status st = make_tma_map(&maps.khi, tb.k_hi, pyr_rows, kBS)) return st;
      if (llsa_status st = make_tma_map(&maps.vhi, tb.v_hi, pyr_rows, kBS)) return st;
      if (llsa_status st = make_tma_map(&maps.klo, tb.k_lo, pyr_rows, kBS)) return st;
      if (llsa_status st = make_tma_map(&maps.vlo, tb.v_lo, pyr_rows, kBS)) return st;
      const uint64_t tiles = (g.n / kTileQ) * units;
      const unsigned grid = (unsigned)(tiles < (uint64_t)num_sms() ? tiles : num_sms());
      tc5_dq_pipe_kernel<<<grid, 320, dqp::kSmem, s>>>(P, maps, units);
      count_launch();
      LLSA_LAUNCH_CHECK("tc5_dq_pipe_kernel");
    }
  }
  if (dq5) LLSA_MARK(mk, "bwd_dq_coarse_tc5", s);
  // levels 1..lim-1 on tcgen05 (row-major), the rest on the key-major kernel
  const uint32_t start = P.rows_on ? P.rl_count : 0;
  // unordered mode: every coarse slot starts at zero and both coarse kernels
  // add into it (rows2 by TMA reductions, tc_kv by red.add), no reduce passes
  if (P.kv_atomic && P.ncl)
    LLSA_CUDA_TRY(cudaMemsetAsync(P.part, 0, (size_t)units * P.part_unit_stride * 4, s));
  if (P.rows_on) {
    const char* r2 = getenv("LLSA_ROWS2");
    const bool persistent = !(r2 && r2[0] == '0');
    TmaMaps qmaps{};
    if (!persistent) P.rows_atomic = 0;
    if (persistent) {
      const uint64_t in_rows = (uint64_t)units * g.n;
      if (llsa_status st = make_tma_map(&qmaps.q, q, in_rows, rows2::kQT)) return st;
      if (llsa_status st = make_tma_map(&qmaps.g, d_out, in_rows, rows2::kQT)) return st;
    }
    if (P.rows_atomic &&
        make_tma_map(&qmaps.o, P.part, units * P.part_unit_stride / kD, kBS, true))
      return LLSA_ERR_CUDA;
    for (uint32_t li = 0; li < P.rl_count; ++li) {
      const uint64_t tasks = (P.rl_tasks[li + 1] - P.rl_tasks[li]) * units;
      const bool lo = P.rl_level[li] >= P.hilo_level;
      if (persistent) {
        const unsigned grid = (unsigned)(tasks < (uint64_t)num_sms() ? tasks : num_sms());
        TcParams Pr = P;
        if (trace_only_rows2()) Pr.trace = P.trace_rows2 && li == 0;
        if (lo)
          tc5_rows2_kernel<true><<<grid, rows2::kThreads, rows2::L<true>::kSmem, s>>>(
              Pr, qmaps, li, units);
        else
          tc5_rows2_kernel<false><<<grid, rows2::kThreads, rows2::L<false>::kSmem, s>>>(
              P, qmaps, li, units);
        count_launch();
        LLSA_LAUNCH_CHECK("tc5_rows2_kernel");
        continue;
      }
      if (lo)
        tc5_kv_rows_kernel<true><<<(unsigned)tasks, 256, rows::Layout<true>::kSmem, s>>>(
            P, li, units);
      else
        tc5_kv_rows_kernel<false><<<(unsigned)tasks, 256, rows::Layout<false>::kSmem, s>>>(
            P, li, units);
      count_launch();
      LLSA_LAUNCH_CHECK("tc5_kv_rows_kernel");
    }
    if (!P.rows_atomic) {
      uint64_t wpu = 0;
      for (uint32_t li = 0; li < P.rl_count; ++li) wpu += g.level_blocks(P.rl_level[li]);
      rows_reduce_kernel<<<(unsigned)(wpu * units), 256, 0, s>>>(P, units, wpu);
      count_launch();
      LLSA_LAUNCH_CHECK("rows_reduce_kernel");
    }
  }
  LLSA_MARK(mk, "bwd_kv_coarse_tc5", s);
  if (start < P.ncl) {
    // slots ascend by level: [start, a) hi-only, [a, ncl) hi + lo
    uint32_t a = start;
    while (a < P.ncl && P.cl_level[a] < P.hilo_level) ++a;
    if (a < P.ncl) {
      const uint64_t tasks = P.cl_tasks[P.ncl] - P.cl_tasks[a];
      const uint64_t warps = tasks * units;
      tc_kv_kernel<2><<<(unsigned)((warps + kKvWarps - 1) / kKvWarps), kKvWarps * 32,
                        KvCfg<true>::Smem, s>>>(P, tasks, units, a);
      count_launch();
      LLSA_LAUNCH_CHECK("tc_kv_kernel<coarse hi+lo>");
    }
    if (a > start) {
      const uint64_t tasks = P.cl_tasks[a] - P.cl_tasks[start];
      const uint64_t warps = tasks * units;
      tc_kv_kernel<1><<<(unsigned)((warps + kKvWarps - 1) / kKvWarps), kKvWarps * 32,
                        KvCfg<true>::Smem, s>>>(P, tasks, units, start);
      count_launch();
      LLSA_LAUNCH_CHECK("tc_kv_kernel<coarse hi>");
    }
    if (!P.kv_atomic) {
      reduce_parts_kernel<<<grid_for(g.n / 16 * kD * units, 256), 256, 0, s>>>(P, units, start,
                                                                              P.ncl);
      count_launch();
      LLSA_LAUNCH_CHECK("reduce_parts_kernel");
    }
  }
  LLSA_MARK(mk, "bwd_kv_coarse", s);
  if (kvf_path(g)) {
    const uint64_t items = (g.n / kBS) * units;
    const unsigned grid = (unsigned)(items < (uint64_t)num_sms() ? items : num_sms());
    tc5_kvf_kernel<<<grid, kvf::kThreads, kvf::kSmem, s>>>(P, units);
    count_launch();
    LLSA_LAUNCH_CHECK("tc5_kvf_kernel");
  } else {
    const uint64_t tasks = g.n / kBS;
    const uint64_t warps = tasks * units;
    tc_kv_kernel<0><<<(unsigned)((warps + kKvWarps - 1) / kKvWarps), kKvWarps * 32,
                      KvCfg<false>::Smem, s>>>(P, tasks, units, 0);
    count_launch();
    LLSA_LAUNCH_CHECK("tc_kv_kernel<fine>");
  }
  LLSA_MARK(mk, "bwd_kv_fine", s);
  return LLSA_OK;
}

}  // namespace llsa_impl

// Debug: copies the pipeline trace recorded by CTA 0 (LLSA_TRACE=1) and resets it.
extern "C" int llsa_debug_trace(unsigned long long* out, int cap) {
  cudaDeviceSynchronize();
  const int n = cap < 8192 ? cap : 8192;
  cudaMemcpyFromSymbol(out, llsa_impl::g_trace, n * sizeof(unsigned long long));
  static unsigned long long zero[8192];
  cudaMemcpyToSymbol(llsa_impl::g_trace, zero, sizeof(zero));
  return n;
}
