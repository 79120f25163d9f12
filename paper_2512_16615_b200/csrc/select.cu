// K2/K3 — coarse-to-fine Top-K block selection, P/src/selection.cpp:21-179.
//
// Scores use the reference's exact fp32 recipe (dot4_exact: 4-lane
// association, no FMA; then scale*dot), so selections are bit-identical to
// the f32 reference.  Top-K is a rank selection: candidate c is kept iff
//   #{c' : s[c'] > s[c]  or  (s[c'] == s[c] and c' < c)} < K,
// which is exactly the (score desc, position asc) order of topk_row
// (selection.cpp:21-38) with its lowest-index tie-break, computed without a
// sort and with float comparisons (−0.0 ties +0.0).  Kept candidates are
// emitted in ascending position order; candidate ids ascend with position
// when the parent row is sorted (always, on the hierarchical path), so rows
// come out ascending as the reference's final std::sort makes them.  A
// user-supplied parent row that is not ascending is detected per CTA and the
// kept ids are then sorted explicitly (selection.cpp:37).
//
// select_level: one CTA per (unit, level-l query block).  All B query rows
// of the block share the same K·B candidate tokens, so the CTA stages those
// rows in shared memory once (row stride d+4 floats: conflict-free float4
// reads) and scores B×K·B pairs from smem.
#include "common.cuh"
#include "internal.h"

namespace llsa_impl {
namespace {

using namespace llsa_dev;

// true when this thread's slice of a parent row is strictly ascending (the
// hierarchical path always produces such rows; ids then ascend with position)
__device__ __forceinline__ bool row_ascending(const uint32_t* prow, uint32_t parent_k) {
  bool ok = true;
  for (uint32_t t = threadIdx.x; t + 1 < parent_k; t += blockDim.x) ok &= prow[t] < prow[t + 1];
  return ok;
}

__device__ __forceinline__ bool beats(float sa, uint32_t a, float sb, uint32_t b) {
  // true when candidate a ranks before candidate b
  return sa > sb || (sa == sb && a < b);
}

// Rank-select over scores[0..C) held in smem; writes selected flags.
__device__ void rank_select(const float* scores, uint32_t C, uint32_t K, uint8_t* sel,
                            uint32_t tid, uint32_t nthr) {
  for (uint32_t c = tid; c < C; c += nthr) {
    const float s = scores[c];
    uint32_t rank = 0;
    for (uint32_t c2 = 0; c2 < C; ++c2) rank += beats(scores[c2], c2, s, c) ? 1u : 0u;
    sel[c] = rank < K ? 1 : 0;
  }
}

__global__ void __launch_bounds__(256) select_coarsest_kernel(
    const float* __restrict__ q, uint64_t q_unit_stride, const float* __restrict__ k,
    uint64_t k_unit_stride, uint32_t rows, uint32_t C, uint32_t d, uint32_t K,
    float scale, uint32_t* __restrict__ out, uint64_t out_unit_stride) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t row = blockIdx.x;
  const uint32_t unit = blockIdx.y;
  float* sq = reinterpret_cast<float*>(smem);                 // d (padded to 4)
  float* scores = sq + ((d + 3) & ~3u);                        // C
  uint8_t* sel = reinterpret_cast<uint8_t*>(scores + C);       // C
  const float* qr = q + unit * q_unit_stride + (uint64_t)row * d;
  const float* ku = k + unit * k_unit_stride;
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) sq[j] = qr[j];
  __syncthreads();
  const bool v4 = (d % 4 == 0) && (reinterpret_cast<uintptr_t>(ku) % 16 == 0);
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    const float* kr = ku + (uint64_t)c * d;
    const float dot = v4 ? dot4_exact_v4(reinterpret_cast<const float4*>(sq),
                                         reinterpret_cast<const float4*>(kr), d / 4)
                         : dot4_exact(sq, kr, d);
    scores[c] = __fmul_rn(scale, dot);
  }
  __syncthreads();
  rank_select(scores, C, K, sel, threadIdx.x, blockDim.x);
  __syncthreads();
  uint32_t* o = out + unit * out_unit_stride + (uint64_t)row * K;
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    if (!sel[c]) continue;
    uint32_t pos = 0;
    for (uint32_t c2 = 0; c2 < c; ++c2) pos += sel[c2];
    o[pos] = c;
  }
}

__global__ void __launch_bounds__(256) select_level_kernel(
    const float* __restrict__ q, uint64_t q_unit_stride, const float* __restrict__ k,
    uint64_t k_unit_stride, const uint32_t* __restrict__ parent,
    uint64_t parent_unit_stride, uint32_t parent_k, uint32_t key_blocks, uint32_t d,
    uint32_t K, float scale, uint32_t B, bool stage_k, uint32_t* __restrict__ out,
    uint64_t out_unit_stride, uint32_t* flag) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t blk = blockIdx.x;   // level-l query block (= parent row)
  const uint32_t unit = blockIdx.y;
  const uint32_t C = parent_k * B;
  const uint32_t ld = (d + 3) & ~3u;           // q row stride
  const uint32_t ldk = ((d + 3) & ~3u) + 4;    // padded k row stride
  uint32_t* ids = reinterpret_cast<uint32_t*>(smem);            // C
  float* sq = reinterpret_cast<float*>(ids + ((C + 3) & ~3u));  // B * ld
  float* scores = sq + (uint64_t)B * ld;                        // B * C
  uint8_t* sel = reinterpret_cast<uint8_t*>(scores + (((uint64_t)B * C + 3) & ~3ull));  // B * C
  float* sk = reinterpret_cast<float*>(sel + (((uint64_t)B * C + 15) & ~15ull));  // C * ldk

  const uint32_t* prow = parent + unit * parent_unit_stride + (uint64_t)blk * parent_k;
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    uint32_t pb = prow[c / B];
    if (pb >= key_blocks) {  // IndexOutOfRange, selection.cpp:125-130
      raise_flag(flag, kErrIndex);
      pb = 0;
    }
    ids[c] = pb * B + c % B;
  }
  const float* qu = q + unit * q_unit_stride + (uint64_t)blk * B * d;
  for (uint32_t e = threadIdx.x; e < B * d; e += blockDim.x)
    sq[(e / d) * ld + e % d] = qu[e];
  const bool asc = __syncthreads_and(row_ascending(prow, parent_k)) != 0;
  const float* ku = k + unit * k_unit_stride;
  if (stage_k) {
    for (uint64_t e = threadIdx.x; e < (uint64_t)C * d; e += blockDim.x) {
      const uint32_t c = (uint32_t)(e / d), j = (uint32_t)(e % d);
      sk[(uint64_t)c * ldk + j] = ku[(uint64_t)ids[c] * d + j];
    }
  }
  __syncthreads();
  const bool v4 = stage_k && (d % 4 == 0);
  for (uint32_t p = threadIdx.x; p < B * C; p += blockDim.x) {
    const uint32_t r = p / C, c = p % C;
    float dot;
    if (v4) {
      dot = dot4_exact_v4(reinterpret_cast<const float4*>(sq + r * ld),
                          reinterpret_cast<const float4*>(sk + (uint64_t)c * ldk), d / 4);
    } else {
      const float* kr = stage_k ? sk + (uint64_t)c * ldk : ku + (uint64_t)ids[c] * d;
      dot = dot4_exact(sq + r * ld, kr, d);
    }
    scores[p] = __fmul_rn(scale, dot);
  }
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < B * C; p += blockDim.x) {
    const uint32_t r = p / C, c = p % C;
    const float* sr = scores + (uint64_t)r * C;
    const float s = sr[c];
    uint32_t rank = 0;
    for (uint32_t c2 = 0; c2 < C; ++c2) rank += beats(sr[c2], c2, s, c) ? 1u : 0u;
    sel[p] = rank < K ? 1 : 0;
  }
  __syncthreads();
  uint32_t* o = out + unit * out_unit_stride + (uint64_t)blk * B * K;
  for (uint32_t p = threadIdx.x; p < B * C; p += blockDim.x) {
    if (!sel[p]) continue;
    const uint32_t r = p / C, c = p % C;
    const uint8_t* sr = sel + (uint64_t)r * C;
    uint32_t pos = 0;
    for (uint32_t c2 = 0; c2 < c; ++c2) pos += sr[c2];
    o[(uint64_t)r * K + pos] = ids[c];
  }
  if (!asc) {  // a user-built parent row out of order: sort like topk_row's std::sort
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < B; r += blockDim.x) {
      uint32_t* orow = o + (uint64_t)r * K;
      for (uint32_t i = 1; i < K; ++i) {
        const uint32_t x = orow[i];
        uint32_t j = i;
        for (; j > 0 && orow[j - 1] > x; --j) orow[j] = orow[j - 1];
        orow[j] = x;
      }
    }
  }
}

// Packed fp32x2 arithmetic (sm_100): two exact IEEE products / sums per
// instruction.  The product is an fma with a -0 addend read from memory, so
// ptxas cannot contract it with the following add (it fuses a plain
// mul.rn.f32x2 + add.rn.f32x2 pair into FFMA2); fma(a, b, -0) rounds the
// exact product once, like mul.rn, including signed zeros.
__device__ __forceinline__ uint64_t mul2_exact(uint64_t a, uint64_t b, uint64_t nz) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(nz));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Top-K of each of the block's B query rows from scores[r * 256 + c] (one
// warp per row; lane owns positions lane*PL .. lane*PL+PL-1): K rounds of a
// warp arg-max over order-preserving keys (score desc, position asc), then
// the kept ids in position order (sorted when the parent row was not).
template <int PL>
__device__ __forceinline__ void topk_rows(const float* scores, const uint32_t* ids, uint32_t C,
                                          uint32_t K, uint32_t B, uint32_t* out_blk,
                                          bool asc) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t r = warp; r < B; r += blockDim.x >> 5) {
    // lane owns positions lane*PL .. lane*PL+PL-1 (contiguous, so position
    // order = (lane, i) order; PL = 4 covers C <= 128 with every lane busy).
    // Scores become order-preserving u32 keys (-0 → +0, the float compare
    // ties them); each round takes the warp max key with redux.sync and,
    // among equal keys, the lowest position (topk_row's lowest-index
    // tie-break), so the selection is exact.
    uint32_t key[PL];
    uint32_t taken = 0;
#pragma unroll
    for (int i = 0; i < PL; ++i) {
      const uint32_t c = lane * PL + i;
      float v = c < C ? scores[r * 256 + c] : 0.f;
      if (v == 0.f) v = 0.f;  // canonical +0
      const uint32_t u = __float_as_uint(v);
      key[i] = c < C ? ((u & 0x80000000u) ? ~u : (u | 0x80000000u)) : 0u;  // valid keys > 0
    }
    for (uint32_t round = 0; round < K; ++round) {
      uint32_t lk = key[0], li = 0;
#pragma unroll
      for (int i = 1; i < PL; ++i)
        if (key[i] > lk) {
          lk = key[i];
          li = i;
        }
      const uint32_t mk = __reduce_max_sync(0xffffffffu, lk);
      const uint32_t mypos = lk == mk && lk != 0u ? lane * PL + li : 0xffffffffu;
      const uint32_t bpos = __reduce_min_sync(0xffffffffu, mypos);
      if (bpos == mypos) {
        taken |= 1u << li;
#pragma unroll
        for (int i = 0; i < PL; ++i)
          if ((uint32_t)i == li) key[i] = 0u;
      }
    }
    const uint32_t cnt = __popc(taken);
    uint32_t pre = cnt;  // inclusive scan of counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= (uint32_t)o) pre += y;
    }
    uint32_t pos = pre - cnt;
    uint32_t* o = out_blk + (uint64_t)r * K;
#pragma unroll
    for (int i = 0; i < PL; ++i)
      if ((taken >> i) & 1u) o[pos++] = ids[lane * PL + i];
    if (!asc) {  // parent row out of order (user-built): rank-sort the K ids
      __syncwarp();
      const uint32_t x = lane < K ? o[lane] : 0u;
      uint32_t rank = 0;
      for (uint32_t j = 0; j < K; ++j) {
        const uint32_t y = __shfl_sync(0xffffffffu, x, j);
        rank += (y < x || (y == x && j < lane)) ? 1u : 0u;
      }
      __syncwarp();
      if (lane < K) o[rank] = x;
    }
  }
}

// Fast variant for d % 4 == 0, B = 16 query rows per block, C = K·B <= 256
// candidates, K <= 32: thread (row r, lane group cg) scores candidates
// cg, cg+16, … with q_r and the candidate rows streamed as float4 from smem
// (4 exact accumulators per pair, same association as detail::dot); then one
// warp per row extracts the top K by K rounds of a warp arg-max over
// (score desc, position asc) and emits the kept positions in ascending order.
template <int CPT>
__global__ void __launch_bounds__(256, 4) select_level_fast_kernel(
    const float* __restrict__ q, uint64_t q_unit_stride, const float* __restrict__ k,
    uint64_t k_unit_stride, const uint32_t* __restrict__ parent, uint64_t parent_unit_stride,
    uint32_t parent_k, uint32_t key_blocks, uint32_t d, uint32_t K, float scale,
    uint32_t* __restrict__ out, uint64_t out_unit_stride, uint32_t* flag, uint64_t negzero2) {
  constexpr uint32_t B = 16;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t blk = blockIdx.x, unit = blockIdx.y;
  const uint32_t C = parent_k * B;
  const uint32_t ld = d + 4;  // padded row stride (floats), keeps 16 B alignment
  uint32_t* ids = reinterpret_cast<uint32_t*>(smem);                  // 256
  float* scores = reinterpret_cast<float*>(ids + 256);                // 16 × 256
  float* sq = scores + 16 * 256;                                      // 16 × ld
  float* sk = sq + 16 * ld;                                           // C × ld
  const uint32_t* prow = parent + unit * parent_unit_stride + (uint64_t)blk * parent_k;
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    uint32_t pb = prow[c / B];
    if (pb >= key_blocks) {
      raise_flag(flag, kErrIndex);
      pb = 0;
    }
    ids[c] = pb * B + c % B;
  }
  const float* qu = q + unit * q_unit_stride + (uint64_t)blk * B * d;
  const uint32_t d4 = d / 4;
  // row / column of flat float4 index e (shift and mask when d/4 is a power of 2)
  const bool pow2 = (d4 & (d4 - 1)) == 0;
  const uint32_t sh = __ffs(d4) - 1;
  auto rc = [&](uint32_t e, uint32_t& r, uint32_t& j) {
    r = pow2 ? e >> sh : e / d4;
    j = pow2 ? e & (d4 - 1) : e % d4;
  };
  for (uint32_t e = threadIdx.x; e < B * d4; e += blockDim.x) {
    uint32_t r, j;
    rc(e, r, j);
    reinterpret_cast<float4*>(sq + r * ld)[j] = reinterpret_cast<const float4*>(qu + r * d)[j];
  }
  const bool asc = __syncthreads_and(row_ascending(prow, parent_k)) != 0;
  // candidate rows: global → smem with cp.async (no register round trip, so
  // a thread's copies are all in flight at once)
  const float* ku = k + unit * k_unit_stride;
  const uint32_t sk_s = (uint32_t)__cvta_generic_to_shared(sk);
  for (uint32_t e = threadIdx.x; e < C * d4; e += blockDim.x) {
    uint32_t c, j;
    rc(e, c, j);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sk_s + (c * ld + 4 * j) * 4),
                 "l"(ku + (uint64_t)ids[c] * d + 4 * j)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  {
    const uint32_t r = threadIdx.x >> 4, cg = threadIdx.x & 15;
    // accumulators (s0, s1) and (s2, s3) of each pair as packed fp32x2: the
    // same per-lane operations and order as detail::dot
    // two passes of CPT/2 candidates: half the accumulator registers, so
    // four CTAs fit per SM without spilling
    constexpr int CH = CPT / 2;
    const ulonglong2* qr = reinterpret_cast<const ulonglong2*>(sq + r * ld);
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      uint64_t acc[CH][2];
#pragma unroll
      for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0ull;
      for (uint32_t j = 0; j < d4; ++j) {
        const ulonglong2 x = qr[j];
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const uint32_t c = cg + 16 * (pass * CH + i);
          if (c < C) {
            const ulonglong2 y = reinterpret_cast<const ulonglong2*>(sk + c * ld)[j];
            acc[i][0] = add2(acc[i][0], mul2_exact(x.x, y.x, negzero2));
            acc[i][1] = add2(acc[i][1], mul2_exact(x.y, y.y, negzero2));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const uint32_t c = cg + 16 * (pass * CH + i);
        if (c < C) {
          const float s0 = __uint_as_float((uint32_t)acc[i][0]);
          const float s1 = __uint_as_float((uint32_t)(acc[i][0] >> 32));
          const float s2 = __uint_as_float((uint32_t)acc[i][1]);
          const float s3 = __uint_as_float((uint32_t)(acc[i][1] >> 32));
          scores[r * 256 + c] = __fmul_rn(scale, __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3)));
        }
      }
    }
  }
  __syncthreads();
  topk_rows<CPT / 2>(scores, ids, C, K, B, out + unit * out_unit_stride + (uint64_t)blk * B * K,
                     asc);
}

// Register-blocked scorer for the hot shape (B = 16, d = 64, C = K·B <= 256):
// thread = candidate, all 16 query rows of the block in registers (16 rows ×
// two packed fp32x2 accumulators).  Per float4 step the thread loads its
// candidate's 16 bytes once (distinct per lane, 4 wavefronts per warp) and
// the 16 query float4s as warp-wide broadcasts, then issues 64 packed exact
// multiply / add instructions: the candidate row is reused 16 times from a
// register instead of being re-read per (row, candidate) pair, so the FP32
// pipe, not shared memory, is the limit.  Same per-pair operations and order
// as detail::dot (bit-exact scores); same top-K as above.
template <int NT>
__global__ void __launch_bounds__(NT, NT == 128 ? 5 : 2) select_level_rb_kernel(
    const float* __restrict__ q, uint64_t q_unit_stride, const float* __restrict__ k,
    uint64_t k_unit_stride, const uint32_t* __restrict__ parent, uint64_t parent_unit_stride,
    uint32_t parent_k, uint32_t key_blocks, uint32_t K, float scale,
    uint32_t* __restrict__ out, uint64_t out_unit_stride, uint32_t* flag, uint64_t negzero2) {
  constexpr uint32_t B = 16, D = 64, LD = D + 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t blk = blockIdx.x, unit = blockIdx.y, tid = threadIdx.x;
  const uint32_t C = parent_k * B;
  uint32_t* ids = reinterpret_cast<uint32_t*>(smem);      // 256
  float* sq = reinterpret_cast<float*>(ids + 256);        // 16 × 64
  float* sk = sq + 16 * D;                                // C × LD
  // the scores (16 × 256) reuse the candidate rows once every dot is done,
  // so a CTA needs ~39 KB instead of ~55 KB (five CTAs per SM instead of four)
  float* scores = sk;
  const uint32_t* prow = parent + unit * parent_unit_stride + (uint64_t)blk * parent_k;
  for (uint32_t c = tid; c < C; c += NT) {
    uint32_t pb = prow[c / B];
    if (pb >= key_blocks) {
      raise_flag(flag, kErrIndex);
      pb = 0;
    }
    ids[c] = pb * B + c % B;
  }
  const uint32_t sq_s = (uint32_t)__cvta_generic_to_shared(sq);
  const float* qu = q + unit * q_unit_stride + (uint64_t)blk * B * D;
  for (uint32_t e = tid; e < B * D / 4; e += NT)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sq_s + e * 16),
                 "l"(qu + 4 * e)
                 : "memory");
  const bool asc = __syncthreads_and(row_ascending(prow, parent_k)) != 0;
  const float* ku = k + unit * k_unit_stride;
  const uint32_t sk_s = (uint32_t)__cvta_generic_to_shared(sk);
  for (uint32_t e = tid; e < C * (D / 4); e += NT) {
    const uint32_t c = e >> 4, j = e & 15;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sk_s + (c * LD + 4 * j) * 4),
                 "l"(ku + (uint64_t)ids[c] * D + 4 * j)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  float sc[B];
  if (tid < C) {
    uint64_t acc[B][2];
#pragma unroll
    for (int r = 0; r < (int)B; ++r) acc[r][0] = acc[r][1] = 0ull;
    const ulonglong2* kr = reinterpret_cast<const ulonglong2*>(sk + tid * LD);
    const ulonglong2* qr = reinterpret_cast<const ulonglong2*>(sq);
#pragma unroll
    for (int j = 0; j < (int)(D / 4); ++j) {
      const ulonglong2 y = kr[j];
#pragma unroll
      for (int r = 0; r < (int)B; ++r) {
        const ulonglong2 x = qr[r * (D / 4) + j];  // same address in every lane: broadcast
        acc[r][0] = add2(acc[r][0], mul2_exact(x.x, y.x, negzero2));
        acc[r][1] = add2(acc[r][1], mul2_exact(x.y, y.y, negzero2));
      }
    }
#pragma unroll
    for (int r = 0; r < (int)B; ++r) {
      const float s0 = __uint_as_float((uint32_t)acc[r][0]);
      const float s1 = __uint_as_float((uint32_t)(acc[r][0] >> 32));
      const float s2 = __uint_as_float((uint32_t)acc[r][1]);
      const float s3 = __uint_as_float((uint32_t)(acc[r][1] >> 32));
      sc[r] = __fmul_rn(scale, __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3)));
    }
  }
  __syncthreads();  // every candidate row has been read: the scores may overwrite them
  if (tid < C) {
#pragma unroll
    for (int r = 0; r < (int)B; ++r) scores[r * 256 + tid] = sc[r];
  }
  __syncthreads();
  topk_rows<NT / 32>(scores, ids, C, K, B, out + unit * out_unit_stride + (uint64_t)blk * B * K,
                     asc);
}

}  // namespace

llsa_status launch_select_coarsest(const float* q, uint64_t q_unit_stride, const float* k,
                                   uint64_t k_unit_stride, uint32_t units, uint32_t rows,
                                   uint32_t cands, uint32_t d, uint32_t K, float scale,
                                   uint32_t* out, uint64_t out_unit_stride, cudaStream_t s) {
  if (rows == 0 || units == 0) return LLSA_OK;
  const size_t smem = sizeof(float) * (((d + 3) & ~3u) + cands) + cands + 16;
  if (smem > 200 * 1024)
    return fail(LLSA_ERR_UNSUPPORTED, "select_coarsest: %u candidates exceed shared memory",
                cands);
  if (smem > 48 * 1024)
    LLSA_CUDA_TRY(cudaFuncSetAttribute(select_coarsest_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
  select_coarsest_kernel<<<dim3(rows, units), 256, smem, s>>>(
      q, q_unit_stride, k, k_unit_stride, rows, cands, d, K, scale, out, out_unit_stride);
  count_launch();
  LLSA_LAUNCH_CHECK("select_coarsest_kernel");
  return LLSA_OK;
}

llsa_status launch_select_level(const float* q, uint64_t q_unit_stride, const float* k,
                                uint64_t k_unit_stride, const uint32_t* parent,
                                uint64_t parent_unit_stride, uint32_t units,
                                uint32_t parent_rows, uint32_t parent_k, uint64_t k_rows,
                                uint32_t d, uint32_t K, float scale, uint32_t B,
                                uint32_t* out, uint64_t out_unit_stride, cudaStream_t s) {
  if (parent_rows == 0 || units == 0) return LLSA_OK;
  const uint64_t C = (uint64_t)parent_k * B;
  if (B == 16 && d % 4 == 0 && d <= 256 && C <= 256 && K <= 32) {
    const uint64_t ld = d + 4;
    const size_t smem = 4 * (256 + 16 * 256 + 16 * ld + C * ld);
    if (smem <= 200 * 1024) {
      const uint32_t key_blocks = (uint32_t)(k_rows / B);
      if (d == 64) {  // the hot shape: register-blocked scorer
        const size_t smem_rb = 4 * (256 + 16 * 64 + (C * 68 > 16 * 256 ? C * 68 : 16 * 256));
        auto rb = C <= 128 ? select_level_rb_kernel<128> : select_level_rb_kernel<256>;
        if (smem_rb > 48 * 1024)
          LLSA_CUDA_TRY(cudaFuncSetAttribute(rb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem_rb));
        rb<<<dim3(parent_rows, units), C <= 128 ? 128 : 256, smem_rb, s>>>(
            q, q_unit_stride, k, k_unit_stride, parent, parent_unit_stride, parent_k,
            key_blocks, K, scale, out, out_unit_stride, device_flag(), 0x8000000080000000ull);
        count_launch();
        LLSA_LAUNCH_CHECK("select_level_rb_kernel");
        return LLSA_OK;
      }
      auto kern = C <= 128 ? select_level_fast_kernel<8> : select_level_fast_kernel<16>;
      if (smem > 48 * 1024)
        LLSA_CUDA_TRY(
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<dim3(parent_rows, units), 256, smem, s>>>(
          q, q_unit_stride, k, k_unit_stride, parent, parent_unit_stride, parent_k, key_blocks,
          d, K, scale, out, out_unit_stride, device_flag(), 0x8000000080000000ull);
      count_launch();
      LLSA_LAUNCH_CHECK("select_level_fast_kernel");
      return LLSA_OK;
    }
  }
  const uint64_t ld = (d + 3) & ~3u, ldk = ld + 4;
  const uint64_t base = 4 * ((C + 3) & ~3ull) + 4 * B * ld + 4 * ((B * C + 3) & ~3ull) +
                        ((B * C + 15) & ~15ull);
  uint64_t smem = base + 4 * C * ldk;
  bool stage = true;
  if (smem > 200 * 1024) {
    stage = false;
    smem = base;
  }
  if (smem > 200 * 1024)
    return fail(LLSA_ERR_UNSUPPORTED, "select_level: block of %u rows x %llu candidates "
                "exceeds shared memory", B, (unsigned long long)C);
  if (smem > 48 * 1024)
    LLSA_CUDA_TRY(cudaFuncSetAttribute(select_level_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
  const uint32_t key_blocks = (uint32_t)(k_rows / B);
  select_level_kernel<<<dim3(parent_rows, units), 256, smem, s>>>(
      q, q_unit_stride, k, k_unit_stride, parent, parent_unit_stride, parent_k, key_blocks,
      d, K, scale, B, stage, out, out_unit_stride, device_flag());
  count_launch();
  LLSA_LAUNCH_CHECK("select_level_kernel");
  return LLSA_OK;
}

}  // namespace llsa_impl
