// K4 — CSR → CSC index transposition (Alg. 2), P/src/indexmap.cpp:14-88.
//
// Same three linear passes as the reference — count, exclusive prefix sum,
// scatter — then each segment is put into the canonical ascending order.
// Instead of the reference's per-segment std::sort, each element's final slot
// is its rank inside the segment (#elements smaller, ties by scatter slot),
// computed by one warp per key block: no second sort pass, deterministic for
// any scatter order.  Integer-only, HBM/latency-bound and tiny (T·K entries).
#include "common.cuh"
#include "internal.h"

namespace llsa_impl {
namespace {

using namespace llsa_dev;

__global__ void count_kernel(const uint32_t* __restrict__ idx, uint64_t idx_unit_stride,
                             uint64_t per_unit, uint32_t units, uint32_t key_blocks,
                             uint32_t* __restrict__ counts, uint32_t* flag) {
  const uint64_t total = per_unit * units;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = e / per_unit, i = e - u * per_unit;
    const uint32_t b = idx[u * idx_unit_stride + i];
    if (b >= key_blocks) {  // indexmap.cpp:28-38
      raise_flag(flag, kErrIndex);
      continue;
    }
    atomicAdd(&counts[u * key_blocks + b], 1u);
  }
}

// One CTA per unit: exclusive scan of counts → offsets[0..key_blocks], and
// the scatter cursors (= offsets) written back over counts.
__global__ void __launch_bounds__(1024) scan_kernel(uint32_t* __restrict__ counts,
                                                    uint32_t key_blocks,
                                                    uint32_t* __restrict__ offsets,
                                                    uint64_t off_unit_stride) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  const uint32_t u = blockIdx.x;
  uint32_t* cnt = counts + (uint64_t)u * key_blocks;
  uint32_t* off = offsets + (uint64_t)u * off_unit_stride;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t base = 0; base < key_blocks; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < key_blocks ? cnt[i] : 0u;
    uint32_t x = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t t = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= (uint32_t)o) t += y;
      }
      warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t excl = carry + (wid ? warp_tot[wid - 1] : 0u) + x - v;
    if (i < key_blocks) {
      off[i] = excl;
      cnt[i] = excl;  // cursor
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[key_blocks] = carry;
}

__global__ void scatter_kernel(const uint32_t* __restrict__ idx, uint64_t idx_unit_stride,
                               uint32_t rows, uint32_t k, uint32_t units,
                               uint32_t key_blocks, uint32_t* __restrict__ cursor,
                               uint32_t* __restrict__ tmp, uint64_t tmp_unit_stride) {
  const uint64_t per_unit = (uint64_t)rows * k;
  const uint64_t total = per_unit * units;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = e / per_unit, i = e - u * per_unit;
    const uint32_t b = idx[u * idx_unit_stride + i];
    if (b >= key_blocks) continue;
    const uint32_t pos = atomicAdd(&cursor[u * key_blocks + b], 1u);
    tmp[u * tmp_unit_stride + pos] = (uint32_t)(i / k);
  }
}

// Long segments (hot key blocks picked by many query blocks: up to T entries)
// would make the per-element rank scan O(len²); a CTA instead sorts them
// cooperatively.  Kernels collect their long segments in a shared list and,
// after a barrier, the whole CTA sorts each one with a bitonic network in the
// "flip" formulation (every compare-exchange puts the minimum at the lower
// index), which lets the sequence stay unpadded: a partner index ≥ len is a
// virtual +inf and its comparison is a no-op.  Row ids are plain integers,
// so no stability question arises.  O(len log² len) per segment.
constexpr uint32_t kLongSeg = 64;     // longer segments take the CTA sort
constexpr uint32_t kSortSmem = 4096;  // sorted in shared memory up to this length

struct LongSeg {
  const uint32_t* src;
  uint32_t* dst;
  uint32_t len;
};

__device__ __forceinline__ void cx(uint32_t* a, uint32_t i, uint32_t j) {
  const uint32_t x = a[i], y = a[j];
  if (y < x) {
    a[i] = y;
    a[j] = x;
  }
}

// whole-CTA sort of src[0..len) into dst (may run in place over dst)
__device__ void cta_sort_segment(const uint32_t* src, uint32_t* dst, uint32_t len,
                                 uint32_t* sbuf) {
  const bool in_smem = len <= kSortSmem;
  uint32_t* a = in_smem ? sbuf : dst;
  for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) a[e] = src[e];
  __syncthreads();
  for (uint32_t k = 2; k < 2 * len; k <<= 1) {
    // flip step: i ↔ i ^ (k - 1) within each k-block
    for (uint32_t t = threadIdx.x; t < (len + 1) / 2 + k; t += blockDim.x) {
      const uint32_t blk = t / (k / 2), off = t % (k / 2);
      const uint32_t i = blk * k + off, j = blk * k + (k - 1 - off);
      if (j < len) cx(a, i, j);
    }
    __syncthreads();
    for (uint32_t h = k / 4; h >= 1; h >>= 1) {  // half-cleaners
      for (uint32_t t = threadIdx.x; t < (len + 1) / 2 + h; t += blockDim.x) {
        const uint32_t blk = t / h, off = t % h;
        const uint32_t i = blk * 2 * h + off, j = i + h;
        if (j < len) cx(a, i, j);
      }
      __syncthreads();
    }
  }
  if (in_smem) {
    for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) dst[e] = a[e];
    __syncthreads();
  }
}

// One warp per (unit, key block): out[off + rank(e)] = tmp[e]; segments past
// kLongSeg entries take the CTA sort.
__global__ void __launch_bounds__(256) segment_order_kernel(
    const uint32_t* __restrict__ tmp, uint64_t tmp_unit_stride,
    const uint32_t* __restrict__ offsets, uint64_t off_unit_stride, uint32_t key_blocks,
    uint32_t units, uint32_t* __restrict__ flat, uint64_t flat_unit_stride) {
  __shared__ LongSeg longs[8];
  __shared__ uint32_t nlong;
  __shared__ uint32_t sbuf[kSortSmem];
  if (threadIdx.x == 0) nlong = 0;
  __syncthreads();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp < (uint64_t)key_blocks * units) {
    const uint64_t u = warp / key_blocks, b = warp - u * key_blocks;
    const uint32_t* off = offsets + u * off_unit_stride;
    const uint32_t s0 = off[b], s1 = off[b + 1];
    const uint32_t* seg = tmp + u * tmp_unit_stride + s0;
    uint32_t* dst = flat + u * flat_unit_stride + s0;
    const uint32_t len = s1 - s0;
    if (len > kLongSeg) {
      if (lane == 0) longs[atomicAdd(&nlong, 1u)] = LongSeg{seg, dst, len};
    } else {
      for (uint32_t e = lane; e < len; e += 32) {
        const uint32_t v = seg[e];
        uint32_t rank = 0;
        for (uint32_t e2 = 0; e2 < len; ++e2) {
          const uint32_t w = seg[e2];
          rank += (w < v || (w == v && e2 < e)) ? 1u : 0u;
        }
        dst[rank] = v;
      }
    }
  }
  __syncthreads();
  for (uint32_t i = 0; i < nlong; ++i) cta_sort_segment(longs[i].src, longs[i].dst, longs[i].len, sbuf);
}

unsigned grid_for(uint64_t threads, int block) {
  uint64_t blocks = (threads + block - 1) / block;
  const uint64_t cap = 148ull * 16;
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

}  // namespace

size_t transpose_ws_bytes(uint32_t units, uint32_t rows, uint32_t k, uint32_t key_blocks) {
  const size_t a = ((size_t)units * key_blocks * 4 + 255) & ~size_t(255);
  const size_t b = ((size_t)units * rows * k * 4 + 255) & ~size_t(255);
  return a + b + 256;
}

llsa_status launch_transpose(const uint32_t* idx, uint64_t idx_unit_stride, uint32_t units,
                             uint32_t rows, uint32_t k, uint32_t key_blocks,
                             uint32_t* offsets, uint64_t off_unit_stride, uint32_t* flat,
                             uint64_t flat_unit_stride, void* ws, cudaStream_t s) {
  if (units == 0) return LLSA_OK;
  uint32_t* counts = static_cast<uint32_t*>(ws);
  uint32_t* tmp = reinterpret_cast<uint32_t*>(
      static_cast<char*>(ws) + (((size_t)units * key_blocks * 4 + 255) & ~size_t(255)));
  const uint64_t per_unit = (uint64_t)rows * k;
  if (key_blocks) LLSA_CUDA_TRY(cudaMemsetAsync(counts, 0, (size_t)units * key_blocks * 4, s));
  if (per_unit && key_blocks) {
    count_kernel<<<grid_for(per_unit * units, 256), 256, 0, s>>>(
        idx, idx_unit_stride, per_unit, units, key_blocks, counts, device_flag());
    count_launch();
    LLSA_LAUNCH_CHECK("count_kernel");
  }
  scan_kernel<<<units, 1024, 0, s>>>(counts, key_blocks, offsets, off_unit_stride);
  count_launch();
  LLSA_LAUNCH_CHECK("scan_kernel");
  if (per_unit == 0 || key_blocks == 0) return LLSA_OK;
  scatter_kernel<<<grid_for(per_unit * units, 256), 256, 0, s>>>(
      idx, idx_unit_stride, rows, k, units, key_blocks, counts, tmp, per_unit);
  count_launch();
  LLSA_LAUNCH_CHECK("scatter_kernel");
  const uint64_t warps = (uint64_t)key_blocks * units;
  segment_order_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(
      tmp, per_unit, offsets, off_unit_stride, key_blocks, units, flat, flat_unit_stride);
  count_launch();
  LLSA_LAUNCH_CHECK("segment_order_kernel");
  return LLSA_OK;
}

}  // namespace llsa_impl

// ---------------------------------------------------------------------------
// All levels at once (the handle path): the same four phases, one launch
// each, blockIdx.y = level; per-level geometry in a by-value table.
// ---------------------------------------------------------------------------
namespace llsa_impl {
namespace {

constexpr int kTrMax = 8;
struct TrAll {
  const uint32_t* idx[kTrMax];
  uint32_t* counts[kTrMax];
  uint32_t* tmp[kTrMax];
  uint32_t* offs[kTrMax];
  uint32_t* flat[kTrMax];
  uint32_t rows[kTrMax], kb[kTrMax];
  uint64_t idx_stride, off_stride, flat_stride;
  uint32_t units, k, levels;
  uint32_t* flag;
};

__global__ void count_all_kernel(TrAll a) {
  const uint32_t l = blockIdx.y;
  const uint64_t per_unit = (uint64_t)a.rows[l] * a.k, total = per_unit * a.units;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = e / per_unit, i = e - u * per_unit;
    const uint32_t b = a.idx[l][u * a.idx_stride + i];
    if (b >= a.kb[l]) {
      raise_flag(a.flag, kErrIndex);
      continue;
    }
    atomicAdd(&a.counts[l][u * a.kb[l] + b], 1u);
  }
}

__global__ void __launch_bounds__(1024) scan_all_kernel(TrAll a) {
  const uint32_t l = blockIdx.y;
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  const uint32_t u = blockIdx.x, kbn = a.kb[l];
  uint32_t* cnt = a.counts[l] + (uint64_t)u * kbn;
  uint32_t* off = a.offs[l] + (uint64_t)u * a.off_stride;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t base = 0; base < kbn; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < kbn ? cnt[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t t = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= (uint32_t)o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const uint32_t excl = carry + (wid ? warp_tot[wid - 1] : 0u) + x - v;
    if (i < kbn) {
      off[i] = excl;
      cnt[i] = excl;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[kbn] = carry;
}

__global__ void scatter_all_kernel(TrAll a) {
  const uint32_t l = blockIdx.y;
  const uint64_t per_unit = (uint64_t)a.rows[l] * a.k, total = per_unit * a.units;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = e / per_unit, i = e - u * per_unit;
    const uint32_t b = a.idx[l][u * a.idx_stride + i];
    if (b >= a.kb[l]) continue;
    const uint32_t pos = atomicAdd(&a.counts[l][u * a.kb[l] + b], 1u);
    a.tmp[l][u * per_unit + pos] = (uint32_t)(i / a.k);
  }
}

// One 8-lane group per key block (four blocks per warp): segments of up to 8
// entries are ranked with group shuffles, up to kLongSeg by the group's lanes
// scanning the segment, longer ones by the CTA sort.
__global__ void __launch_bounds__(256) segment_order_all_kernel(TrAll a) {
  __shared__ LongSeg longs[32];
  __shared__ uint32_t nlong;
  __shared__ uint32_t sbuf[kSortSmem];
  if (threadIdx.x == 0) nlong = 0;
  __syncthreads();
  const uint32_t l = blockIdx.y;
  const uint64_t grp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 3;
  const uint32_t sl = threadIdx.x & 7;
  const uint64_t nb = (uint64_t)a.kb[l] * a.units;
  const bool live = grp < nb;
  uint32_t len = 0, s0 = 0;
  const uint32_t* seg = nullptr;
  uint32_t* dst = nullptr;
  if (live) {
    const uint64_t u = grp / a.kb[l], b = grp - u * a.kb[l];
    const uint32_t* off = a.offs[l] + u * a.off_stride;
    s0 = off[b];
    len = off[b + 1] - s0;
    seg = a.tmp[l] + u * (uint64_t)a.rows[l] * a.k + s0;
    dst = a.flat[l] + u * a.flat_stride + s0;
  }
  // the group's 8 lanes share len, so the branches below are group-uniform;
  // shuffles run over the whole warp with width 8
  const bool small = len <= 8;
  const uint32_t v = (live && small && sl < len) ? seg[sl] : 0xffffffffu;
  uint32_t rank = 0;
  for (uint32_t e2 = 0; e2 < 8; ++e2) {
    const uint32_t w = __shfl_sync(0xffffffffu, v, e2, 8);
    rank += (e2 < len && (w < v || (w == v && e2 < sl))) ? 1u : 0u;
  }
  if (live && small && sl < len) dst[rank] = v;
  if (live && !small && len <= kLongSeg) {
    for (uint32_t e = sl; e < len; e += 8) {
      const uint32_t x = seg[e];
      uint32_t r = 0;
      for (uint32_t e2 = 0; e2 < len; ++e2) {
        const uint32_t w = seg[e2];
        r += (w < x || (w == x && e2 < e)) ? 1u : 0u;
      }
      dst[r] = x;
    }
  } else if (live && len > kLongSeg && sl == 0) {
    longs[atomicAdd(&nlong, 1u)] = LongSeg{seg, dst, len};
  }
  __syncthreads();
  for (uint32_t i = 0; i < nlong; ++i) cta_sort_segment(longs[i].src, longs[i].dst, longs[i].len, sbuf);
}

}  // namespace

bool transpose_all_fused_ok(const Geometry& g) { return g.L >= 1 && g.L <= kTrMax; }

size_t transpose_all_fused_ws(const Geometry& g, uint32_t units) {
  size_t b = 256;
  for (uint32_t l = 0; l < g.L; ++l) {
    b += ((size_t)units * g.level_blocks(l) * 4 + 255) & ~size_t(255);
    b += ((size_t)units * g.level_blocks(l) * g.K * 4 + 255) & ~size_t(255);
  }
  return b;
}

llsa_status transpose_all_fused(const Geometry& g, uint32_t units, const uint32_t* tables,
                                uint32_t* offs, uint32_t* flat, void* ws, cudaStream_t s) {
  TrAll a{};
  char* p = static_cast<char*>(ws);
  size_t cbytes = 0;
  uint64_t maxe = 0, maxkb = 0;
  for (uint32_t l = 0; l < g.L; ++l) {  // counts of every level are contiguous (one memset)
    a.counts[l] = reinterpret_cast<uint32_t*>(p + cbytes);
    cbytes += ((size_t)units * g.level_blocks(l) * 4 + 255) & ~size_t(255);
  }
  size_t tb = cbytes;
  for (uint32_t l = 0; l < g.L; ++l) {
    const uint64_t rows = g.level_blocks(l), kb = g.level_blocks(l);  // square per level
    a.tmp[l] = reinterpret_cast<uint32_t*>(p + tb);
    tb += ((size_t)units * rows * g.K * 4 + 255) & ~size_t(255);
    a.idx[l] = tables + g.table_off[l];
    a.offs[l] = offs + g.csc_off_off[l];
    a.flat[l] = flat + g.csc_flat_off[l];
    a.rows[l] = (uint32_t)rows;
    a.kb[l] = (uint32_t)kb;
    maxe = rows * g.K > maxe ? rows * g.K : maxe;
    maxkb = kb > maxkb ? kb : maxkb;
  }
  a.idx_stride = g.table_entries;
  a.off_stride = g.csc_off_entries;
  a.flat_stride = g.csc_flat_entries;
  a.units = units;
  a.k = g.K;
  a.levels = g.L;
  a.flag = device_flag();
  LLSA_CUDA_TRY(cudaMemsetAsync(ws, 0, cbytes, s));
  const dim3 ge(grid_for(maxe * units, 256), g.L);
  count_all_kernel<<<ge, 256, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("count_all_kernel");
  scan_all_kernel<<<dim3(units, g.L), 1024, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("scan_all_kernel");
  scatter_all_kernel<<<ge, 256, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("scatter_all_kernel");
  const uint64_t groups = maxkb * units;  // 8 lanes per key block
  segment_order_all_kernel<<<dim3((unsigned)((groups * 8 + 255) / 256), g.L), 256, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("segment_order_all_kernel");
  return LLSA_OK;
}

}  // namespace llsa_impl

// ---------------------------------------------------------------------------
// Mask-based key→query lookup: the measured baseline of the key/value
// backward (SURVEY.md §8(f) row 2, P/src/oracle.cpp:365-501).  Per level a
// dense query-block × key-block bit mask is built from the tables, and every
// key block scans its whole mask column — O(T_q·T_k) per level instead of
// the CSR→CSC pass's O(T·K).  The column scan visits rows in ascending order,
// so it emits the same canonical CSC as llsa_transpose_all and the same
// key-major backward kernels then consume it.
// ---------------------------------------------------------------------------
namespace llsa_impl {
namespace {

struct MaskAll {
  const uint32_t* idx[kTrMax];
  uint32_t* mask[kTrMax];   // [units][T_q][words]
  uint32_t* offs[kTrMax];
  uint32_t* flat[kTrMax];
  uint32_t rows[kTrMax], kb[kTrMax], words[kTrMax];
  uint64_t idx_stride, off_stride, flat_stride, mask_stride[kTrMax];
  uint32_t units, k;
  uint32_t* flag;
};

__global__ void mask_build_kernel(MaskAll a) {
  const uint32_t l = blockIdx.y;
  const uint64_t per_unit = (uint64_t)a.rows[l] * a.k, total = per_unit * a.units;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = e / per_unit, i = e - u * per_unit, row = i / a.k;
    const uint32_t b = a.idx[l][u * a.idx_stride + i];
    if (b >= a.kb[l]) {
      raise_flag(a.flag, kErrIndex);
      continue;
    }
    atomicOr(&a.mask[l][u * a.mask_stride[l] + row * a.words[l] + (b >> 5)], 1u << (b & 31));
  }
}

// thread = (unit, key block): count (pass 0) or emit (pass 1) its column.
__global__ void mask_scan_kernel(MaskAll a, int pass) {
  const uint32_t l = blockIdx.y;
  const uint64_t total = (uint64_t)a.kb[l] * a.units;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = t / a.kb[l], b = t - u * a.kb[l];
    const uint32_t* m = a.mask[l] + u * a.mask_stride[l] + (b >> 5);
    const uint32_t bit = 1u << (b & 31);
    uint32_t* off = a.offs[l] + u * a.off_stride;
    if (pass == 0) {
      uint32_t c = 0;
      for (uint32_t i = 0; i < a.rows[l]; ++i) c += (m[(uint64_t)i * a.words[l]] & bit) ? 1u : 0u;
      off[b] = c;  // count, turned into offsets by the scan
    } else {
      uint32_t* dst = a.flat[l] + u * a.flat_stride + off[b];
      for (uint32_t i = 0; i < a.rows[l]; ++i)
        if (m[(uint64_t)i * a.words[l]] & bit) *dst++ = i;
    }
  }
}

// in-place exclusive scan of counts[0..kb) → offsets[0..kb]; CTA = (unit, level)
__global__ void __launch_bounds__(1024) mask_offsets_kernel(MaskAll a) {
  const uint32_t l = blockIdx.y, u = blockIdx.x, kbn = a.kb[l];
  uint32_t* off = a.offs[l] + (uint64_t)u * a.off_stride;
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t base = 0; base < kbn; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < kbn ? off[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t t = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= (uint32_t)o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const uint32_t excl = carry + (wid ? warp_tot[wid - 1] : 0u) + x - v;
    if (i < kbn) off[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[kbn] = carry;
}

}  // namespace

size_t mask_lookup_ws_bytes(const Geometry& g, uint32_t units) {
  size_t b = 256;
  for (uint32_t l = 0; l < g.L && l < (uint32_t)kTrMax; ++l)
    b += ((size_t)units * g.level_blocks(l) * ((g.level_blocks(l) + 31) / 32) * 4 + 255) &
         ~size_t(255);
  return b;
}

llsa_status mask_lookup(const Geometry& g, uint32_t units, const uint32_t* tables,
                        uint32_t* offs, uint32_t* flat, void* ws, cudaStream_t s) {
  if (g.L > (uint32_t)kTrMax) return fail(LLSA_ERR_UNSUPPORTED, "too many levels");
  MaskAll a{};
  char* p = static_cast<char*>(ws);
  size_t mb = 0;
  uint64_t maxe = 0, maxkb = 0;
  for (uint32_t l = 0; l < g.L; ++l) {
    const uint64_t t = g.level_blocks(l);
    a.words[l] = (uint32_t)((t + 31) / 32);
    a.mask_stride[l] = t * a.words[l];
    a.mask[l] = reinterpret_cast<uint32_t*>(p + mb);
    mb += ((size_t)units * a.mask_stride[l] * 4 + 255) & ~size_t(255);
    a.idx[l] = tables + g.table_off[l];
    a.offs[l] = offs + g.csc_off_off[l];
    a.flat[l] = flat + g.csc_flat_off[l];
    a.rows[l] = (uint32_t)t;
    a.kb[l] = (uint32_t)t;
    maxe = t * g.K > maxe ? t * g.K : maxe;
    maxkb = t > maxkb ? t : maxkb;
  }
  a.idx_stride = g.table_entries;
  a.off_stride = g.csc_off_entries;
  a.flat_stride = g.csc_flat_entries;
  a.units = units;
  a.k = g.K;
  a.flag = device_flag();
  LLSA_CUDA_TRY(cudaMemsetAsync(ws, 0, mb, s));
  mask_build_kernel<<<dim3(grid_for(maxe * units, 256), g.L), 256, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("mask_build_kernel");
  const dim3 gs(grid_for(maxkb * units, 128), g.L);
  mask_scan_kernel<<<gs, 128, 0, s>>>(a, 0);
  count_launch();
  LLSA_LAUNCH_CHECK("mask_scan_kernel");
  mask_offsets_kernel<<<dim3(units, g.L), 1024, 0, s>>>(a);
  count_launch();
  LLSA_LAUNCH_CHECK("mask_offsets_kernel");
  mask_scan_kernel<<<gs, 128, 0, s>>>(a, 1);
  count_launch();
  LLSA_LAUNCH_CHECK("mask_scan_kernel");
  return LLSA_OK;
}

}  // namespace llsa_impl

// ---------------------------------------------------------------------------
// CSC → CSR: the per-level selection tables rebuilt from the key→query lists
// (kv_backward receives only the transposed lists, attention_grad.hpp:32-37,
// while the tensor-core backward walks the query-major tables as well).
// Every query block appears K times per level; its row is filled by atomic
// cursors and then sorted ascending (the tables' canonical order,
// selection.cpp:37), so the result is deterministic.
// ---------------------------------------------------------------------------
namespace llsa_impl {
namespace {

__global__ void csc_scatter_kernel(const uint32_t* __restrict__ offs,
                                   const uint32_t* __restrict__ flat, uint32_t units,
                                   uint32_t key_blocks, uint32_t rows, uint32_t K,
                                   uint64_t off_stride, uint64_t flat_stride,
                                   uint64_t tab_stride, uint32_t* __restrict__ cursor,
                                   uint32_t* __restrict__ tables, uint32_t* flag) {
  const uint64_t total = (uint64_t)units * key_blocks;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = t / key_blocks, b = t - u * key_blocks;
    const uint32_t* o = offs + u * off_stride;
    const uint32_t s0 = o[b], s1 = o[b + 1];
    if (s1 < s0 || s1 > rows * K) {
      raise_flag(flag, kErrIndex);
      continue;
    }
    for (uint32_t e = s0; e < s1; ++e) {
      const uint32_t q = flat[u * flat_stride + e];
      if (q >= rows) {
        raise_flag(flag, kErrIndex);
        continue;
      }
      const uint32_t pos = atomicAdd(&cursor[u * rows + q], 1u);
      if (pos >= K) {
        raise_flag(flag, kErrIndex);
        continue;
      }
      tables[u * tab_stride + (uint64_t)q * K + pos] = (uint32_t)b;
    }
  }
}

__global__ void row_sort_kernel(uint32_t* __restrict__ tables, uint32_t units, uint32_t rows,
                                uint32_t K, uint64_t tab_stride,
                                const uint32_t* __restrict__ cursor, uint32_t* flag) {
  const uint64_t total = (uint64_t)units * rows;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = t / rows, r = t - u * rows;
    if (cursor[t] != K) raise_flag(flag, kErrIndex);  // a query block not listed K times
    uint32_t* row = tables + u * tab_stride + r * K;
    for (uint32_t i = 1; i < K; ++i) {
      const uint32_t x = row[i];
      uint32_t j = i;
      for (; j > 0 && row[j - 1] > x; --j) row[j] = row[j - 1];
      row[j] = x;
    }
  }
}

}  // namespace

size_t tables_from_csc_ws(const Geometry& g, uint32_t units) {
  size_t rows = 0;
  for (uint32_t l = 0; l < g.L; ++l) rows += g.level_blocks(l);
  return ((size_t)units * rows * 4 + 255) & ~size_t(255);
}

llsa_status tables_from_csc(const Geometry& g, uint32_t units, const uint32_t* offs,
                            const uint32_t* flat, uint32_t* tables, void* ws, cudaStream_t s) {
  uint32_t* cursor = static_cast<uint32_t*>(ws);
  LLSA_CUDA_TRY(cudaMemsetAsync(cursor, 0, tables_from_csc_ws(g, units), s));
  size_t crow = 0;
  for (uint32_t l = 0; l < g.L; ++l) {
    const uint32_t rows = (uint32_t)g.level_blocks(l);  // query blocks = key blocks per level
    uint32_t* cur = cursor + (size_t)units * crow;
    csc_scatter_kernel<<<grid_for((uint64_t)units * rows, 256), 256, 0, s>>>(
        offs + g.csc_off_off[l], flat + g.csc_flat_off[l], units, rows, rows, g.K,
        g.csc_off_entries, g.csc_flat_entries, g.table_entries, cur,
        tables + g.table_off[l], device_flag());
    count_launch();
    LLSA_LAUNCH_CHECK("csc_scatter_kernel");
    row_sort_kernel<<<grid_for((uint64_t)units * rows, 256), 256, 0, s>>>(
        tables + g.table_off[l], units, rows, g.K, g.table_entries, cur, device_flag());
    count_launch();
    LLSA_LAUNCH_CHECK("row_sort_kernel");
    crow += rows;
  }
  return LLSA_OK;
}

}  // namespace llsa_impl
