// The reference operator API (namespace llsa, include/llsa/*.hpp) on top of
// the C ABI (include/llsa_cuda.h).  Each call validates on the host exactly
// where and how the reference throws (file:line cited per function), copies
// host FeatureMatrix data to device buffers, runs the GPU kernels, copies the
// results back and turns device-side errors into the same typed exceptions.
// Unmodified reference callers compile and link against this library.
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <ostream>
#include <string>
#include <vector>

#include "llsa/attention.hpp"
#include "llsa/attention_grad.hpp"
#include "llsa/config.hpp"
#include "llsa/errors.hpp"
#include "llsa/indexmap.hpp"
#include "llsa/parallel.hpp"
#include "llsa/pyramid.hpp"
#include "llsa/selection.hpp"
#include "llsa/types.hpp"
#include "llsa_cuda.h"

namespace llsa {

void throw_status(int st) {
  const std::string msg = llsa_last_error();
  switch (st) {
    case LLSA_OK: return;
    case LLSA_ERR_CONFIG: throw ConfigError(msg);
    case LLSA_ERR_DIVISIBILITY: throw DivisibilityError(msg);
    case LLSA_ERR_LEVEL: throw LevelError(msg);
    case LLSA_ERR_TOPK: throw TopKError(msg);
    case LLSA_ERR_SHAPE: throw ShapeMismatch(msg);
    case LLSA_ERR_INDEX_RANGE: throw IndexOutOfRange(msg);
    case LLSA_ERR_NONFINITE: throw NonFiniteError(msg);
    case LLSA_ERR_STALE_STATE: throw StaleState(msg);
    case LLSA_ERR_FORMAT: throw FormatError(msg);
    case LLSA_ERR_IO: throw IoError(msg);
    case LLSA_ERR_PRECISION: throw PrecisionError(msg);
    case LLSA_ERR_NOT_SQUARE_BLOCK: throw NotSquareBlock(msg);
    case LLSA_ERR_ORACLE_CAP: throw OracleCapExceeded(msg);
    default: throw DeviceError(std::string(llsa_status_name(static_cast<llsa_status>(st))) +
                               ": " + msg);
  }
}

namespace {

void ck(llsa_status s) {
  if (s != LLSA_OK) throw_status(s);
}
void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}
// Wait for the GPU and raise what the kernels flagged (IndexOutOfRange,
// NonFiniteError), as the reference does when its loops finish.
void finish() { ck(llsa_sync_status(nullptr)); }

// Device scratch for the host-buffer API: a process-wide caching pool keyed
// by power-of-two size class, so a call sequence reuses device memory instead
// of paying cudaMalloc/cudaFree (an implicit device synchronisation) per
// call.  Cached blocks are kept up to kPoolCap bytes; beyond that they are
// returned to the driver.
class DevicePool {
 public:
  static DevicePool& get() {
    static DevicePool* pool = new DevicePool();  // intentionally leaked: no teardown-order hazards
    return *pool;
  }
  void* acquire(std::size_t bytes, std::size_t* cls_out) {
    const std::size_t cls = std::bit_ceil(std::max<std::size_t>(bytes, 256));
    *cls_out = cls;
    {
      std::lock_guard<std::mutex> g(mu_);
      auto it = free_.find(cls);
      if (it != free_.end() && !it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        cached_ -= cls;
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, cls);
    if (e != cudaSuccess) {  // release the cache once and retry
      trim();
      (void)cudaGetLastError();
      e = cudaMalloc(&p, cls);
    }
    ckc(e, "cudaMalloc");
    return p;
  }
  void release(void* p, std::size_t cls) {
    {
      std::lock_guard<std::mutex> g(mu_);
      if (cached_ + cls <= kPoolCap) {
        free_[cls].push_back(p);
        cached_ += cls;
        return;
      }
    }
    cudaFree(p);
  }
  void trim() {
    std::lock_guard<std::mutex> g(mu_);
    for (auto& [cls, v] : free_)
      for (void* p : v) cudaFree(p);
    free_.clear();
    cached_ = 0;
  }

 private:
  static constexpr std::size_t kPoolCap = std::size_t(4) << 30;
  std::mutex mu_;
  std::map<std::size_t, std::vector<void*>> free_;
  std::size_t cached_ = 0;
};

template <typename T>
class DevBuf {
 public:
  explicit DevBuf(std::size_t n) : n_(n) {
    if (n_) p_ = static_cast<T*>(DevicePool::get().acquire(n_ * sizeof(T), &cls_));
  }
  DevBuf(const T* host, std::size_t n) : DevBuf(n) { upload(host); }
  ~DevBuf() {
    if (p_) DevicePool::get().release(p_, cls_);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  T* get() const { return p_; }
  void upload(const T* host) {
    if (n_) ckc(cudaMemcpy(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  }
  void download(T* host) const {
    if (n_) ckc(cudaMemcpy(host, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0, cls_ = 0;
};

llsa_config to_c(const LLSAConfig& c) {
  llsa_config r{};
  r.n = c.n;
  r.d = c.d;
  r.block_size = c.block_size;
  r.top_k = c.top_k;
  r.levels = c.levels;
  r.enrich_levels = c.enrich_levels;
  r.softmax_scale = static_cast<float>(c.softmax_scale);
  r.reweight_mode = static_cast<uint32_t>(c.reweight_mode);
  r.safe_softmax = c.safe_softmax ? 1u : 0u;
  return r;
}

// Levels 1..L of a pyramid concatenated ([pyr_rows][d]); levels missing from
// a shallower pyramid are left zero (the plan never reads them).
std::vector<real> concat_levels(const Pyramid& p, const ValidatedConfig& cfg) {
  std::vector<real> out;
  out.reserve(static_cast<std::size_t>(llsa_pyramid_rows(cfg.n(), cfg.block_size(),
                                                         cfg.levels())) * cfg.d());
  for (std::uint32_t l = 1; l <= cfg.levels(); ++l) {
    const std::size_t want = static_cast<std::size_t>(cfg.level_tokens(l)) * cfg.d();
    if (l < p.levels.size() && p.level(l).size() == want) {
      out.insert(out.end(), p.level(l).data(), p.level(l).data() + want);
    } else {
      out.insert(out.end(), want, real(0));
    }
  }
  return out;
}

// Per-level tables concatenated in the C-ABI layout (zeros where a level's
// table is absent or of another shape; only validated levels are read).
std::vector<std::uint32_t> concat_tables(const SelectionResult& sel, const ValidatedConfig& cfg) {
  std::vector<std::uint32_t> out;
  for (std::uint32_t l = 0; l < cfg.levels(); ++l) {
    const std::size_t want = static_cast<std::size_t>(cfg.level_blocks(l)) * cfg.top_k();
    if (l < sel.per_level.size() && sel.per_level[l].indices.size() == want) {
      out.insert(out.end(), sel.per_level[l].indices.begin(), sel.per_level[l].indices.end());
    } else {
      out.insert(out.end(), want, 0u);
    }
  }
  return out;
}

void concat_csc(const std::vector<TransposedIndices>& tr, const ValidatedConfig& cfg,
                std::vector<std::uint32_t>& offs, std::vector<std::uint32_t>& flat) {
  for (std::uint32_t l = 0; l < cfg.levels(); ++l) {
    const std::size_t kb = cfg.level_blocks(l);
    const std::size_t nf = kb * cfg.top_k();
    if (l < tr.size() && tr[l].offsets.size() == kb + 1 && tr[l].flat_queries.size() == nf) {
      offs.insert(offs.end(), tr[l].offsets.begin(), tr[l].offsets.end());
      flat.insert(flat.end(), tr[l].flat_queries.begin(), tr[l].flat_queries.end());
    } else {
      offs.insert(offs.end(), kb + 1, 0u);
      flat.insert(flat.end(), nf, 0u);
    }
  }
}

void fnv(std::uint64_t& h, std::uint64_t w) {
  h ^= w;
  h *= 0x100000001b3ULL;
}

void fnv_matrix(std::uint64_t& h, const FeatureMatrix& m) {
  fnv(h, m.rows());
  fnv(h, m.cols());
  for (std::size_t i = 0; i < m.size(); ++i) fnv(h, std::bit_cast<std::uint32_t>(m.data()[i]));
}

std::uint32_t deepest_level(const EnrichedKVPlan& plan) {
  std::uint32_t top = 0;
  for (const PlanEntry& e : plan.entries) top = std::max(top, e.level);
  return top;
}

void check_saved(const FeatureMatrix& d_out, const ForwardState& saved,
                 const ValidatedConfig& cfg) {
  // P/src/attention_grad.cpp:75-86
  const std::size_t n = cfg.n(), d = cfg.d();
  if (d_out.rows() != n || d_out.cols() != d) throw ShapeMismatch("cotangent must be n x d");
  if (saved.output.rows() != n || saved.output.cols() != d || saved.row_max.size() != n ||
      saved.row_denom.size() != n)
    throw ShapeMismatch("saved forward state has wrong dimensions");
}

std::uint64_t kv_macs(const std::vector<TransposedIndices>& tr, const ValidatedConfig& cfg) {
  // P/src/attention_grad.cpp:114,164,198
  const std::uint64_t n = cfg.n(), d = cfg.d(), B = cfg.block_size();
  std::uint64_t m = 2 * n * d;
  const std::uint32_t lim = std::min(cfg.enrich_levels() + 1, cfg.levels());
  for (std::uint32_t l = 0; l < lim; ++l)
    m += std::uint64_t(tr[l].flat_queries.size()) * cfg.pow_block(l + 1) * B * 4 * d;
  if (cfg.enrich_levels() == cfg.levels()) m += n * cfg.level_tokens(cfg.levels()) * 4 * d;
  return m;
}

}  // namespace

// ---- types -----------------------------------------------------------------
FeatureMatrix::FeatureMatrix(std::size_t rows, std::size_t cols)
    : n_rows_(rows), n_cols_(cols), data_(rows * cols, real(0)) {}

FeatureMatrix FeatureMatrix::from_values(std::size_t rows, std::size_t cols,
                                         std::vector<real> values) {
  if (values.size() != rows * cols)
    throw ShapeMismatch("matrix buffer holds " + std::to_string(values.size()) +
                        " values, expected " + std::to_string(rows * cols));
  FeatureMatrix m;
  m.n_rows_ = rows;
  m.n_cols_ = cols;
  m.data_ = std::move(values);
  if (!m.all_finite()) throw NonFiniteError("matrix contains NaN or infinite values");
  return m;
}

bool FeatureMatrix::all_finite() const noexcept {
  return std::all_of(data_.begin(), data_.end(), [](real v) { return std::isfinite(v); });
}

real max_abs_diff(const FeatureMatrix& a, const FeatureMatrix& b) {
  if (!a.same_shape(b)) throw ShapeMismatch("max_abs_diff: shapes differ");
  real worst = 0;
  for (std::size_t i = 0; i < a.size(); ++i)
    worst = std::max(worst, std::abs(a.data()[i] - b.data()[i]));
  return worst;
}

// ---- config ----------------------------------------------------------------
const char* to_string(ReweightMode mode) {
  return mode == ReweightMode::ScaleKV ? "scalekv" : "logitbias";
}

std::uint32_t max_levels(std::uint64_t n, std::uint32_t block_size) {
  return llsa_max_levels(n, block_size);
}

ValidatedConfig validate_config(const LLSAConfig& cfg) {
  const llsa_config c = to_c(cfg);
  float scale = 0.f;
  ck(llsa_validate_config(&c, &scale, nullptr));
  ValidatedConfig v;
  v.raw_ = cfg;
  v.scale_ = cfg.softmax_scale > real(0) ? cfg.softmax_scale : static_cast<real>(scale);
  v.powers_.assign(cfg.levels + 2, 1);
  for (std::uint32_t l = 1; l < v.powers_.size(); ++l)
    v.powers_[l] = v.powers_[l - 1] * cfg.block_size;
  return v;
}

std::uint32_t effective_block_count(const ValidatedConfig& cfg) {
  const llsa_config c = to_c(cfg.raw());
  std::uint32_t e = 0;
  ck(llsa_validate_config(&c, nullptr, &e));
  return e;
}

// ---- parallel (host knob only) --------------------------------------------
namespace {
unsigned g_threads = 0;
}
void set_thread_count(unsigned count) { g_threads = count; }
unsigned thread_count() { return g_threads ? g_threads : 1; }
void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& body) {
  if (n) body(0, n);
}
std::uint64_t parallel_sum(std::size_t n,
                           const std::function<std::uint64_t(std::size_t, std::size_t)>& body) {
  return n ? body(0, n) : 0;
}

// ---- pyramid (P/src/pyramid.cpp:11-64) -------------------------------------
Pyramid build_pyramid(const FeatureMatrix& x, std::uint32_t block_size, std::uint32_t levels) {
  if (block_size < 2) throw DivisibilityError("block size must be at least 2");
  std::size_t rows = x.rows();
  for (std::uint32_t l = 1; l <= levels; ++l) {
    if (rows % block_size != 0)
      throw DivisibilityError("level " + std::to_string(l - 1) + " has " + std::to_string(rows) +
                              " rows, not a multiple of block size " +
                              std::to_string(block_size));
    rows /= block_size;
  }
  Pyramid p;
  p.levels.reserve(levels + 1);
  p.levels.push_back(x);
  const std::uint64_t pr = llsa_pyramid_rows(x.rows(), block_size, levels);
  if (levels == 0) return p;
  DevBuf<real> dx(x.data(), x.size());
  DevBuf<real> dout(pr * x.cols());
  ck(llsa_build_pyramid(dx.get(), LLSA_F32, 1, x.rows(), static_cast<std::uint32_t>(x.cols()),
                        block_size, levels, dout.get(), nullptr));
  finish();
  std::vector<real> host(pr * x.cols());
  dout.download(host.data());
  std::size_t off = 0, r = x.rows();
  for (std::uint32_t l = 1; l <= levels; ++l) {
    r /= block_size;
    FeatureMatrix m(r, x.cols());
    std::copy(host.begin() + off, host.begin() + off + m.size(), m.data());
    off += m.size();
    p.levels.push_back(std::move(m));
  }
  return p;
}

FeatureMatrix pool_backward(const FeatureMatrix& d_coarse, std::uint32_t block_size,
                            std::uint32_t hops) {
  if (hops == 0) return d_coarse;
  if (block_size < 2) throw DivisibilityError("block size must be at least 2");
  std::size_t group = 1;
  for (std::uint32_t h = 0; h < hops; ++h) group *= block_size;
  FeatureMatrix fine(d_coarse.rows() * group, d_coarse.cols());
  if (fine.empty()) return fine;
  DevBuf<real> g(d_coarse.data(), d_coarse.size());
  DevBuf<real> o(fine.size());
  ck(llsa_pool_backward(g.get(), 1, d_coarse.rows(), static_cast<std::uint32_t>(d_coarse.cols()),
                        block_size, hops, o.get(), nullptr));
  finish();
  o.download(fine.data());
  return fine;
}

// ---- selection (P/src/selection.cpp:42-189) --------------------------------
LevelIndices select_coarsest(const FeatureMatrix& q_top, const FeatureMatrix& k_top,
                             std::uint32_t top_k, real scale, std::uint32_t out_level,
                             std::uint64_t* mul_accs) {
  if (q_top.cols() != k_top.cols())
    throw ShapeMismatch("coarsest selection: query/key widths differ");
  const auto cands = static_cast<std::uint32_t>(k_top.rows());
  if (top_k < 1 || top_k > cands)
    throw TopKError("top_k " + std::to_string(top_k) + " outside [1, " + std::to_string(cands) +
                    "]");
  LevelIndices out;
  out.level = out_level;
  out.query_blocks = static_cast<std::uint32_t>(q_top.rows());
  out.k = top_k;
  out.indices.resize(std::size_t(out.query_blocks) * top_k);
  if (!out.indices.empty()) {
    DevBuf<real> q(q_top.data(), q_top.size()), k(k_top.data(), k_top.size());
    DevBuf<std::uint32_t> o(out.indices.size());
    ck(llsa_select_coarsest(q.get(), k.get(), 1, out.query_blocks, cands,
                            static_cast<std::uint32_t>(q_top.cols()), top_k, scale, o.get(),
                            nullptr));
    finish();
    o.download(out.indices.data());
  }
  if (mul_accs) *mul_accs += std::uint64_t(q_top.rows()) * cands * q_top.cols();
  return out;
}

LevelIndices select_level(const FeatureMatrix& q_level, const FeatureMatrix& k_level,
                          const LevelIndices& parent, std::uint32_t top_k, real scale,
                          std::uint32_t block_size, std::uint64_t* mul_accs) {
  if (parent.level == 0) throw LevelError("select_level needs a parent table at level >= 1");
  if (q_level.cols() != k_level.cols())
    throw ShapeMismatch("level selection: query/key widths differ");
  if (q_level.rows() != std::size_t(parent.query_blocks) * block_size)
    throw ShapeMismatch("level selection: expected " +
                        std::to_string(std::size_t(parent.query_blocks) * block_size) +
                        " query tokens, got " + std::to_string(q_level.rows()));
  if (block_size == 0 || k_level.rows() % block_size != 0)
    throw ShapeMismatch("level selection: key token count not a multiple of the block size");
  const std::uint32_t cands = parent.k * block_size;
  if (top_k < 1 || top_k > cands)
    throw TopKError("top_k " + std::to_string(top_k) + " outside [1, " + std::to_string(cands) +
                    "]");
  const auto key_blocks = static_cast<std::uint32_t>(k_level.rows() / block_size);
  for (std::uint32_t idx : parent.indices)
    if (idx >= key_blocks)
      throw IndexOutOfRange("parent index " + std::to_string(idx) + " >= key block count " +
                            std::to_string(key_blocks));
  LevelIndices out;
  out.level = parent.level - 1;
  out.query_blocks = static_cast<std::uint32_t>(q_level.rows());
  out.k = top_k;
  out.indices.resize(std::size_t(out.query_blocks) * top_k);
  if (!out.indices.empty()) {
    DevBuf<real> q(q_level.data(), q_level.size()), k(k_level.data(), k_level.size());
    DevBuf<std::uint32_t> par(parent.indices.data(), parent.indices.size());
    DevBuf<std::uint32_t> o(out.indices.size());
    ck(llsa_select_level(q.get(), k.get(), par.get(), 1, parent.level, parent.query_blocks,
                         parent.k, k_level.rows(), static_cast<std::uint32_t>(q_level.cols()),
                         top_k, scale, block_size, o.get(), nullptr));
    finish();
    o.download(out.indices.data());
  }
  if (mul_accs) *mul_accs += std::uint64_t(q_level.rows()) * cands * q_level.cols();
  return out;
}

SelectionResult hierarchical_topk(const Pyramid& pyr_q, const Pyramid& pyr_k,
                                  const ValidatedConfig& cfg) {
  const std::uint32_t levels = cfg.levels();
  if (pyr_q.depth() < levels || pyr_k.depth() < levels)
    throw ShapeMismatch("pyramids are shallower than the configured levels");
  for (std::uint32_t l = 0; l <= levels; ++l)
    if (pyr_q.level(l).rows() != cfg.level_tokens(l) ||
        pyr_k.level(l).rows() != cfg.level_tokens(l) || pyr_q.level(l).cols() != cfg.d() ||
        pyr_k.level(l).cols() != cfg.d())
      throw ShapeMismatch("pyramid level " + std::to_string(l) + " disagrees with the config");
  const llsa_config c = to_c(cfg.raw());
  const std::vector<real> hq = concat_levels(pyr_q, cfg), hk = concat_levels(pyr_k, cfg);
  DevBuf<real> dq(hq.data(), hq.size()), dk(hk.data(), hk.size());
  DevBuf<std::uint32_t> tables(llsa_table_entries(&c));
  ck(llsa_hierarchical_topk(&c, 1, dq.get(), dk.get(), tables.get(), nullptr));
  finish();
  std::vector<std::uint32_t> host(llsa_table_entries(&c));
  tables.download(host.data());
  SelectionResult sel;
  sel.coarsest_full = true;
  sel.mul_accs = llsa_select_mul_accs(&c);
  std::size_t off = 0;
  for (std::uint32_t l = 0; l < levels; ++l) {
    LevelIndices t;
    t.level = l;
    t.query_blocks = cfg.level_blocks(l);
    t.k = cfg.top_k();
    t.indices.assign(host.begin() + off, host.begin() + off + std::size_t(t.query_blocks) * t.k);
    off += t.indices.size();
    sel.per_level.push_back(std::move(t));
  }
  return sel;
}

void dump_selection(const SelectionResult& sel, std::ostream& out) {
  for (const LevelIndices& t : sel.per_level)
    for (std::uint32_t i = 0; i < t.query_blocks; ++i) {
      out << "level " << t.level << " / row " << i << ":";
      for (std::uint32_t idx : t.row(i)) out << ' ' << idx;
      out << '\n';
    }
}

// ---- CSR → CSC (P/src/indexmap.cpp:14-88) -----------------------------------
TransposedIndices transpose_indices(const LevelIndices& idx, std::uint32_t key_blocks) {
  for (std::uint32_t b : idx.indices)
    if (b >= key_blocks)
      throw IndexOutOfRange("selection entry >= key block count " + std::to_string(key_blocks));
  TransposedIndices out;
  out.key_blocks = key_blocks;
  out.offsets.assign(std::size_t(key_blocks) + 1, 0u);
  out.flat_queries.resize(idx.indices.size());
  const std::uint32_t rows = idx.k ? static_cast<std::uint32_t>(idx.indices.size() / idx.k) : 0;
  const std::size_t wsb = llsa_transpose_workspace_bytes(1, rows, idx.k, key_blocks);
  DevBuf<char> ws(wsb);
  DevBuf<std::uint32_t> din(idx.indices.data(), idx.indices.size());
  DevBuf<std::uint32_t> doffs(out.offsets.size()), dflat(out.flat_queries.size());
  ck(llsa_transpose_indices(din.get(), 1, rows, idx.k, key_blocks, doffs.get(), dflat.get(),
                            ws.get(), wsb, nullptr));
  finish();
  doffs.download(out.offsets.data());
  dflat.download(out.flat_queries.data());
  return out;
}

std::vector<TransposedIndices> transpose_all(const SelectionResult& sel,
                                             const ValidatedConfig& cfg) {
  if (sel.per_level.size() != cfg.levels())
    throw ShapeMismatch("selection has " + std::to_string(sel.per_level.size()) +
                        " levels, config expects " + std::to_string(cfg.levels()));
  std::vector<TransposedIndices> out;
  out.reserve(cfg.levels());
  for (std::uint32_t l = 0; l < cfg.levels(); ++l)
    out.push_back(transpose_indices(sel.per_level[l], cfg.level_blocks(l)));
  return out;
}

// ---- plan + forward (P/src/attention.cpp:80-219) ----------------------------
EnrichedKVPlan build_plan(const SelectionResult& sel, const ValidatedConfig& cfg) {
  if (sel.per_level.size() != cfg.levels())
    throw ShapeMismatch("selection depth disagrees with the config");
  const std::uint32_t lim = std::min(cfg.enrich_levels() + 1, cfg.levels());
  for (std::uint32_t l = 0; l < lim; ++l) {
    const LevelIndices& t = sel.per_level[l];
    if (t.level != l || t.k != cfg.top_k() || t.query_blocks != cfg.n() / cfg.pow_block(l + 1))
      throw ShapeMismatch("selection table at level " + std::to_string(l) +
                          " disagrees with the config");
  }
  const llsa_config c = to_c(cfg.raw());
  EnrichedKVPlan plan;
  plan.fine_blocks = cfg.fine_blocks();
  plan.entries_per_block = effective_block_count(cfg);
  const std::size_t total = std::size_t(plan.fine_blocks) * plan.entries_per_block;
  const std::vector<std::uint32_t> tables = concat_tables(sel, cfg);
  DevBuf<std::uint32_t> dt(tables.data(), tables.size());
  DevBuf<std::uint32_t> lv(total), bl(total);
  DevBuf<real> w(total);
  ck(llsa_build_plan(&c, 1, dt.get(), lv.get(), bl.get(), w.get(), nullptr));
  finish();
  std::vector<std::uint32_t> hl(total), hb(total);
  std::vector<real> hw(total);
  lv.download(hl.data());
  bl.download(hb.data());
  w.download(hw.data());
  plan.entries.resize(total);
  for (std::size_t i = 0; i < total; ++i) plan.entries[i] = PlanEntry{hl[i], hb[i], hw[i]};
  return plan;
}

std::uint64_t input_checksum(const FeatureMatrix& q, const FeatureMatrix& k,
                             const FeatureMatrix& v, const EnrichedKVPlan& plan,
                             const ValidatedConfig& cfg) {
  std::uint64_t h = 0xcbf29ce484222325ULL;
  fnv(h, cfg.n());
  fnv(h, cfg.d());
  fnv(h, cfg.block_size());
  fnv(h, cfg.top_k());
  fnv(h, cfg.levels());
  fnv(h, cfg.enrich_levels());
  fnv(h, static_cast<std::uint64_t>(cfg.mode()));
  fnv(h, cfg.safe_softmax() ? 1 : 0);
  fnv(h, std::bit_cast<std::uint64_t>(static_cast<double>(cfg.scale())));
  fnv(h, plan.fine_blocks);
  fnv(h, plan.entries_per_block);
  fnv_matrix(h, q);
  fnv_matrix(h, k);
  fnv_matrix(h, v);
  return h;
}

namespace {

// check_forward_shapes, P/src/attention.cpp:38-77
void check_forward(const FeatureMatrix& q, const FeatureMatrix& k, const FeatureMatrix& v,
                   const Pyramid& pyr_k, const Pyramid& pyr_v, const EnrichedKVPlan& plan,
                   const ValidatedConfig& cfg) {
  const std::size_t n = cfg.n(), d = cfg.d();
  if (q.rows() != n || q.cols() != d || k.rows() != n || k.cols() != d || v.rows() != n ||
      v.cols() != d)
    throw ShapeMismatch("q/k/v must be n x d for the validated config");
  if (plan.fine_blocks != cfg.fine_blocks())
    throw ShapeMismatch("plan covers " + std::to_string(plan.fine_blocks) +
                        " fine blocks, config has " + std::to_string(cfg.fine_blocks()));
  const std::uint32_t need = deepest_level(plan);
  if (pyr_k.levels.empty() || pyr_v.levels.empty() || pyr_k.depth() < need ||
      pyr_v.depth() < need)
    throw ShapeMismatch("pyramids are shallower than the plan's levels");
  for (std::uint32_t l = 0; l <= need; ++l) {
    const std::size_t rows = pyr_k.level(l).rows();
    if (rows != pyr_v.level(l).rows() || pyr_k.level(l).cols() != d ||
        pyr_v.level(l).cols() != d || rows % cfg.block_size() != 0)
      throw ShapeMismatch("pyramid level " + std::to_string(l) + " has inconsistent shape");
  }
  for (const PlanEntry& e : plan.entries)
    if (std::size_t(e.block + 1) * cfg.block_size() > pyr_k.level(e.level).rows())
      throw IndexOutOfRange("plan names key block " + std::to_string(e.block) +
                            " beyond level " + std::to_string(e.level));
}

struct DevPlan {
  DevBuf<std::uint32_t> level, block;
  DevBuf<real> weight;
  explicit DevPlan(const EnrichedKVPlan& p)
      : level(p.entries.size()), block(p.entries.size()), weight(p.entries.size()) {
    std::vector<std::uint32_t> l(p.entries.size()), b(p.entries.size());
    std::vector<real> w(p.entries.size());
    for (std::size_t i = 0; i < p.entries.size(); ++i) {
      l[i] = p.entries[i].level;
      b[i] = p.entries[i].block;
      w[i] = p.entries[i].weight;
    }
    level.upload(l.data());
    block.upload(b.data());
    weight.upload(w.data());
  }
};

}  // namespace

ForwardState llsa_forward(const FeatureMatrix& q, const FeatureMatrix& k, const FeatureMatrix& v,
                          const Pyramid& pyr_k, const Pyramid& pyr_v, const EnrichedKVPlan& plan,
                          const ValidatedConfig& cfg) {
  check_forward(q, k, v, pyr_k, pyr_v, plan, cfg);
  const std::size_t n = cfg.n(), d = cfg.d();
  const llsa_config c = to_c(cfg.raw());
  ForwardState st;
  st.output = FeatureMatrix(n, d);
  st.row_max.assign(n, real(0));
  st.row_denom.assign(n, real(0));
  st.input_checksum = input_checksum(q, k, v, plan, cfg);
  st.mul_accs = std::uint64_t(n) * plan.entries_per_block * cfg.block_size() * d;
  const std::vector<real> hk = concat_levels(pyr_k, cfg), hv = concat_levels(pyr_v, cfg);
  DevBuf<real> dq(q.data(), q.size()), dk(k.data(), k.size()), dv(v.data(), v.size());
  DevBuf<real> pk(hk.data(), hk.size()), pv(hv.data(), hv.size());
  DevPlan dp(plan);
  DevBuf<real> out(n * d), rm(n), rd(n);
  ck(llsa_forward_plan(&c, 1, LLSA_F32, dq.get(), dk.get(), dv.get(), pk.get(), pv.get(),
                       dp.level.get(), dp.block.get(), dp.weight.get(), plan.entries_per_block,
                       out.get(), rm.get(), rd.get(), nullptr));
  finish();  // NonFiniteError, attention.cpp:215-217
  out.download(st.output.data());
  rm.download(st.row_max.data());
  rd.download(st.row_denom.data());
  return st;
}

// ---- backward (P/src/attention_grad.cpp:90-265) -----------------------------
void kv_backward(const FeatureMatrix& d_out, const ForwardState& saved, const FeatureMatrix& q,
                 const Pyramid& pyr_k, const Pyramid& pyr_v,
                 const std::vector<TransposedIndices>& transposed, const ValidatedConfig& cfg,
                 FeatureMatrix& dk, FeatureMatrix& dv, std::uint64_t* mul_accs) {
  check_saved(d_out, saved, cfg);
  if (q.rows() != cfg.n() || q.cols() != cfg.d()) throw ShapeMismatch("q must be n x d");
  if (transposed.size() != cfg.levels())
    throw ShapeMismatch("expected one transposed table per level");
  const std::uint32_t lim = std::min(cfg.enrich_levels() + 1, cfg.levels());
  for (std::uint32_t l = 0; l < lim; ++l)
    if (transposed[l].key_blocks != cfg.level_blocks(l))
      throw ShapeMismatch("transposed table at level " + std::to_string(l) +
                          " disagrees with the config");
  const std::size_t n = cfg.n(), d = cfg.d();
  const llsa_config c = to_c(cfg.raw());
  dk = FeatureMatrix(n, d);
  dv = FeatureMatrix(n, d);
  std::vector<std::uint32_t> ho, hf;
  concat_csc(transposed, cfg, ho, hf);
  const std::vector<real> hk = concat_levels(pyr_k, cfg), hv = concat_levels(pyr_v, cfg);
  DevBuf<real> g(d_out.data(), d_out.size()), o(saved.output.data(), saved.output.size());
  DevBuf<real> rm(saved.row_max.data(), n), rd(saved.row_denom.data(), n);
  DevBuf<real> dq_(q.data(), q.size());
  DevBuf<real> k0(pyr_k.level(0).data(), pyr_k.level(0).size());
  DevBuf<real> v0(pyr_v.level(0).data(), pyr_v.level(0).size());
  DevBuf<real> pk(hk.data(), hk.size()), pv(hv.data(), hv.size());
  DevBuf<std::uint32_t> offs(ho.data(), ho.size()), flat(hf.data(), hf.size());
  DevBuf<real> ok(n * d), ov(n * d);
  const std::size_t wsb = llsa_backward_workspace_bytes(&c, 1);
  DevBuf<char> ws(wsb);
  ck(llsa_kv_backward(&c, 1, LLSA_F32, g.get(), o.get(), rm.get(), rd.get(), dq_.get(), pk.get(),
                      pv.get(), k0.get(), v0.get(), offs.get(), flat.get(), ok.get(), ov.get(),
                      ws.get(), wsb, nullptr));
  finish();
  ok.download(dk.data());
  ov.download(dv.data());
  if (mul_accs) *mul_accs += kv_macs(transposed, cfg);
}

GradientSet llsa_backward(const FeatureMatrix& d_out, const ForwardState& saved,
                          const FeatureMatrix& q, const FeatureMatrix& k, const FeatureMatrix& v,
                          const Pyramid& pyr_k, const Pyramid& pyr_v, const EnrichedKVPlan& plan,
                          const std::vector<TransposedIndices>& transposed,
                          const ValidatedConfig& cfg, std::uint64_t* mul_accs) {
  check_saved(d_out, saved, cfg);
  if (saved.input_checksum != input_checksum(q, k, v, plan, cfg))
    throw StaleState("saved forward state was computed from different inputs");
  if (q.rows() != cfg.n() || q.cols() != cfg.d()) throw ShapeMismatch("q must be n x d");
  if (transposed.size() != cfg.levels())
    throw ShapeMismatch("expected one transposed table per level");
  const std::uint32_t lim = std::min(cfg.enrich_levels() + 1, cfg.levels());
  for (std::uint32_t l = 0; l < lim; ++l)
    if (transposed[l].key_blocks != cfg.level_blocks(l))
      throw ShapeMismatch("transposed table at level " + std::to_string(l) +
                          " disagrees with the config");
  const std::size_t n = cfg.n(), d = cfg.d();
  const llsa_config c = to_c(cfg.raw());
  GradientSet gs;
  gs.dq = FeatureMatrix(n, d);
  gs.dk = FeatureMatrix(n, d);
  gs.dv = FeatureMatrix(n, d);
  std::vector<std::uint32_t> ho, hf;
  concat_csc(transposed, cfg, ho, hf);
  const std::vector<real> hk = concat_levels(pyr_k, cfg), hv = concat_levels(pyr_v, cfg);
  DevBuf<real> g(d_out.data(), d_out.size()), o(saved.output.data(), saved.output.size());
  DevBuf<real> rm(saved.row_max.data(), n), rd(saved.row_denom.data(), n);
  DevBuf<real> dq_(q.data(), q.size()), dk_(k.data(), k.size()), dv_(v.data(), v.size());
  DevBuf<real> pk(hk.data(), hk.size()), pv(hv.data(), hv.size());
  DevBuf<std::uint32_t> offs(ho.data(), ho.size()), flat(hf.data(), hf.size());
  DevPlan dp(plan);
  DevBuf<real> oq(n * d), ok(n * d), ov(n * d);
  const std::size_t wsb = llsa_backward_workspace_bytes(&c, 1);
  DevBuf<char> ws(wsb);
  ck(llsa_backward_plan(&c, 1, LLSA_F32, g.get(), o.get(), rm.get(), rd.get(), dq_.get(),
                        dk_.get(), dv_.get(), pk.get(), pv.get(), dp.level.get(),
                        dp.block.get(), dp.weight.get(), plan.entries_per_block, offs.get(),
                        flat.get(), oq.get(), ok.get(), ov.get(), ws.get(), wsb, nullptr));
  finish();
  oq.download(gs.dq.data());
  ok.download(gs.dk.data());
  ov.download(gs.dv.data());
  if (mul_accs)
    *mul_accs += std::uint64_t(n) * plan.entries_per_block * cfg.block_size() * 3 * d +
                 2 * n * d + kv_macs(transposed, cfg);
  return gs;
}

}  // namespace llsa
