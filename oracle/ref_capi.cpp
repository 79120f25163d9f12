// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C wrapper around the UNMODIFIED reference library (/root/reference/proj),
// compiled by oracle/Makefile into oracle/_ref/libllsa_ref{32,64}.so.  It lets
// the Python tests and bench.py's reference arm drive the reference's own
// operator API (build_pyramid → hierarchical_topk → build_plan → llsa_forward
// → transpose_all → llsa_backward) on float buffers.  Only
// tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) may load the resulting library.
//
// Every entry point returns 0 or a status code equal to include/llsa_cuda.h's
// llsa_status for the reference exception type that was thrown.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "llsa/attention.hpp"
#include "llsa/attention_grad.hpp"
#include "llsa/config.hpp"
#include "llsa/errors.hpp"
#include "llsa/indexmap.hpp"
#include "llsa/oracle.hpp"
#include "llsa/parallel.hpp"
#include "llsa/pyramid.hpp"
#include "llsa/reorder2d.hpp"
#include "llsa/selection.hpp"
#include "llsa/tensorio.hpp"

using namespace llsa;

namespace {

thread_local std::string g_err;

// Same numbering as llsa_status in include/llsa_cuda.h.
int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const DivisibilityError*>(&e)) return 2;
  if (dynamic_cast<const LevelError*>(&e)) return 3;
  if (dynamic_cast<const TopKError*>(&e)) return 4;
  if (dynamic_cast<const ShapeMismatch*>(&e)) return 5;
  if (dynamic_cast<const IndexOutOfRange*>(&e)) return 6;
  if (dynamic_cast<const NonFiniteError*>(&e)) return 7;
  if (dynamic_cast<const StaleState*>(&e)) return 8;
  if (dynamic_cast<const FormatError*>(&e)) return 9;
  if (dynamic_cast<const IoError*>(&e)) return 10;
  if (dynamic_cast<const PrecisionError*>(&e)) return 11;
  if (dynamic_cast<const NotSquareBlock*>(&e)) return 12;
  if (dynamic_cast<const OracleCapExceeded*>(&e)) return 13;
  return 99;
}

FeatureMatrix to_fm(const float* p, std::size_t rows, std::size_t cols) {
  FeatureMatrix m(rows, cols);
  for (std::size_t i = 0; i < rows * cols; ++i) m.data()[i] = real(p[i]);
  return m;
}

void from_fm(const FeatureMatrix& m, float* out) {
  for (std::size_t i = 0; i < m.size(); ++i) out[i] = float(m.data()[i]);
}

struct RawCfg {
  std::uint64_t n;
  std::uint32_t d, block_size, top_k, levels, enrich_levels;
  float softmax_scale;
  std::uint32_t reweight_mode, safe_softmax;
};

LLSAConfig to_cfg(const RawCfg* c) {
  LLSAConfig cfg;
  cfg.n = c->n;
  cfg.d = c->d;
  cfg.block_size = c->block_size;
  cfg.top_k = c->top_k;
  cfg.levels = c->levels;
  cfg.enrich_levels = c->enrich_levels;
  cfg.softmax_scale = real(c->softmax_scale);
  cfg.reweight_mode = c->reweight_mode ? ReweightMode::LogitBias
                                       : ReweightMode::ScaleKV;
  cfg.safe_softmax = c->safe_softmax != 0;
  return cfg;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now() - t0)
      .count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_real_bytes() { return int(sizeof(real)); }
void ref_set_threads(unsigned t) { set_thread_count(t); }
unsigned ref_threads() { return thread_count(); }

// build_reorder (reorder2d.cpp:11-69): forward / inverse, height*width each.
int ref_build_reorder(std::uint32_t h, std::uint32_t w, std::uint32_t b, std::uint32_t* fwd,
                      std::uint32_t* inv) {
  try {
    const Permutation p = build_reorder(h, w, b);
    std::copy(p.forward.begin(), p.forward.end(), fwd);
    std::copy(p.inverse.begin(), p.inverse.end(), inv);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

std::uint32_t ref_max_levels(std::uint64_t n, std::uint32_t b) {
  return max_levels(n, b);
}

// Validates; on success writes the resolved scale and E.
int ref_validate(const RawCfg* c, float* scale, std::uint32_t* eff) {
  try {
    const ValidatedConfig v = validate_config(to_cfg(c));
    if (scale) *scale = float(v.scale());
    if (eff) *eff = effective_block_count(v);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

void ref_gen_random(float* out, std::size_t rows, std::size_t cols,
                    std::uint64_t seed, int uniform) {
  const FeatureMatrix m = gen_random(
      rows, cols, seed, uniform ? Distribution::Uniform01 : Distribution::StdNormal);
  from_fm(m, out);
}

// levels_out: concatenated levels 1..L, each (rows/B^l) x cols.
int ref_build_pyramid(const float* x, std::size_t rows, std::size_t cols,
                      std::uint32_t b, std::uint32_t levels, float* levels_out) {
  try {
    const Pyramid p = build_pyramid(to_fm(x, rows, cols), b, levels);
    float* o = levels_out;
    for (std::uint32_t l = 1; l <= levels; ++l) {
      from_fm(p.level(l), o);
      o += p.level(l).size();
    }
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_pool_backward(const float* g, std::size_t rows, std::size_t cols,
                      std::uint32_t b, std::uint32_t hops, float* out) {
  try {
    from_fm(pool_backward(to_fm(g, rows, cols), b, hops), out);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_select_coarsest(const float* q, std::size_t q_rows, const float* k,
                        std::size_t k_rows, std::size_t d, std::uint32_t top_k,
                        float scale, std::uint32_t* out, std::uint64_t* macs) {
  try {
    const LevelIndices t = select_coarsest(to_fm(q, q_rows, d), to_fm(k, k_rows, d),
                                           top_k, real(scale), 0, macs);
    std::copy(t.indices.begin(), t.indices.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_select_level(const float* q, std::size_t q_rows, const float* k,
                     std::size_t k_rows, std::size_t d, const std::uint32_t* parent,
                     std::uint32_t parent_level, std::uint32_t parent_rows,
                     std::uint32_t parent_k, std::uint32_t top_k, float scale,
                     std::uint32_t b, std::uint32_t* out, std::uint64_t* macs) {
  try {
    LevelIndices p;
    p.level = parent_level;
    p.query_blocks = parent_rows;
    p.k = parent_k;
    p.indices.assign(parent, parent + std::size_t(parent_rows) * parent_k);
    const LevelIndices t = select_level(to_fm(q, q_rows, d), to_fm(k, k_rows, d), p,
                                        top_k, real(scale), b, macs);
    std::copy(t.indices.begin(), t.indices.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_transpose(const std::uint32_t* idx, std::uint32_t rows, std::uint32_t k,
                  std::uint32_t key_blocks, std::uint32_t* offsets,
                  std::uint32_t* flat) {
  try {
    LevelIndices t;
    t.level = 0;
    t.query_blocks = rows;
    t.k = k;
    t.indices.assign(idx, idx + std::size_t(rows) * k);
    const TransposedIndices tr = transpose_indices(t, key_blocks);
    std::copy(tr.offsets.begin(), tr.offsets.end(), offsets);
    std::copy(tr.flat_queries.begin(), tr.flat_queries.end(), flat);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Whole per-unit path exactly as SURVEY.md §3(1).  Any output pointer may be
// null.  Layouts:
//   pyr_{q,k,v}: levels 1..L concatenated; tables: per_level 0..L-1
//   concatenated ([N/B^(l+1)][K] each); csc_offsets: per level (T_l+1)
//   concatenated; csc_flat: per level (T_l*K) concatenated; plan_{level,block}
//   and plan_weight: [N/B][E].
// stage_ms (8 doubles, optional): pyramids, select, plan, forward, transpose,
// backward, total, dense-unused.
int ref_run_pipeline(const RawCfg* c, const float* q, const float* k,
                     const float* v, const float* d_out, float* pyr_q,
                     float* pyr_k, float* pyr_v, std::uint32_t* tables,
                     std::uint32_t* plan_level, std::uint32_t* plan_block,
                     float* plan_weight, float* out, float* row_max,
                     float* row_denom, std::uint64_t* checksum,
                     std::uint32_t* csc_offsets, std::uint32_t* csc_flat,
                     float* dq, float* dk, float* dv, std::uint64_t* macs,
                     double* stage_ms) {
  try {
    using clk = std::chrono::steady_clock;
    const ValidatedConfig cfg = validate_config(to_cfg(c));
    const std::size_t n = cfg.n(), d = cfg.d();
    const FeatureMatrix fq = to_fm(q, n, d), fk = to_fm(k, n, d), fv = to_fm(v, n, d);
    double st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const auto t_all = clk::now();

    auto t0 = clk::now();
    const Pyramid pq = build_pyramid(fq, cfg.block_size(), cfg.levels());
    const Pyramid pk = build_pyramid(fk, cfg.block_size(), cfg.levels());
    const Pyramid pv = build_pyramid(fv, cfg.block_size(), cfg.levels());
    st[0] = ms_since(t0);

    t0 = clk::now();
    const SelectionResult sel = hierarchical_topk(pq, pk, cfg);
    st[1] = ms_since(t0);

    t0 = clk::now();
    const EnrichedKVPlan plan = build_plan(sel, cfg);
    st[2] = ms_since(t0);

    t0 = clk::now();
    const ForwardState fwd = llsa_forward(fq, fk, fv, pk, pv, plan, cfg);
    st[3] = ms_since(t0);

    std::uint64_t mac_total = sel.mul_accs + fwd.mul_accs;
    if (d_out) {
      t0 = clk::now();
      const std::vector<TransposedIndices> tr = transpose_all(sel, cfg);
      st[4] = ms_since(t0);
      t0 = clk::now();
      std::uint64_t bmacs = 0;
      const GradientSet g = llsa_backward(to_fm(d_out, n, d), fwd, fq, fk, fv, pk,
                                          pv, plan, tr, cfg, &bmacs);
      st[5] = ms_since(t0);
      mac_total += bmacs;
      if (dq) from_fm(g.dq, dq);
      if (dk) from_fm(g.dk, dk);
      if (dv) from_fm(g.dv, dv);
      if (csc_offsets && csc_flat) {
        std::uint32_t* po = csc_offsets;
        std::uint32_t* pf = csc_flat;
        for (const TransposedIndices& t : tr) {
          std::copy(t.offsets.begin(), t.offsets.end(), po);
          po += t.offsets.size();
          std::copy(t.flat_queries.begin(), t.flat_queries.end(), pf);
          pf += t.flat_queries.size();
        }
      }
    }
    st[6] = ms_since(t_all);

    auto dump_pyr = [&](const Pyramid& p, float* o) {
      if (!o) return;
      for (std::uint32_t l = 1; l <= cfg.levels(); ++l) {
        from_fm(p.level(l), o);
        o += p.level(l).size();
      }
    };
    dump_pyr(pq, pyr_q);
    dump_pyr(pk, pyr_k);
    dump_pyr(pv, pyr_v);
    if (tables) {
      std::uint32_t* o = tables;
      for (const LevelIndices& t : sel.per_level) {
        std::copy(t.indices.begin(), t.indices.end(), o);
        o += t.indices.size();
      }
    }
    for (std::size_t i = 0; i < plan.entries.size(); ++i) {
      if (plan_level) plan_level[i] = plan.entries[i].level;
      if (plan_block) plan_block[i] = plan.entries[i].block;
      if (plan_weight) plan_weight[i] = float(plan.entries[i].weight);
    }
    if (out) from_fm(fwd.output, out);
    for (std::size_t t = 0; t < n; ++t) {
      if (row_max) row_max[t] = float(fwd.row_max[t]);
      if (row_denom) row_denom[t] = float(fwd.row_denom[t]);
    }
    if (checksum) *checksum = fwd.input_checksum;
    if (macs) *macs = mac_total;
    if (stage_ms) std::copy(st, st + 8, stage_ms);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// Independent slow references from the reference's own oracle module
// (capped at 2048 rows there): effective_attention and mask_backward.
int ref_oracle_effective(const RawCfg* c, const float* q, const float* k,
                         const float* v, float* out) {
  try {
    const ValidatedConfig cfg = validate_config(to_cfg(c));
    const std::size_t n = cfg.n(), d = cfg.d();
    const FeatureMatrix fq = to_fm(q, n, d), fk = to_fm(k, n, d), fv = to_fm(v, n, d);
    const Pyramid pq = build_pyramid(fq, cfg.block_size(), cfg.levels());
    const Pyramid pk = build_pyramid(fk, cfg.block_size(), cfg.levels());
    const Pyramid pv = build_pyramid(fv, cfg.block_size(), cfg.levels());
    const SelectionResult sel = hierarchical_topk(pq, pk, cfg);
    const EnrichedKVPlan plan = build_plan(sel, cfg);
    from_fm(oracle::effective_attention(fq, fk, fv, pk, pv, plan, cfg), out);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_oracle_dense(const float* q, const float* k, const float* v,
                     std::size_t n, std::size_t d, float scale, float* out) {
  try {
    from_fm(oracle::dense_attention(to_fm(q, n, d), to_fm(k, n, d), to_fm(v, n, d),
                                    real(scale)),
            out);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

}  // extern "C"
