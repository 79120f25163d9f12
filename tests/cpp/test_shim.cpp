// C++ parity tests of the drop-in library (libllsa.so, include/llsa/*.hpp):
// the reference's operator API called exactly as the reference's own unit
// tests call it (P/tests/test_*.cpp), with known answers transcribed from
// them and independent dense references written here.  Runs on the GPU.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "llsa/attention.hpp"
#include "llsa/attention_grad.hpp"
#include "llsa/config.hpp"
#include "llsa/errors.hpp"
#include "llsa/indexmap.hpp"
#include "llsa/pyramid.hpp"
#include "llsa/selection.hpp"
#include "llsa/tensorio.hpp"

using namespace llsa;

namespace {

LLSAConfig cfg_of(std::uint64_t n, std::uint32_t d, std::uint32_t b, std::uint32_t k,
                  std::uint32_t levels, std::uint32_t enrich,
                  ReweightMode mode = ReweightMode::ScaleKV) {
  LLSAConfig c;
  c.n = n;
  c.d = d;
  c.block_size = b;
  c.top_k = k;
  c.levels = levels;
  c.enrich_levels = enrich;
  c.reweight_mode = mode;
  return c;
}

FeatureMatrix column(std::vector<real> v) {
  const std::size_t n = v.size();
  return FeatureMatrix::from_values(n, 1, std::move(v));
}

struct Case {
  FeatureMatrix q, k, v, g;
  Pyramid pk, pv;
  SelectionResult sel;
  EnrichedKVPlan plan;
  std::vector<TransposedIndices> tr;
};

Case make_case(const ValidatedConfig& cfg, std::uint64_t seed) {
  Case c;
  c.q = gen_random(cfg.n(), cfg.d(), seed);
  c.k = gen_random(cfg.n(), cfg.d(), seed + 1);
  c.v = gen_random(cfg.n(), cfg.d(), seed + 2);
  c.g = gen_random(cfg.n(), cfg.d(), seed + 3);
  const Pyramid pq = build_pyramid(c.q, cfg.block_size(), cfg.levels());
  c.pk = build_pyramid(c.k, cfg.block_size(), cfg.levels());
  c.pv = build_pyramid(c.v, cfg.block_size(), cfg.levels());
  c.sel = hierarchical_topk(pq, c.pk, cfg);
  c.plan = build_plan(c.sel, cfg);
  c.tr = transpose_all(c.sel, cfg);
  return c;
}

// Plain dense softmax attention and its gradient in double (independent of
// the library).
void dense(const FeatureMatrix& q, const FeatureMatrix& k, const FeatureMatrix& v,
           const FeatureMatrix& g, double scale, std::vector<double>& o,
           std::vector<double>& dq, std::vector<double>& dk, std::vector<double>& dv) {
  const std::size_t n = q.rows(), d = q.cols();
  o.assign(n * d, 0);
  dq.assign(n * d, 0);
  dk.assign(n * d, 0);
  dv.assign(n * d, 0);
  std::vector<double> p(n), dp(n);
  for (std::size_t t = 0; t < n; ++t) {
    double mx = -1e300;
    for (std::size_t j = 0; j < n; ++j) {
      double s = 0;
      for (std::size_t c = 0; c < d; ++c) s += double(q.at(t, c)) * k.at(j, c);
      p[j] = scale * s;
      mx = std::max(mx, p[j]);
    }
    double den = 0;
    for (std::size_t j = 0; j < n; ++j) den += (p[j] = std::exp(p[j] - mx));
    double rs = 0;
    for (std::size_t j = 0; j < n; ++j) {
      p[j] /= den;
      dp[j] = 0;
      for (std::size_t c = 0; c < d; ++c) {
        o[t * d + c] += p[j] * v.at(j, c);
        dp[j] += double(g.at(t, c)) * v.at(j, c);
      }
      rs += p[j] * dp[j];
    }
    for (std::size_t j = 0; j < n; ++j) {
      const double ds = p[j] * (dp[j] - rs);
      for (std::size_t c = 0; c < d; ++c) {
        dq[t * d + c] += scale * ds * k.at(j, c);
        dk[j * d + c] += scale * ds * q.at(t, c);
        dv[j * d + c] += p[j] * g.at(t, c);
      }
    }
  }
}

double max_rel(const FeatureMatrix& a, const std::vector<double>& ref) {
  double mx = 0, md = 0;
  for (std::size_t i = 0; i < ref.size(); ++i) {
    mx = std::max(mx, std::fabs(ref[i]));
    md = std::max(md, std::fabs(double(a.data()[i]) - ref[i]));
  }
  return md / (mx > 0 ? mx : 1);
}

}  // namespace

TEST_CASE("max_levels and validation match the reference's known answers") {
  CHECK(max_levels(65536, 16) == 3);
  CHECK(max_levels(65535, 16) == 2);
  CHECK(max_levels(16384, 16) == 2);
  CHECK(max_levels(8, 4) == 0);
  CHECK_THROWS_AS(validate_config(cfg_of(0, 4, 4, 1, 1, 0)), ConfigError);
  CHECK_THROWS_AS(validate_config(cfg_of(64, 4, 4, 1, 3, 0)), LevelError);
  CHECK_THROWS_AS(validate_config(cfg_of(100, 4, 3, 1, 2, 0)), DivisibilityError);
  CHECK_THROWS_AS(validate_config(cfg_of(4096, 4, 16, 17, 2, 0)), TopKError);
  CHECK(effective_block_count(validate_config(cfg_of(16384, 64, 16, 8, 2, 2))) == 20);
  CHECK(effective_block_count(validate_config(cfg_of(16384, 64, 16, 8, 2, 0))) == 8);
  CHECK(validate_config(cfg_of(64, 16, 4, 2, 1, 0)).scale() == doctest::Approx(0.25));
  CHECK(std::string(to_string(ReweightMode::LogitBias)) == "logitbias");
}

TEST_CASE("pooling known answers and adjoint") {
  const Pyramid p = build_pyramid(column({1, 3, 5, 7}), 2, 1);
  REQUIRE(p.depth() == 1);
  CHECK(p.level(1).at(0, 0) == real(2));
  CHECK(p.level(1).at(1, 0) == real(6));
  std::vector<real> ramp(16);
  std::iota(ramp.begin(), ramp.end(), real(0));
  const Pyramid p2 = build_pyramid(column(ramp), 2, 2);
  CHECK(p2.level(2).at(0, 0) == real(1.5));
  CHECK(p2.level(2).at(3, 0) == real(13.5));
  CHECK_THROWS_AS(build_pyramid(column({1, 2, 3, 4, 5, 6}), 2, 2), DivisibilityError);
  const FeatureMatrix one = pool_backward(column({6}), 2, 1);
  CHECK(one.rows() == 2);
  CHECK(one.at(1, 0) == real(3));
  const FeatureMatrix x = gen_random(64, 4, 11);
  const Pyramid px = build_pyramid(x, 4, 2);
  const FeatureMatrix y = gen_random(4, 4, 102);
  const FeatureMatrix yt = pool_backward(y, 4, 2);
  double lhs = 0, rhs = 0;
  for (std::size_t i = 0; i < y.size(); ++i) lhs += double(px.level(2).data()[i]) * y.data()[i];
  for (std::size_t i = 0; i < x.size(); ++i) rhs += double(x.data()[i]) * yt.data()[i];
  CHECK(std::fabs(lhs - rhs) <= 1e-5 * (1 + std::fabs(lhs)));
}

TEST_CASE("selection: ties, keep-all, refinement and argument errors") {
  FeatureMatrix k(10, 3);
  for (std::size_t r = 0; r < 10; ++r)
    for (std::size_t c = 0; c < 3; ++c) k.at(r, c) = real(c + 1);
  const LevelIndices ties = select_coarsest(gen_random(4, 3, 77), k, 4, real(1), 0);
  for (std::uint32_t i = 0; i < 4; ++i)
    for (std::uint32_t j = 0; j < 4; ++j) CHECK(ties.row(i)[j] == j);
  const LevelIndices all = select_coarsest(gen_random(6, 4, 1), gen_random(8, 4, 2), 8, 1, 0);
  for (std::uint32_t i = 0; i < 6; ++i)
    for (std::uint32_t j = 0; j < 8; ++j) CHECK(all.row(i)[j] == j);
  LevelIndices parent;
  parent.level = 1;
  parent.query_blocks = 4;
  parent.k = 2;
  parent.indices = {0, 2, 1, 3, 0, 1, 2, 3};
  const FeatureMatrix q = gen_random(16, 4, 5), kk = gen_random(16, 4, 6);
  const LevelIndices out = select_level(q, kk, parent, 3, real(0.7), 4);
  for (std::uint32_t t = 0; t < 16; ++t)
    for (std::uint32_t idx : out.row(t)) {
      const auto pr = parent.row(t / 4);
      CHECK(std::find(pr.begin(), pr.end(), idx / 4) != pr.end());
    }
  LevelIndices bad = parent;
  bad.indices[3] = 4;
  CHECK_THROWS_AS(select_level(q, kk, bad, 2, 1, 4), IndexOutOfRange);
  LevelIndices fine = parent;
  fine.level = 0;
  CHECK_THROWS_AS(select_level(q, kk, fine, 2, 1, 4), LevelError);
  CHECK_THROWS_AS(select_level(q, kk, parent, 9, 1, 4), TopKError);
  CHECK_THROWS_AS(select_coarsest(q, gen_random(16, 5, 1), 2, 1, 0), ShapeMismatch);
}

TEST_CASE("transposition known answers") {
  LevelIndices t;
  t.query_blocks = 4;
  t.k = 1;
  t.indices = {1, 0, 1, 3};
  const TransposedIndices out = transpose_indices(t, 4);
  CHECK(out.offsets == std::vector<std::uint32_t>{0, 1, 3, 3, 4});
  CHECK(out.flat_queries == std::vector<std::uint32_t>{1, 0, 2, 3});
  t.indices = {0, 5, 1, 1};
  CHECK_THROWS_AS(transpose_indices(t, 4), IndexOutOfRange);
}

TEST_CASE("plan composition, dump format and the input checksum") {
  const ValidatedConfig cfg = validate_config(cfg_of(16384, 4, 16, 8, 2, 2));
  const Case c = make_case(cfg, 11);
  CHECK(c.plan.entries_per_block == 20);
  for (std::uint32_t i : {0u, 17u, 1023u}) {
    const auto e = c.plan.block(i);
    CHECK(e[0].block == c.sel.per_level[0].row(i)[0]);
    CHECK(e[8].level == 1);
    CHECK(e[8].block == c.sel.per_level[1].row(i / 16)[0]);
    CHECK(e[8].weight == real(16));
    CHECK(e[19].level == 2);
    CHECK(e[19].block == 3);
  }
  SelectionResult s;
  LevelIndices t0;
  t0.query_blocks = 2;
  t0.k = 2;
  t0.indices = {0, 3, 1, 2};
  s.per_level = {t0};
  std::ostringstream os;
  dump_selection(s, os);
  CHECK(os.str() == "level 0 / row 0: 0 3\nlevel 0 / row 1: 1 2\n");
  FeatureMatrix v2 = c.v;
  v2.at(3, 1) += real(1e-3);
  CHECK(input_checksum(c.q, c.k, c.v, c.plan, cfg) != input_checksum(c.q, c.k, v2, c.plan, cfg));
}

TEST_CASE("keeping every block reproduces dense attention and its gradient") {
  const ValidatedConfig cfg = validate_config(cfg_of(64, 8, 4, 16, 1, 0));
  const Case c = make_case(cfg, 19);
  const ForwardState st = llsa_forward(c.q, c.k, c.v, c.pk, c.pv, c.plan, cfg);
  const GradientSet gs =
      llsa_backward(c.g, st, c.q, c.k, c.v, c.pk, c.pv, c.plan, c.tr, cfg);
  std::vector<double> o, dq, dk, dv;
  dense(c.q, c.k, c.v, c.g, cfg.scale(), o, dq, dk, dv);
  CHECK(max_rel(st.output, o) <= 1e-5);
  CHECK(max_rel(gs.dq, dq) <= 1e-4);
  CHECK(max_rel(gs.dk, dk) <= 1e-4);
  CHECK(max_rel(gs.dv, dv) <= 1e-4);
}

TEST_CASE("constant values collapse the output; overflow needs rescaling") {
  LLSAConfig raw = cfg_of(128, 8, 4, 2, 2, 2, ReweightMode::LogitBias);
  const ValidatedConfig cfg = validate_config(raw);
  Case c = make_case(cfg, 17);
  for (std::size_t i = 0; i < c.v.size(); ++i) c.v.data()[i] = real(0.7);
  c.pv = build_pyramid(c.v, 4, 2);
  const ForwardState st = llsa_forward(c.q, c.k, c.v, c.pk, c.pv, c.plan, cfg);
  for (std::size_t i = 0; i < st.output.size(); ++i)
    CHECK(std::fabs(st.output.data()[i] - real(0.7)) <= real(1e-5));

  LLSAConfig r2 = cfg_of(16, 8, 4, 2, 1, 0);
  r2.safe_softmax = false;
  const ValidatedConfig plain = validate_config(r2);
  r2.safe_softmax = true;
  const ValidatedConfig safe = validate_config(r2);
  FeatureMatrix q(16, 8), k(16, 8);
  for (std::size_t i = 0; i < q.size(); ++i) q.data()[i] = real(300);
  for (std::size_t i = 0; i < k.size(); ++i) k.data()[i] = real(1);
  const FeatureMatrix v = gen_random(16, 8, 31);
  const Pyramid pq = build_pyramid(q, 4, 1), pk = build_pyramid(k, 4, 1),
                pv = build_pyramid(v, 4, 1);
  const EnrichedKVPlan plan = build_plan(hierarchical_topk(pq, pk, plain), plain);
  CHECK_THROWS_AS(llsa_forward(q, k, v, pk, pv, plan, plain), NonFiniteError);
  const ForwardState ok = llsa_forward(q, k, v, pk, pv, plan, safe);
  for (std::size_t i = 0; i < ok.output.size(); ++i) CHECK(std::isfinite(ok.output.data()[i]));
}

TEST_CASE("forward and backward validate inputs; stale state is rejected") {
  const ValidatedConfig cfg = validate_config(cfg_of(64, 4, 4, 2, 2, 2));
  Case c = make_case(cfg, 53);
  EnrichedKVPlan bad = c.plan;
  bad.entries[0].block = 999;
  CHECK_THROWS_AS(llsa_forward(c.q, c.k, c.v, c.pk, c.pv, bad, cfg), IndexOutOfRange);
  CHECK_THROWS_AS(llsa_forward(gen_random(32, 4, 54), c.k, c.v, c.pk, c.pv, c.plan, cfg),
                  ShapeMismatch);
  const ForwardState st = llsa_forward(c.q, c.k, c.v, c.pk, c.pv, c.plan, cfg);
  FeatureMatrix zero(cfg.n(), cfg.d());
  const GradientSet z = llsa_backward(zero, st, c.q, c.k, c.v, c.pk, c.pv, c.plan, c.tr, cfg);
  for (const FeatureMatrix* m : {&z.dq, &z.dk, &z.dv})
    for (std::size_t i = 0; i < m->size(); ++i) CHECK(m->data()[i] == real(0));
  FeatureMatrix q2 = c.q;
  q2.at(5, 2) += real(0.25);
  CHECK_THROWS_AS(llsa_backward(c.g, st, q2, c.k, c.v, c.pk, c.pv, c.plan, c.tr, cfg),
                  StaleState);
  std::vector<TransposedIndices> few(c.tr.begin(), c.tr.end() - 1);
  FeatureMatrix dk, dv;
  CHECK_THROWS_AS(kv_backward(c.g, st, c.q, c.pk, c.pv, few, cfg, dk, dv), ShapeMismatch);
  CHECK_THROWS_AS(llsa_backward(gen_random(64, 3, 33), st, c.q, c.k, c.v, c.pk, c.pv, c.plan,
                                c.tr, cfg),
                  ShapeMismatch);
}

TEST_CASE("work counters are analytic") {
  const ValidatedConfig cfg = validate_config(cfg_of(256, 8, 4, 2, 2, 2));
  const Case c = make_case(cfg, 41);
  const ForwardState st = llsa_forward(c.q, c.k, c.v, c.pk, c.pv, c.plan, cfg);
  CHECK(st.mul_accs == std::uint64_t(256) * c.plan.entries_per_block * 4 * 8);
  std::uint64_t kv = 0;
  FeatureMatrix dk, dv;
  kv_backward(c.g, st, c.q, c.pk, c.pv, c.tr, cfg, dk, dv, &kv);
  std::uint64_t expect = 2 * 256 * 8;
  for (std::uint32_t l = 0; l < 2; ++l)
    expect += std::uint64_t(c.tr[l].flat_queries.size()) * cfg.pow_block(l + 1) * 4 * 4 * 8;
  expect += std::uint64_t(256) * cfg.level_tokens(2) * 4 * 8;
  CHECK(kv == expect);
}

TEST_CASE("FMAT round trip and deterministic streams") {
  const FeatureMatrix m = gen_random(3, 5, 9);
  const std::string path = "/tmp/llsa_shim_test.fmat";
  write_tensor(path, m);
  const FeatureMatrix r = read_tensor(path);
  CHECK(r.rows() == 3);
  CHECK(max_abs_diff(m, r) == real(0));
  CHECK(max_abs_diff(gen_random(4, 4, 123), gen_random(4, 4, 123)) == real(0));
  std::remove(path.c_str());
  CHECK_THROWS_AS(read_tensor("/nonexistent/x.fmat"), IoError);
}
