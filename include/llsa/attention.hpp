// Enriched plan + streaming attention forward (B200 build of
// P/include/llsa/attention.hpp).  GPU kernels: attn_simt.cu (any shape) and
// attn_tc.cu (d = 64, B = 16, bf16 — reached through llsa_handle_*).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "llsa/config.hpp"
#include "llsa/pyramid.hpp"
#include "llsa/selection.hpp"
#include "llsa/types.hpp"

namespace llsa {

struct PlanEntry {
  std::uint32_t level = 0;
  std::uint32_t block = 0;
  real weight = real(1);
};

struct EnrichedKVPlan {
  std::uint32_t fine_blocks = 0;
  std::uint32_t entries_per_block = 0;
  std::vector<PlanEntry> entries;  // fine_blocks × entries_per_block

  std::span<const PlanEntry> block(std::uint32_t i) const {
    return {entries.data() + static_cast<std::size_t>(i) * entries_per_block,
            entries_per_block};
  }
};

EnrichedKVPlan build_plan(const SelectionResult& sel, const ValidatedConfig& cfg);

struct ForwardState {
  FeatureMatrix output;
  std::vector<real> row_max;
  std::vector<real> row_denom;
  std::uint64_t mul_accs = 0;
  std::uint64_t input_checksum = 0;
};

// FNV-1a over config, plan shape and the raw bits of q, k, v — bit-compatible
// with the reference's f32 build (P/src/attention.cpp:18-34,124-143).
std::uint64_t input_checksum(const FeatureMatrix& q, const FeatureMatrix& k,
                             const FeatureMatrix& v, const EnrichedKVPlan& plan,
                             const ValidatedConfig& cfg);

ForwardState llsa_forward(const FeatureMatrix& q, const FeatureMatrix& k,
                          const FeatureMatrix& v, const Pyramid& pyr_k, const Pyramid& pyr_v,
                          const EnrichedKVPlan& plan, const ValidatedConfig& cfg);

}  // namespace llsa
