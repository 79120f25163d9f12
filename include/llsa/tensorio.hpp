// FMAT tensor files and the deterministic generator (B200 build of
// P/include/llsa/tensorio.hpp; same byte format and streams).
//   offset 0 "FMAT" | 4 u32 version (1) | 8 u32 dtype (0 f32, 1 f64)
//   | 12 u64 rows | 20 u64 cols | 28 payload, row-major, little-endian
#pragma once

#include <cstdint>
#include <string>

#include "llsa/types.hpp"

namespace llsa {

inline constexpr std::uint32_t kTensorVersion = 1;
inline constexpr std::uint32_t kDtypeF32 = 0;
inline constexpr std::uint32_t kDtypeF64 = 1;
inline constexpr std::size_t kTensorHeaderBytes = 28;

void write_tensor(const std::string& path, const FeatureMatrix& m);
FeatureMatrix read_tensor(const std::string& path);

enum class Distribution { StdNormal, Uniform01 };

// splitmix64-seeded xoshiro256++; Box-Muller for StdNormal.
FeatureMatrix gen_random(std::size_t rows, std::size_t cols, std::uint64_t seed,
                         Distribution dist = Distribution::StdNormal);

}  // namespace llsa
