// Worker-count knob kept for source compatibility with the reference
// (P/include/llsa/parallel.hpp).  The B200 build runs every operator on the
// GPU, so the count only affects the host-side helpers (none are parallel);
// results never depend on it.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>

namespace llsa {

void set_thread_count(unsigned count);
unsigned thread_count();

// Serial host loop with the reference's contract (body(begin, end) over a
// partition of [0, n)); provided for callers that use it directly.
void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& body);
std::uint64_t parallel_sum(std::size_t n,
                           const std::function<std::uint64_t(std::size_t, std::size_t)>& body);

}  // namespace llsa
