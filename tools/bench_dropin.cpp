// End to end through the C++ drop-in (include/llsa/*.hpp → libllsa.so), the
// way a reference caller uses the reference library: host FeatureMatrix in,
// host results out, every call copying its operands to the GPU and back
// (real = float: the reference's LLSA_SINGLE_PRECISION semantics, general
// fp32 kernels).  One step = the reference bench's path per unit
// (bench.cpp run_scaling: pyramids, hierarchical_topk, build_plan,
// llsa_forward, transpose_all, llsa_backward) for every unit of the C3
// workload.  Prints one JSON line.
//   build: tools/bench_dropin.sh;  run: tools/bench_dropin [units] [steps]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "llsa/attention.hpp"
#include "llsa/attention_grad.hpp"
#include "llsa/config.hpp"
#include "llsa/indexmap.hpp"
#include "llsa/pyramid.hpp"
#include "llsa/selection.hpp"
#include "llsa/tensorio.hpp"

using namespace llsa;
using Clock = std::chrono::steady_clock;

int main(int argc, char** argv) {
  const unsigned units = argc > 1 ? (unsigned)atoi(argv[1]) : 16;
  const int steps = argc > 2 ? atoi(argv[2]) : 2;
  LLSAConfig c;
  c.n = 65536;
  c.d = 64;
  c.block_size = 16;
  c.top_k = 8;
  c.levels = 3;
  c.enrich_levels = 3;
  const ValidatedConfig cfg = validate_config(c);
  struct Unit {
    FeatureMatrix q, k, v, g;
  };
  std::vector<Unit> in(units);
  for (unsigned u = 0; u < units; ++u) {
    const std::uint64_t s = 42 + 4 * u;  // bench.cpp:270-273 seeding
    in[u] = {gen_random(c.n, c.d, s), gen_random(c.n, c.d, s + 1), gen_random(c.n, c.d, s + 2),
             gen_random(c.n, c.d, s + 3)};
  }
  double checksum = 0;
  auto step = [&]() {
    for (const Unit& x : in) {
      const Pyramid pq = build_pyramid(x.q, cfg.block_size(), cfg.levels());
      const Pyramid pk = build_pyramid(x.k, cfg.block_size(), cfg.levels());
      const Pyramid pv = build_pyramid(x.v, cfg.block_size(), cfg.levels());
      const SelectionResult sel = hierarchical_topk(pq, pk, cfg);
      const EnrichedKVPlan plan = build_plan(sel, cfg);
      const ForwardState st = llsa_forward(x.q, x.k, x.v, pk, pv, plan, cfg);
      const auto tr = transpose_all(sel, cfg);
      const GradientSet gs = llsa_backward(x.g, st, x.q, x.k, x.v, pk, pv, plan, tr, cfg);
      checksum += gs.dq.data()[0] + st.output.data()[0];
    }
  };
  step();  // warm-up (CUDA context, first allocations)
  std::vector<double> ms;
  for (int i = 0; i < steps; ++i) {
    const auto t0 = Clock::now();
    step();
    ms.push_back(std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
  }
  double mean = 0;
  for (double m : ms) mean += m;
  mean /= ms.size();
  std::printf("{\"path\": \"C++ drop-in (include/llsa/*.hpp -> libllsa.so), host FeatureMatrix "
              "in/out, fp32\", \"units\": %u, \"steps\": %d, \"ms_per_step\": %.3f, "
              "\"ms_per_unit\": %.3f, \"checksum\": %.6g}\n",
              units, steps, mean, mean / units, checksum);
  return 0;
}
