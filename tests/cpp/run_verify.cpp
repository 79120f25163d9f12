// TEST INFRASTRUCTURE: runs the reference's own oracle-equivalence harness
// (llsa::bench::run_verify, P/src/bench.cpp:154-247 — its seven checks) on
// whichever library it is linked against (oracle/Makefile: the B200 drop-in
// libllsa.so, or the reference's f32 library for the allowlist), then the
// negative control (corrupt_roundtrip must make transpose-roundtrip fail).
// Prints one line per check; exit code = number of failed checks.
#include <cstdio>

#include "llsa/bench.hpp"

int main() {
  using namespace llsa;
  int failed = 0;
  for (const bench::VerifyCheck& c : bench::run_verify()) {
    std::printf("[%s] %s error %.3g tolerance %.3g\n", c.pass ? "PASS" : "FAIL", c.name.c_str(),
                c.error, c.tolerance);
    failed += c.pass ? 0 : 1;
  }
  bench::VerifyOptions neg;
  neg.corrupt_roundtrip = true;
  bool caught = false;
  for (const bench::VerifyCheck& c : bench::run_verify(neg))
    if (c.name == "transpose-roundtrip") caught = !c.pass;
  std::printf("[%s] negative-control corrupt_roundtrip detected\n", caught ? "PASS" : "FAIL");
  failed += caught ? 0 : 1;
  std::printf("%d failed\n", failed);
  return failed;
}
