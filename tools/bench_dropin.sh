#!/bin/bash
# Builds tools/bench_dropin against the drop-in headers and library.
ROOT=$(cd "$(dirname "$0")/.." && pwd)
g++ -std=c++20 -O2 -I"$ROOT/include" -o "$ROOT/tools/bench_dropin" "$ROOT/tools/bench_dropin.cpp" \
    -L"$ROOT/paper_2512_16615_b200/lib" -lllsa -Wl,-rpath,"$ROOT/paper_2512_16615_b200/lib"
