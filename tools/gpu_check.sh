#!/bin/bash
# GPU round trip used during development: parity tests, then a short bench.
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -8
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/bench.log 2>&1
grep -o '"value": [0-9.]*' gpurun_out/bench.log | head -1
grep -o '"stages_ms[^}]*}' gpurun_out/bench.log
