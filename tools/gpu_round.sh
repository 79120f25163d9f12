#!/bin/bash
# One gpurun call: GPU tests (parity log kept), then the default bench line.
set -u
mkdir -p gpurun_out
export LLSA_PARITY_LOG=gpurun_out/parity.jsonl
rm -f "$LLSA_PARITY_LOG"
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -5 gpurun_out/gputest.log
if [ "${SKIP_BENCH:-0}" != 1 ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
fi
