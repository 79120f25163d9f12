#!/bin/bash
# Full GPU round trip: every GPU test (parity log kept), sanitizers, bench line.
mkdir -p gpurun_out
export LLSA_PARITY_LOG=gpurun_out/parity.jsonl
rm -f "$LLSA_PARITY_LOG"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/gputest.log; grep -E "^FAILED" gpurun_out/gputest.log | head
[ "${SANITIZE:-1}" = 1 ] && bash tools/sanitize.sh
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['stages_ms'], d['roofline'], d['e2e'], d['cpu_baseline'])"
