#!/bin/bash
# One gpurun call for the round's evidence: every GPU test (parity log),
# sanitizers, the full bench line, the ncu launch list + full-set capture,
# every BASELINE config, the DiT step.  Outputs under gpurun_out/.
mkdir -p gpurun_out
bash tools/gpu_full.sh > gpurun_out/full.log 2>&1
bash tools/profile_round.sh > gpurun_out/prof.log 2>&1
bash tools/bench_configs.sh > gpurun_out/configs.log 2>&1
timeout 900 python tools/dit_step_bench.py > gpurun_out/dit.json 2> gpurun_out/dit.err
cat gpurun_out/full.log | cut -c1-300; tail -3 gpurun_out/prof.log; cat gpurun_out/configs.log
