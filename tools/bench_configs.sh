#!/bin/bash
# Every BASELINE.json config as a bench line on one GPU:
# gpurun_out/configs.jsonl, one JSON line per preset.
mkdir -p gpurun_out
out=gpurun_out/configs.jsonl; rm -f $out
for c in C2 C3 C4 C5-K4-Le3 C5-K8-Le3 C5-K16-Le3 C5-K4-Le0 C5-K8-Le0 C5-K16-Le0; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-dense \
    --no-cpu-baseline ${EXTRA:-} > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  echo "$c rc=$?"; cat gpurun_out/cfg_$c.json >> $out
done
