#!/bin/bash
# Dev: N short bench runs back to back (stage times per run) for A/B noise checks.
for r in $(seq 1 ${N:-3}); do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/rep$r.log 2>&1
  echo "run $r $(grep -o '"value": [0-9.]*' gpurun_out/rep$r.log | head -1) $(grep -o '"stages_ms[^}]*}' gpurun_out/rep$r.log)"
done
