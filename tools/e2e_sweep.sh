#!/bin/bash
# Dev: e2e (host buffers) per-step time vs the number of pipelined steps timed.
for n in 10 30; do
  LLSA_E2E_STEPS=$n timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/e2e$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e$n.json')); print($n, d['e2e']['value'], {k: v.get('value') for k, v in d.get('e2e_variants', {}).items()})"
done
