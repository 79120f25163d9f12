#!/bin/bash
# Dev: e2e (host buffers) with one or two copy streams per direction.
for sp in 0 1; do
  LLSA_E2E_SPLIT=$sp timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/e2e_s$sp.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_s$sp.json')); print('split=$sp', d['e2e']['value'], {k: v.get('value') for k, v in d.get('e2e_variants', {}).items()})"
done
