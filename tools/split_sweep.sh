#!/bin/bash
# Dev: coarsest-level key-major split size sweep (queries per task).
for q in ${QS:-512 1024 2048 4096}; do
  LLSA_KV_SPLIT_Q=$q timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/s$q.log 2>&1
  echo "q=$q $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/s$q.log | head -1) $(grep -o '"bwd_kv_coarse": [0-9.]*' gpurun_out/s$q.log)"
done
