for u in 2 4 8 16 32; do
  timeout 300 python bench.py --units $u --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/u$u.log 2>&1
  echo "units=$u $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/u$u.log | head -1) $(grep -o '"stages_ms[^}]*}' gpurun_out/u$u.log)"
done
