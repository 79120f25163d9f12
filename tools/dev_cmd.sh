LLSA_DETERMINISTIC=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/det.log 2>&1
echo "det $(grep -o '"value": [0-9.]*' gpurun_out/det.log | head -1) $(grep -o '"stages_ms[^}]*}' gpurun_out/det.log)"
bash tools/trace_rows2.sh > gpurun_out/rows2_table.txt 2>&1
head -34 gpurun_out/rows2_table.txt
