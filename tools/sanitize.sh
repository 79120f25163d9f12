#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over one handle step at
# C2 (N=16384, L=2) and C3 (N=65536, L=3), one unit each: every kernel of the
# tensor-core path runs (tc5_fwd, tc5_dqf, tc5_rows2<0/1>, tc_kv<2>, tc5_kvf,
# transpose, select, compress).  Output: gpurun_out/sanitize_<tool>_<cfg>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for cfg in "16384 2" "65536 3"; do
    set -- $cfg
    log=gpurun_out/sanitize_${tool}_n$1.log
    timeout 900 compute-sanitizer --tool $tool \
      python tools/memcheck_c3.py $1 $2 1 > $log 2>&1
    echo "$tool n=$1 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $log | tail -2 | tr '\n' ' ')"
  done
done
