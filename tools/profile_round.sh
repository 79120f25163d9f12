#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): the launch list of two
# steps (per-launch times, cold and serialised under ncu) and one --set full
# capture of every hot kernel of a step; summaries go to gpurun_out/.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"tc5_|select_level_rb|pyr12|rows_reduce|segment_order|tc_kv_kernel|scatter_all|count_all|scan_all|reduce_parts" \
    -s 20 -c 14 -o gpurun_out/prof python tools/profile_step.py --steps 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof.ncu-rep > gpurun_out/prof_summary.md
python tools/make_traffic.py gpurun_out/prof.ncu-rep > /dev/null
cp profiles/kernel_traffic.json gpurun_out/kernel_traffic.json
tail -20 gpurun_out/prof_summary.md
