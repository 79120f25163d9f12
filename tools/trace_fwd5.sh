#!/bin/bash
# Dev (GPU box): trace build, CTA 0's tc5_fwd_kernel per-tile timeline.
LLSA_NVCC_EXTRA=-DLLSA_TRACE_EVENTS python -m paper_2512_16615_b200._build --force > /dev/null 2>&1
TRACE_TMAX=32 python tools/trace_fwd.py fwd > gpurun_out/trace_fwd.txt 2>&1
