#!/bin/bash
# Dev (GPU box): trace build, CTA 0's tc5_dqf_kernel timeline (kvf disabled so
# it does not overwrite the roles), chunk-indexed events.
LLSA_NVCC_EXTRA=-DLLSA_TRACE_EVENTS python -m paper_2512_16615_b200._build --force > /dev/null 2>&1
TRACE_TMAX=32 python tools/trace_fwd.py bwd dq > gpurun_out/trace_dqf.txt 2>&1
