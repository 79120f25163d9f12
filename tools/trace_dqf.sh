#!/bin/bash
# Dev (GPU box): trace build, CTA 0's tc5_dqf_kernel timeline (kvf disabled so
# it does not overwrite the roles), chunk-indexed events.
LLSA_NVCC_EXTRA=-DLLSA_TRACE_EVENTS python -m paper_2512_16615_b200._build --force > /dev/null 2>&1
TRACE_TMAX=32 python tools/trace_fwd.py bwd dq > gpurun_out/trace_dqf.txt 2>&1
python - <<'PY'
import re, collections
ev = collections.defaultdict(dict)
for line in open("gpurun_out/trace_dqf.txt"):
    m = re.match(r"\s*(\d+)\s+(\S+) tile\s+(\d+) ev (\d+)", line)
    if m:
        t, role, c, e = int(m[1]), m[2], int(m[3]), int(m[4])
        ev[(role, e)][c] = t
keys = sorted(ev)
base = min(min(d.values()) for d in ev.values())
print("chunk " + " ".join(f"{r}{e:>2}".rjust(11) for r, e in keys))
for c in range(32):
    print(f"{c:5d} " + " ".join((str(ev[k][c] - base) if c in ev[k] else "").rjust(11) for k in keys))
PY
