#!/bin/bash
# Dev (GPU box): rebuild with the pipeline trace events compiled in, then
# print CTA 0's kvf timeline (chunk-indexed events) for steady-state chunks.
LLSA_NVCC_EXTRA=-DLLSA_TRACE_EVENTS python -m paper_2512_16615_b200._build --force > /dev/null 2>&1
TRACE_TMAX=32 python tools/trace_fwd.py bwd kv > gpurun_out/trace_bwd.txt 2>&1
python - <<'PY'
import re, collections
ev = collections.defaultdict(dict)
for line in open("gpurun_out/trace_bwd.txt"):
    m = re.match(r"\s*(\d+)\s+(\S+) tile\s+(\d+) ev (\d+)", line)
    if m:
        t, role, c, e = int(m[1]), m[2], int(m[3]), int(m[4])
        ev[(role, e)][c] = t
keys = sorted(ev)
print("chunk " + " ".join(f"{r}{e:>2}".rjust(11) for r, e in keys))
base = min(min(d.values()) for d in ev.values())
for c in range(32):
    print(f"{c:5d} " + " ".join((str(ev[k][c] - base) if c in ev[k] else "").rjust(11) for k in keys))
PY
