#!/bin/bash
# Dev (GPU box): trace build, CTA 0's level-1 tc5_rows2 timeline (tile-indexed
# events; LLSA_TRACE_ONLY=rows2 leaves every other kernel untraced).
LLSA_NVCC_EXTRA=-DLLSA_TRACE_EVENTS python -m paper_2512_16615_b200._build --force > /dev/null 2>&1
LLSA_TRACE_ONLY=rows2 TRACE_TMAX=32 python tools/trace_fwd.py bwd > gpurun_out/trace_rows2.txt 2>&1
python - <<'PY'
import re, collections
ev = collections.defaultdict(dict)
names = {"prod": "keys", "2": "qtma", "S": "S", "softmax": "smax", "dQ/dKV": "acc"}
for line in open("gpurun_out/trace_rows2.txt"):
    m = re.match(r"\s*(\d+)\s+(\S+) tile\s+(\d+) ev (\d+)", line)
    if m:
        t, role, c, e = int(m[1]), m[2], int(m[3]), int(m[4])
        ev[(names.get(role, role), e)][c] = t
keys = sorted(ev)
base = min(min(d.values()) for d in ev.values())
print("tile  " + " ".join(f"{r}{e:>2}".rjust(9) for r, e in keys))
for c in range(32):
    print(f"{c:5d} " + " ".join((str(ev[k][c] - base) if c in ev[k] else "").rjust(9) for k in keys))
PY
