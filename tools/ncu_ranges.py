"""Warp-stall samples of one kernel aggregated over SASS index ranges, with the
distinctive opcodes of each range (to map ranges to kernel phases).
Usage: python tools/ncu_ranges.py rep kernel_regex [bucket]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
bucket = int(sys.argv[3]) if len(sys.argv) > 3 else 100
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
isrc, ist = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[ist].isdigit()]
tot = sum(int(r[ist]) for r in body)
KEY = ("HMMA", "UTCHMMA", "UTCBAR", "LDTM", "MUFU", "SYNCS", "LDGSTS", "UTMALDG", "STS", "LDSM",
       "STG", "BAR", "LDG", "F2FP")
for b in range(0, len(body), bucket):
    seg = body[b:b + bucket]
    s = sum(int(r[ist]) for r in seg)
    ex = sum(int(r[iex] or 0) for r in seg)
    ops = collections.Counter()
    for r in seg:
        op = r[isrc].strip().split()
        op = [o for o in op if not o.startswith("@")]
        if op:
            base = op[0].split(".")[0]
            if base in KEY:
                ops[base] += 1
    print(f"[{b:5d}-{b + len(seg) - 1:5d}] {s / tot * 100:5.1f}%  exec {ex:>10}  " +
          " ".join(f"{k}:{v}" for k, v in ops.most_common(6)))
