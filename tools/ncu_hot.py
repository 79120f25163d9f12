"""Top SASS lines by warp-stall samples for one kernel of an ncu report.
Usage: python tools/ncu_hot.py rep.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index(
    "Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[ist].isdigit()]
tot = sum(int(r[ist]) for r in body)
print("total samples", tot, "instructions", len(body))
for i, r in sorted(enumerate(body), key=lambda x: -int(x[1][ist]))[:n]:
    print(f"{int(r[ist]) / tot * 100:5.1f}%  [{i:5d}] {r[isrc].strip()[:90]}")
