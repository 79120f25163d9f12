"""Dynamic opcode histogram (instructions executed) of a SASS index range of one
kernel in an ncu report.  Usage: python tools/ncu_ops.py rep kernel lo hi"""
import collections
import csv
import io
import subprocess
import sys

rep, kern, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[ist].isdigit()]
c = collections.Counter()
st = collections.Counter()
for r in body[lo:hi]:
    op = [o for o in r[isrc].strip().split() if not o.startswith("@")]
    if not op:
        continue
    k = op[0].rstrip(";")
    c[k] += int(r[iex] or 0)
    st[k] += int(r[ist] or 0)
tot = sum(c.values())
print("total", tot)
for k, v in c.most_common(30):
    print(f"{v:>12} {v / tot * 100:5.1f}%  stall {st[k]:>6}  {k}")
