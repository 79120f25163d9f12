"""Writes profiles/kernel_traffic.json from ncu --set full reports: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per launch of each kernel, and
per bench stage (sum over the stage's kernels, one launch each).  bench.py
reports the dominant stage's figure as roofline.traffic.
Usage: python tools/make_traffic.py rep1.ncu-rep [rep2 ...]"""
import csv
import io
import json
import os
import subprocess
import sys

STAGES = {  # bench stage -> kernel name prefixes (one launch each per step)
    "fwd_attention": ["tc5_fwd_kernel"],
    "bwd_dq": ["tc5_dqf_kernel"],
    # levels 1 and 2 both run the hi + lo variant since round 2: two launches
    "bwd_kv_coarse_tc5": ["tc5_rows2_kernel<1>", "tc5_rows2_kernel<1>#2", "rows_reduce_kernel"],
    "compress": ["pyr12_kernel"],
    "bwd_kv_coarse": ["tc_kv_kernel<2>", "reduce_parts_kernel"],
    "bwd_kv_fine": ["tc5_kvf_kernel"],
    "select": ["select_coarsest_kernel", "select_level_rb_kernel<128>"],
    "transpose": ["count_all_kernel", "scan_all_kernel", "scatter_all_kernel",
                  "segment_order_all_kernel"],
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def kernels(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    c = {h: i for i, h in enumerate(hdr)}
    out = {}
    for r in rows[2:]:
        name = r[c["Kernel Name"]].split("(")[0].replace("void ", "")
        name = name.split("::")[-1]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[c[m]].replace(",", "")) * SCALE.get(units[c[m]], 1)
        # first capture of each launch in order; the second launch of the same
        # kernel within a step is "<name>#2"
        key = name if name not in out else f"{name}#2"
        out.setdefault(key, b)
    return out


def main(reps):
    per = {}
    for rep in reps:
        for k, v in kernels(rep).items():
            per.setdefault(k, v)
    stages = {}
    for st, ks in STAGES.items():
        if all(k in per for k in ks):
            stages[st] = sum(per[k] for k in ks)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", "kernel_traffic.json")
    with open(path, "w") as f:
        json.dump({"source": [os.path.basename(r) for r in reps],
                   "note": "DRAM bytes per launch from ncu --set full (cold cache, replayed)",
                   "kernels": per, "stages": stages}, f, indent=1, sort_keys=True)
    print(json.dumps(stages, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
