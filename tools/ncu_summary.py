"""Summarises an ncu report (--page raw) into one markdown row per kernel:
time, DRAM bytes, tensor-pipe %, issue/occupancy figures, top stall reasons.
Usage: python tools/ncu_summary.py gpurun_out/x.ncu-rep"""
import csv
import io
import subprocess
import sys

M = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "tensor_%": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_%": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_%": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "xu_%": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_%": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lsu_%": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram_%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_")
             and h.endswith(".ratio")]
    if not stall:
        stall = [h for h in hdr if "warp_issue_stalled" in h and h.endswith("_per_warp_active.pct")]
    print("| kernel | " + " | ".join(M) + " | top stalls |")
    print("|---" * (len(M) + 2) + "|")
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("llsa_impl::<unnamed>::", "")
        name = name.replace("void ", "")
        vals = []
        for k, m in M.items():
            v = r[col[m]] if m in col else ""
            try:
                f = float(v.replace(",", ""))
                u = units[col[m]]
                if k.endswith("_MB"):
                    f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
                if k == "time_us":
                    f = f * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
                vals.append(f"{f:.1f}")
            except ValueError:
                vals.append(v)
        st = []
        for h in stall:
            try:
                st.append((float(r[col[h]].replace(",", "")), h))
            except ValueError:
                pass
        st.sort(reverse=True)
        top = ", ".join(f"{h.split('stalled_')[1].split('_per')[0].split('.')[0]} {v:.1f}"
                        for v, h in st[:3])
        print(f"| {name} | " + " | ".join(vals) + f" | {top} |")


if __name__ == "__main__":
    main(sys.argv[1])
