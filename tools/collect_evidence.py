"""Dev: copies one tools/round_evidence.sh run (gpurun_out/) into profiles/:
bench line (profiles/r2_bench_line_v<N>.json), launch list, kernel traffic,
DiT step, parity table, BASELINE configs, and refreshes the tables inside
profiles/r2_ncu_v2.md and profiles/r2_sanitizer.md (current line refs).
Usage: python tools/collect_evidence.py <N>"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(R, "gpurun_out"), os.path.join(R, "profiles")
v = sys.argv[1]
shutil.copy(f"{G}/bench.json", f"{P}/r2_bench_line_v{v}.json")
shutil.copy(f"{G}/launches.csv", f"{P}/r2_launches_v3.csv")
shutil.copy(f"{G}/kernel_traffic.json", f"{P}/kernel_traffic.json")
shutil.copy(f"{G}/dit.json", f"{P}/r2_dit_step.json")
subprocess.run([sys.executable, f"{R}/tools/parity_json.py", f"{G}/parity.jsonl",
                f"{P}/r2_parity.json"], check=True)
# BASELINE configs
doc = json.load(open(f"{P}/r2_configs.json"))
lines = []
for ln in open(f"{G}/configs.jsonl"):
    if not ln.strip():
        continue
    d = json.loads(ln)
    c, r = d["config"], d["roofline"]
    lines.append({"preset": c["preset"], "baseline": c.get("baseline_config"),
                  "units": c["units_per_gpu"], "ms_per_step": round(d["ms_per_step"], 4),
                  "ms_per_unit": round(d["ms_per_step"] / c["units_per_gpu"], 5),
                  "stages_ms": d["stages_ms"], "effective_tflops": round(d["effective_tflops"], 1),
                  "roofline": {k: r[k] for k in ("kernel", "bound", "frac", "tensor_frac",
                                                  "hbm_frac")},
                  "clocks": d["clocks"]})
doc["lines"] = lines
json.dump(doc, open(f"{P}/r2_configs.json", "w"), indent=1)
# ncu tables
rows = list(csv.reader(open(f"{P}/r2_launches_v3.csv")))
h0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[h0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[h0 + 1:]:
    if len(r) <= vi:
        continue
    n = r[ki]
    name = (n.split("(")[0].replace("void ", "").replace("llsa_impl::<unnamed>::", "")
            if "llsa_impl" in n else n[:60])
    agg.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1000)
tot = sum(sum(x) for x in agg.values())
tbl = "\n".join(f"| {n} | {len(x)} | {sum(x):.1f} | {100 * sum(x) / tot:.1f} % |"
                for n, x in sorted(agg.items(), key=lambda kv: -sum(kv[1])))
summ = open(f"{G}/prof_summary.md").read().strip().splitlines()
mt = "\n".join(summ[next(i for i, ln in enumerate(summ) if ln.startswith("| kernel")):])
nd = open(f"{P}/r2_ncu_v2.md").read()
i, j = nd.index("| kernel | launches (2 steps)"), nd.index("## Per-kernel metrics")
nd = nd[:i] + "| kernel | launches (2 steps) | µs (2 steps) | share |\n|---|---|---|---|\n" + \
    tbl + "\n\n" + nd[j:]
i, j = nd.index("| kernel | time_us"), nd.index("## Reading")
nd = nd[:i] + mt + "\n\n" + nd[j:]
open(f"{P}/r2_ncu_v2.md", "w").write(nd)
# sanitizer summary table + verbatim racecheck lines
def summ_of(f):
    m = re.findall(r"(ERROR SUMMARY: \d+ errors|RACECHECK SUMMARY: [^\n]*)", open(f).read())
    return m[-1] if m else "?"
sd = open(f"{P}/r2_sanitizer.md").read()
trows = "\n".join(f"| {t} | {summ_of(f'{G}/sanitize_{t}_n16384.log')} | "
                  f"{summ_of(f'{G}/sanitize_{t}_n65536.log')} |"
                  for t in ("memcheck", "racecheck", "synccheck"))
i, j = sd.index("| tool | C2 | C3 |"), sd.index("## racecheck reports")
sd = sd[:i] + "| tool | C2 | C3 |\n|---|---|---|\n" + trows + "\n\n" + sd[j:]
race = "\n".join(ln.rstrip() for ln in open(f"{G}/sanitize_racecheck_n65536.log")
                 if "Race reported" in ln or "and Write access" in ln)
i = sd.index("```\n") + 4
j = sd.index("```", i)
sd = sd[:i] + race + "\n" + sd[j:]
# the hazard explanations, with the current source line numbers
src = open(f"{R}/paper_2512_16615_b200/csrc/attn_tc.cu").read().splitlines()


def ln(pat, start=0):
    return next(i + 1 for i, t in enumerate(src) if i >= start and pat in t)


k0 = ln("tc5_kvf_kernel(const __grid_constant__")
r_lo = ln("const uint32_t lo0 = fact[fs * kFactWords], hi0", k0)
r_ids = ln("const uint32_t ids0 = fact[fs * kFactWords + 4 + lane];", k0)
w_kb = ln("fact[j * kFactWords + 3] = (uint32_t)(id % nkb);", k0)
w_qb = ln("fact[j * kFactWords + 4 + lane] = qb;", k0)
w_wait = ln("if (it >= (uint32_t)kFactSlots) mbar_wait(bar(FACTE + j)", k0)
w_arr = ln("if (lane == 0) mbar_arrive(bar(FACTF + j));", k0)
g_wait = ln("mbar_wait(bar(FACTF + fs), (it / kFactSlots) & 1);", k0)
g_arr = ln("if (lane == 0) mbar_arrive(bar(FACTE + fs));", k0)
e_wait = ln("mbar_wait(bar(FACTF + fs), (it / kFactSlots) & 1);", g_wait)
e_arr = ln("if (lane == 0) mbar_arrive(bar(FACTE + fs));", g_arr)
d0 = ln("tc5_dqf_kernel(const __grid_constant__")
d_wait = ln("mbar_wait(bar(DREADY + ts), (i / kStatSlots) & 1);", d0)
d_read = ln("const float lse = stat[ts * 256 + row], Drow", d0)
d_w1 = ln("stat[ts * 256 + fw * 16 + rr] = lse_r;", d0)
d_arr = ln("mbar_arrive(bar(DREADY + ts));", d0)
prose = (
    f"* `tc5_kvf_kernel` `attn_tc.cu:{r_lo}/{r_ids}` (the gather warps read the item-facts "
    f"ring) vs `:{w_kb}/{w_qb}` (the facts warp writes it): the writer waits `FACTE[slot]` "
    f"before every write (`:{w_wait}`); the readers — the four gather warps and the four "
    f"epilogue warps — arrive on `FACTE[slot]` after `__syncwarp()` once they hold the words "
    f"in registers (`:{g_arr}`, `:{e_arr}`), and wait `FACTF[slot]` (`:{g_wait}`, "
    f"`:{e_wait}`), which the writer arrives after its stores (`:{w_arr}`). A full/empty "
    f"ring.\n"
    f"* `tc5_dqf_kernel` `attn_tc.cu:{d_read}` (coarse warps read the tile's LSE / D) vs "
    f"`:{d_w1}-{d_w1 + 1}` (fine warps write them for a later tile): until round 2 this "
    f"two-slot ring had no ordering of the refill after the read — a real race (a 128-unit "
    f"batch showed garbage dq in a few units, DESIGN §4).  The ring now has three slots "
    f"(`DREADY`, `:{d_wait}` / `:{d_arr}`); the fine warps, at most two tiles ahead "
    f"(bounded by `FFREE`), never refill an unread slot, and racecheck no longer reports "
    f"the pair.\n\n")
i = sd.index("* `tc5_kvf_kernel` `attn_tc.cu:")
j = sd.index("memcheck and synccheck: 0 errors")
sd = sd[:i] + prose + sd[j:]
open(f"{P}/r2_sanitizer.md", "w").write(sd)
b = json.load(open(f"{G}/bench.json"))
print("bench", b["value"], "e2e", b["e2e"]["value"], "ref", b["cpu_baseline"]["value"],
      "dense", b["dense_sdpa"]["speedup_fwd"], b["dense_sdpa"]["speedup_fwd_bwd"])
print("configs", [(x["preset"], x["ms_per_step"]) for x in lines])
print("racecheck refs", sorted(set(re.findall(r"attn_tc.cu:(\d+)", race))))
