#!/usr/bin/env python
"""LLSA hot-path benchmark (BASELINE.json metric: "LLSA fwd+bwd ms at
N=65536 (256² px tokens) and % of tensor/HBM roofline").

One step = the whole path on `units` = 16 (batch·head) units per GPU:
compress → select → attention forward → CSR→CSC transpose → backward, at
N=65536, d=64, B=16, K=8, L=3 (= "4 levels"), L_e=L, ScaleKV, bf16 inputs,
synthetic N(0,1) data resident in HBM.  Multi-GPU (torchrun): every rank runs
its own 16 units (weak scaling over batch; no collective on the data path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl llsa|reference]

Prints ONE JSON line on rank 0 (see the task contract; DESIGN.md §Measurement
explains every field).  `--impl reference` times the reference CPU library
(oracle/_ref, built from /root/reference) with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TOK, D, B, K, LEVELS = 65536, 64, 16, 8, 3
UNITS_PER_GPU = 16
METRIC = "LLSA fwd+bwd ms at N=65536 (256² px tokens) and % of tensor/HBM roofline"

# BASELINE.json configs as bench presets (SURVEY.md §8 resolves "levels": the
# reference's `levels` L = max_levels(N, 16); C5's "5 levels" is inadmissible
# at N = 262144, so L = 3 = max).  C1 (N = 4096, fp32, 1 head) is the CPU
# reference's own case and a parity test, not a bench line.
PRESETS = {
    "C2": dict(n=16384, levels=2, top_k=8, enrich_levels=2, units=16, global_units=0,
               baseline="configs[1]: N=16384, 3 levels, 16 heads, bf16 fwd+bwd"),
    "C3": dict(n=65536, levels=3, top_k=8, enrich_levels=3, units=16, global_units=0,
               baseline="configs[2]: N=65536, 4 levels, 16 heads (headline metric)"),
    "C4": dict(n=65536, levels=3, top_k=8, enrich_levels=3, units=16, global_units=128,
               baseline="configs[3]: N=65536 fwd+bwd, batch 8 x 16 heads over 1/2/4/8 GPUs"),
}
for _k in (4, 8, 16):
    for _le in (3, 0):
        PRESETS[f"C5-K{_k}-Le{_le}"] = dict(
            n=262144, levels=3, top_k=_k, enrich_levels=_le, units=16, global_units=0,
            baseline=f"configs[4]: N=262144, K={_k}, "
                     f"{'full' if _le == 3 else 'no'} KV enrichment")


def _peaks() -> tuple[dict, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback"


def _geometry(n: int, L: int, k: int = K, b: int = B, le: int | None = None):
    le = L if le is None else le
    lim = min(le + 1, L)
    top = n // b ** (L + 1) if le == L else 0      # coarsest blocks every query sees
    E = k * lim + top
    return {"E": E, "P": n * E * b,                # (query, key) pairs per unit, P = N·E·B
            "P_fine": n * k * b,                   # level 0
            "P_coarse": n * k * b * (lim - 1),     # levels 1 .. lim-1 (selected)
            "P_top": n * top * b}                  # coarsest level (all N queries)


def algorithmic_work(n: int, L: int, units: int, le: int | None = None, k: int = K) -> dict:
    """Algorithmic work per timed stage for `units` units: SURVEY.md §8(d)'s
    per-unit figures, split per kernel as DESIGN.md §3 states them.  bytes are
    the minimum HBM traffic with bf16 tensors in and out (§8(d)); bytes_f32out
    the same with the fp32 outputs this build writes (O, dq, dk, dv)."""
    g = _geometry(n, L, k, le=le)
    d, Nd, N = D, n * D, n
    pyr_rows = sum(n // B ** l for l in range(1, L + 1))
    sel_macs = (n // B ** L) ** 2 * d + sum((n // B ** l) * k * B * d for l in range(1, L))
    tr_entries = sum((n // B ** (l + 1)) * k for l in range(L))
    w = {
        # read q, k, v (bf16); write the fp32 pooled levels of the three
        "compress": {"flops": 0, "bytes": 3 * Nd * 2 + 3 * pyr_rows * d * 4},
        # exact fp32 scores (2 flops per MAC) over the pooled q, k
        "select": {"flops": 2 * sel_macs, "bytes": 2 * pyr_rows * d * 4 + tr_entries * 4},
        # QK^T + PV = 4·d·P; read Q, K, V, write O + LSE (8·N·d + 4·N; + row_max and
        # row_denom = 8·N·d + 8·N as stored)
        "fwd_attention": {"flops": 4 * d * g["P"], "bytes": 8 * Nd + 8 * N,
                          "bytes_f32out": 6 * Nd + 4 * Nd + 8 * N},
        # CSR → CSC: read the tables, write offsets + lists (int32)
        "transpose": {"flops": 0, "bytes": 3 * 4 * tr_entries},
        # S, dP, dQ over every pair (6·d·P); read Q, K, V, O, dO, LSE; write dq, D
        "bwd_dq": {"flops": 6 * d * g["P"], "bytes": 12 * Nd + 8 * N,
                   "bytes_f32out": 8 * Nd + 4 * Nd + 4 * Nd + 8 * N},
        # S, dP, dK', dV' over the selected coarse pairs (levels 1..L_e); read Q, dO,
        # LSE, D once; the pooled K', V' rows and gradients are small
        "bwd_kv_coarse_tc5": {"flops": 8 * d * g["P_coarse"],
                              "bytes": 4 * Nd + 8 * N + 4 * pyr_rows * d * 2},
        # coarsest level against all N queries: read Q, dO, LSE, D
        "bwd_kv_coarse": {"flops": 8 * d * g["P_top"], "bytes": 4 * Nd + 8 * N},
        # S, dP, dK, dV over the fine pairs (8·d·P_fine); read Q, K, V, dO, LSE, D,
        # write dK, dV (12·N·d + 8·N; fp32 dK, dV: 16·N·d + 8·N)
        "bwd_kv_fine": {"flops": 8 * d * g["P_fine"], "bytes": 12 * Nd + 8 * N,
                        "bytes_f32out": 8 * Nd + 8 * Nd + 8 * N},
    }
    for v in w.values():
        v["flops"] *= units
        v["bytes"] *= units
        if "bytes_f32out" in v:
            v["bytes_f32out"] *= units
    # whole-path totals (§8(d)): forward 4·d·P, backward 10·d·P FLOP;
    # forward 8·N·d + 4·N, backward 16·N·d + 8·N bytes
    w["fwd_total"] = {"flops": units * 4 * d * g["P"], "bytes": units * (8 * Nd + 4 * N)}
    w["bwd_total"] = {"flops": units * 10 * d * g["P"], "bytes": units * (16 * Nd + 8 * N)}
    w["pairs"], w["E"] = units * g["P"], g["E"]
    return w


def stage_roofline(name: str, ms: float, W: dict, peaks: dict) -> dict | None:
    """Tensor and HBM fractions of one stage; `bound` is the roof its
    algorithmic work hits first (max of the two ideal times)."""
    wk = W.get(name)
    if not wk or ms <= 0:
        return None
    pt, ph = peaks["bf16_tflops"], peaks["hbm_gbs"]
    tflops = wk["flops"] / (ms * 1e-3) / 1e12
    gbs = wk["bytes"] / (ms * 1e-3) / 1e9
    t_tc = wk["flops"] / (pt * 1e12)
    t_hbm = wk["bytes"] / (ph * 1e9)
    r = {"ms": round(ms, 4), "flops": wk["flops"], "bytes": wk["bytes"],
         "tflops": round(tflops, 2), "tensor_frac": round(tflops / pt, 4),
         "gbs": round(gbs, 1), "hbm_frac": round(gbs / ph, 4),
         "bound": "tensor" if t_tc >= t_hbm else "hbm",
         "ideal_ms": round(max(t_tc, t_hbm) * 1e3, 4)}
    if "bytes_f32out" in wk:
        r["hbm_frac_f32out"] = round(wk["bytes_f32out"] / (ms * 1e-3) / 1e9 / ph, 4)
    tr = _traffic(name)
    if tr:
        r["traffic"] = tr
        r["traffic_over_algorithmic"] = round(tr / wk["bytes"], 3)
    return r


class ClockSampler:
    """Samples SM clocks + throttle reasons via NVML during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            pass
        self.period = period_s
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                c = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((c, r))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self._t.join(timeout=1)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1): "gpu_idle",
            getattr(nv, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2): "app_clocks",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonSyncBoost", 0x10): "sync_boost",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80):
                "hw_power_brake_slowdown",
        }
        seen = 0
        for _, r in self.samples:
            seen |= r
        reasons = sorted(v for k, v in names.items() if seen & k)
        return {"sm_mhz": statistics.median(c for c, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference CPU arm
# ---------------------------------------------------------------------------
def reference_sample(steps: int, warmup: int, n: int = N_TOK, L: int = LEVELS,
                     units: int = UNITS_PER_GPU, k: int = K, le: int | None = None) -> dict:
    """Times the reference library (oracle/_ref: the unmodified reference
    compiled from its sources, f32 build) on the WHOLE step: all `units`
    units, each through the reference's full path (compress, select, plan,
    forward, transpose, backward), the units run concurrently on host threads
    (the library is reentrant; its own parallel_for uses every core inside
    each call), so a step is the same work as the GPU arm's step."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import REF_SO, Config, OracleC, Reference, unit_inputs
    cfg = Config(n, D, B, k, L, L if le is None else le)
    if os.path.exists(REF_SO[32]):
        be = Reference(32)
        be.set_threads(0)
        kind, cores = "reference", be.threads()
        kw = {"want_outputs": False}
    else:  # reference not compiled on this box: the C restatement (1 thread per unit)
        be = OracleC()
        kind, cores = "port", os.cpu_count() or 1
        kw = {}
    ins = [unit_inputs(cfg, u, backend=be) for u in range(units)]
    pool = ThreadPoolExecutor(max_workers=units)

    def one_step():
        list(pool.map(lambda x: be.run(cfg, *x, **kw), ins))

    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        one_step()
        dt = (time.perf_counter() - t0) * 1e3
        if i >= warmup:
            times.append(dt)
    pool.shutdown()
    per_step = statistics.fmean(times)   # total / steps, like the GPU arm
    return {"value": per_step, "unit": "ms", "cores": cores, "kind": kind,
            "sample": f"all {units} units per step (N={n}, L={L}, K={k}, fwd+bwd incl. "
                      f"compress/select/plan/transpose), units concurrent on host threads, "
                      f"mean of {steps} step(s) after {warmup} warm-up; "
                      f"{os.cpu_count()} host CPUs",
            "steps": steps, "warmup": warmup, "median_ms": statistics.median(times)}


# ---------------------------------------------------------------------------
# dense comparator (north star: >= 28x faster than dense FlashAttention-style
# attention at the same shape)
# ---------------------------------------------------------------------------
def dense_sdpa(n: int, units: int, dev, steps: int = 3, warmup: int = 2) -> dict:
    """torch scaled_dot_product_attention (bf16, [1, units, n, 64], non-causal;
    the fused flash / cuDNN kernel torch picks on this GPU), timed with CUDA
    events: forward only and forward+backward.  Library kernels, reported
    beside the LLSA numbers, never as them."""
    import torch
    import torch.nn.functional as F
    shape = (1, units, n, D)
    q, k, v, g = (torch.randn(shape, device=dev, dtype=torch.bfloat16) for _ in range(4))
    qr, kr, vr = (t.clone().requires_grad_(True) for t in (q, k, v))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    with torch.no_grad():
        for _ in range(warmup):
            F.scaled_dot_product_attention(q, k, v)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            F.scaled_dot_product_attention(q, k, v)
        e1.record()
        torch.cuda.synchronize()
    res["fwd_ms"] = e0.elapsed_time(e1) / steps
    for _ in range(warmup):
        F.scaled_dot_product_attention(qr, kr, vr).backward(g)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        F.scaled_dot_product_attention(qr, kr, vr).backward(g)
    e1.record()
    torch.cuda.synchronize()
    res["fwd_bwd_ms"] = e0.elapsed_time(e1) / steps
    flops_fwd = 4.0 * n * n * D * units
    res["fwd_tflops"] = flops_fwd / (res["fwd_ms"] * 1e-3) / 1e12
    res["fwd_bwd_tflops"] = 3.5 * flops_fwd / (res["fwd_bwd_ms"] * 1e-3) / 1e12
    res["impl"] = "torch.nn.functional.scaled_dot_product_attention (bf16, non-causal)"
    del q, k, v, g, qr, kr, vr
    torch.cuda.empty_cache()
    return res


def _traffic(stage: str):
    """DRAM bytes per launch of a stage's dominant kernel from the committed ncu
    capture (profiles/kernel_traffic.json, dram__bytes_read.sum +
    dram__bytes_write.sum), or None."""
    p = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return t.get("stages", {}).get(stage)
    except (OSError, ValueError):
        return None


def run_e2e(kind: str, h, inputs, cfg, dev, stream, steps: int, barrier, max_over_ranks
            ) -> dict:
    """End to end through the C ABI with HOST buffers: every step copies its
    inputs (q, k, v, dO bf16) H2D from pinned memory, runs the whole path and
    copies its results (O, dq, dk, dv) D2H.  Steps are software-pipelined over
    three streams with double-buffered device sets, so H2D of step i+1 and D2H
    of step i-1 overlap step i's kernels (PCIe is full duplex) and the steady
    state is bound by the larger transfer.  Up to 30 pipelined steps are
    timed (LLSA_E2E_STEPS, bounded by --steps) so the pipeline fill and drain
    (one transfer + one compute) weigh little in the per-step figure.
      handle_bf16_out  llsa_handle_forward_ex / backward_ex, bf16 results
      handle_f32_out   llsa_handle_forward / backward, fp32 results
      staged_c_abi     the reference-shaped staged entry points (llsa_build_pyramid
                       x3, llsa_hierarchical_topk, llsa_forward, llsa_transpose_all,
                       llsa_backward; bf16 inputs run the same tensor-core kernels),
                       fp32 results as the reference's ForwardState / GradientSet"""
    import torch

    import paper_2512_16615_b200 as llsa
    q, k, v, dO = inputs
    shape = q.shape
    odt = torch.bfloat16 if kind == "handle_bf16_out" else torch.float32
    hq, hk, hv, hdo = (t.cpu().pin_memory() for t in (q, k, v, dO))
    hout = [tuple(torch.empty(shape, dtype=odt).pin_memory() for _ in range(4))
            for _ in range(2)]
    din = [tuple(t.clone() for t in (q, k, v, dO)) for _ in range(2)]
    dres = [tuple(torch.empty(shape, device=dev, dtype=odt) for _ in range(4))
            for _ in range(2)]
    vc = llsa.validate_config(cfg)
    s_h2d, s_cmp, s_d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_free = [ev(), ev()]     # compute of the step that last used din[b] is done
    res_free = [ev(), ev()]    # D2H of the step that last used dres[b] is done
    for e_ in in_free + res_free:
        e_.record(stream)

    def compute(q_, k_, v_, g_, o_, dq_, dk_, dv_):
        if kind != "staged_c_abi":
            h.forward(q_, k_, v_, o_)
            h.backward(g_, q_, k_, v_, o_, dq_, dk_, dv_)
            return
        L = vc.levels
        pq, pk, pv = (llsa.build_pyramid(t, vc.block_size, L) for t in (q_, k_, v_))
        tables = llsa.hierarchical_topk(pq, pk, vc)
        st = llsa.llsa_forward(q_, k_, v_, pk, pv, tables, vc, check_finite=False)
        tr = llsa.transpose_all(tables, vc)
        gq, gk, gv = llsa.llsa_backward(g_, st, q_, k_, v_, pk, pv, tables, tr, vc)
        for d_, s_ in zip((o_, dq_, dk_, dv_), (st.output, gq, gk, gv)):
            d_.copy_(s_)

    def e2e_steps(n_steps):
        for i in range(n_steps):
            b = i & 1
            h2d_done, cmp_done = ev(), ev()
            with torch.cuda.stream(s_h2d):
                s_h2d.wait_event(in_free[b])
                for d_, h_ in zip(din[b], (hq, hk, hv, hdo)):
                    d_.copy_(h_, non_blocking=True)
                h2d_done.record(s_h2d)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(h2d_done)
                s_cmp.wait_event(res_free[b])
                compute(*din[b], *dres[b])
                cmp_done.record(s_cmp)
                in_free[b] = ev()
                in_free[b].record(s_cmp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(cmp_done)
                for h_, d_ in zip(hout[b], dres[b]):
                    h_.copy_(d_, non_blocking=True)
                res_free[b] = ev()
                res_free[b].record(s_d2h)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps(2)
    torch.cuda.synchronize()
    llsa.sync_status()
    n_e2e = max(3, min(steps, int(os.environ.get("LLSA_E2E_STEPS", "30"))))
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for s_ in (s_h2d, s_cmp, s_d2h):
        s_.wait_event(e0)
    e2e_steps(n_e2e)
    for s_ in (s_h2d, s_cmp, s_d2h):
        stream.wait_stream(s_)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    llsa.sync_status()
    ms = max_over_ranks(e0.elapsed_time(e1) / n_e2e)
    esz = 2 if odt == torch.bfloat16 else 4
    res = {"value": ms, "unit": "ms", "h2d_bytes_per_step": 4 * q.numel() * 2,
           "d2h_bytes_per_step": 4 * q.numel() * esz, "steps": n_e2e,
           "outputs": str(odt).replace("torch.", ""),
           "path": {"handle_bf16_out": "llsa_handle_forward_ex/backward_ex (C ABI), bf16 O/dq/"
                                       "dk/dv",
                    "handle_f32_out": "llsa_handle_forward/backward (C ABI), fp32 O/dq/dk/dv",
                    "staged_c_abi": "staged reference-shaped C ABI (llsa_build_pyramid, "
                                    "llsa_hierarchical_topk, llsa_forward, llsa_transpose_all, "
                                    "llsa_backward), fp32 O/dq/dk/dv"}[kind]
           + "; pinned host buffers, H2D / kernels / D2H pipelined over three streams"}
    del din, dres, hout
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------------------
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="llsa", choices=["llsa", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(PRESETS),
                    help="BASELINE.json workload preset (SURVEY.md §8 C2..C5); C3 is the "
                         "headline metric's config")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--levels", type=int, default=None)
    ap.add_argument("--top-k", type=int, default=None)
    ap.add_argument("--enrich-levels", type=int, default=None)
    ap.add_argument("--units", type=int, default=None,
                    help="units per GPU (weak scaling, default)")
    ap.add_argument("--global-units", type=int, default=None,
                    help="fixed total units split over the GPUs (strong scaling, e.g. 128 "
                         "for BASELINE C4 = batch 8 x 16 heads)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of a captured CUDA graph")
    ap.add_argument("--no-dense", action="store_true",
                    help="skip the dense SDPA comparator")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    preset = PRESETS[args.config]
    for key in ("n", "levels", "top_k", "enrich_levels", "units", "global_units"):
        if getattr(args, key) is None:
            setattr(args, key, preset[key])

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2512_16615_b200.sharding import shard_units
    scaling = "weak"
    if args.global_units:
        args.units = shard_units(args.global_units, world, rank)[1]
        scaling = "strong"
    cfg_json = {"workload": f"LLSA fwd+bwd ({args.config}), N={args.n}, {args.units} units "
                            f"(batch·head) per GPU, d=64, B=16, K={args.top_k}, "
                            f"L={args.levels}, L_e={args.enrich_levels}, ScaleKV, bf16 in / "
                            "fp32 out",
                "preset": args.config, "baseline_config": preset["baseline"],
                "n": args.n, "d": D, "block_size": B, "top_k": args.top_k,
                "levels": args.levels, "enrich_levels": args.enrich_levels,
                "units_per_gpu": args.units,
                "global_units": args.global_units or args.units * world,
                "parallelism": f"batch*head units sharded over {world} GPU(s), no collective",
                "l2": "inputs larger than L2 (4 x units x N x 64 bf16 per step)"}

    if args.impl == "reference":
        if rank != 0:
            return
        # a CPU library has nothing to warm beyond page faults: one warm-up step
        r = reference_sample(args.steps, 1, args.n, args.levels, args.units, args.top_k,
                             args.enrich_levels)
        line = {"metric": METRIC, "value": r["value"], "unit": "ms", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": 1,
                "warmup_requested": args.warmup,
                "ms_per_step": r["value"], "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference gen_random "
                "N(0,1), bf16-rounded)", "config": cfg_json,
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": "ms", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "gpu_launches": 0}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    import paper_2512_16615_b200 as llsa

    # LLSA_BENCH_SHARE_GPU=1: ranks share the visible GPUs round-robin and
    # talk over gloo (a multi-rank dry run of this launch path on a box with
    # fewer GPUs than ranks; NCCL needs one GPU per rank).  The data path has
    # no collective either way.
    share = os.environ.get("LLSA_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(torch.cuda.device_count(), 1)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    units = args.units
    n = args.n

    def barrier():
        if world > 1:
            dist.barrier()

    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    shape = (units, n, D)
    q, k, v, dO = (torch.randn(shape, generator=gen, device=dev).to(torch.bfloat16)
                   for _ in range(4))
    cfg = llsa.LLSAConfig(n, D, B, args.top_k, args.levels, args.enrich_levels)
    h = llsa.LLSAHandle(cfg, units, torch.bfloat16)
    h.enable_timing(True)
    out = torch.empty(shape, device=dev, dtype=torch.float32)
    dq, dk, dv = (torch.empty(shape, device=dev, dtype=torch.float32) for _ in range(3))
    stream = torch.cuda.current_stream()

    def step():
        h.forward(q, k, v, out)
        lf = h.last_launches
        h.backward(dO, q, k, v, out, dq, dk, dv)
        return lf + h.last_launches

    for _ in range(args.warmup):
        launches = step()
    llsa.sync_status()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # per-stage breakdown: an eager pass with the handle's stage events on
    h.enable_timing(True)  # reset the event ring
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        launches = step()
    e1.record(stream)
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / args.steps
    stages = h.stage_times()
    llsa.sync_status()

    # the timed region: the step's launch sequence captured once as a CUDA
    # graph and replayed (static shapes, as in a training loop), which
    # removes the host launch gaps between the ~30 kernels of a step
    graph = None
    if not args.no_graph:
        h.enable_timing(False)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
        llsa.sync_status()

    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    llsa.sync_status()
    from paper_2512_16615_b200.sharding import max_over_ranks
    ms = max_over_ranks(ms)

    # secondary: the same step with bf16 results (O, dq, dk, dv written as
    # bf16 by the kernels, llsa_handle_*_ex) — what a bf16 training step and
    # the e2e line use; the headline keeps the reference's fp32 results
    ms_bf16 = None
    if graph is not None:
        out16, dq16, dk16, dv16 = (torch.empty(shape, device=dev, dtype=torch.bfloat16)
                                   for _ in range(4))

        def step16():
            h.forward(q, k, v, out16)
            h.backward(dO, q, k, v, out16, dq16, dk16, dv16)

        for _ in range(2):
            step16()
        g16 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g16):
            step16()
        g16.replay()
        torch.cuda.synchronize()
        llsa.sync_status()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            g16.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_bf16 = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        llsa.sync_status()

    # ---- roofline: every stage, and the dominant one as the headline --------
    peaks, peak_src = _peaks()
    W = algorithmic_work(n, args.levels, units, args.enrich_levels, args.top_k)
    per_stage = {s_: stage_roofline(s_, t_, W, peaks) for s_, t_ in stages}
    per_stage = {k_: v_ for k_, v_ in per_stage.items() if v_}
    dom_name = max(per_stage, key=lambda s_: per_stage[s_]["ms"]) if per_stage else "?"
    dr = per_stage.get(dom_name, {})
    if dr.get("bound") == "tensor":
        roof = {"bound": "tensor", "achieved": dr["tflops"], "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": dr["tensor_frac"]}
    else:
        roof = {"bound": "hbm", "achieved": dr.get("gbs"), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": dr.get("hbm_frac")}
    roof["traffic"] = dr.get("traffic")
    roof.update({"kernel": dom_name, "kernel_ms": dr.get("ms"),
                 "algorithmic_bytes": dr.get("bytes"), "algorithmic_flops": dr.get("flops"),
                 "tensor_frac": dr.get("tensor_frac"), "hbm_frac": dr.get("hbm_frac"),
                 "traffic_over_algorithmic": dr.get("traffic_over_algorithmic"),
                 "peak_source": f"{peak_src} (MEASURED_PEAKS.json, burst)",
                 "work_model": "SURVEY.md §8(d) per-unit bytes / FLOPs x units, per kernel "
                               "as DESIGN.md §3; bench.algorithmic_work"})
    total_flops = W["fwd_total"]["flops"] + W["bwd_total"]["flops"]
    ideal_ms = sum(max(W[k_]["flops"] / (peaks["bf16_tflops"] * 1e12),
                       W[k_]["bytes"] / (peaks["hbm_gbs"] * 1e9))
                   for k_ in ("fwd_total", "bwd_total")) * 1e3

    # ---- end to end through the C ABI with host buffers -----------------------
    # Every step copies its inputs H2D from pinned host memory and its results
    # (O, dq, dk, dv fp32) D2H.  Steps are software-pipelined over three
    # streams with double-buffered device sets: H2D of step i+1 and D2H of
    # step i-1 overlap step i's kernels (PCIe is full duplex), so the
    # steady state is bound by the larger transfer, not by their sum.
    e2e, e2e_variants = None, {}
    if not args.no_e2e:
        e2e_variants = {k_: run_e2e(k_, h, (q, k, v, dO), cfg, dev, stream, args.steps,
                                    barrier, max_over_ranks)
                        for k_ in ("handle_bf16_out", "handle_f32_out", "staged_c_abi")}
        e2e = dict(e2e_variants["handle_bf16_out"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = reference_sample(1, 0, n, args.levels, units, args.top_k, args.enrich_levels)
            cpu = {k_: r[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "ms", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {ex}"}

    dense = None
    if rank == 0 and not args.no_dense:
        try:
            dense = dense_sdpa(n, units, dev)
            fwd_only = sum(t_ for s_, t_ in stages
                           if s_ in ("compress", "select", "compress+select", "fwd_prep",
                                     "fwd_attention"))
            dense["llsa_fwd_ms"] = fwd_only
            dense["speedup_fwd"] = dense["fwd_ms"] / fwd_only if fwd_only else None
            dense["speedup_fwd_bwd"] = dense["fwd_bwd_ms"] / ms
        except Exception as ex:  # noqa: BLE001
            dense = {"unavailable": str(ex)[:200]}

    if rank == 0:
        line = {"metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": False, "scaling": scaling, "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic (torch.randn N(0,1) -> bf16, resident in "
                "HBM)", "config": cfg_json,
                "units_per_s": (args.global_units or units * world) / (ms * 1e-3),
                "effective_tflops": total_flops / (ms * 1e-3) / 1e12,
                "ideal_ms": ideal_ms,
                "roofline": roof,
                "stages_ms": {s: round(t_, 4) for s, t_ in stages},
                "stages_roofline": per_stage,
                "eager_ms_per_step": eager_ms,
                "ms_per_step_bf16_outputs": ms_bf16,
                "timed_launch_mode": "cuda_graph_replay" if graph is not None else "eager",
                "tensor_cores": h.uses_tensor_cores,
                "cpu_baseline": cpu, "e2e": e2e, "e2e_variants": e2e_variants, "dense_sdpa": dense, "gpu_launches": launches * args.steps,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
