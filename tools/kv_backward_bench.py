"""Key/value backward: CSC lookup vs the dense-mask baseline on the GPU, over
N (the reference's run_kv_backward_bench, bench.cpp:371-385, and the paper's
Fig. 7 claim "CSC stays flat, the mask degrades").  Both paths share the key-
major backward kernels; they differ in how each key block finds its queries:
CSR→CSC (count/scan/scatter/order, O(T·K)) vs a dense query-block × key-block
mask scanned per column (O(T^2)).  bf16, d = 64, B = 16: both run the
production tensor-core kernels (tc5_kvf, tc5_rows2, tc_kv); `--units` units
(default 16, as the bench).  Times are CUDA events per call (index build +
backward), median of 5 after 2 warm-ups; K = 8, L = max_levels.

  python tools/kv_backward_bench.py > profiles/kv_backward_mask_vs_csc.json
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


units = int(sys.argv[sys.argv.index("--units") + 1]) if "--units" in sys.argv else 16
rows = []
for n in (4096, 16384, 65536, 262144):
    L = llsa.max_levels(n, 16)
    cfg = llsa.validate_config(llsa.LLSAConfig(n, 64, 16, 8, L, L))
    q, k, v, g = (torch.randn(units, n, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
    pq, pk, pv = (llsa.build_pyramid(t, 16, L) for t in (q, k, v))
    tables = llsa.hierarchical_topk(pq, pk, cfg)
    st = llsa.llsa_forward(q, k, v, pk, pv, tables, cfg)

    def csc():
        tr = llsa.transpose_all(tables, cfg)
        return llsa.kv_backward(g, st, q, k, v, pk, pv, tr, cfg)

    def mask():
        return llsa.mask_kv_backward(g, st, q, k, v, pk, pv, tables, cfg)

    a, b = csc(), mask()
    llsa.sync_status()
    same = bool(torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]))
    t_csc, t_mask = timed(csc), timed(mask)
    rows.append({"n": n, "levels": L, "csc_ms": t_csc, "mask_ms": t_mask,
                 "csc_ns_per_token": t_csc * 1e6 / (n * units),
                 "mask_ns_per_token": t_mask * 1e6 / (n * units),
                 "mask_over_csc": t_mask / t_csc, "identical": same})
    print(json.dumps(rows[-1]), file=sys.stderr)
print(json.dumps({"bench": "kv_backward CSC vs dense mask (GPU, tensor-core kv kernels)",
                  "units": units, "d": 64, "B": 16, "K": 8, "rows": rows}, indent=1))
