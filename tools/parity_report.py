"""Prints the tensor-core path's error against the oracle (the C restatement
of the reference, fp32) at the BASELINE shapes: max|Δ|/max|ref|, relative
Frobenius and worst-row relative for O, dq, dk, dv, LSE, and the number of
selection rows that differ (must be 0).  Used for DESIGN.md's precision table."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402
from oracle import Config, OracleC, lse, rel_err, unit_inputs  # noqa: E402

oc = OracleC()
cases = [("C2 N=16384 L=2 ScaleKV", Config(16384, 64, 16, 8, 2, 2), True),
         ("C2 N=16384 L=2 LogitBias", Config(16384, 64, 16, 8, 2, 2, reweight_mode=1), True),
         ("C3 N=65536 L=3 ScaleKV", Config(65536, 64, 16, 8, 3, 3), "--full" in sys.argv),
         ("C3' N=65536 L=2 ScaleKV", Config(65536, 64, 16, 8, 2, 2), False),
         ("C5 N=262144 L=3 K=8", Config(262144, 64, 16, 8, 3, 3), False)]
rows = []
for name, cfg, bwd in cases:
    q, k, v, dO = unit_inputs(cfg, 0, backend=oc)
    t0 = time.time()
    ref = oc.run(cfg, q, k, v, dO if bwd else None)
    T = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)[None]  # noqa: E731
    h = llsa.LLSAHandle(llsa.LLSAConfig(cfg.n, 64, 16, cfg.top_k, cfg.levels,
                                        cfg.enrich_levels, reweight_mode=cfg.reweight_mode), 1)
    out = h.forward(T(q), T(k), T(v))
    tabs = h.view("tables")[0].cpu().numpy().astype(np.uint32)
    r = {"case": name, "tensor_cores": h.uses_tensor_cores,
         "table_rows_differing": int((tabs != ref.tables).reshape(-1, cfg.top_k).any(1).sum()),
         "out": rel_err(out[0].cpu().numpy(), ref.out)}
    m, d = h.view("row_max")[0].cpu().numpy(), h.view("row_denom")[0].cpu().numpy()
    r["lse_max_abs"] = float(np.abs(lse(m, d) - lse(ref.row_max, ref.row_denom)).max())
    if bwd:
        g = h.backward(T(dO), T(q), T(k), T(v), out)
        for nm, a, b in zip(("dq", "dk", "dv"), g, (ref.dq, ref.dk, ref.dv)):
            r[nm] = rel_err(a[0].cpu().numpy(), b)
    llsa.sync_status()
    r["oracle_s"] = round(time.time() - t0, 1)
    rows.append(r)
    print(json.dumps(r), flush=True)
