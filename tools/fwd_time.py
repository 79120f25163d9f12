"""Development timing of the attention forward / backward stages at the
bench shape (16 x 65536, d 64, B 16, K 8, L 3): median ms of the handle's
forward and backward over a few repetitions.  Env toggles (LLSA_DBG, ...)
are read per call, so variants can be compared in one process:
    python tools/fwd_time.py 0 64 24     # LLSA_DBG values to compare
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402

units, n = 16, 65536
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, dO = (torch.randn(units, n, 64, device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(4))
h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, 8, 3, 3), units)
out = torch.empty(units, n, 64, device="cuda")
grads = [torch.empty(units, n, 64, device="cuda") for _ in range(3)]
lc = llsa.LLSAConfig(n, 64, 16, 8, 3, 3)
vc = llsa.validate_config(lc)
pq, pk, pv = (llsa.build_pyramid(t, 16, 3) for t in (q, k, v))
ref = llsa.llsa_forward(q, k, v, pk, pv, llsa.hierarchical_topk(pq, pk, vc), vc).output
for dbg in (sys.argv[1:] or ["0"]):
    os.environ["LLSA_DBG"] = dbg
    ts_f, ts_b = [], []
    for it in range(12):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        h.forward(q, k, v, out)
        e1.record()
        h.backward(dO, q, k, v, out, *grads)
        e2.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts_f.append(e0.elapsed_time(e1))
            ts_b.append(e1.elapsed_time(e2))
    ts_f.sort()
    ts_b.sort()
    d = (out - ref).abs().max().item()
    print(f"LLSA_DBG={dbg:>4}: forward {ts_f[len(ts_f) // 2]:.4f} ms  backward "
          f"{ts_b[len(ts_b) // 2]:.4f} ms  max|out - simt| {d:.3e}", flush=True)
