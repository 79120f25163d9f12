"""Dev: one handle forward + backward for compute-sanitizer.
Usage: python tools/memcheck_c3.py [n] [levels] [units] [top_k] [enrich_levels]
(default C3, 1 unit, K = 8, L_e = L)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
L = int(sys.argv[2]) if len(sys.argv) > 2 else 3
units = int(sys.argv[3]) if len(sys.argv) > 3 else 1
K = int(sys.argv[4]) if len(sys.argv) > 4 else 8
Le = int(sys.argv[5]) if len(sys.argv) > 5 else L
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v, dO = (torch.randn(units, n, 64, device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(4))
h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, K, L, Le), units, torch.bfloat16)
out = h.forward(q, k, v)
dq, dk, dv = h.backward(dO, q, k, v, out)
llsa.sync_status()
torch.cuda.synchronize()
print(f"n={n} L={L} units={units} K={K} Le={Le} ok", float(out.abs().mean()), float(dq.abs().mean()), float(dk.abs().mean()))
