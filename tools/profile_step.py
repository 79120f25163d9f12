"""Runs `--steps` LLSA fwd+bwd steps of the bench workload for profilers
(ncu).  Not a benchmark: numbers printed under a profiler are meaningless."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--levels", type=int, default=3)
ap.add_argument("--units", type=int, default=16)
a = ap.parse_args()
shape = (a.units, a.n, 64)
q, k, v, dO = (torch.randn(shape, device="cuda").to(torch.bfloat16) for _ in range(4))
h = llsa.LLSAHandle(llsa.LLSAConfig(a.n, 64, 16, 8, a.levels, a.levels), a.units)
out = torch.empty(shape, device="cuda")
g = [torch.empty(shape, device="cuda") for _ in range(3)]
for _ in range(a.steps):
    h.forward(q, k, v, out)
    h.backward(dO, q, k, v, out, *g)
torch.cuda.synchronize()
llsa.sync_status()
print("done", h.uses_tensor_cores)
