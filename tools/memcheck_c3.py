"""Dev: one C3-size handle forward + backward (1 unit) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402

n = 65536
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v, dO = (torch.randn(1, n, 64, device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(4))
h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, 8, 3, 3), 1, torch.bfloat16)
out = h.forward(q, k, v)
dq, dk, dv = h.backward(dO, q, k, v, out)
llsa.sync_status()
torch.cuda.synchronize()
print("c3 ok", float(out.abs().mean()), float(dq.abs().mean()), float(dk.abs().mean()))
