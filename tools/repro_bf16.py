"""Dev: handle bf16-output mode at C3 (units from argv) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16615_b200 as llsa
units = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
L = 3 if n >= 65536 else 2
q, k, v, g = (torch.randn(units, n, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, 8, L, L), units)
o = h.forward(q, k, v, out_dtype=torch.bfloat16); torch.cuda.synchronize(); print("fwd ok", flush=True)
gr = h.backward(g, q, k, v, o); torch.cuda.synchronize(); print("bwd ok", flush=True)
o32 = h.forward(q, k, v); gr32 = h.backward(g, q, k, v, o32); torch.cuda.synchronize()
print("equal", torch.equal(o, o32.bfloat16()), [torch.equal(a, b.bfloat16()) for a, b in zip(gr, gr32)])
