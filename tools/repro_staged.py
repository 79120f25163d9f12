"""Dev: staged C-ABI tensor-core path at C3 vs the handle (units from argv)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16615_b200 as llsa
units = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
L = 3 if n >= 65536 else 2
q, k, v, g = (torch.randn(units, n, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
cfg = llsa.LLSAConfig(n, 64, 16, 8, L, L)
vc = llsa.validate_config(cfg)
h = llsa.LLSAHandle(cfg, units)
o = h.forward(q, k, v); gr = h.backward(g, q, k, v, o); torch.cuda.synchronize()
pq, pk, pv = (llsa.build_pyramid(t, 16, L) for t in (q, k, v))
tables = llsa.hierarchical_topk(pq, pk, vc)
print("tables eq", torch.equal(tables.view(-1), h.view("tables").view(-1)), flush=True)
st = llsa.llsa_forward(q, k, v, pk, pv, tables, vc)
print("fwd eq", torch.equal(st.output, o), flush=True)
tr = llsa.transpose_all(tables, vc)
print("csc eq", torch.equal(tr[0].view(-1), h.view("csc_offsets").view(-1)),
      torch.equal(tr[1].view(-1), h.view("csc_flat").view(-1)), tr[0].shape, tr[1].shape, flush=True)
dq, dk, dv = llsa.llsa_backward(g, st, q, k, v, pk, pv, tables, tr, vc)
torch.cuda.synchronize()
print("bwd eq", torch.equal(dq, gr[0]), torch.equal(dk, gr[1]), torch.equal(dv, gr[2]), flush=True)
