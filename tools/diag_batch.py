"""Dev: 128-unit handle vs one-unit handles in the ordered mode (which
tensor differs, by how much) and 128-unit run-to-run equality."""
import os
import sys

os.environ["LLSA_DETERMINISTIC"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402

a = [int(x) for x in sys.argv[1:]] + [None] * 5
units, n, L = a[0] or 128, a[1] or 65536, a[2] or 3
K, Le = a[3] or 8, a[4] if a[4] is not None else L
g = torch.Generator(device="cuda").manual_seed(44)
q, k, v, dO = (torch.randn(units, n, 64, device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(4))
lc = llsa.LLSAConfig(n, 64, 16, K, L, Le)
print(f"units={units} n={n} L={L} K={K} Le={Le}")
hm = llsa.LLSAHandle(lc, units, torch.bfloat16)
out = hm.forward(q, k, v, out_dtype=torch.bfloat16)
gr = hm.backward(dO, q, k, v, out)
gr = [x.clone() for x in gr]
out2 = hm.forward(q, k, v, out_dtype=torch.bfloat16)
gr2 = hm.backward(dO, q, k, v, out2)
print("rerun equal:", torch.equal(out, out2), [torch.equal(a, b) for a, b in zip(gr, gr2)])
h1 = llsa.LLSAHandle(lc, 1, torch.bfloat16)
bad = []
for u in range(units):
    sl = slice(u, u + 1)
    o1 = h1.forward(q[sl], k[sl], v[sl], out_dtype=torch.bfloat16)
    g1 = h1.backward(dO[sl], q[sl], k[sl], v[sl], o1)
    eq = [torch.equal(out[sl], o1)] + [torch.equal(a[sl], b) for a, b in zip(gr, g1)]
    if not all(eq):
        d = [float((a[sl].float() - b.float()).abs().max()) for a, b in zip(gr, g1)]
        bad.append((u, eq, d))
print("units differing:", len(bad), bad[:8])
llsa.sync_status()
