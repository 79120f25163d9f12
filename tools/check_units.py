"""Debug: single-unit handle forward vs the SIMT path; error statistics."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402
from oracle import rel_err  # noqa: E402

n = 65536
for seed in (0, 7):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(1, n, 64, device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(3))
    lc = llsa.LLSAConfig(n, 64, 16, 8, 3, 3)
    vc = llsa.validate_config(lc)
    h = llsa.LLSAHandle(lc, 1, torch.bfloat16)
    out = h.forward(q, k, v).clone()
    pq, pk, pv = (llsa.build_pyramid(t, 16, 3) for t in (q, k, v))
    tab = llsa.hierarchical_topk(pq, pk, vc)
    simt = llsa.llsa_forward(q, k, v, pk, pv, tab, vc).output
    a, b = out[0].cpu().numpy(), simt[0].cpu().numpy()
    e = rel_err(a, b)
    d = np.abs(a - b)
    r, c = np.unravel_index(np.argmax(d), d.shape)
    rows = np.argsort(-d.max(axis=1))[:8]
    print(f"seed {seed}: {e} max|ref| {np.abs(b).max():.3f} worst ({r},{c}) got {a[r, c]:.4f} "
          f"want {b[r, c]:.4f}; worst rows {rows.tolist()} row errs {d.max(axis=1)[rows].round(3).tolist()}")
    print("  rows with err > 0.05:", int((d.max(axis=1) > 0.05).sum()), "of", n)
