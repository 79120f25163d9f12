"""Diagnostic (test infrastructure): where do the tcgen05 path's errors vs the
compiled reference concentrate?  Prints per-row statistics for one config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_16615_b200 as llsa
from oracle import Config, Reference, unit_inputs, lse

def main(n, K, L, Le, mode=0):
    cfg = Config(n, 64, 16, K, L, Le, reweight_mode=mode)
    ref = Reference(32); ref.set_threads(os.cpu_count())
    q, k, v, dO = unit_inputs(cfg, 0, bf16=True, backend=ref)
    r = ref.run(cfg, q, k, v, dO)
    T = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)[None]
    h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, K, L, Le, reweight_mode=mode), 1, torch.bfloat16)
    out = h.forward(T(q), T(k), T(v)); dq, dk, dv = h.backward(T(dO), T(q), T(k), T(v), out)
    rm = h.view("row_max")[0].cpu().numpy(); rd = h.view("row_denom")[0].cpu().numpy()
    el = np.abs(lse(rm, rd) - lse(r.row_max, r.row_denom))
    print(f"cfg n={n} K={K} L={L} Le={Le} mode={mode}")
    print("LSE err: max %.3e  p99 %.3e  median %.3e" % (el.max(), np.percentile(el, 99), np.median(el)))
    idx = np.argsort(-el)[:8]
    for i in idx:
        print("  row %6d lse_ref %.4f lse_gpu %.4f  ref m %.4f d %.4f | gpu m %.4f d %.4f" % (
            i, lse(r.row_max, r.row_denom)[i], lse(rm, rd)[i], r.row_max[i], r.row_denom[i], rm[i], rd[i]))
    for name, g, w in (("out", out, r.out), ("dq", dq, r.dq), ("dk", dk, r.dk)):
        g = g[0].cpu().numpy().astype(np.float64); w = w.astype(np.float64)
        rn = np.linalg.norm(w, axis=1); en = np.linalg.norm(g - w, axis=1)
        rel = en / np.maximum(rn, 1e-30)
        bad = np.argsort(-rel)[:6]
        print(f"{name}: row-rel max {rel.max():.3e}, p99 {np.percentile(rel,99):.3e}; worst rows:")
        for i in bad:
            print("   row %6d rel %.3e |ref| %.3e |err| %.3e  ref denom %.4f  row-median|ref| %.3e" % (
                i, rel[i], rn[i], en[i], r.row_denom[i], np.median(rn)))

if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
