"""Debug: runs one forward with LLSA_TRACE=1 and prints CTA 0's pipeline
timeline (role, tile, event, cycle offset).  Needs a build with the events
compiled in:  LLSA_NVCC_EXTRA=-DLLSA_TRACE_EVENTS python -m
paper_2512_16615_b200._build --force"""
import ctypes as C
import os
import sys

os.environ["LLSA_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402

units, n = 16, 65536
q, k, v = (torch.randn(units, n, 64, device="cuda").to(torch.bfloat16) for _ in range(3))
h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, 8, 3, 3), units)
out = torch.empty(units, n, 64, device="cuda")
lib = llsa._lib.load()
buf = (C.c_ulonglong * 8192)()
which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
if which == "bwd" and len(sys.argv) > 2:
    os.environ.update({"LLSA_KVF": "0"} if sys.argv[2] == "dq" else
                      {"LLSA_DQF": "0"} if sys.argv[2] == "kv" else {})
dO = torch.randn_like(q)
g = [torch.empty(units, n, 64, device="cuda") for _ in range(3)]
for it in range(2):
    if which == "fwd":
        lib.llsa_debug_trace(buf, 8192)  # reset
    h.forward(q, k, v, out)
    torch.cuda.synchronize()
    if which == "bwd":
        lib.llsa_debug_trace(buf, 8192)  # reset
        h.backward(dO, q, k, v, out, *g)
        torch.cuda.synchronize()
cnt = lib.llsa_debug_trace(buf, 8192)
ev = []
for idx, x in enumerate(buf[:cnt]):
    if x >> 63:
        ev.append((idx // 1024, (idx // 32) % 32, idx % 32, x & 0x7FFFFFFFFFFFFFFF))
t0 = min(e[3] for e in ev)
names = {0: "coars6", 1: "Kprod", 2: "Vprod", 3: "MMA", 4: "coarse", 5: "fine", 6: "coars4", 7: "coars5"} if which == "fwd" else {1: "prod", 3: "S", 4: "softmax", 5: "fine", 6: "dQ/dKV", 7: "c-epi"}
ev.sort(key=lambda e: e[3])
for r, t, e, c in ev:
    if t < int(os.environ.get("TRACE_TMAX", "8")):
        print(f"{c - t0:>9} {names.get(r, r):>6} tile {t:3d} ev {e}")
