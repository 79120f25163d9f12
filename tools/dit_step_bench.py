"""A DiT-style transformer block's training step with LLSA attention
(the paper's setting, §4) against the same
block with dense attention (torch SDPA, flash/cuDNN).

Block (bf16, pre-norm): x + Wo·Attn(LN(x)·Wqkv) then x + MLP(LN(x)), MLP
1024 → 4096 → 1024 (GELU); 16 heads of d = 64; N = 65536 tokens (256² px),
batch 1.  LLSA: `LLSAAttention(n=65536)` (B = 16, K = 8, L = 3, L_e = 3);
q, k, v in the token order the block produces (an image sequence would be
laid out by the 2-D hierarchical curve once, llsa.build_reorder).  One step =
forward + backward of the block (loss = mean of the output), timed with CUDA
events after warm-up; the attention call alone is timed the same way.
Random-init weights, synthetic N(0,1) input.

  python tools/dit_step_bench.py > profiles/r2_dit_step.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import paper_2512_16615_b200 as llsa  # noqa: E402

N, C, H, D = 65536, 1024, 16, 64


class Block(torch.nn.Module):
    def __init__(self, attn: str):
        super().__init__()
        self.ln1 = torch.nn.LayerNorm(C)
        self.qkv = torch.nn.Linear(C, 3 * C)
        self.proj = torch.nn.Linear(C, C)
        self.ln2 = torch.nn.LayerNorm(C)
        self.fc1 = torch.nn.Linear(C, 4 * C)
        self.fc2 = torch.nn.Linear(4 * C, C)
        self.kind = attn
        self.llsa = llsa.LLSAAttention(n=N, d=D) if attn == "llsa" else None

    def attend(self, q, k, v):
        if self.kind == "llsa":
            return self.llsa(q, k, v)
        return F.scaled_dot_product_attention(q, k, v)

    def forward(self, x):
        b = x.shape[0]
        qkv = self.qkv(self.ln1(x)).view(b, N, 3, H, D).permute(2, 0, 3, 1, 4)
        q, k, v = (t.contiguous() for t in qkv)
        a = self.attend(q, k, v).transpose(1, 2).reshape(b, N, C)
        x = x + self.proj(a)
        return x + self.fc2(F.gelu(self.fc1(self.ln2(x))))


def timed(fn, steps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    torch.manual_seed(0)
    dev = "cuda"
    res = {"block": f"pre-norm DiT block, N={N}, C={C}, {H} heads x d={D}, MLP 4x, bf16, "
                    "batch 1", "rows": {}}
    x = torch.randn(1, N, C, device=dev, dtype=torch.bfloat16)
    for kind in ("llsa", "dense_sdpa"):
        blk = Block(kind).to(dev, torch.bfloat16)

        def step():
            blk.zero_grad(set_to_none=True)
            xr = x.detach().requires_grad_(True)
            blk(xr).float().mean().backward()

        q, k, v = (torch.randn(1, H, N, D, device=dev, dtype=torch.bfloat16,
                               requires_grad=True) for _ in range(3))
        g = torch.randn(1, H, N, D, device=dev, dtype=torch.bfloat16)

        def attn_step():
            blk.attend(q, k, v).backward(g)

        step_ms = timed(step)
        attn_ms = timed(attn_step)
        res["rows"][kind] = {"step_ms": step_ms, "attention_fwd_bwd_ms": attn_ms,
                             "attention_share": attn_ms / step_ms}
        print(json.dumps({kind: res["rows"][kind]}), file=sys.stderr)
        del blk
        torch.cuda.empty_cache()
    r = res["rows"]
    res["speedup_step"] = r["dense_sdpa"]["step_ms"] / r["llsa"]["step_ms"]
    res["speedup_attention"] = r["dense_sdpa"]["attention_fwd_bwd_ms"] / \
        r["llsa"]["attention_fwd_bwd_ms"]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
