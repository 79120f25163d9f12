"""torch.autograd wrapper around the fused LLSA path (the DiT caller of the
paper's training setting).

    attn = LLSAAttention(n=65536, d=64, heads=16)   # one handle per layer
    y = attn(q, k, v)            # q, k, v: [batch, heads, n, 64] bf16, CUDA
    y.float().sum().backward()

Forward = compress → select → sparse attention (tensor cores for d=64,
B=16, bf16); backward = CSR→CSC transpose → mask-free dq/dk/dv.  Top-K
indices carry no gradient (attention_grad.hpp:39-40).  The handle keeps the
selection and softmax statistics of its latest forward; a backward against an
older forward raises StaleState, like the reference's checksum guard
(attention_grad.cpp:213-216).
"""
from __future__ import annotations

import torch

from ._lib import StaleState
from .ops import LLSAConfig, LLSAHandle


class _LLSAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, module):
        units = q.shape[0] * q.shape[1]
        h = module._handle_for(units, q)
        x = [t.reshape(units, t.shape[-2], t.shape[-1]).contiguous() for t in (q, k, v)]
        # outputs in the input dtype straight from the handle (bf16 mode keeps
        # the fp32 O the backward needs inside the handle)
        out = h.forward(*x, out_dtype=q.dtype)
        module._generation += 1
        ctx.module, ctx.generation, ctx.shape = module, module._generation, q.shape
        ctx.save_for_backward(*x, out)
        return out.view(q.shape)

    @staticmethod
    def backward(ctx, grad):
        q, k, v, out = ctx.saved_tensors
        m = ctx.module
        if ctx.generation != m._generation:
            raise StaleState("LLSA backward after a newer forward on the same layer")
        g = grad.reshape(out.shape).to(q.dtype).contiguous()
        dq, dk, dv = m._handle.backward(g, q, k, v, out)
        shape = ctx.shape
        return dq.view(shape), dk.view(shape), dv.view(shape), None


class LLSAAttention(torch.nn.Module):
    """Log-linear sparse attention over [batch, heads, n, d] tensors."""

    def __init__(self, n: int, d: int = 64, block_size: int = 16, top_k: int = 8,
                 levels: int | None = None, enrich_levels: int | None = None,
                 softmax_scale: float = 0.0, reweight_mode: int = 0):
        super().__init__()
        from .ops import max_levels
        L = levels if levels is not None else max_levels(n, block_size)
        self.cfg = LLSAConfig(n, d, block_size, top_k, L,
                              L if enrich_levels is None else enrich_levels, softmax_scale,
                              reweight_mode, True)
        self._handle: LLSAHandle | None = None
        self._generation = 0

    def _handle_for(self, units: int, like: torch.Tensor) -> LLSAHandle:
        h = self._handle
        if h is None or h.units != units or h.dtype != like.dtype or \
                h.device != like.device:
            with torch.cuda.device(like.device):
                self._handle = LLSAHandle(self.cfg, units, like.dtype)
        return self._handle

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        if q.dim() != 4 or q.shape != k.shape or q.shape != v.shape:
            raise ValueError("q, k, v must share shape [batch, heads, n, d]")
        if tuple(q.shape[-2:]) != (self.cfg.n, self.cfg.d):
            raise ValueError(f"q, k, v must be [batch, heads, {self.cfg.n}, {self.cfg.d}] for "
                             f"this layer, got {tuple(q.shape)}")
        if q.dtype not in (torch.bfloat16, torch.float32) or k.dtype != q.dtype or \
                v.dtype != q.dtype:
            raise ValueError("q, k, v must all be bfloat16 or all float32 "
                             f"(got {q.dtype}, {k.dtype}, {v.dtype})")
        return _LLSAFunction.apply(q, k, v, self)
