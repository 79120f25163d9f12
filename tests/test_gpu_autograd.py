"""Autograd wrapper and dense-limit checks on the tensor-core path."""
import pytest
import torch

import paper_2512_16615_b200 as llsa

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _rel(a, b):
    return float((a.float() - b.float()).abs().max() / b.float().abs().max())


def test_full_selection_equals_dense_sdpa():
    # acceptance A2 (P/tests/acceptance.cpp:282-295) on the tensor-core path:
    # one level, every fine block selected → plain softmax attention.
    n = 1024
    torch.manual_seed(0)
    q, k, v, g = (torch.randn(2, 2, n, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
    attn = llsa.LLSAAttention(n, 64, 16, top_k=n // 16, levels=1, enrich_levels=0)
    qs, ks, vs = (t.detach().clone().requires_grad_(True) for t in (q, k, v))
    y = attn(qs, ks, vs)
    assert attn._handle.uses_tensor_cores
    y.backward(g)
    qd, kd, vd = (t.detach().float().requires_grad_(True) for t in (q, k, v))
    ref = torch.nn.functional.scaled_dot_product_attention(qd, kd, vd, scale=0.125)
    ref.backward(g.float())
    assert _rel(y, ref) < 2e-2
    for a, b in ((qs.grad, qd.grad), (ks.grad, kd.grad), (vs.grad, vd.grad)):
        assert _rel(a, b) < 2e-2


def test_autograd_matches_handle_and_guards_staleness(deterministic):
    n = 4096
    q, k, v, g = (torch.randn(1, 2, n, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
    attn = llsa.LLSAAttention(n)
    qs, ks, vs = (t.clone().requires_grad_(True) for t in (q, k, v))
    y = attn(qs, ks, vs)
    y.backward(g)
    h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, 8, 2, 2), 2)
    out = h.forward(q.view(2, n, 64), k.view(2, n, 64), v.view(2, n, 64))
    dq, dk, dv = h.backward(g.view(2, n, 64), q.view(2, n, 64), k.view(2, n, 64),
                            v.view(2, n, 64), out)
    assert torch.equal(y.view(2, n, 64), out.to(torch.bfloat16))
    assert torch.equal(qs.grad.view(2, n, 64), dq.to(torch.bfloat16))
    assert torch.equal(vs.grad.view(2, n, 64), dv.to(torch.bfloat16))
    y1 = attn(qs, ks, vs)
    attn(qs, ks, vs)                      # a newer forward on the same layer
    with pytest.raises(llsa.StaleState):
        y1.backward(g)


def test_handle_bf16_outputs_are_rounded_fp32_outputs(deterministic):
    # llsa_handle_forward_ex / backward_ex with bf16 results: exactly the
    # fp32 results rounded to bf16 (RNE); a backward against any other output
    # buffer than the latest forward's raises StaleState
    n = 16384
    q, k, v, g = (torch.randn(2, n, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
    cfg = llsa.LLSAConfig(n, 64, 16, 8, 2, 2)
    h = llsa.LLSAHandle(cfg, 2)
    out32 = h.forward(q, k, v)
    grads32 = h.backward(g, q, k, v, out32)
    out16 = h.forward(q, k, v, out_dtype=torch.bfloat16)
    assert out16.dtype == torch.bfloat16
    assert torch.equal(out16, out32.to(torch.bfloat16))
    grads16 = h.backward(g, q, k, v, out16)
    for a, b in zip(grads16, grads32):
        assert a.dtype == torch.bfloat16 and torch.equal(a, b.to(torch.bfloat16))
    with pytest.raises(llsa.StaleState):
        h.backward(g, q, k, v, out16.clone())
    with pytest.raises(llsa.ShapeMismatch):
        h.forward(q[:1], k[:1], v[:1])
    with pytest.raises(llsa.ArgumentError):
        h.forward(q.half(), k.half(), v.half())


@pytest.mark.parametrize("n,L,K", [(65536, 3, 16), (65536, 3, 8)])
def test_bf16_outputs_equal_rounded_fp32_on_multi_pass_forward(deterministic, n, L, K):
    # K = 16 at L = 3: 33 coarse entries run as two tcgen05 forward passes; the
    # bf16 copy is written by the final pass's epilogue only
    q, k, v, g = (torch.randn(2, n, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
    h = llsa.LLSAHandle(llsa.LLSAConfig(n, 64, 16, K, L, L), 2)
    out32 = h.forward(q, k, v)
    grads32 = h.backward(g, q, k, v, out32)
    out16 = h.forward(q, k, v, out_dtype=torch.bfloat16)
    assert torch.equal(out16, out32.to(torch.bfloat16))
    grads16 = h.backward(g, q, k, v, out16)
    for a, b in zip(grads16, grads32):
        assert torch.equal(a, b.to(torch.bfloat16))
    llsa.sync_status()
