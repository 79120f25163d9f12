"""2-D reordering (SURVEY.md §8(f) row 3, P/src/reorder2d.cpp): the host curve
from the C ABI against the reference library and the C oracle (CPU), and the
GPU gather / gather-fused pyramid against the oracle (bit-exact)."""
import numpy as np
import pytest
import torch

import paper_2512_16615_b200 as llsa
from oracle import REF_SO, OracleC, Reference

SHAPES = [(1, 1, 4), (2, 2, 4), (4, 4, 4), (8, 8, 4), (12, 8, 4), (64, 128, 16),
          (48, 48, 16), (256, 256, 16), (96, 64, 4), (27, 27, 9)]
BAD = [((4, 4, 8), llsa.NotSquareBlock), ((4, 4, 2), llsa.NotSquareBlock),
       ((4, 4, 0), llsa.NotSquareBlock), ((3, 5, 4), llsa.DivisibilityError),
       ((0, 4, 4), llsa.DivisibilityError), ((4, 0, 16), llsa.DivisibilityError)]


@pytest.mark.parametrize("h,w,b", SHAPES)
def test_curve_matches_oracle_and_reference(h, w, b):
    fwd, inv = llsa.build_reorder(h, w, b)
    code, fo, io = OracleC().build_reorder(h, w, b)
    assert code == 0
    assert np.array_equal(fwd, fo) and np.array_equal(inv, io)
    assert np.array_equal(np.sort(fwd), np.arange(h * w))        # a bijection
    assert np.array_equal(inv[fwd], np.arange(h * w))
    import os
    if os.path.exists(REF_SO[32]):
        code, fr, ir = Reference(32).build_reorder(h, w, b)
        assert code == 0 and np.array_equal(fwd, fr) and np.array_equal(inv, ir)


@pytest.mark.parametrize("args,exc", BAD)
def test_invalid_geometry_raises_the_reference_type(args, exc):
    with pytest.raises(exc):
        llsa.build_reorder(*args)
    assert OracleC().build_reorder(*args)[0] == exc.code


def test_blocks_are_spatial_patches():
    # every aligned run of B positions is one s x s patch (reorder2d.hpp:21-26)
    h = w = 64
    fwd, _ = llsa.build_reorder(h, w, 16)
    ys, xs = fwd // w, fwd % w
    for start in range(0, h * w, 16):
        y, x = ys[start:start + 16], xs[start:start + 16]
        assert y.max() - y.min() == 3 and x.max() - x.min() == 3


gpu = pytest.mark.gpu
needs_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


@gpu
@needs_cuda
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d", [64, 6])
def test_apply_permutation_gathers_rows(dtype, d):
    h = w = 32
    fwd, inv = llsa.build_reorder(h, w, 16)
    x = torch.randn(3, h * w, d, device="cuda").to(dtype)
    f = torch.from_numpy(fwd.astype(np.int64)).cuda()
    i = torch.from_numpy(inv.astype(np.int64)).cuda()
    y = llsa.apply_permutation(x, f)
    llsa.sync_status()
    assert torch.equal(y, x[:, f])
    assert torch.equal(llsa.apply_permutation(y, i), x)          # Inverse undoes Forward


@gpu
@needs_cuda
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_pyramid_of_reordered_image_is_fused_gather_bit_exact(dtype):
    h = w = 64
    n, B, L = h * w, 16, 2
    fwd, _ = llsa.build_reorder(h, w, B)
    x = torch.randn(2, n, 64, device="cuda").to(dtype)
    f = torch.from_numpy(fwd.astype(np.int64)).cuda()
    got = llsa.build_pyramid_permuted(x, f, B, L)
    ref = llsa.build_pyramid(x[:, f].contiguous(), B, L)
    llsa.sync_status()
    assert torch.equal(got, ref)
    # ... and the oracle agrees (pooling of the gathered rows, pyramid.cpp:31-37)
    oc = OracleC()
    for u in range(2):
        xs = x[u].float().cpu().numpy()[fwd]
        want = oc.build_pyramid(xs, B, L).reshape(-1, 64)
        assert np.array_equal(got[u].cpu().numpy(), want)


@gpu
@needs_cuda
def test_reordered_pooling_equals_spatial_pooling():
    # the paper's claim (acceptance.cpp:307-386): pooling the reordered
    # sequence by B = s^2 is s x s average pooling of the image
    h = w = 64
    fwd, inv = llsa.build_reorder(h, w, 16)
    img = torch.randn(1, h * w, 64, device="cuda")
    pyr = llsa.build_pyramid_permuted(img, torch.from_numpy(fwd.astype(np.int64)).cuda(), 16, 1)
    pooled = torch.nn.functional.avg_pool2d(img.view(1, h, w, 64).permute(0, 3, 1, 2), 4)
    half_fwd, _ = llsa.build_reorder(h // 4, w // 4, 16)
    spatial = pooled.permute(0, 2, 3, 1).reshape(1, (h // 4) * (w // 4), 64)[:, half_fwd]
    assert torch.allclose(pyr, spatial, atol=1e-5, rtol=1e-5)
