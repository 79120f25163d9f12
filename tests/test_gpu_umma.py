"""tcgen05 primitive self-test (csrc/selftest/umma_selftest.cu): one
128 x N x 64 bf16 GEMM through K-major / MN-major SW128 descriptors with the
accumulator in TMEM, against torch."""
import ctypes as C
import os

import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                  "paper_2512_16615_b200", "build", "libllsa_umma_selftest.so")


@pytest.mark.parametrize("n,lbo", [(64, 8192), (128, 8192), (80, 8192), (80, 24576),
                                   (128, 16384)])
@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_umma_gemm(n, lbo, a_mn, b_mn):
    lib = C.CDLL(SO)
    torch.manual_seed(n + 2 * a_mn + b_mn)
    A = torch.randn(128, 64, device="cuda").to(torch.bfloat16)   # [m][k]
    B = torch.randn(64, n, device="cuda").to(torch.bfloat16)     # [k][n]
    a_in = A.t().contiguous() if a_mn else A                      # MN-major: [k][m]
    b_in = B.contiguous() if b_mn else B.t().contiguous()         # K-major: [n][k]
    d = torch.empty(128, n, device="cuda")
    rc = lib.llsa_umma_selftest(C.c_void_p(a_in.data_ptr()), C.c_void_p(b_in.data_ptr()),
                                C.c_void_p(d.data_ptr()), n, a_mn, b_mn, lbo,
                                C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    ref = A.float() @ B.float()
    assert torch.allclose(d, ref, atol=1e-3, rtol=1e-3), (d - ref).abs().max().item()


def test_tmem_store_from_mma_fragments():
    # tcgen05.st.16x256b writes 16 lanes x 8 columns in the m16n8 accumulator
    # layout (the fine warps stage partial results in TMEM this way)
    lib = C.CDLL(SO)
    out = torch.zeros(128, 32, device="cuda")
    assert lib.llsa_umma_frag_selftest(C.c_void_p(out.data_ptr()),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    torch.cuda.synchronize()
    lane = torch.arange(128, device="cuda").float()[:, None]
    col = torch.arange(32, device="cuda").float()[None, :]
    assert torch.equal(out, lane * 100 + col)
