"""tcgen05/TMA GEMM (BF16 in, fp32 TMEM accumulation) against a torch fp32
reference of the same product, through the C ABI (poetx_matmul)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    from paper_2603_05500_b200 import _native as N

    N.lib()
    assert N.lib().poetx_tc_enabled() == 1
    return N


def matmul(N, a, b, trans_b):
    M, K = a.shape
    Nn = b.shape[0] if trans_b else b.shape[1]
    c = torch.empty((M, Nn), dtype=torch.bfloat16, device="cuda")
    N.call("poetx_matmul", N.BF16, M, Nn, K, a.data_ptr(), K, 0, b.data_ptr(), b.shape[1], int(trans_b),
           c.data_ptr(), Nn, 0, N.stream_ptr())
    return c


@pytest.mark.parametrize("M,Nn,K", [(128, 256, 64), (256, 512, 128), (300, 544, 1000), (1024, 768, 2048),
                                    (8192, 2048, 2048)])
@pytest.mark.parametrize("trans_b", [0, 1])
def test_tc_gemm_matches_fp32_reference(N, M, Nn, K, trans_b):
    g = torch.Generator("cuda").manual_seed(M + Nn + K)
    a = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn((Nn, K) if trans_b else (K, Nn), device="cuda", generator=g).to(torch.bfloat16)
    before = N.launch_count()
    c = matmul(N, a, b, trans_b)
    assert N.launch_count() == before + 1
    ref = a.float() @ (b.float().t() if trans_b else b.float())
    err = (c.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    # bf16 output rounding (2^-8 relative) dominates
    assert err <= 8e-3 * max(1.0, scale), (err, scale)


@pytest.mark.parametrize("b,nb,T", [(64, 8, 1024), (128, 6, 300), (256, 8, 8192), (256, 22, 512)])
@pytest.mark.parametrize("transpose", [False, True])
def test_tc_blockdiag_apply(N, b, nb, T, transpose):
    import paper_2603_05500_b200 as P

    g = torch.Generator("cuda").manual_seed(b + T)
    x = torch.randn((T, nb * b), device="cuda", generator=g).to(torch.bfloat16)
    G = (0.1 * torch.randn((nb, b, b), device="cuda", generator=g)).to(torch.bfloat16)
    y = P.apply_to_features(P.BlockDiagonalFactor(G), x, transpose=transpose)
    Gf = G.float().transpose(1, 2) if transpose else G.float()
    ref = torch.einsum("tsi,sij->tsj", x.float().view(T, nb, b), Gf).reshape(T, nb * b)
    err = (y.float() - ref).abs().max().item()
    assert err <= 8e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("b,nb,T", [(64, 8, 1024), (128, 3, 77), (256, 8, 8192), (256, 22, 520)])
def test_tc_segmented_outer(N, b, nb, T):
    import paper_2603_05500_b200 as P

    g = torch.Generator("cuda").manual_seed(b * T)
    x = torch.randn((T, nb * b), device="cuda", generator=g).to(torch.bfloat16)
    y = torch.randn((T, nb * b), device="cuda", generator=g).to(torch.bfloat16)
    out = P.segmented_outer(x, y, b)
    assert out.dtype == torch.float32
    ref = torch.einsum("tsi,tsj->sij", x.float().view(T, nb, b), y.float().view(T, nb, b))
    err = (out - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err
    # deterministic: bitwise identical on repeat
    assert torch.equal(out, P.segmented_outer(x, y, b))
