"""tcgen05/TMA GEMM (BF16 in, fp32 TMEM accumulation) against a torch fp32
reference of the same product, through the C ABI (poetx_matmul)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def setp(packed, a):
    """Write values into a layer's packed parameters in place, whether they
    are host numpy arrays (numpy-constructed layer) or device tensors."""
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    if isinstance(packed, np.ndarray):
        packed[...] = np.asarray(a, dtype=packed.dtype)
    else:
        packed.copy_(torch.from_numpy(np.ascontiguousarray(a)).to(packed))


def host(a):
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


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


@pytest.mark.parametrize("M,Nn,K", [(256, 256, 64), (512, 768, 320), (8192, 5632, 2048), (8192, 2048, 5632)])
@pytest.mark.parametrize("trans_b", [0, 1])
@pytest.mark.parametrize("pair", [1, 0], ids=["cta_pair", "single_cta"])
def test_tc_gemm_pair_and_single_cta(N, M, Nn, K, trans_b, pair):
    """The CTA-pair (cta_group::2) kernel and the single-CTA kernel agree with
    the fp32 reference and with each other bit-for-bit (same K order)."""
    g = torch.Generator("cuda").manual_seed(7 * M + Nn + K)
    a = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn((Nn, K) if trans_b else (K, Nn), device="cuda", generator=g).to(torch.bfloat16)
    N.lib().poetx_set_gemm_pair_enabled(pair)
    try:
        c = matmul(N, a, b, trans_b)
        N.lib().poetx_set_gemm_pair_enabled(1 - pair)
        c2 = matmul(N, a, b, trans_b)
    finally:
        N.lib().poetx_set_gemm_pair_enabled(1)
    ref = a.float() @ (b.float().t() if trans_b else b.float())
    err = (c.float() - ref).abs().max().item()
    assert err <= 8e-3 * max(1.0, ref.abs().max().item()), err
    assert torch.equal(c, c2)


@pytest.mark.parametrize("b,nb,T", [(64, 8, 1024), (128, 6, 300), (256, 8, 8192), (256, 22, 512), (256, 3, 300),
                                    (256, 1, 64)])
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


@pytest.mark.parametrize("b,nb,scale", [(256, 12, 0.01), (128, 5, 0.02), (64, 9, 0.03)])
def test_tc_cnp_vs_oracle(N, b, nb, scale):
    """BF16 tensor-core CNP (forward G and packed backward) against the float64
    oracle restatement of cnp.py, at the bf16 tolerance 2e-2."""
    import numpy as np

    import paper_2603_05500_b200 as P
    from oracle import poetx_oracle as O

    r = np.random.default_rng(b + nb)
    packed = scale * r.standard_normal((nb, b * (b - 1) // 2))
    dg = r.standard_normal((nb, b, b))
    q = O.skew_from_packed(packed, b)
    g_ref, cache = O.cnp_forward(q, 3)
    dp_ref = O.packed_grad_from_skew_grad(O.cnp_backward(cache, dg, 3))
    g16, qq2, g32 = P.cnp_forward_tc(torch.from_numpy(packed).float().cuda(), b, want_fp32=True)
    for g in (g16, g32):
        err = np.abs(g.double().cpu().numpy() - g_ref).max()
        assert err <= 2e-2 * max(1.0, np.abs(g_ref).max()), err
    # fp32 G keeps the fine structure: G - I against the oracle
    d_err = np.abs((g32.double().cpu().numpy() - g_ref)).max() / np.abs(g_ref - np.eye(b)).max()
    assert d_err <= 2e-2, d_err
    dp = P.cnp_backward_tc(qq2, torch.from_numpy(dg).float().cuda())
    err = np.abs(dp.double().cpu().numpy() - dp_ref).max()
    assert err <= 2e-2 * max(1.0, np.abs(dp_ref).max()), err
    acc = P.cnp_backward_tc(qq2, torch.from_numpy(dg).float().cuda(), out=dp.clone(), accumulate=True)
    assert torch.allclose(acc, 2 * dp, rtol=1e-6, atol=1e-6)


def test_layer_backward_dg_matches_packed(N):
    """poetx_layer_backward_dg + batched TC CNP backward == per-layer backward."""
    import paper_2603_05500_b200 as P

    m, n, b, T = 512, 768, 256, 640
    base = torch.randn((m, n), device="cuda").div(m ** 0.5).bfloat16()
    layer = P.PoetLinearLayer(base, b, P.Rng(3))
    layer.q_r.packed.normal_(0, 0.01)
    layer.q_p.packed.normal_(0, 0.01)
    x = torch.randn((T, m), device="cuda").bfloat16()
    dz = torch.randn((T, n), device="cuda").bfloat16()
    z, cache = layer.forward(x)
    g_ref = layer.backward(cache, dz)
    # dG path
    f = cache.factors
    dgr = torch.empty((m // b, b, b), device="cuda")
    dgp = torch.empty((n // b, b, b), device="cuda")
    dx = torch.empty_like(x)
    d = layer._desc()
    ws, wsb = N.workspace(N.lib().poetx_layer_workspace_bytes(d, T))
    N.call("poetx_layer_backward_dg", d, f.struct, T, x.data_ptr(), dz.data_ptr(), cache.saved_mm2.data_ptr(),
           dx.data_ptr(), dgr.data_ptr(), dgp.data_ptr(), 0, 0, ws, wsb, N.stream_ptr())
    assert torch.equal(dx, g_ref.x)
    _, qq2r, _ = P.cnp_forward_tc(f.packed_r, b)
    _, qq2p, _ = P.cnp_forward_tc(f.packed_p, b)
    gr = P.cnp_backward_tc(qq2r, dgr)
    gp = P.cnp_backward_tc(qq2p, dgp)
    for got, want in ((gr, g_ref.q_r), (gp, g_ref.q_p)):
        err = (got - want).abs().max().item()
        assert err <= 2e-2 * max(1.0, want.abs().max().item()), err


@pytest.mark.parametrize("K", [64, 192, 256, 320, 448, 512, 640, 2048])
@pytest.mark.parametrize("ms", [1, 2])
def test_pair_gemm_k_edges_of_the_tile_head_and_tail(N, K, ms):
    """512-row pair tiles run the first min(K blocks, stages) K blocks on
    sub-tile 0 first and the last up to 3 on sub-tile 0 first again
    (POETX_PAIR_TAIL): K from one 64-wide block (head only) through
    head + 1, head + tail with no middle, and long middles, against torch
    fp32; 256-row tiles alongside.  Several tiles per CTA pair (M = 8192 on
    74 pairs) so the head / tail hand-over between tiles is exercised."""
    M, Nn = 8192, 1024
    g = torch.Generator("cuda").manual_seed(K * 7 + ms)
    a = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn((K, Nn), device="cuda", generator=g).to(torch.bfloat16)
    N.lib().poetx_set_gemm_pair_ms(ms)
    try:
        c = matmul(N, a, b, 0)
        torch.cuda.synchronize()
    finally:
        N.lib().poetx_set_gemm_pair_ms(0)
    ref = a.float() @ b.float()
    err = float((c.float() - ref).abs().max() / ref.abs().max())
    assert err < 1e-2, err
