"""Fused row operators of the decoder block (csrc/model_ops.cu, row_pipe.cu)
against plain PyTorch fp32 references of the same op: RMSNorm + feature
gathers, SwiGLU through composed index maps, RoPE after the output scatter,
residual scatter-add, feature permutation -- forward and backward."""

import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(8192, 2048, 5632), (300, 512, 1408), (1, 256, 768), (77, 1024, 2816)]


@pytest.fixture
def N():
    from paper_2603_05500_b200 import _native as N

    return N


def _bf(t):
    return t.to(torch.bfloat16)


def _close(got, ref, tol=1e-2):
    err = (got.float() - ref.float()).abs().max().item()
    assert err <= tol * max(1.0, ref.float().abs().max().item()), err


def _perm(n, g):
    return torch.randperm(n, generator=g).int().cuda()


@pytest.mark.parametrize("T,d,f", SHAPES)
def test_permute_cols_exact(N, T, d, f):
    from paper_2603_05500_b200.trainer import _permute_cols

    g = torch.Generator().manual_seed(T + d)
    for dim in (d, f):
        x = _bf(torch.randn(T, dim)).cuda()
        idx = _perm(dim, g)
        assert torch.equal(_permute_cols(x, idx), x[:, idx.long()])


@pytest.mark.parametrize("T,d,f", SHAPES)
@pytest.mark.parametrize("K", [1, 2, 3])
def test_rmsnorm_gather_fwd_bwd(N, T, d, f, K):
    from paper_2603_05500_b200.trainer import _RMSNormGather

    g = torch.Generator().manual_seed(K * 7 + T)
    h = _bf(torch.randn(T, d)).cuda()
    w = (1 + 0.1 * torch.randn(d)).cuda()
    fwds = [_perm(d, g) for _ in range(K)]
    invs = [torch.argsort(p.long()).int() for p in fwds]
    hh = h.clone().requires_grad_(True)
    ww = w.clone().requires_grad_(True)
    outs = _RMSNormGather.apply(hh, ww, fwds, invs)
    # reference in fp32
    hr = h.float().clone().requires_grad_(True)
    wr = w.clone().requires_grad_(True)
    y = hr * torch.rsqrt(hr.pow(2).mean(-1, keepdim=True) + 1e-6) * wr
    refs = [y[:, p.long()] for p in fwds] + [hr]
    for o, r in zip(outs, refs):
        _close(o, r)
    dus = [_bf(torch.randn(T, d)).cuda() for _ in range(K + 1)]
    torch.autograd.backward(outs, dus)
    torch.autograd.backward(refs, [u.float() for u in dus])
    _close(hh.grad, hr.grad, 2e-2)
    _close(ww.grad, wr.grad, 2e-2)


@pytest.mark.parametrize("T,d,f", SHAPES)
def test_swiglu_gather_fwd_bwd(N, T, d, f):
    from paper_2603_05500_b200.trainer import _SwiGLUGather

    g = torch.Generator().manual_seed(f + T)
    fg, fu, fd = _perm(f, g).long(), _perm(f, g).long(), _perm(f, g).long()
    ig, iu, idn = torch.argsort(fg), torch.argsort(fu), torch.argsort(fd)
    maps = {"cg": ig[fd], "cu": iu[fd], "A": idn[fg], "B": iu[fg], "C": idn[fu], "D": ig[fu]}
    maps = {k: v.int().contiguous() for k, v in maps.items()}
    vg = _bf(torch.randn(T, f)).cuda()
    vu = _bf(torch.randn(T, f)).cuda()
    a, b = vg.clone().requires_grad_(True), vu.clone().requires_grad_(True)
    out = _SwiGLUGather.apply(a, b, maps)
    ar, br = vg.float().clone().requires_grad_(True), vu.float().clone().requires_grad_(True)
    zg, zu = ar[:, ig], br[:, iu]          # output scatters of gate / up
    ref = (torch.nn.functional.silu(zg) * zu)[:, fd]  # input gather of down
    _close(out, ref)
    du = _bf(torch.randn(T, f)).cuda()
    out.backward(du)
    ref.backward(du.float())
    _close(a.grad, ar.grad, 2e-2)
    _close(b.grad, br.grad, 2e-2)


@pytest.mark.parametrize("T,d,f", [(8192, 2048, 0), (512, 1024, 0), (64, 512, 0)])
def test_rope_scatter_fwd_bwd(N, T, d, f):
    from paper_2603_05500_b200.trainer import _RopeScatter

    S = 256 if T % 256 == 0 else 64
    hd = 64
    H = d // hd
    g = torch.Generator().manual_seed(d + T)
    fwd = _perm(d, g)
    inv = torch.argsort(fwd.long()).int()
    ang = torch.outer(torch.arange(S).float(), 1.0 / (10000 ** (torch.arange(0, hd, 2).float() / hd))).cuda()
    cos, sin = ang.cos().contiguous(), ang.sin().contiguous()
    v = _bf(torch.randn(T, d)).cuda()
    vv = v.clone().requires_grad_(True)
    out = _RopeScatter.apply(vv, inv, fwd, cos, sin, S, H, hd)
    vr = v.float().clone().requires_grad_(True)
    z = vr[:, inv.long()].view(T // S, S, H, hd)
    x1, x2 = z[..., : hd // 2], z[..., hd // 2:]
    c, s = cos.view(1, S, 1, hd // 2), sin.view(1, S, 1, hd // 2)
    ref = torch.cat((x1 * c - x2 * s, x2 * c + x1 * s), -1).reshape(T, d)
    _close(out, ref)
    dout = _bf(torch.randn(T, d)).cuda()
    out.backward(dout)
    ref.backward(dout.float())
    _close(vv.grad, vr.grad, 2e-2)


@pytest.mark.parametrize("T,d,f", SHAPES)
def test_scatter_add(N, T, d, f):
    from paper_2603_05500_b200.trainer import _ScatterAdd

    g = torch.Generator().manual_seed(d * 3 + T)
    fwd = _perm(d, g)
    inv = torch.argsort(fwd.long()).int()
    h = _bf(torch.randn(T, d)).cuda()
    v = _bf(torch.randn(T, d)).cuda()
    out = _ScatterAdd.apply(h, v, inv, fwd)
    _close(out, h.float() + v.float()[:, inv.long()], 1e-2)


@pytest.mark.parametrize("T,V", [(8192, 32000), (37, 64), (1, 128)])
def test_fused_cross_entropy(N, T, V):
    """Fused bf16 cross-entropy head vs torch's fp32 cross_entropy."""
    from paper_2603_05500_b200.trainer import _CrossEntropy

    g = torch.Generator().manual_seed(T + V)
    logits = (3 * torch.randn(T, V, generator=g)).to(torch.bfloat16).cuda()
    tgt = torch.randint(0, V, (T,), generator=g).cuda()
    a = logits.clone().requires_grad_(True)
    loss = _CrossEntropy.apply(a, tgt)
    r = logits.float().clone().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(r, tgt)
    assert abs(loss.item() - ref.item()) <= 1e-5 * max(1.0, abs(ref.item()))
    (2.0 * loss).backward()
    (2.0 * ref).backward()
    _close(a.grad, r.grad, 1e-2)


@pytest.mark.parametrize("T,V,d", [(8192, 32000, 2048), (300, 50, 512), (7, 3, 256)])
def test_embedding_fwd_bwd(N, T, V, d):
    """Fused embedding (gather + bf16 cast; sorted-run table gradient added in
    place) against F.embedding in fp32; repeated tokens included."""
    from paper_2603_05500_b200.trainer import _Embedding

    g = torch.Generator().manual_seed(T + V)
    tok = torch.randint(0, V, (T,), generator=g).cuda()
    table = torch.randn(V, d, generator=g).cuda()
    gbuf = torch.randn(V, d, generator=g).cuda()  # accumulates onto existing content
    base = gbuf.clone()
    t = table.clone().requires_grad_(True)
    out = _Embedding.apply(tok, t, gbuf)
    ref = torch.nn.functional.embedding(tok, table)
    assert torch.equal(out, ref.to(torch.bfloat16))
    dh = _bf(torch.randn(T, d, generator=g)).cuda()
    out.backward(dh)
    tr = table.clone().requires_grad_(True)
    torch.nn.functional.embedding(tok, tr).backward(dh.float())
    _close(gbuf - base, tr.grad, 1e-5)
    first = gbuf.clone()
    gbuf.copy_(base)
    _Embedding.apply(tok, t, gbuf).backward(dh)
    assert torch.equal(gbuf, first)  # deterministic: bitwise the same result again


@pytest.mark.parametrize("T,d,f", SHAPES)
def test_swiglu_16bit_maps_bitwise_equal_to_32bit(N, T, d, f):
    """The 16-bit-map SwiGLU kernels (half the index bytes) produce exactly
    the 32-bit-map results, forward and backward."""
    from paper_2603_05500_b200.trainer import _SwiGLUGather

    g = torch.Generator().manual_seed(f + T + 1)
    fg, fu, fd = _perm(f, g).long(), _perm(f, g).long(), _perm(f, g).long()
    ig, iu, idn = torch.argsort(fg), torch.argsort(fu), torch.argsort(fd)
    m32 = {"cg": ig[fd], "cu": iu[fd], "A": idn[fg], "B": iu[fg], "C": idn[fu], "D": ig[fu]}
    m32 = {k: v.int().contiguous() for k, v in m32.items()}
    m16 = dict(m32, **{k + "16": torch.from_numpy(v.cpu().numpy().astype("uint16")).cuda() for k, v in m32.items()})
    vg = _bf(torch.randn(T, f)).cuda()
    vu = _bf(torch.randn(T, f)).cuda()
    du = _bf(torch.randn(T, f)).cuda()
    res = []
    for maps in (m32, m16):
        a, b = vg.clone().requires_grad_(True), vu.clone().requires_grad_(True)
        out = _SwiGLUGather.apply(a, b, maps)
        out.backward(du)
        res.append((out, a.grad, b.grad))
    for x, y in zip(*res):
        assert torch.equal(x, y)
