"""POET-XQ dequantization fused into the GEMM producer (
reference layer.py:188-210, quant.py:22-74).

The pair GEMM takes the frozen weight's int8 codes directly: warps of each
CTA turn a TMA-loaded int8 stage into the bf16 B operand (code * row scale,
ONE bf16 rounding).  That is exactly what the standalone dequantizer writes,
so every product must be BIT-IDENTICAL to dequantize + the bf16 GEMM:

* ``poetx_matmul_q8`` both ways (mm2 ``a . W``: scale per K row; adjoint
  ``a . W^T``: scale per N row), 256- and 512-row pair tiles;
* the forward weight fold ``bd(G_R) PM`` of a quantized layer
  (``poetx_layer_weight_fold``, grouped pair GEMM) against dequantize + the
  same fold of the bf16 weight;
* a quantized bf16 layer's forward / backward at b = 256 against a float64
  oracle at the bf16 tolerance, and a POET-XQ Llama trainer run with the
  fused path against the same run with ``POETX_Q8_GEMM=0`` (dequantize
  everywhere): bitwise equal losses and parameters.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def N():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2603_05500_b200 import _native as N

    N.lib()
    return N


def dequant(N, codes, scales):
    rows, cols = codes.shape
    out = torch.empty((rows, cols), dtype=torch.bfloat16, device="cuda")
    N.call("poetx_dequantize_rows", N.BF16, rows, cols, cols, codes.data_ptr(), scales.data_ptr(), None, None,
           out.data_ptr(), N.stream_ptr())
    return out


@pytest.mark.parametrize("M,Nn,K", [(256, 512, 768), (1024, 768, 512), (2048, 1024, 1024), (640, 256, 320)])
@pytest.mark.parametrize("transB", [0, 1])
def test_matmul_q8_bitwise_equal_to_dequantize_then_gemm(N, M, Nn, K, transB):
    g = torch.Generator(device="cuda").manual_seed(M + Nn + K + transB)
    a = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    rows, cols = (Nn, K) if transB else (K, Nn)
    codes = torch.randint(-127, 128, (rows, cols), device="cuda", generator=g, dtype=torch.int8)
    scales = torch.rand(rows, device="cuda", generator=g) * 0.02 + 1e-3
    w = dequant(N, codes, scales)
    want = torch.empty((M, Nn), dtype=torch.bfloat16, device="cuda")
    N.call("poetx_matmul", N.BF16, M, Nn, K, a.data_ptr(), K, 0, w.data_ptr(), cols, transB, want.data_ptr(), Nn, 0,
           N.stream_ptr())
    got = torch.empty_like(want)
    N.call("poetx_matmul_q8", M, Nn, K, a.data_ptr(), K, codes.data_ptr(), cols, transB, scales.data_ptr(),
           got.data_ptr(), Nn, N.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    ref = a.float() @ (w.float().t() if transB else w.float())
    assert float((got.float() - ref).abs().max()) <= 1e-2 * float(ref.abs().max())


def test_matmul_q8_rejects_untiled_shapes(N):
    from paper_2603_05500_b200.errors import ShapeError

    a = torch.zeros((128, 64), device="cuda", dtype=torch.bfloat16)
    codes = torch.zeros((64, 96), device="cuda", dtype=torch.int8)
    s = torch.ones(64, device="cuda")
    c = torch.empty((128, 96), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ShapeError):
        N.call("poetx_matmul_q8", 128, 96, 64, a.data_ptr(), 64, codes.data_ptr(), 96, 0, s.data_ptr(), c.data_ptr(),
               96, N.stream_ptr())


def _quant_layer(P, m, n, seed):
    r = np.random.default_rng(seed)
    base = torch.from_numpy(r.standard_normal((m, n)) / np.sqrt(m)).to(torch.bfloat16)
    lay = P.PoetLinearLayer(base, 256, P.Rng.keyed(seed, "q8"), variant="mem")
    lay.quantize_base()
    lay.q_r.packed.copy_(torch.from_numpy(0.01 * r.standard_normal(tuple(lay.q_r.packed.shape))))
    lay.q_p.packed.copy_(torch.from_numpy(0.01 * r.standard_normal(tuple(lay.q_p.packed.shape))))
    return lay, r


def test_quantized_weight_fold_bitwise(N):
    """bd(G_R) . PM with PM as int8 codes in the grouped pair GEMM == the same
    fold of the dequantized bf16 weight."""
    m, n, b = 1024, 768, 256
    g = torch.Generator(device="cuda").manual_seed(5)
    codes = torch.randint(-127, 128, (m, n), device="cuda", generator=g, dtype=torch.int8)
    scales = torch.rand(m, device="cuda", generator=g) * 0.02 + 1e-3
    g_r = (torch.eye(b, device="cuda") + 0.05 * torch.randn((m // b, b, b), device="cuda", generator=g)).to(torch.bfloat16)
    w = dequant(N, codes, scales)
    want = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    N.call("poetx_apply_to_weight_rows", N.BF16, m // b, b, n, g_r.data_ptr(), 0, w.data_ptr(), want.data_ptr(),
           N.stream_ptr())
    d = N.LayerDesc()
    d.dtype, d.variant, d.neumann_k, d.m, d.n, d.b = N.BF16, N.MEM, 3, m, n, b
    d.fold_weight = 1
    d.pm_codes, d.pm_scales = codes.data_ptr(), scales.data_ptr()
    f = N.LayerFactors(None, None, None, None, g_r.data_ptr(), g_r.data_ptr(), None, None)
    got = torch.empty_like(want)
    ws, wsb = N.workspace(int(N.lib().poetx_layer_workspace_bytes(d, 0)))
    N.call("poetx_layer_weight_fold", d, f, 0, got.data_ptr(), ws, wsb, N.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_quantized_transposed_out_fold(N):
    """W1^T = (PM bd(G_P))^T straight from the codes (which = 1 of a POET-XQ
    layer at b = 256) against the transposed fold of the dequantized weight
    (bf16 output: within one bf16 rounding)."""
    m, n, b = 768, 1024, 256
    g = torch.Generator(device="cuda").manual_seed(9)
    codes = torch.randint(-127, 128, (m, n), device="cuda", generator=g, dtype=torch.int8)
    scales = torch.rand(m, device="cuda", generator=g) * 0.02 + 1e-3
    g_p = (torch.eye(b, device="cuda") + 0.05 * torch.randn((n // b, b, b), device="cuda", generator=g)).to(torch.bfloat16)
    w = dequant(N, codes, scales).float()
    want = torch.einsum("jsk,ski->jsi", w.view(m, n // b, b), g_p.float()).reshape(m, n).t()
    d = N.LayerDesc()
    d.dtype, d.variant, d.neumann_k, d.m, d.n, d.b = N.BF16, N.MEM, 3, m, n, b
    d.fold_weight = 1
    d.pm_codes, d.pm_scales = codes.data_ptr(), scales.data_ptr()
    f = N.LayerFactors(None, None, None, None, g_p.data_ptr(), g_p.data_ptr(), None, None)
    got = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
    ws, wsb = N.workspace(int(N.lib().poetx_layer_workspace_bytes(d, 0)))
    N.call("poetx_layer_weight_fold", d, f, 1, got.data_ptr(), ws, wsb, N.stream_ptr())
    torch.cuda.synchronize()
    assert float((got.float() - want).abs().max()) <= 2 ** -8 * float(want.abs().max())


@pytest.mark.parametrize("fold", [True, False], ids=["weight_folded", "activation_side"])
def test_quantized_bf16_layer_b256_vs_float64_oracle(fold):
    """A POET-XQ bf16 layer at b = 256 (the shapes where the fused int8 GEMM
    and fold run) against the float64 oracle on the dequantized base."""
    import paper_2603_05500_b200 as P
    from oracle import poetx_oracle as O

    m, n, T = 512, 768, 256
    lay, r = _quant_layer(P, m, n, 17)
    lay.fold_weight = fold
    x = torch.from_numpy(r.standard_normal((T, m))).cuda().to(torch.bfloat16)
    dz = torch.from_numpy(r.standard_normal((T, n))).cuda().to(torch.bfloat16)
    z, cache = lay.forward(x)
    gr = lay.backward(cache, dz)
    base = lay.base.dequantize() if hasattr(lay.base, "dequantize") else lay.base
    ref = O.OracleLayer(base.double().cpu().numpy(), 256, lay.perm_in.forward, lay.perm_out.forward)
    ref.q_r[...] = lay.q_r.packed.double().cpu().numpy()
    ref.q_p[...] = lay.q_p.packed.double().cpu().numpy()
    with O.blas_products():
        z_ref, c = ref.forward(x.double().cpu().numpy())
        g_r, g_p, dx = ref.backward(c, dz.double().cpu().numpy())
    for got, want in ((z, z_ref), (gr.x, dx), (gr.q_r, g_r), (gr.q_p, g_p)):
        got = got.double().cpu().numpy()
        assert float(np.abs(got - want).max()) <= 2e-2 * max(1.0, float(np.abs(want).max()))


_TRAIN = r"""
import hashlib, json, sys, torch
sys.path.insert(0, %r)
from paper_2603_05500_b200.trainer import Trainer, LlamaConfig
cfg = LlamaConfig(name="xq-test", d=512, f=1536, layers=2, heads=8, block=256, vocab=2048, seq=128,
                  variant="mem", quantized=True)
tr = Trainer(cfg, 4, seed=3, merge_gap=0)
g = torch.Generator().manual_seed(0)
losses = []
for i in range(3):
    t = torch.randint(0, cfg.vocab, (4, cfg.seq + 1), generator=g).cuda()
    losses.append(float(tr.step(t[:, :-1], t[:, 1:])))
torch.cuda.synchronize()
h = hashlib.sha256(tr.model.poet.param.detach().cpu().numpy().tobytes()).hexdigest()
print(json.dumps({"losses": losses, "poet": h}))
"""


def test_xq_trainer_fused_int8_path_bitwise_equal_to_dequantize_path():
    out = {}
    for flag in ("2", "0"):  # 2: every product that can takes the codes (main GEMMs included)
        env = dict(os.environ, POETX_Q8_GEMM=flag)
        res = subprocess.run([sys.executable, "-c", _TRAIN % ROOT], capture_output=True, text=True, env=env,
                             timeout=600, cwd=ROOT)
        assert res.returncode == 0, res.stderr[-3000:]
        out[flag] = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["2"] == out["0"], out
    assert all(x == x for x in out["2"]["losses"])
