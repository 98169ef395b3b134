"""POET-XQ on the device (csrc/quant.cu, quantized layer paths) against the
oracle pinned to the reference (tests/golden/quant.npz)."""

import os

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

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold():
    return dict(np.load(os.path.join(GOLD, "quant.npz")))


@pytest.mark.parametrize("tag", ["gauss_f32", "gauss_f64", "ties_f64", "wide_f32"])
def test_device_quantize_bitwise(tag):
    import paper_2603_05500_b200 as P

    d = gold()
    q = P.QuantizedMatrix.quantize(torch.from_numpy(d[f"q_{tag}_w"]).cuda())
    assert np.array_equal(q.codes.cpu().numpy(), d[f"q_{tag}_codes"])
    assert np.array_equal(q.scales.cpu().numpy(), d[f"q_{tag}_scales"])
    # dequantization: codes in the scale type times the row scale (quant.py:50-61)
    want = d[f"q_{tag}_codes"].astype(d[f"q_{tag}_scales"].dtype) * d[f"q_{tag}_scales"][:, None]
    assert np.array_equal(q.dequantize().cpu().numpy(), want)
    k = q.shape[0] - 1
    assert np.array_equal(q.dequant_row(k).cpu().numpy(), want[k])
    assert np.array_equal(q.dequant_col(2).cpu().numpy(), want[:, 2])


def test_gather_commutes_with_dequantize():
    import paper_2603_05500_b200 as P

    w = torch.randn(64, 96, device="cuda")
    q = P.QuantizedMatrix.quantize(w)
    ri, ci = np.random.default_rng(1).permutation(64), np.random.default_rng(2).permutation(96)
    g = q.gather(ri, ci)
    assert torch.equal(g.dequantize(), q.dequantize()[torch.from_numpy(ri).cuda()][:, torch.from_numpy(ci).cuda()])


def test_quantize_requires_mem_variant():
    import paper_2603_05500_b200 as P
    from paper_2603_05500_b200.trainer import PoetLinear, PoetStack

    lay = P.init_layer(16, 16, 4, P.Rng.keyed(1, "q"), variant="fast")
    with pytest.raises(P.ConfigError, match="mem variant"):
        lay.quantize_base()
    st = PoetStack([("x.r", 4), ("x.p", 4)], 4, torch.device("cuda"))
    with pytest.raises(P.ConfigError, match="mem variant"):
        PoetLinear("x", 16, 16, st, P.Rng.keyed(1, "q"), variant="fast", quantized=True)


@pytest.mark.parametrize("tag,tol", [("f32", 1e-5), ("f64", 1e-10)])
def test_quantized_layer_matches_oracle(tag, tol):
    """Forward, backward through the int8 base (dequantized per call) and the
    requantizing merge, against the reference's numbers."""
    import paper_2603_05500_b200 as P
    from paper_2603_05500_b200.permute import PermutationMap

    d = gold()
    lay = P.PoetLinearLayer(d[f"l_{tag}_base"], 8, P.Rng(0), variant="mem")
    lay.set_permutations(PermutationMap.from_forward(d[f"l_{tag}_perm_in"]),
                         PermutationMap.from_forward(d[f"l_{tag}_perm_out"]))
    lay.quantize_base()
    assert lay.quantized and isinstance(lay.base, P.QuantizedMatrix)
    setp(lay.q_r.packed, d[f"l_{tag}_q_r"])
    setp(lay.q_p.packed, d[f"l_{tag}_q_p"])
    z, cache = lay.forward(d[f"l_{tag}_x"])
    g = lay.backward(cache, d[f"l_{tag}_dz"])
    for got, key in ((z, "z"), (g.q_r, "gr"), (g.q_p, "gp"), (g.x, "dx")):
        want = d[f"l_{tag}_{key}"]
        assert np.abs(np.asarray(got) - want).max() <= tol * max(1.0, np.abs(want).max()), key
    # merge: the device folds in its own accumulation order, so codes may move
    # by one step at a rounding boundary; the reference's own bound applies
    # (<= half a scale against the float shadow, test_layer.py:370-388)
    lay.set_permutations(PermutationMap.from_forward(d[f"l_{tag}_perm_in"]),
                         PermutationMap.from_forward(d[f"l_{tag}_perm_out"]))
    shadow = host(lay.materialize_weight()).astype(np.float64)

    new_in, new_out = d[f"l_{tag}_new_perm_in"], d[f"l_{tag}_new_perm_out"]
    import paper_2603_05500_b200.layer as L

    orig = L.sample_permutation
    seq = iter([PermutationMap.from_forward(new_in), PermutationMap.from_forward(new_out)])
    L.sample_permutation = lambda n, rng: next(seq)
    try:
        lay.merge_and_reinit(None)
    finally:
        L.sample_permutation = orig
    codes = lay.base.codes.cpu().numpy()
    scales = lay.base.scales.cpu().numpy()
    assert np.array_equal(lay.perm_in.forward, new_in)
    got = lay.base.dequantize().double().cpu().numpy()
    assert np.all(np.abs(got - shadow) <= scales[:, None] / 2.0 + 1e-9 * np.abs(shadow).max())
    same = np.mean(codes == d[f"l_{tag}_merged_codes"])
    assert same >= 0.995, same
    assert np.allclose(scales, d[f"l_{tag}_merged_scales"], rtol=1e-5)
    assert np.all(host(lay.q_r.packed) == 0)


def test_quantized_llama_trains_and_checkpoints(tmp_path):
    """Llama-60M POET-XQ (mem, int8 frozen weights): loss falls through a
    merge, the frozen weight takes half the bytes, and a PXK1 round trip
    (base_codes / base_scales, runner.py:159-161) resumes bitwise."""
    from paper_2603_05500_b200.trainer import Trainer, llama_config

    cfg = llama_config("llama-60m", layers=2, seq=64, variant="mem", quantized=True)
    toks = [torch.randint(0, 64, (4, cfg.seq + 1), generator=torch.Generator().manual_seed(i)).cuda()
            for i in range(6)]
    tr = Trainer(cfg, 4, seed=1, merge_gap=3, base_lr=3e-3)
    lay = tr.model.poet_layers()[0]
    assert lay.quantized and lay.premerged is None and lay.codes.dtype == torch.int8
    losses = [float(tr.step(t[:, :-1], t[:, 1:])) for t in toks[:3]]
    tr.save_checkpoint(str(tmp_path / "q.pxk1"))
    rest = [float(tr.step(t[:, :-1], t[:, 1:])) for t in toks[3:]]
    assert losses[-1] < losses[0] and all(x == x for x in rest)
    assert lay.merge_count == 2
    b = Trainer(cfg, 4, seed=1, merge_gap=3, base_lr=3e-3)
    b.load_checkpoint(str(tmp_path / "q.pxk1"))
    again = [float(b.step(t[:, :-1], t[:, 1:])) for t in toks[3:]]
    assert again == rest
    for x, y in zip(tr.model.poet_layers(), b.model.poet_layers()):
        assert torch.equal(x.codes, y.codes) and torch.equal(x.scales, y.scales)
