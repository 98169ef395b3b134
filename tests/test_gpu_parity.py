"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference's golden vectors.

Tolerances use the reference's metric max|got - want| <= tol * max(1, max|want|)
(reference tests/test_layer.py:54,62,75):
  * float64 path: 1e-10 (the reference's own layer oracle bound);
  * float32 path: 1e-5 (north star / reference test_layer.py:62);
  * bf16 path: 2e-2 against the float64 oracle (north star);
  * permutations and other index work: bit-exact.
"""

import os

import numpy as np
import pytest
import torch

from oracle import poetx_oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def close(got, want, tol):
    got = got.detach().cpu().double().numpy() if isinstance(got, torch.Tensor) else np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    err = float(np.max(np.abs(got - want))) if got.size else 0.0
    bound = tol * max(1.0, float(np.max(np.abs(want))) if want.size else 1.0)
    assert err <= bound, f"max err {err:.3e} > {bound:.3e}"
    return err


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2603_05500_b200 as P

    P._native.lib()
    return P


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()

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



# ------------------------------------------------------------------- CNP ----


@pytest.mark.parametrize("tag", ["k3_f64", "k3_f32", "k2_f64", "k5_f64", "k3_b64_f32"])
def test_cnp_golden(P, tag):
    d = load("cnp.npz")
    packed, dg, k = d[f"{tag}/packed"], d[f"{tag}/dg"], int(d[f"{tag}/k"][0])
    nb, pairs = packed.shape
    b = int(round((1 + np.sqrt(1 + 8 * pairs)) / 2))
    tol = 1e-12 if packed.dtype == np.float64 else 1e-5
    q = P.skew_from_packed(P.SkewParams(nb, b, dev(packed)))
    assert np.array_equal(q.cpu().numpy(), O.skew_from_packed(packed, b))
    g, cache = P.cnp_forward(q, k)
    close(g, d[f"{tag}/g"], tol)
    dq = P.cnp_backward(cache, dev(dg))
    close(P.packed_grad_from_skew_grad(dq), d[f"{tag}/dpacked"], tol)


def test_cnp_frozen_values_and_identity(P):
    g, _ = P.cnp_forward(P.skew_from_packed(P.SkewParams(1, 2, dev(np.array([[0.1]])))), 3)
    g = g.cpu().numpy()
    assert abs(g[0, 0, 0] - 0.9801) <= 1e-12 and abs(g[0, 0, 1] - 0.198) <= 1e-12
    assert abs(g[0, 1, 0] + 0.198) <= 1e-12 and abs(g[0, 1, 1] - 0.9801) <= 1e-12
    for k in (1, 2, 3, 5):
        gz, _ = P.cnp_forward(torch.zeros((4, 5, 5), dtype=torch.float64, device="cuda"), k)
        assert torch.equal(gz, torch.eye(5, dtype=torch.float64, device="cuda").expand(4, 5, 5))


@pytest.mark.parametrize("b,nb,scale", [(64, 8, 0.01), (256, 4, 0.005), (128, 3, 0.02)])
def test_cnp_fp32_large_blocks_vs_oracle(P, b, nb, scale):
    r = np.random.default_rng(b)
    packed = (scale * r.standard_normal((nb, b * (b - 1) // 2))).astype(np.float64)
    dg = r.standard_normal((nb, b, b))
    q64 = O.skew_from_packed(packed, b)
    g64, c64 = O.cnp_forward(q64, 3)
    dp64 = O.packed_grad_from_skew_grad(O.cnp_backward(c64, dg, 3))
    p32 = dev(packed.astype(np.float32))
    g, cache = P.cnp_forward(P.skew_from_packed(P.SkewParams(nb, b, p32)), 3)
    close(g, g64, 1e-5)
    dq = P.cnp_backward(cache, dev(dg.astype(np.float32)))
    close(P.packed_grad_from_skew_grad(dq), dp64, 1e-5)


def test_orthogonality_bound_wide_regime(P):
    """reference tests/test_cnp.py:115-128: ||G^T G - I||_F <= 1e-2 for
    ||Q||_2 in [0.01, 0.2], b in {2,4,8,16}; plus <= 1e-5 at 0.03."""
    rng = np.random.default_rng(0)
    for trial in range(30):
        b = (2, 4, 8, 16)[trial % 4]
        nb = 1 + trial % 4
        scale = 0.01 + 0.19 * rng.random()
        q = O.skew_from_packed(rng.standard_normal((nb, b * (b - 1) // 2)), b)
        top = max(np.linalg.norm(q[i], 2) for i in range(nb))
        q = q * (scale / top)
        g, _ = P.cnp_forward(dev(q), 3)
        err = P.orthogonality_error(g)
        assert err <= 1e-2
        assert abs(err - O.orthogonality_error(O.cnp_forward(q, 3)[0])) <= 1e-9
    q = O.skew_from_packed(rng.standard_normal((4, 28)), 8)
    q *= 0.03 / max(np.linalg.norm(q[i], 2) for i in range(4))
    g, _ = P.cnp_forward(dev(q), 3)
    assert P.orthogonality_error(g) <= 1e-5
    c = P.cayley_exact(dev(q))
    assert float(torch.linalg.norm(g - c)) <= 1e-5


# --------------------------------------------------------- permutations ----


def test_permutation_products_exact(P):
    rng = P.Rng(7)
    for n in (1, 7, 64, 513):
        pm = P.sample_permutation(n, rng)
        w = np.random.default_rng(n).standard_normal((n, n))
        x = np.random.default_rng(n + 1).standard_normal((3, n)).astype(np.float32)
        for direction in ("forward", "inverse"):
            assert np.array_equal(P.permute_rows(w, pm, direction),
                                  O.permute_rows(w, pm.forward, pm.inverse, direction))
            assert np.array_equal(P.permute_cols(w, pm, direction),
                                  O.permute_cols(w, pm.forward, pm.inverse, direction))
            assert np.array_equal(P.permute_features(x, pm, direction),
                                  O.permute_cols(x, pm.forward, pm.inverse, direction))
        xb = dev(x).to(torch.bfloat16)
        got = P.permute_features(xb, pm, "inverse")
        assert torch.equal(got, xb[:, torch.from_numpy(pm.forward).long().cuda()])


def test_premerge_entrywise(P):
    rng = P.Rng(21)
    rp, cp = P.sample_permutation(6, rng), P.sample_permutation(8, rng)
    w = np.random.default_rng(1).standard_normal((6, 8))
    got = P.premerge_weight(w, rp, cp)
    assert np.array_equal(got, O.premerge(w, rp.forward, cp.forward))


# ------------------------------------------------------- block-diagonal ----


@pytest.mark.parametrize("dt,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
def test_blockdiag_ops_vs_oracle(P, dt, tol):
    r = np.random.default_rng(3)
    for nb, b, T in ((4, 3, 5), (8, 64, 1024), (3, 16, 77)):
        g = r.standard_normal((nb, b, b)).astype(dt)
        x = r.standard_normal((T, nb * b)).astype(dt)
        y = r.standard_normal((T, nb * b)).astype(dt)
        f = P.BlockDiagonalFactor(dev(g))
        for tr in (False, True):
            close(P.apply_to_features(f, dev(x), transpose=tr), O.apply_to_features(g, x, tr), tol)
        w = r.standard_normal((nb * b, 9)).astype(dt)
        close(P.apply_to_weight_rows(f, dev(w)), O.apply_to_weight_rows(g, w), tol)
        close(P.apply_to_weight_rows(f, dev(w), transpose=True), O.apply_to_weight_rows(g, w, True), tol)
        close(P.segmented_outer(dev(x), dev(y), b), O.segmented_outer(x, y, b), tol * max(1, T / 64))


def test_orthogonality_error_matches(P):
    c, s = np.cos(0.3), np.sin(0.3)
    rot = np.array([[[c, s], [-s, c]], [[1.0, 0.0], [0.0, 1.0]]])
    assert P.orthogonality_error(dev(rot)) <= 1e-15
    assert P.orthogonality_error(dev(2.0 * rot)) > 1.0


# ---------------------------------------------------------------- layer ----


def _gpu_layer(P, d, tag, variant, dtype=None):
    base = d[f"{tag}/base"]
    m, n, b = (int(v) for v in d[f"{tag}/meta"][:3])
    layer = P.PoetLinearLayer(base if dtype is None else torch.from_numpy(base).to(dtype), b, P.Rng(0),
                              variant=variant)
    layer.set_permutations(P.PermutationMap.from_forward(d[f"{tag}/perm_in"]),
                           P.PermutationMap.from_forward(d[f"{tag}/perm_out"]))
    setp(layer.q_r.packed, d[f"{tag}/q_r"])
    setp(layer.q_p.packed, d[f"{tag}/q_p"])
    return layer


@pytest.mark.parametrize("tag,variant", [("small_f64_fast", "fast"), ("small_f64_mem", "mem"),
                                         ("small_f32_fast", "fast"), ("mid_f32_fast", "fast")])
def test_layer_golden(P, tag, variant):
    d = load("layer.npz")
    tol = 1e-10 if d[f"{tag}/base"].dtype == np.float64 else 1e-5
    layer = _gpu_layer(P, d, tag, variant)
    assert isinstance(layer.base, np.ndarray) and layer.dtype == d[f"{tag}/base"].dtype  # numpy in, numpy out
    assert np.array_equal(layer.base, d[f"{tag}/base"])  # PM round trip exact
    z, cache = layer.forward(d[f"{tag}/x"])
    close(z, d[f"{tag}/z"], tol)
    grads = layer.backward(cache, d[f"{tag}/dz"])
    close(grads.q_r, d[f"{tag}/gq_r"], tol)
    close(grads.q_p, d[f"{tag}/gq_p"], tol)
    close(grads.x, d[f"{tag}/dx"], tol)
    with pytest.raises(P.StateError):
        layer.backward(cache, d[f"{tag}/dz"])
    seed = int(d[f"{tag}/meta"][4])
    packed_ref = layer.q_r.packed
    audit = layer.merge_and_reinit(P.Rng.keyed(seed, "merge", 1, 0))
    assert layer.q_r.packed is packed_ref and not bool(packed_ref.any())
    assert np.array_equal(layer.perm_in.forward, d[f"{tag}/new_perm_in"])
    assert np.array_equal(layer.perm_out.forward, d[f"{tag}/new_perm_out"])
    close(layer.base, d[f"{tag}/merged_base"], tol)
    close(np.array([audit.orth_err_r, audit.orth_err_p]), d[f"{tag}/orth_err"], 1e-6)
    z2, _ = layer.forward(d[f"{tag}/x"])
    close(z2, d[f"{tag}/z_after_merge"], tol)


def test_cfg1_layer_vs_oracle(P):
    """BASELINE configs[0]: 512x512, b=64, k=3, fp32, 1024 tokens."""
    base, fi, fo, q_r, q_p, x, dz = O.cfg1_inputs()
    ref = O.OracleLayer(base, 64, fi, fo)
    ref.q_r[...] = q_r
    ref.q_p[...] = q_p
    z_ref, cache = ref.forward(x)
    gr_ref, gp_ref, dx_ref = ref.backward(cache, dz)
    for variant in ("fast", "mem"):
        layer = P.PoetLinearLayer(base, 64, P.Rng(0), variant=variant)
        layer.set_permutations(P.PermutationMap.from_forward(fi), P.PermutationMap.from_forward(fo))
        setp(layer.q_r.packed, q_r)
        setp(layer.q_p.packed, q_p)
        z, c = layer.forward(dev(x))
        close(z, z_ref, 1e-5)
        g = layer.backward(c, dev(dz))
        close(g.q_r, gr_ref, 1e-5)
        close(g.q_p, gp_ref, 1e-5)
        close(g.x, dx_ref, 1e-5)


def test_fast_and_mem_bitwise_on_gpu(P):
    base = np.random.default_rng(7).standard_normal((64, 96)).astype(np.float32)
    out = []
    for variant in ("fast", "mem"):
        layer = P.PoetLinearLayer(base, 16, P.Rng.keyed(7, "p"), variant=variant)
        setp(layer.q_r.packed, 0.05 * np.random.default_rng(1).standard_normal(layer.q_r.packed.shape))
        setp(layer.q_p.packed, 0.05 * np.random.default_rng(2).standard_normal(layer.q_p.packed.shape))
        x = dev(np.random.default_rng(9).standard_normal((33, 64)).astype(np.float32))
        dz = dev(np.random.default_rng(10).standard_normal((33, 96)).astype(np.float32))
        z, c = layer.forward(x)
        g = layer.backward(c, dz)
        out.append((z, g))
    (za, ga), (zb, gb) = out
    assert torch.equal(za, zb)
    assert torch.equal(ga.q_r, gb.q_r) and torch.equal(ga.q_p, gb.q_p) and torch.equal(ga.x, gb.x)


def test_layer_backward_finite_differences_f64(P):
    """reference tests/test_layer.py:104-142 on the GPU float64 path."""
    layer = P.init_layer(8, 12, 4, P.Rng.keyed(0, "layer"), dtype=np.float64)
    rng = np.random.default_rng(3)
    setp(layer.q_r.packed, 0.15 * rng.standard_normal(tuple(layer.q_r.packed.shape)))
    setp(layer.q_p.packed, 0.15 * rng.standard_normal(tuple(layer.q_p.packed.shape)))
    x = rng.standard_normal((3, 8))
    mask = rng.standard_normal((3, 12))
    z, cache = layer.forward(x)
    grads = layer.backward(cache, mask)
    h = 1e-6
    for attr, got in (("q_r", grads.q_r), ("q_p", grads.q_p)):
        packed = getattr(layer, attr).packed
        flat = packed.reshape(-1)  # a view (host numpy array: numpy-constructed layer)
        fd = np.zeros(flat.shape[0])
        for i in range(flat.shape[0]):
            keep = float(flat[i])
            flat[i] = keep + h
            up = float(np.sum(mask * layer.forward(x)[0]))
            flat[i] = keep - h
            dn = float(np.sum(mask * layer.forward(x)[0]))
            flat[i] = keep
            fd[i] = (up - dn) / (2 * h)
        close(got.reshape(-1), fd, 1e-6)


def test_zero_params_reproduce_base_weight(P):
    for dt, tol in ((np.float64, 1e-12), (np.float32, 1e-5)):
        layer = P.init_layer(8, 12, 4, P.Rng.keyed(0, "layer"), dtype=dt)
        x = np.random.default_rng(2).standard_normal((5, 8)).astype(dt)
        z, _ = layer.forward(x)
        close(z, x @ host(layer.base), tol)


def test_merge_preserves_function_and_materialize(P):
    layer = P.init_layer(64, 32, 8, P.Rng.keyed(14, "layer"), dtype=np.float64)
    rng = np.random.default_rng(14)
    setp(layer.q_r.packed, 0.1 * rng.standard_normal(tuple(layer.q_r.packed.shape)))
    setp(layer.q_p.packed, 0.1 * rng.standard_normal(tuple(layer.q_p.packed.shape)))
    x = rng.standard_normal((5, 64))
    z0, _ = layer.forward(x)
    w_eff = host(layer.materialize_weight())
    close(x @ w_eff, z0, 1e-11)
    old = layer.perm_in.forward.copy()
    layer.merge_and_reinit(P.Rng.keyed(16, "merge"))
    z1, _ = layer.forward(x)
    close(z1, z0, 1e-11)
    assert layer.merge_count == 1 and not np.array_equal(old, layer.perm_in.forward)


def test_merge_sv_drift(P):
    """reference tests/test_layer.py:271-286."""
    layer = P.init_layer(64, 64, 8, P.Rng.keyed(21, "drift"), dtype=np.float64)
    rng = np.random.default_rng(22)
    setp(layer.q_r.packed, 0.012 * rng.standard_normal(tuple(layer.q_r.packed.shape)))
    setp(layer.q_p.packed, 0.012 * rng.standard_normal(tuple(layer.q_p.packed.shape)))
    audit = layer.merge_and_reinit(P.Rng.keyed(23, "m"), compute_sv_drift=True)
    assert audit.sv_drift <= 1e-3
    setp(layer.q_r.packed, 0.012 * rng.standard_normal(tuple(layer.q_r.packed.shape)))
    setp(layer.q_p.packed, 0.012 * rng.standard_normal(tuple(layer.q_p.packed.shape)))
    audit2 = layer.merge_and_reinit(P.Rng.keyed(25, "m"), use_exact_cayley=True, compute_sv_drift=True)
    assert audit2.sv_drift <= 1e-9 and audit2.orth_err_r <= 1e-11


# --------------------------------------------------------------- bf16 path ----


@pytest.mark.parametrize("m,n,b,T,variant,quant", [
    (512, 512, 64, 1024, "fast", False), (256, 768, 128, 512, "fast", False), (1024, 512, 256, 384, "fast", False),
    (512, 768, 256, 77, "fast", False), (768, 512, 256, 300, "mem", False), (512, 1024, 256, 130, "mem", True),
    (256, 256, 64, 33, "mem", True)])
@pytest.mark.parametrize("fold", [True, False], ids=["weight_folded", "activation_side"])
def test_bf16_layer_vs_oracle(P, m, n, b, T, variant, quant, fold):
    """bf16 layer (tensor-core path: block factors folded into the weight or
    applied to the activations, CTA-pair GEMMs; ragged T; mem variant; int8
    base) against the float64 oracle."""
    r = np.random.default_rng(m + n + T)
    base = (r.standard_normal((m, n)) / np.sqrt(m))
    layer = P.PoetLinearLayer(torch.from_numpy(base).to(torch.bfloat16), b, P.Rng(5), variant=variant)
    layer.fold_weight = fold
    if quant:
        layer.quantize_base()
        base_q = layer.base.dequantize().double().cpu().numpy()  # the int8 weight the GPU holds
    else:
        base_q = layer.base.double().cpu().numpy()  # bf16-rounded weight the GPU really holds
    q_r = 0.01 * r.standard_normal(tuple(layer.q_r.packed.shape))
    q_p = 0.01 * r.standard_normal(tuple(layer.q_p.packed.shape))
    setp(layer.q_r.packed, q_r)
    setp(layer.q_p.packed, q_p)
    x = r.standard_normal((T, m))
    dz = r.standard_normal((T, n))
    xb = dev(x).to(torch.bfloat16)
    dzb = dev(dz).to(torch.bfloat16)
    ref = O.OracleLayer(base_q, b, layer.perm_in.forward, layer.perm_out.forward)
    ref.q_r[...] = q_r
    ref.q_p[...] = q_p
    z_ref, c = ref.forward(xb.double().cpu().numpy())
    gr, gp, dx = ref.backward(c, dzb.double().cpu().numpy())
    z, cache = layer.forward(xb)
    close(z, z_ref, 2e-2)
    g = layer.backward(cache, dzb)
    close(g.x, dx, 2e-2)
    close(g.q_r, gr, 2e-2)
    close(g.q_p, gp, 2e-2)


# ------------------------------------------------------------------ AdamW ----


def test_adamw_transcript_bitwise(P):
    d = load("optim.npz")
    for tag in ("float32", "float64"):
        s = P.ScheduleConfig(base_lr=0.05, total_steps=1000, warmup_steps=10, weight_decay=0.01)
        params = {k: dev(d[f"{tag}/p0/{k}"]) for k in ("a", "b")}
        st = P.adamw_init(params)
        for t in range(5):
            grads = {k: dev(d[f"{tag}/g{t}/{k}"]) for k in ("a", "b")}
            thr = P.clip_threshold_at(t, t if t < 3 else None, s)
            norm = P.global_clip(grads, thr)
            assert abs(norm - d[f"{tag}/norms"][t]) <= 1e-12 * norm
            P.adamw_step(params, grads, st, P.lr_at(t + 10, s, poet=True), s)
            for k in ("a", "b"):
                assert np.array_equal(params[k].cpu().numpy(), d[f"{tag}/p{t + 1}/{k}"]), (tag, t, k)


def test_adamw_nonfinite_aborts(P):
    s = P.ScheduleConfig(base_lr=0.1, total_steps=100)
    p = {"w": torch.ones(2, dtype=torch.float64, device="cuda")}
    st = P.adamw_init(p)
    with pytest.raises(P.NumericsError):
        P.adamw_step(p, {"w": torch.tensor([float("nan"), 0.0], dtype=torch.float64, device="cuda")}, st, 0.1, s)
    with pytest.raises(P.NumericsError):
        P.global_clip({"a": torch.tensor([float("inf"), 1.0], device="cuda")}, 1.0)


def test_fused_clip_adamw_matches_two_step(P):
    s = P.ScheduleConfig(base_lr=0.05, total_steps=1000)
    r = np.random.default_rng(0)
    p0 = r.standard_normal(1000).astype(np.float32)
    g0 = r.standard_normal(1000).astype(np.float32)
    pa, ga = dev(p0), dev(g0)
    st = P.adamw_init({"w": pa})
    P.global_clip({"w": ga}, 0.5)
    P.adamw_step({"w": pa}, {"w": ga}, st, 0.01, s)
    pb, gb = dev(p0), dev(g0)
    mb, vb = torch.zeros_like(pb), torch.zeros_like(pb)
    P.fused_clip_adamw([([pb], [gb], [mb], [vb], 0.01, 1)], 0.5, s)
    assert torch.equal(pa, pb)
