"""Pin the CPU oracle against golden vectors produced by the reference.

These run without a GPU.  Every comparison is bitwise: the oracle keeps
the reference's fixed accumulation order and its numpy Philox stream.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import poetx_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def keyed(seed, *tags):
    return O.numpy_rng(seed, O.keyed_stream(*tags))


@pytest.mark.parametrize("tag", ["k3_f64", "k3_f32", "k2_f64", "k5_f64", "k3_b64_f32"])
def test_cnp_bitwise(tag):
    d = load("cnp.npz")
    packed, dg, k = d[f"{tag}/packed"], d[f"{tag}/dg"], int(d[f"{tag}/k"][0])
    b = int((1 + np.sqrt(1 + 8 * packed.shape[1])) / 2)
    q = O.skew_from_packed(packed, b)
    g, cache = O.cnp_forward(q, k)
    dq = O.cnp_backward(cache, dg, k)
    assert np.array_equal(g, d[f"{tag}/g"])
    assert np.array_equal(O.packed_grad_from_skew_grad(dq), d[f"{tag}/dpacked"])


def test_cnp_frozen_planar_rotation():
    # reference tests/test_cnp.py:56-65
    g, _ = O.cnp_forward(O.skew_from_packed(np.array([[0.1]]), 2), 3)
    assert abs(g[0, 0, 0] - 0.9801) <= 1e-12 and abs(g[0, 0, 1] - 0.198) <= 1e-12
    assert abs(g[0, 1, 0] + 0.198) <= 1e-12


def test_packing_order():
    # reference tests/test_cnp.py:38-42
    q = O.skew_from_packed(np.array([[1.0, 2.0, 3.0]]), 3)
    assert np.array_equal(q[0], [[0, 1, 2], [-1, 0, 3], [-2, -3, 0]])


def test_permutations_numpy_and_pure_python():
    d = load("perm.npz")
    for i, n in enumerate((1, 2, 16, 64, 512, 2048, 5632, 5461)):
        want = d[f"merge_{n}"]
        r = keyed(99, "merge", 400 * (i + 1), i)
        assert np.array_equal(r.permutation(n).astype(np.int32), want)
        gen = O.PhiloxPy(99, O.keyed_stream("merge", 400 * (i + 1), i))
        assert np.array_equal(O.philox_permutation_py(gen, n), want)
    r = keyed(5, "init", "reg", 0)
    r.standard_normal((3, 7))
    gen = O.PhiloxPy(state=r.bit_generator.state)
    assert np.array_equal(O.philox_permutation_py(gen, 37), d["after_normal_a"])
    assert np.array_equal(O.philox_permutation_py(gen, 1000), d["after_normal_b"])


def test_inverse_of_2_0_1():
    # reference tests/test_permute.py:24-27
    assert np.array_equal(O.invert(np.array([2, 0, 1], dtype=np.int32)), [1, 2, 0])


def _layer_from(d, tag, variant):
    layer = O.OracleLayer(d[f"{tag}/base"], int(d[f"{tag}/meta"][2]), d[f"{tag}/perm_in"],
                          d[f"{tag}/perm_out"], variant=variant)
    layer.q_r[...] = d[f"{tag}/q_r"]
    layer.q_p[...] = d[f"{tag}/q_p"]
    return layer


@pytest.mark.parametrize("tag,variant", [("small_f64_fast", "fast"), ("small_f64_mem", "mem"),
                                         ("small_f32_fast", "fast"), ("mid_f32_fast", "fast")])
def test_layer_bitwise(tag, variant):
    d = load("layer.npz")
    layer = _layer_from(d, tag, variant)
    z, cache = layer.forward(d[f"{tag}/x"])
    gr, gp, dx = layer.backward(cache, d[f"{tag}/dz"])
    assert np.array_equal(z, d[f"{tag}/z"])
    assert np.array_equal(gr, d[f"{tag}/gq_r"])
    assert np.array_equal(gp, d[f"{tag}/gq_p"])
    assert np.array_equal(dx, d[f"{tag}/dx"])
    seed = int(d[f"{tag}/meta"][4])
    r = keyed(seed, "merge", 1, 0)
    new_in = r.permutation(layer.m).astype(np.int32)
    new_out = r.permutation(layer.n).astype(np.int32)
    err = layer.merge_and_reinit(new_in, new_out)
    assert np.array_equal(layer.base, d[f"{tag}/merged_base"])
    assert np.array_equal(new_in, d[f"{tag}/new_perm_in"])
    assert np.array_equal(np.array(err), d[f"{tag}/orth_err"])
    z2, _ = layer.forward(d[f"{tag}/x"])
    assert np.array_equal(z2, d[f"{tag}/z_after_merge"])


cfg1_inputs = O.cfg1_inputs


def test_cfg1_checksums():
    d = load("cfg1.npz")
    base, fi, fo, q_r, q_p, x, dz = cfg1_inputs()
    assert sha(base) == str(d["cfg1/base/sha256"])
    assert np.array_equal(fi, d["cfg1/perm_in"]) and np.array_equal(fo, d["cfg1/perm_out"])
    layer = O.OracleLayer(base, 64, fi, fo)
    layer.q_r[...] = q_r
    layer.q_p[...] = q_p
    z, cache = layer.forward(x)
    gr, gp, dx = layer.backward(cache, dz)
    for name, v in (("z", z), ("gq_r", gr), ("gq_p", gp), ("dx", dx)):
        assert sha(v) == str(d[f"cfg1/{name}/sha256"]), name


def test_optim_transcript_bitwise():
    d = load("optim.npz")
    for tag in ("float32", "float64"):
        params = {k: d[f"{tag}/p0/{k}"].copy() for k in ("a", "b")}
        m = {k: np.zeros_like(v) for k, v in params.items()}
        v = {k: np.zeros_like(x) for k, x in params.items()}
        t = 0
        norms = []
        for s in range(5):
            grads = {k: d[f"{tag}/g{s}/{k}"].copy() for k in ("a", "b")}
            thr = O.clip_threshold_at(s, s if s < 3 else None)
            norms.append(O.global_clip(grads, thr))
            lr = O.lr_at(s + 10, 0.05, 1000, warmup_steps=10, poet=True)
            t = O.adamw_step(params, grads, m, v, t, lr)
            for k in ("a", "b"):
                assert np.array_equal(params[k], d[f"{tag}/p{s + 1}/{k}"]), (tag, s, k)
        assert np.array_equal(np.array(norms), d[f"{tag}/norms"])
    steps = d["lr_steps"]
    assert np.array_equal([O.lr_at(int(k), 0.08, 3000, 100) for k in steps], d["lr"])
    assert np.array_equal([O.lr_at(int(k), 0.08, 3000, 100, poet=True) for k in steps], d["lr_poet"])


# -- POET-XQ (quant.py, quantized layer paths) --------------------------------


@pytest.mark.parametrize("tag", ["gauss_f32", "gauss_f64", "ties_f64", "wide_f32"])
def test_quantize_rows_bitwise(tag):
    d = load("quant.npz")
    codes, scales = O.quantize_rows(d[f"q_{tag}_w"])
    assert codes.dtype == np.int8 and scales.dtype == d[f"q_{tag}_w"].dtype
    assert np.array_equal(codes, d[f"q_{tag}_codes"])
    assert np.array_equal(scales, d[f"q_{tag}_scales"])


@pytest.mark.parametrize("tag", ["f32", "f64"])
def test_quantized_layer_bitwise(tag):
    d = load("quant.npz")
    lay = O.OracleLayer(d[f"l_{tag}_base"], 8, d[f"l_{tag}_perm_in"], d[f"l_{tag}_perm_out"], variant="mem",
                        quantized=True)
    lay.q_r[...] = d[f"l_{tag}_q_r"]
    lay.q_p[...] = d[f"l_{tag}_q_p"]
    z, cache = lay.forward(d[f"l_{tag}_x"])
    gr, gp, dx = lay.backward(cache, d[f"l_{tag}_dz"])
    for got, key in ((z, "z"), (gr, "gr"), (gp, "gp"), (dx, "dx")):
        assert np.array_equal(got, d[f"l_{tag}_{key}"]), key
    lay.merge_and_reinit(d[f"l_{tag}_new_perm_in"], d[f"l_{tag}_new_perm_out"])
    assert np.array_equal(lay.codes, d[f"l_{tag}_merged_codes"])
    assert np.array_equal(lay.scales, d[f"l_{tag}_merged_scales"])


@pytest.mark.parametrize("tag", ["square", "tall", "wide", "rank6", "single", "graded"])
def test_jacobi_singular_values_bitwise(tag):
    """linalg.svd_singular_values restated: bitwise against the reference."""
    g = load("spectrum.npz")
    sv, ok, _ = O.svd_singular_values(g[f"a_{tag}"])
    assert ok
    assert np.array_equal(sv, g[f"sv_{tag}"])
