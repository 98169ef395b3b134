"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference lives at /root/reference and is
importable there; it does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Small cases store full tensors; the config-1
case (512x512, b=64, T=1024, fp32 -- BASELINE.json configs[0]) stores the
SHA-256 of each output's bytes plus its float64 sum, because the inputs are
regenerated from keyed seeds and the oracle reproduces the reference
bitwise.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import poetx  # noqa: E402  (the reference)
from poetx.cnp import SkewParams, cnp_backward, cnp_forward, packed_grad_from_skew_grad, skew_from_packed  # noqa: E402
from poetx.layer import init_layer  # noqa: E402
from poetx.linalg import Rng  # noqa: E402
from poetx.optim import ScheduleConfig, adamw_init, adamw_step, clip_threshold_at, global_clip, lr_at  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cnp_cases():
    out = {}
    for tag, (nb, b, k, dt, scale) in {
        "k3_f64": (3, 8, 3, np.float64, 0.3),
        "k3_f32": (4, 16, 3, np.float32, 0.05),
        "k2_f64": (2, 6, 2, np.float64, 0.3),
        "k5_f64": (2, 5, 5, np.float64, 0.2),
        "k3_b64_f32": (8, 64, 3, np.float32, 0.01),
    }.items():
        rng = Rng.keyed(7, "golden", "cnp", tag)
        packed = (scale * rng.normal((nb, b * (b - 1) // 2))).astype(dt)
        dg = rng.normal((nb, b, b)).astype(dt)
        q = skew_from_packed(SkewParams(nb, b, packed))
        g, cache = cnp_forward(q, k)
        dq = cnp_backward(cache, dg)
        out[f"{tag}/packed"] = packed
        out[f"{tag}/dg"] = dg
        out[f"{tag}/k"] = np.array([k])
        out[f"{tag}/g"] = g
        out[f"{tag}/dpacked"] = packed_grad_from_skew_grad(dq)
    np.savez_compressed(os.path.join(OUT, "cnp.npz"), **out)


def layer_case(tag, m, n, b, T, dt, variant, scale, seed, store_full=True):
    layer = init_layer(m, n, b, Rng.keyed(seed, "layer"), dtype=dt, variant=variant)
    prng = Rng.keyed(seed, "packed")
    layer.q_r.packed[...] = (scale * prng.normal(layer.q_r.packed.shape)).astype(dt)
    layer.q_p.packed[...] = (scale * prng.normal(layer.q_p.packed.shape)).astype(dt)
    d = Rng.keyed(seed, "data")
    x = d.normal((T, m)).astype(dt)
    dz = d.normal((T, n)).astype(dt)
    z, cache = layer.forward(x)
    grads = layer.backward(cache, dz)
    rec = {
        "z": z, "dx": grads.x, "gq_r": grads.q_r, "gq_p": grads.q_p,
    }
    inputs = {
        "base": layer.base.copy(), "perm_in": layer.perm_in.forward.copy(),
        "perm_out": layer.perm_out.forward.copy(), "q_r": layer.q_r.packed.copy(),
        "q_p": layer.q_p.packed.copy(), "x": x, "dz": dz,
    }
    audit = layer.merge_and_reinit(Rng.keyed(seed, "merge", 1, 0))
    rec["merged_base"] = layer.base.copy()
    rec["new_perm_in"] = layer.perm_in.forward.copy()
    rec["new_perm_out"] = layer.perm_out.forward.copy()
    rec["orth_err"] = np.array([audit.orth_err_r, audit.orth_err_p])
    z2, _ = layer.forward(x)
    rec["z_after_merge"] = z2
    out = {}
    if store_full:
        for k, v in {**inputs, **rec}.items():
            out[f"{tag}/{k}"] = v
    else:
        for k, v in rec.items():
            out[f"{tag}/{k}/sha256"] = np.array(sha(v))
            out[f"{tag}/{k}/sum64"] = np.array([float(np.sum(np.asarray(v, dtype=np.float64)))])
        for k in ("perm_in", "perm_out"):
            out[f"{tag}/{k}"] = inputs[k]
        out[f"{tag}/base/sha256"] = np.array(sha(inputs["base"]))
    out[f"{tag}/meta"] = np.array([m, n, b, T, seed])
    return out


def layer_cases():
    out = {}
    out.update(layer_case("small_f64_fast", 16, 24, 4, 6, np.float64, "fast", 0.1, 11))
    out.update(layer_case("small_f64_mem", 16, 24, 4, 6, np.float64, "mem", 0.1, 12))
    out.update(layer_case("small_f32_fast", 32, 16, 8, 5, np.float32, "fast", 0.05, 13))
    out.update(layer_case("mid_f32_fast", 128, 192, 16, 48, np.float32, "fast", 0.02, 14))
    np.savez_compressed(os.path.join(OUT, "layer.npz"), **out)
    cfg1 = layer_case("cfg1", 512, 512, 64, 1024, np.float32, "fast", 0.01, 2603, store_full=False)
    np.savez_compressed(os.path.join(OUT, "cfg1.npz"), **cfg1)


def perm_cases():
    out = {}
    for i, n in enumerate((1, 2, 16, 64, 512, 2048, 5632, 5461)):
        out[f"merge_{n}"] = Rng.keyed(99, "merge", 400 * (i + 1), i).permutation(n).astype(np.int32)
    # two consecutive draws sharing the uint32 buffer, after a gaussian draw
    r = Rng.keyed(5, "init", "reg", 0)
    r.normal((3, 7))
    out["after_normal_a"] = r.permutation(37).astype(np.int32)
    out["after_normal_b"] = r.permutation(1000).astype(np.int32)
    np.savez_compressed(os.path.join(OUT, "perm.npz"), **out)


def optim_cases():
    out = {}
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        s = ScheduleConfig(base_lr=0.05, total_steps=1000, warmup_steps=10, weight_decay=0.01)
        rng = Rng.keyed(3, "golden", "adamw", tag)
        params = {"a": rng.normal((4, 33)).astype(dt), "b": rng.normal((257,)).astype(dt)}
        out[f"{tag}/p0/a"] = params["a"].copy()
        out[f"{tag}/p0/b"] = params["b"].copy()
        st = adamw_init(params)
        norms = []
        for t in range(5):
            grads = {k: (0.3 * rng.normal(p.shape)).astype(dt) for k, p in params.items()}
            out[f"{tag}/g{t}/a"] = grads["a"].copy()
            out[f"{tag}/g{t}/b"] = grads["b"].copy()
            thr = clip_threshold_at(t, t if t < 3 else None, s)
            norms.append(global_clip(grads, thr))
            adamw_step(params, grads, st, lr_at(t + 10, s, poet=True), s)
            out[f"{tag}/p{t + 1}/a"] = params["a"].copy()
            out[f"{tag}/p{t + 1}/b"] = params["b"].copy()
        out[f"{tag}/norms"] = np.array(norms)
    s = ScheduleConfig(base_lr=0.08, total_steps=3000, warmup_steps=100)
    steps = np.array([0, 1, 50, 99, 100, 101, 500, 1500, 2999, 3000, 4000])
    out["lr"] = np.array([lr_at(int(k), s) for k in steps])
    out["lr_poet"] = np.array([lr_at(int(k), s, poet=True) for k in steps])
    out["lr_steps"] = steps
    out["clip"] = np.array([clip_threshold_at(g, k, s) for g, k in ((500, 0), (500, 5), (500, 10), (1999, 0), (2000, 0))])
    out["clip_none"] = np.array([clip_threshold_at(500, None, s)])
    np.savez_compressed(os.path.join(OUT, "optim.npz"), **out)


if __name__ == "__main__":
    print("reference poetx", poetx.__version__, "numpy", np.__version__)
    cnp_cases()
    perm_cases()
    optim_cases()
    layer_cases()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
