"""Golden vectors for POET-XQ (quant.py, layer.py quantized paths) from the
REFERENCE.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_quant.py

Writes tests/golden/quant.npz: per-row quantization of assorted matrices
(codes, scales), and a quantized mem-variant layer's forward, backward and
merge (float32 and float64)."""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from poetx.layer import init_layer  # noqa: E402  (the reference)
from poetx.linalg import Rng  # noqa: E402
from poetx.quant import QuantizedMatrix  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
out = {}
r = Rng.keyed(77, "quant")
mats = {
    "gauss_f32": r.normal((24, 40)).astype(np.float32),
    "gauss_f64": r.normal((16, 33)),
    "ties_f64": np.array([[127.0, 63.5, -63.5, 0.5, -0.5, 1.5, 2.5, 0.0],
                          [0.0] * 8, [1e-30, -2e-30, 3e-30, 0, 0, 0, 0, 0]]),
    "wide_f32": (r.normal((8, 512)) * np.linspace(1e-3, 1e3, 8)[:, None]).astype(np.float32),
}
for tag, w in mats.items():
    q = QuantizedMatrix.quantize(w)
    out[f"q_{tag}_w"] = w
    out[f"q_{tag}_codes"] = q.codes
    out[f"q_{tag}_scales"] = q.scales
for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
    layer = init_layer(32, 48, 8, Rng.keyed(5, "qlayer", tag), dtype=dt, variant="mem")
    out[f"l_{tag}_base"] = layer.base.copy()
    out[f"l_{tag}_perm_in"] = layer.perm_in.forward.astype(np.int32)
    out[f"l_{tag}_perm_out"] = layer.perm_out.forward.astype(np.int32)
    layer.quantize_base()
    prng = Rng.keyed(5, "qpacked", tag)
    layer.q_r.packed[...] = (0.05 * prng.normal(layer.q_r.packed.shape)).astype(dt)
    layer.q_p.packed[...] = (0.05 * prng.normal(layer.q_p.packed.shape)).astype(dt)
    out[f"l_{tag}_q_r"] = layer.q_r.packed.copy()
    out[f"l_{tag}_q_p"] = layer.q_p.packed.copy()
    x = prng.normal((10, 32)).astype(dt)
    dz = prng.normal((10, 48)).astype(dt)
    z, cache = layer.forward(x)
    g = layer.backward(cache, dz)
    out[f"l_{tag}_x"], out[f"l_{tag}_dz"] = x, dz
    out[f"l_{tag}_z"], out[f"l_{tag}_gr"], out[f"l_{tag}_gp"], out[f"l_{tag}_dx"] = z, g.q_r, g.q_p, g.x
    layer.merge_and_reinit(Rng.keyed(5, "qmerge", tag))
    out[f"l_{tag}_merged_codes"] = layer.base.codes
    out[f"l_{tag}_merged_scales"] = layer.base.scales
    out[f"l_{tag}_new_perm_in"] = layer.perm_in.forward.astype(np.int32)
    out[f"l_{tag}_new_perm_out"] = layer.perm_out.forward.astype(np.int32)
np.savez_compressed(os.path.join(OUT, "quant.npz"), **out)
print("wrote quant.npz with", len(out), "arrays")
