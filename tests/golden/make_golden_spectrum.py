"""Golden vectors for the device spectrum audit from the
REFERENCE.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_spectrum.py

Writes tests/golden/spectrum.npz: svd_singular_values (linalg.py:166-218) of
assorted matrices (square, tall, wide, rank-deficient, a skew block stack),
and the rows of run_spectrum_audit (runner.py:452-529) for small cnp / cayley
configurations in float64 and float32."""

import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from poetx.config import TrainConfig  # noqa: E402  (the reference)
from poetx.linalg import Rng, svd_singular_values  # noqa: E402
from poetx.runner import run_spectrum_audit  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
out = {}
r = Rng.keyed(11, "spectrum")
low = r.normal((40, 6)) @ r.normal((6, 24))
skew = r.normal((5, 16, 16)) * 0.05
skew = skew - skew.transpose(0, 2, 1)
mats = {"square": r.normal((32, 32)), "tall": r.normal((50, 20)), "wide": r.normal((12, 45)),
        "rank6": low, "single": r.normal((7, 1)), "graded": np.diag(np.logspace(0, -8, 10)) @ r.normal((10, 10))}
for k, a in mats.items():
    out[f"a_{k}"] = a
    out[f"sv_{k}"] = svd_singular_values(a)
out["a_skew"] = skew
out["sv_skew"] = np.stack([svd_singular_values(b) for b in skew])

CASES = {
    "cnp64": dict(audit_dim=32, block_size=8, audit_merges=3, audit_steps=3, audit_mode="cnp", precision=64,
                  batch_size=16, seed=3, audit_lr=1e-2),
    "cayley64": dict(audit_dim=32, block_size=8, audit_merges=3, audit_steps=3, audit_mode="cayley", precision=64,
                     batch_size=16, seed=4, audit_lr=1e-2),
    "cnp32": dict(audit_dim=24, block_size=4, audit_merges=2, audit_steps=4, audit_mode="cnp", precision=32,
                  batch_size=8, seed=5, audit_lr=1e-2),
}
audits = {}
for name, kw in CASES.items():
    with tempfile.TemporaryDirectory() as d:
        res = run_spectrum_audit(TrainConfig(out_dir=d, **kw))
        with open(os.path.join(d, "spectrum_audit.csv")) as fh:
            csv_text = fh.read()
    audits[name] = {"config": kw, "rows": res["rows"], "csv": csv_text}
out["audits_json"] = np.frombuffer(json.dumps(audits).encode(), dtype=np.uint8)
np.savez_compressed(os.path.join(OUT, "spectrum.npz"), **out)
print("wrote", os.path.join(OUT, "spectrum.npz"))
