"""Golden PXK1 file written by the REFERENCE's save_checkpoint
(checkpoint.py:41-65), for the byte-compatibility tests of
paper_2603_05500_b200.checkpoint.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_pxk1.py

Writes tests/golden/ref_small.pxk1 and the same tensors (in order) to
tests/golden/ref_small_pxk1.npz, plus the config text to .txt."""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from poetx.checkpoint import save_checkpoint  # noqa: E402  (the reference)

OUT = os.path.dirname(os.path.abspath(__file__))
r = np.random.default_rng(2603)
tensors = {
    "progress/step": np.array([40], dtype=np.uint32),
    "progress/steps_since_merge": np.array([0xFFFFFFFF], dtype=np.uint32),
    "progress/sv_drift": np.array([1.5e-4], dtype=np.float64),
    "param/layer0.q_r": r.standard_normal((2, 6)).astype(np.float32),
    "param/embed": r.standard_normal((5, 3)),
    "layer/layer0/base_codes": r.integers(-127, 128, size=(4, 8)).astype(np.int8),
    "layer/layer0/perm_in": r.permutation(8).astype(np.uint32),
    "scalar/rank0": np.asarray(np.float32(3.25)),
    "empty/zero_len": np.zeros((0, 4), dtype=np.float32),
}
config = "run: ünicode ✓\nblock_size = 4\n"
save_checkpoint(os.path.join(OUT, "ref_small.pxk1"), tensors, config)
np.savez(os.path.join(OUT, "ref_small_pxk1.npz"), **tensors)
with open(os.path.join(OUT, "ref_small_pxk1.txt"), "w", encoding="utf-8") as f:
    f.write(config)
print("wrote ref_small.pxk1", os.path.getsize(os.path.join(OUT, "ref_small.pxk1")), "bytes")
