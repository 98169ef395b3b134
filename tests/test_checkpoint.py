"""PXK1 container (checkpoint.py:1-116): byte compatibility with a file the
reference itself wrote (tests/golden/make_golden_pxk1.py), byte-exact round
trips, and the reference's error behaviour; on the GPU, a resumed Llama
training run continues bitwise identically."""

import os

import numpy as np
import pytest

from paper_2603_05500_b200.checkpoint import load_checkpoint, save_checkpoint
from paper_2603_05500_b200.errors import CheckpointError, ShapeError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    with np.load(os.path.join(GOLD, "ref_small_pxk1.npz")) as z:
        tensors = {k: z[k] for k in z.files}
    with open(os.path.join(GOLD, "ref_small_pxk1.txt"), encoding="utf-8") as f:
        cfg = f.read()
    return tensors, cfg


def test_reads_reference_written_file():
    want, cfg = _golden()
    got, text = load_checkpoint(os.path.join(GOLD, "ref_small.pxk1"))
    assert text == cfg
    assert list(got) == list(want)
    for k in want:
        assert got[k].dtype == want[k].dtype and got[k].shape == want[k].shape
        assert got[k].tobytes() == want[k].tobytes()
    assert got["scalar/rank0"].ndim == 0


def test_writes_reference_bytes(tmp_path):
    tensors, cfg = _golden()
    out = tmp_path / "ours.pxk1"
    save_checkpoint(str(out), tensors, cfg)
    with open(os.path.join(GOLD, "ref_small.pxk1"), "rb") as f:
        assert out.read_bytes() == f.read()


def test_roundtrip_and_writable_copies(tmp_path):
    r = np.random.default_rng(0)
    t = {"a": r.standard_normal((3, 4)).astype(np.float32), "b": np.arange(5, dtype=np.uint32),
         "c": np.array([], dtype=np.int8), "d": np.float64(2.5) * np.ones(())}
    p = tmp_path / "sub" / "x.pxk1"
    save_checkpoint(str(p), t, "cfg")
    got, cfg = load_checkpoint(str(p))
    assert cfg == "cfg" and list(got) == list(t)
    for k in t:
        assert got[k].tobytes() == np.asarray(t[k]).tobytes()
    got["a"][0, 0] = 7.0  # writable copy


def test_errors(tmp_path):
    with pytest.raises(ShapeError):
        save_checkpoint(str(tmp_path / "bad.pxk1"), {"x": np.zeros(2, dtype=np.int64)}, "")
    with pytest.raises(CheckpointError, match="not found"):
        load_checkpoint(str(tmp_path / "missing.pxk1"))
    good = tmp_path / "g.pxk1"
    save_checkpoint(str(good), {"x": np.arange(6, dtype=np.float32).reshape(2, 3)}, "c")
    raw = good.read_bytes()
    (tmp_path / "magic.pxk1").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(CheckpointError, match="bad magic"):
        load_checkpoint(str(tmp_path / "magic.pxk1"))
    (tmp_path / "ver.pxk1").write_bytes(raw[:4] + b"\x02\x00" + raw[6:])
    with pytest.raises(CheckpointError, match="unsupported checkpoint version"):
        load_checkpoint(str(tmp_path / "ver.pxk1"))
    for cut in range(1, len(raw)):
        (tmp_path / "cut.pxk1").write_bytes(raw[:cut])
        with pytest.raises(CheckpointError):
            load_checkpoint(str(tmp_path / "cut.pxk1"))
    (tmp_path / "tail.pxk1").write_bytes(raw + b"\x00")
    with pytest.raises(CheckpointError, match="trailing"):
        load_checkpoint(str(tmp_path / "tail.pxk1"))


@pytest.mark.gpu
def test_resume_is_bitwise_identical(tmp_path):
    """Train 6 steps straight, or 3 steps -> PXK1 -> fresh trainer -> 3 steps
    (a merge happens at step 4 in both): identical losses and parameters."""
    import torch

    from paper_2603_05500_b200.trainer import Trainer, llama_config

    cfg = llama_config("llama-60m", layers=2, seq=64)
    toks = [torch.randint(0, cfg.vocab, (4, cfg.seq + 1), generator=torch.Generator().manual_seed(i)).cuda()
            for i in range(6)]
    full = Trainer(cfg, 4, seed=3, merge_gap=4, base_lr=3e-3)
    lf = [float(full.step(t[:, :-1], t[:, 1:])) for t in toks]
    a = Trainer(cfg, 4, seed=3, merge_gap=4, base_lr=3e-3)
    la = [float(a.step(t[:, :-1], t[:, 1:])) for t in toks[:3]]
    a.save_checkpoint(str(tmp_path / "mid.pxk1"), "llama-60m test", tokens=3 * 4 * 64)
    # same config (the merge RNG is keyed on the config seed); all state is
    # scrambled first so everything must come from the file
    b = Trainer(cfg, 4, seed=3, merge_gap=4, base_lr=3e-3)
    for grp in (b.model.poet, b.model.dense):
        for buf in (grp.param, grp.m, grp.v):
            buf.normal_()
    for lay in b.model.poet_layers():
        lay.premerged.normal_()
    tokens, text = b.load_checkpoint(str(tmp_path / "mid.pxk1"))
    assert tokens == 768 and text == "llama-60m test" and b.step_idx == 3
    lb = [float(b.step(t[:, :-1], t[:, 1:])) for t in toks[3:]]
    assert la + lb == lf
    for x, y in ((full.model.poet, b.model.poet), (full.model.dense, b.model.dense)):
        assert torch.equal(x.param, y.param) and torch.equal(x.m, y.m) and torch.equal(x.v, y.v)
    for lx, ly in zip(full.model.poet_layers(), b.model.poet_layers()):
        assert torch.equal(lx.premerged, ly.premerged)
        assert np.array_equal(lx.perm_in.forward, ly.perm_in.forward)
        assert lx.merge_count == ly.merge_count
