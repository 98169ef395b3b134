"""Device spectrum audit (csrc/svd.cu, audit.py) against
golden vectors the reference produced (tests/golden/make_golden_spectrum.py):
Jacobi singular values, the ConvergenceError contract, and the rows of
run_spectrum_audit for CNP and exact-Cayley merges in float64 and float32."""

import json
import os
import types

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spectrum.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.mark.parametrize("tag", ["square", "tall", "wide", "rank6", "single", "graded"])
def test_singular_values_match_reference(gold, tag):
    from paper_2603_05500_b200 import singular_values

    a, ref = gold[f"a_{tag}"], gold[f"sv_{tag}"]
    sv = singular_values(torch.from_numpy(a).cuda()).cpu().numpy()
    assert sv.shape == ref.shape
    # different (round-robin) pair order: equal to the Jacobi tolerance
    assert np.max(np.abs(sv - ref)) <= 1e-10 * max(1.0, ref[0]), np.max(np.abs(sv - ref))


def test_singular_values_batched_skew_blocks(gold):
    from paper_2603_05500_b200 import singular_values, spectral_norm

    a, ref = gold["a_skew"], gold["sv_skew"]
    sv = singular_values(a).cpu().numpy()
    assert np.max(np.abs(sv - ref)) <= 1e-12
    assert abs(spectral_norm(a) - ref[:, 0].max()) <= 1e-12


def test_singular_values_float32_input_and_empty():
    from paper_2603_05500_b200 import singular_values

    a = torch.randn(20, 9, device="cuda")
    ref = np.linalg.svd(a.double().cpu().numpy(), compute_uv=False)
    assert np.max(np.abs(singular_values(a).cpu().numpy() - ref)) <= 1e-10 * ref[0]
    assert singular_values(torch.zeros(5, 0, device="cuda")).shape == (0,)


def test_singular_values_convergence_error():
    from paper_2603_05500_b200 import ConvergenceError, singular_values

    a = torch.randn(48, 48, dtype=torch.float64, device="cuda")
    with pytest.raises(ConvergenceError) as e:
        singular_values(a, max_sweeps=1)
    assert e.value.residual > 1e-10


def _cfg(kw, out_dir):
    base = dict(variant="fast", neumann_k=3, base_lr=5e-4, total_steps=1000, warmup_steps=100, min_lr_ratio=0.01,
                poet_lr_scale=0.5, weight_decay=0.01, clip_norm=1.0, post_merge_clip_start=0.01,
                post_merge_clip_ramp=10, post_merge_clip_window=2000, adam_beta1=0.9, adam_beta2=0.999,
                adam_eps=1e-8, out_dir=str(out_dir))
    base.update(kw)
    return types.SimpleNamespace(**base)


@pytest.mark.parametrize("case", ["cnp64", "cayley64", "cnp32"])
def test_spectrum_audit_matches_reference(gold, case, tmp_path):
    from paper_2603_05500_b200 import spectrum_audit

    audits = json.loads(bytes(gold["audits_json"]).decode())
    ref = audits[case]
    res = spectrum_audit(_cfg(ref["config"], tmp_path), verbose=False)
    f64 = ref["config"]["precision"] == 64
    rtol, atol = (1e-6, 1e-12) if f64 else (5e-3, 1e-6)
    assert len(res["rows"]) == len(ref["rows"])
    for got, want in zip(res["rows"], ref["rows"]):
        assert got["merge"] == want["merge"]
        for key in ("loss", "max_q_norm", "orth_err_r", "orth_err_p", "per_merge_drift", "cumulative_drift"):
            g, w = got[key], want[key]
            assert abs(g - w) <= atol + rtol * abs(w), (case, got["merge"], key, g, w)
    with open(res["report_path"]) as fh:
        lines = fh.read().splitlines()
    ref_lines = ref["csv"].splitlines()
    assert lines[0] == ref_lines[0] and len(lines) == len(ref_lines)
