"""CPU-side checks of the native library and host logic (no GPU needed):
the C ABI loads and exports every symbol include/poetx_b200.h declares,
the H1 Philox sampler is bit-exact with numpy, host schedules match the
reference's golden values."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import poetx_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "poetx_b200.h")


def _header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(poetx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2603_05500_b200 import _native as N

    lib = N.lib()
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding declares a signature for every one of them
    assert set(syms) == set(N.EXPORTED_SYMBOLS)
    assert lib.poetx_abi_version() == N.ABI_VERSION == 3


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2603_05500_b200", "libpoetx_b200.so")
    blob = open(so, "rb").read()
    assert b"sm_100a" in blob


@pytest.mark.parametrize("n", [1, 2, 3, 16, 64, 512, 2048, 5461, 5632, 14336])
def test_native_permutation_bit_exact_with_numpy(n):
    from paper_2603_05500_b200 import Rng

    for step, idx in ((400, 0), (800, 3), (1200, 17)):
        want = O.numpy_rng(11, O.keyed_stream("merge", step, idx)).permutation(n)
        got = Rng.keyed(11, "merge", step, idx).permutation(n)
        assert np.array_equal(got, want)


def test_native_permutation_shares_stream_with_normal_draws():
    """init_layer draw order: W (gaussian), then pi_in, then pi_out from ONE
    stream (layer.py:335-340, 139-140)."""
    from paper_2603_05500_b200 import Rng

    ref = O.numpy_rng(5, O.keyed_stream("init", "reg", 0))
    mine = Rng.keyed(5, "init", "reg", 0)
    assert np.array_equal(ref.standard_normal((3, 7)), mine.normal((3, 7)))
    for n in (37, 1000, 1):
        assert np.array_equal(ref.permutation(n), mine.permutation(n))
    assert np.array_equal(ref.standard_normal(5), mine.normal(5))


def test_native_permutation_golden():
    from paper_2603_05500_b200 import Rng

    d = dict(np.load(os.path.join(ROOT, "tests", "golden", "perm.npz")))
    for i, n in enumerate((1, 2, 16, 64, 512, 2048, 5632, 5461)):
        got = Rng.keyed(99, "merge", 400 * (i + 1), i).permutation(n)
        assert np.array_equal(got, d[f"merge_{n}"])


def test_sample_permutation_inverse_and_errors():
    from paper_2603_05500_b200 import PermutationMap, Rng, ShapeError, sample_permutation

    pm = sample_permutation(33, Rng(3))
    assert np.array_equal(pm.forward[pm.inverse], np.arange(33))
    assert np.array_equal(PermutationMap.from_forward([2, 0, 1]).inverse, [1, 2, 0])
    with pytest.raises(ShapeError):
        sample_permutation(0, Rng(0))
    with pytest.raises(ShapeError):
        PermutationMap.from_forward([0, 0, 2])


def test_schedule_matches_reference_golden():
    from paper_2603_05500_b200 import ScheduleConfig, clip_threshold_at, lr_at

    d = dict(np.load(os.path.join(ROOT, "tests", "golden", "optim.npz")))
    s = ScheduleConfig(base_lr=0.08, total_steps=3000, warmup_steps=100)
    assert [lr_at(int(k), s) for k in d["lr_steps"]] == list(d["lr"])
    assert [lr_at(int(k), s, poet=True) for k in d["lr_steps"]] == list(d["lr_poet"])
    got = [clip_threshold_at(g, k, s) for g, k in ((500, 0), (500, 5), (500, 10), (1999, 0), (2000, 0))]
    assert got == list(d["clip"])
    assert clip_threshold_at(500, None, s) == d["clip_none"][0]


def test_error_codes_map_to_reference_exceptions():
    from paper_2603_05500_b200 import _native as N
    from paper_2603_05500_b200.errors import ConfigError, ShapeError

    st = N.PhiloxState()
    with pytest.raises(ShapeError):
        N.call("poetx_philox_permutation", ctypes.byref(st), 0, None, None)
    d = N.LayerDesc()
    d.dtype, d.variant, d.neumann_k, d.m, d.n, d.b = 0, 0, 3, 10, 8, 4
    with pytest.raises(ConfigError, match="divisible by block_size"):
        N.call("poetx_layer_factors", d, N.LayerFactors(), None, 0, None)


def test_quantized_descriptor_requires_mem_variant():
    """POET-XQ is mem-variant only (layer.py:169-177): the C ABI rejects a
    quantized descriptor on the fast variant with the reference's error."""
    from paper_2603_05500_b200 import _native as N
    from paper_2603_05500_b200.errors import ConfigError

    d = N.LayerDesc()
    d.dtype, d.variant, d.neumann_k, d.m, d.n, d.b = N.F32, N.FAST, 3, 8, 8, 4
    d.pm_codes, d.pm_scales = 16, 16  # any non-NULL pointers: validation fails first
    with pytest.raises(ConfigError, match="quantized base requires the mem variant"):
        N.call("poetx_layer_factors", d, N.LayerFactors(), None, 0, None)


def test_weight_folding_rule(monkeypatch):
    """Reassociated products only where they measured faster:
    Llama-1B at 8192 tokens; not Llama-350M, not Llama-8B at 1024 tokens;
    POETX_REASSOC forces either way."""
    from paper_2603_05500_b200.trainer import llama_config, weight_folding_pays

    monkeypatch.delenv("POETX_REASSOC", raising=False)
    assert weight_folding_pays(llama_config("llama-1b"), 32)
    assert not weight_folding_pays(llama_config("llama-350m"), 32)
    assert not weight_folding_pays(llama_config("llama-8b"), 1)
    assert weight_folding_pays(llama_config("llama-8b"), 8)
    monkeypatch.setenv("POETX_REASSOC", "0")
    assert not weight_folding_pays(llama_config("llama-1b"), 32)
    monkeypatch.setenv("POETX_REASSOC", "1")
    assert weight_folding_pays(llama_config("llama-350m"), 32)
