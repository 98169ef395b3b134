"""Keyed counter-based RNG with the reference's semantics
(linalg.py:264-294 `Rng`).

Normal draws (init-time weights, host data) come from numpy's
Generator(Philox) exactly as in the reference.  Permutations -- the
quantity that must be bit-exact on the training path -- are drawn by the
native H1 sampler (csrc/philox.cpp) from the same Philox state, which is
synchronised back into the numpy generator so interleaved draws keep one
stream, as in the reference (layer.py:335-340: W, then pi_in, then pi_out).
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np

from . import _native as N

_MASK64 = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int, stream: int = 0):
        self.seed = int(seed) & _MASK64
        self.stream = int(stream) & _MASK64
        key = np.array([self.seed, self.stream], dtype=np.uint64)
        self._gen = np.random.Generator(np.random.Philox(key=key))

    @classmethod
    def keyed(cls, seed: int, *tags) -> "Rng":
        text = "/".join(str(t) for t in tags)
        digest = hashlib.blake2b(text.encode("utf-8"), digest_size=8).digest()
        return cls(seed, int.from_bytes(digest, "little"))

    def normal(self, shape) -> np.ndarray:
        """Standard normal draws, always float64 (host)."""
        return self._gen.standard_normal(shape)

    def integers(self, low: int, high: int, size=None) -> np.ndarray:
        return self._gen.integers(low, high, size=size)

    # -- native permutation sampling --------------------------------------------

    def permutation_with_inverse(self, n: int):
        return native_permutation(self._gen, n)

    def permutation(self, n: int) -> np.ndarray:
        """Same values as numpy's Generator.permutation(n) (int64)."""
        return self.permutation_with_inverse(n)[0].astype(np.int64)


def _export(gen: np.random.Generator) -> N.PhiloxState:
    s = gen.bit_generator.state
    st = N.PhiloxState()
    for i in range(4):
        st.counter[i] = int(s["state"]["counter"][i])
        st.buffer[i] = int(s["buffer"][i])
    st.key[0] = int(s["state"]["key"][0])
    st.key[1] = int(s["state"]["key"][1])
    st.buffer_pos = int(s["buffer_pos"])
    st.has_uint32 = int(s["has_uint32"])
    st.uinteger = int(s["uinteger"])
    return st


def _import(gen: np.random.Generator, st: N.PhiloxState) -> None:
    gen.bit_generator.state = {
        "bit_generator": "Philox",
        "state": {
            "counter": np.array([st.counter[i] for i in range(4)], dtype=np.uint64),
            "key": np.array([st.key[0], st.key[1]], dtype=np.uint64),
        },
        "buffer": np.array([st.buffer[i] for i in range(4)], dtype=np.uint64),
        "buffer_pos": int(st.buffer_pos),
        "has_uint32": int(st.has_uint32),
        "uinteger": int(st.uinteger),
    }


def is_philox(gen) -> bool:
    return isinstance(gen, np.random.Generator) and isinstance(gen.bit_generator, np.random.Philox)


def native_permutation(gen: np.random.Generator, n: int):
    """Generator.permutation(n) of a numpy Philox generator, drawn by the
    native H1 sampler from (and written back into) the generator's state:
    bit-exact with numpy, so a reference ``poetx.linalg.Rng`` (whose
    ``_gen`` is such a generator) can be passed to this package directly.
    Returns (forward, inverse) int32."""
    n = int(n)
    fwd = np.empty(max(n, 0), dtype=np.int32)
    inv = np.empty(max(n, 0), dtype=np.int32)
    st = _export(gen)
    N.call("poetx_philox_permutation", C.byref(st), n, fwd.ctypes.data, inv.ctypes.data)
    _import(gen, st)
    return fwd, inv
