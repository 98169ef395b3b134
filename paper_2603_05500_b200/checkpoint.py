"""PXK1 checkpoint container and training-state (de)serialisation
(SURVEY §8f-2), byte-compatible with the reference (checkpoint.py:1-116,
runner.py:144-228).

Container, little-endian: b"PXK1", u16 version (1), u32 config length +
UTF-8 config text, u32 tensor count, then per tensor: u16 name length +
UTF-8 name, u8 dtype code (0 f64, 1 f32, 2 i8, 3 u32), u8 ndim, u64 dims,
raw C-order data.  Round trips are byte-exact and keep tensor order.

Tensor names follow the reference's runner: ``progress/*``, ``param/<name>``,
``layer/<name>/{base,perm_in,perm_out,merge_count}``,
``opt/{poet,dense}/{t,m/<name>,v/<name>}``.  The device keeps only the
premerged bf16 weight; ``base`` is recovered by the exact inverse gather
``W[r, c] = PM[pi_in^-1(r), pi_out^-1(c)]`` and stored as float32 (every
bf16 value is exact in float32), so save -> load -> premerge reproduces the
device weight bit for bit and a resumed run continues bitwise identically.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .errors import CheckpointError, ShapeError
from .permute import PermutationMap

MAGIC = b"PXK1"
VERSION = 1
NO_MERGE = 0xFFFFFFFF  # steps_since_merge before the first merge (runner.py:45)

_DTYPES = ((np.dtype("<f8"), 0), (np.dtype("<f4"), 1), (np.dtype("i1"), 2), (np.dtype("<u4"), 3))
_CODE = {dt: code for dt, code in _DTYPES}
_FROM_CODE = {code: dt for dt, code in _DTYPES}


def _host(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        a = a.detach()
        if a.dtype == torch.bfloat16:
            a = a.float()
        a = a.cpu().numpy()
    return np.asarray(a)


def save_checkpoint(path: str, tensors: dict, config_text: str) -> None:
    """Write a PXK1 file (numpy arrays or torch tensors; bf16 is widened to f32)."""
    parts = [MAGIC, struct.pack("<H", VERSION)]
    cfg = config_text.encode("utf-8")
    parts += [struct.pack("<I", len(cfg)), cfg, struct.pack("<I", len(tensors))]
    for name, value in tensors.items():
        arr = _host(value)
        code = _CODE.get(arr.dtype.newbyteorder("<") if arr.dtype.byteorder == ">" else arr.dtype)
        if code is None:
            raise ShapeError(f"tensor {name!r} has unsupported dtype {arr.dtype}")
        key = name.encode("utf-8")
        parts += [struct.pack("<H", len(key)), key, struct.pack("<BB", code, arr.ndim),
                  struct.pack(f"<{arr.ndim}Q", *arr.shape),
                  np.ascontiguousarray(arr, dtype=_FROM_CODE[code]).tobytes()]
    out = Path(path)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_bytes(b"".join(parts))


def load_checkpoint(path: str):
    """-> (dict of numpy arrays in stored order, config text)."""
    p = Path(path)
    if not p.is_file():
        raise CheckpointError(f"checkpoint not found: {path}")
    raw = memoryview(p.read_bytes())
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(raw):
            raise CheckpointError(f"truncated checkpoint: {path}")
        out = raw[pos:pos + n]
        pos += n
        return out

    def unpack(fmt):
        return struct.unpack(fmt, take(struct.calcsize(fmt)))

    if bytes(take(4)) != MAGIC:
        raise CheckpointError(f"bad magic in {path}; not a checkpoint file")
    (version,) = unpack("<H")
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version} in {path}")
    (cfg_len,) = unpack("<I")
    config_text = bytes(take(cfg_len)).decode("utf-8")
    (count,) = unpack("<I")
    tensors = {}
    for _ in range(count):
        (name_len,) = unpack("<H")
        name = bytes(take(name_len)).decode("utf-8")
        code, ndim = unpack("<BB")
        if code not in _FROM_CODE:
            raise CheckpointError(f"unknown dtype code {code} for tensor {name!r} in {path}")
        dims = unpack(f"<{ndim}Q") if ndim else ()
        dt = _FROM_CODE[code]
        size = int(np.prod(dims, dtype=np.int64)) * dt.itemsize
        tensors[name] = np.frombuffer(take(size), dtype=dt).reshape(dims).copy()
    if pos != len(raw):
        raise CheckpointError(f"trailing bytes after tensor table in {path}")
    return tensors, config_text


# ------------------------------------------------------------ layer state --


def _get(tensors: dict, name: str) -> np.ndarray:
    if name not in tensors:
        raise CheckpointError(f"checkpoint missing tensor {name!r}")
    return tensors[name]


def _restore(dst: torch.Tensor, name: str, tensors: dict) -> None:
    src = _get(tensors, name)
    want = tuple(dst.shape)
    if tuple(src.shape) != want or src.dtype != np.dtype(str(dst.dtype).replace("torch.", "")):
        raise CheckpointError(f"tensor {name!r} mismatch: stored {src.dtype}{src.shape}, "
                              f"expected {dst.dtype}{want}")
    dst.copy_(torch.from_numpy(src))


def unpermuted_weight(premerged: torch.Tensor, perm_in: PermutationMap, perm_out: PermutationMap) -> torch.Tensor:
    """W[r, c] = PM[pi_in^-1(r), pi_out^-1(c)] (exact gather, same dtype)."""
    m, n = premerged.shape
    ri, ci = perm_in.device(premerged.device)[1], perm_out.device(premerged.device)[1]
    w = torch.empty_like(premerged)
    N.call("poetx_gather2d", N.dtype_code(premerged.dtype), m, n, ri.data_ptr(), ci.data_ptr(),
           premerged.data_ptr(), w.data_ptr(), N.stream_ptr(premerged.device))
    return w


def trainer_tensors(trainer, tokens: int = 0, sv_drift: float = 0.0) -> dict:
    """The Llama trainer's full training state under the reference's names."""
    model = trainer.model
    since = NO_MERGE if trainer.since_merge is None else trainer.since_merge
    t = {
        "progress/step": np.array([trainer.step_idx], dtype=np.uint32),
        "progress/tokens": np.array([tokens], dtype=np.uint32),
        "progress/steps_since_merge": np.array([since], dtype=np.uint32),
        "progress/sv_drift": np.array([sv_drift], dtype=np.float64),
    }
    for tag, grp, name, off, n, shape in _named_slices(model):
        t[f"param/{name}"] = grp.param[off:off + n].view(shape)
    for lay in model.poet_layers():
        key = f"layer/{lay.name}"
        if getattr(lay, "quantized", False):  # W's codes / scales (runner.py:159-161)
            ri, ci = lay.perm_in.device(lay.device)[1], lay.perm_out.device(lay.device)[1]
            codes = torch.empty_like(lay.codes)
            scales = torch.empty_like(lay.scales)
            N.call("poetx_quant_gather", N.BF16, lay.m, lay.n, lay.n, ri.data_ptr(), ci.data_ptr(), lay.codes.data_ptr(),
                   lay.scales.data_ptr(), codes.data_ptr(), scales.data_ptr(), N.stream_ptr(lay.device))
            t[f"{key}/base_codes"] = codes
            t[f"{key}/base_scales"] = scales
        else:
            t[f"{key}/base"] = unpermuted_weight(lay.premerged, lay.perm_in, lay.perm_out)
        t[f"{key}/perm_in"] = lay.perm_in.forward.astype(np.uint32)
        t[f"{key}/perm_out"] = lay.perm_out.forward.astype(np.uint32)
        t[f"{key}/merge_count"] = np.array([lay.merge_count], dtype=np.uint32)
    # moments keyed by the parameter name with the parameter's shape, as the
    # reference's AdamWState dicts are (runner.py:166-172)
    t["opt/poet/t"] = np.array([model.poet.t], dtype=np.uint32)
    t["opt/dense/t"] = np.array([model.dense.t], dtype=np.uint32)
    for tag, grp, name, off, n, shape in _named_slices(model):
        t[f"opt/{tag}/m/{name}"] = grp.m[off:off + n].view(shape)
    for tag, grp, name, off, n, shape in _named_slices(model):
        t[f"opt/{tag}/v/{name}"] = grp.v[off:off + n].view(shape)
    return t


def _named_slices(model):
    """(group tag, FlatGroup, reference parameter name, offset, numel, shape)
    for every trainable tensor: POET packed stacks as ``<layer>.q_r`` /
    ``<layer>.q_p`` (nb, pairs); dense tensors with their 2-D shapes."""
    out = []
    for lay in model.poet_layers():
        for side, packed in (("r", lay.packed_r), ("p", lay.packed_p)):
            off, n = model.poet.offsets[f"{lay.name}.{side}"]
            out.append(("poet", model.poet, f"{lay.name}.q_{side}", off, n, tuple(packed.shape)))
    d = model.cfg.d
    for name, (off, n) in model.dense.offsets.items():
        shape = (n // d, d) if name in ("embed", "head") else (n,)
        out.append(("dense", model.dense, name, off, n, shape))
    return out


def restore_trainer(trainer, tensors: dict) -> int:
    """Install a state written by ``trainer_tensors`` (same model shape);
    returns the stored token count."""
    model = trainer.model
    for tag, grp, name, off, n, shape in _named_slices(model):
        _restore(grp.param[off:off + n].view(shape), f"param/{name}", tensors)
    for lay in model.poet_layers():
        key = f"layer/{lay.name}"
        pin = PermutationMap.from_forward(_get(tensors, f"{key}/perm_in").astype(np.int32))
        pout = PermutationMap.from_forward(_get(tensors, f"{key}/perm_out").astype(np.int32))
        if getattr(lay, "quantized", False):
            codes, scales = tensors.get(f"{key}/base_codes"), tensors.get(f"{key}/base_scales")
            if codes is None or scales is None:
                raise CheckpointError(f"checkpoint missing quantized base for {lay.name}")
            lay.install_quantized(torch.from_numpy(codes), torch.from_numpy(scales), pin, pout)
        else:
            base = _get(tensors, f"{key}/base")
            if base.shape != (lay.m, lay.n):
                raise CheckpointError(f"tensor {key}/base mismatch: stored {base.shape}, expected {(lay.m, lay.n)}")
            lay.install(torch.from_numpy(base).to(lay.device).to(torch.bfloat16), pin, pout)
        lay.merge_count = int(_get(tensors, f"{key}/merge_count")[0])
    model.refresh_maps()
    for tag, grp in (("poet", model.poet), ("dense", model.dense)):
        grp.t = int(_get(tensors, f"opt/{tag}/t")[0])
    for tag, grp, name, off, n, shape in _named_slices(model):
        _restore(grp.m[off:off + n].view(shape), f"opt/{tag}/m/{name}", tensors)
        _restore(grp.v[off:off + n].view(shape), f"opt/{tag}/v/{name}", tensors)
    trainer.step_idx = int(_get(tensors, "progress/step")[0])
    since = int(_get(tensors, "progress/steps_since_merge")[0])
    trainer.since_merge = None if since == NO_MERGE else since
    return int(_get(tensors, "progress/tokens")[0])
