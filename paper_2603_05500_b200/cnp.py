"""Cayley-Neumann parameterization on the GPU (reference cnp.py).

Packed strict-upper-triangle skew parameters (row-major pair order,
cnp.py:66-68) unpack to Q; the factor is G = (I + Q)(I + sum_{i<=k} Q^i),
for k = 3 regrouped as G = 2(Q + Q^2 + Q^2 Q) + Q^2 Q^2 + I (three block
products, Q^2 cached) with the six-product closed-form backward
(cnp.py:128-145).  All arithmetic runs in libpoetx_b200 kernels; numpy
inputs are accepted for drop-in use and come back as numpy.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, ShapeError


def num_pairs(block_dim: int) -> int:
    return block_dim * (block_dim - 1) // 2


def _to_dev(a, dtype=None):
    if isinstance(a, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        return (t if dtype is None else t.to(dtype)), True
    return a, False


def _out(t, was_np):
    return t.cpu().numpy() if was_np else t


@dataclass
class SkewParams:
    """Packed skew-symmetric parameters for a stack of blocks (cnp.py:42-59).
    ``packed`` (num_blocks, b(b-1)/2) is a device tensor, or a host numpy
    array kept as is (numpy-constructed layers: the optimizer and the caller
    mutate it in place, as with the reference)."""

    num_blocks: int
    block_dim: int
    packed: torch.Tensor

    def __post_init__(self):
        want = (self.num_blocks, num_pairs(self.block_dim))
        if tuple(self.packed.shape) != want:
            raise ShapeError(f"packed shape {tuple(self.packed.shape)}, expected {want}")

    @classmethod
    def zeros(cls, num_blocks: int, block_dim: int, dtype=torch.float64, device="cuda") -> "SkewParams":
        if num_blocks < 1 or block_dim < 1:
            raise ShapeError(f"bad block layout ({num_blocks}, {block_dim})")
        return cls(num_blocks, block_dim,
                   torch.zeros((num_blocks, num_pairs(block_dim)), dtype=dtype, device=device))


def _pdtype(t: torch.Tensor) -> int:
    if t.dtype not in (torch.float32, torch.float64):
        raise ShapeError(f"CNP dtype must be float32 or float64, got {t.dtype}")
    return N.dtype_code(t.dtype)


def skew_from_packed(params: SkewParams):
    """Unpack to a (num_blocks, b, b) skew-symmetric stack (cnp.py:71-78)."""
    p, was_np = _to_dev(params.packed)
    p = p.contiguous()
    b = params.block_dim
    q = torch.empty((params.num_blocks, b, b), dtype=p.dtype, device=p.device)
    N.call("poetx_skew_from_packed", _pdtype(p), params.num_blocks, b, p.data_ptr(), q.data_ptr(),
           N.stream_ptr(p.device))
    return _out(q, was_np)


def packed_grad_from_skew_grad(dq):
    """g_ij = dQ_ij - dQ_ji (cnp.py:81-86)."""
    dq, was_np = _to_dev(dq)
    if dq.ndim != 3 or dq.shape[1] != dq.shape[2]:
        raise ShapeError(f"expected a square block stack, got {tuple(dq.shape)}")
    nb, b, _ = dq.shape
    g = torch.empty((nb, num_pairs(b)), dtype=dq.dtype, device=dq.device)
    N.call("poetx_packed_grad_from_skew_grad", _pdtype(dq), nb, b, dq.contiguous().data_ptr(),
           g.data_ptr(), 0, N.stream_ptr(dq.device))
    return _out(g, was_np)


@dataclass
class CnpCache:
    """Saved operands for the backward pass (cnp.py:89-96)."""

    k: int
    q: torch.Tensor
    qsq: torch.Tensor | None  # k == 3 fast path
    powers: list | None = None  # generic path: recomputed on device from q


def cnp_forward(q, neumann_k: int = 3):
    """Blockwise truncated Cayley transform -> (g, cache) (cnp.py:99-125)."""
    q, was_np = _to_dev(q)
    if q.ndim != 3 or q.shape[1] != q.shape[2]:
        raise ShapeError(f"expected a square block stack, got {tuple(q.shape)}")
    if neumann_k < 1:
        raise ConfigError(f"neumann_k must be >= 1, got {neumann_k}")
    q = q.contiguous()
    nb, b, _ = q.shape
    dt = _pdtype(q)
    g = torch.empty_like(q)
    qsq = torch.empty_like(q) if neumann_k == 3 else None
    ws, wsb = N.workspace(N.lib().poetx_cnp_workspace_bytes(dt, nb, b, neumann_k), q.device)
    N.call("poetx_cnp_forward", dt, nb, b, neumann_k, q.data_ptr(), None, g.data_ptr(), None,
           N.ptr(qsq), ws, wsb, N.stream_ptr(q.device))
    cache = CnpCache(k=neumann_k, q=q, qsq=qsq)
    if was_np:
        return g.cpu().numpy(), cache
    return g, cache


def cnp_backward(cache: CnpCache, dg):
    """Adjoint w.r.t. the full Q stack (cnp.py:128-158); project with
    packed_grad_from_skew_grad."""
    dg, was_np = _to_dev(dg)
    if tuple(dg.shape) != tuple(cache.q.shape):
        raise ShapeError(f"cotangent shape {tuple(dg.shape)} does not match Q {tuple(cache.q.shape)}")
    q = cache.q
    nb, b, _ = q.shape
    dt = _pdtype(q)
    dg = dg.to(q.dtype).contiguous()
    dq = torch.empty_like(q)
    ws, wsb = N.workspace(N.lib().poetx_cnp_workspace_bytes(dt, nb, b, cache.k), q.device)
    N.call("poetx_cnp_backward", dt, nb, b, cache.k, q.data_ptr(), None, N.ptr(cache.qsq),
           dg.data_ptr(), dq.data_ptr(), None, 0, ws, wsb, N.stream_ptr(q.device))
    return _out(dq, was_np)


def cayley_exact(q):
    """Exact Cayley transform (I + Q)(I - Q)^{-1}, blockwise, solved in float64
    (cnp.py:161-176).  Audit / merge-hook only: uses torch.linalg.solve."""
    q, was_np = _to_dev(q)
    if q.ndim != 3 or q.shape[1] != q.shape[2]:
        raise ShapeError(f"expected a square block stack, got {tuple(q.shape)}")
    q64 = q.to(torch.float64)
    eye = torch.eye(q.shape[1], dtype=torch.float64, device=q.device).expand_as(q64)
    lhs = (eye - q64).transpose(1, 2)
    rhs = (eye + q64).transpose(1, 2)
    sol = torch.linalg.solve(lhs, rhs).transpose(1, 2).contiguous().to(q.dtype)
    return _out(sol, was_np)


# ----------------------------------------------------- BF16 tensor-core path --


def cnp_forward_tc(packed: torch.Tensor, block_dim: int, want_fp32: bool = False):
    """Tensor-core CNP (k = 3) for the BF16 path over a whole stack of blocks:
    packed fp32 (nb, b(b-1)/2) -> (G bf16 (nb, b, b), cache [Q | Q^2] bf16,
    G fp32 or None).  Same algebra as cnp_forward (cnp.py:109-116)."""
    if packed.dtype != torch.float32 or packed.ndim != 2 or packed.shape[1] != num_pairs(block_dim):
        raise ShapeError(f"packed must be float32 (nb, {num_pairs(block_dim)}), got {tuple(packed.shape)}")
    nb, b = packed.shape[0], block_dim
    dev = packed.device
    qq2 = torch.empty((nb, b, 2 * b), dtype=torch.bfloat16, device=dev)
    g16 = torch.empty((nb, b, b), dtype=torch.bfloat16, device=dev)
    g32 = torch.empty((nb, b, b), dtype=torch.float32, device=dev) if want_fp32 else None
    ws, wsb = N.workspace(N.lib().poetx_cnp_tc_workspace_bytes(nb, b), dev)
    N.call("poetx_cnp_forward_tc", nb, b, packed.contiguous().data_ptr(), qq2.data_ptr(), g16.data_ptr(),
           N.ptr(g32), ws, wsb, N.stream_ptr(dev))
    return g16, qq2, g32


def cnp_backward_tc(qq2: torch.Tensor, dg: torch.Tensor, out: torch.Tensor | None = None,
                    accumulate: bool = False) -> torch.Tensor:
    """Tensor-core closed-form backward (cnp.py:136-145 regrouped) fused with
    the packed projection (cnp.py:81-86): dG fp32 (nb, b, b) -> packed grad."""
    nb, b, _ = qq2.shape
    if tuple(dg.shape) != (nb, b, b) or dg.dtype != torch.float32:
        raise ShapeError(f"dG must be float32 {(nb, b, b)}, got {tuple(dg.shape)} {dg.dtype}")
    if out is None:
        out = torch.empty((nb, num_pairs(b)), dtype=torch.float32, device=qq2.device)
    ws, wsb = N.workspace(N.lib().poetx_cnp_tc_workspace_bytes(nb, b), qq2.device)
    N.call("poetx_cnp_backward_tc", nb, b, qq2.data_ptr(), dg.contiguous().data_ptr(), out.data_ptr(),
           int(accumulate), ws, wsb, N.stream_ptr(qq2.device))
    return out
