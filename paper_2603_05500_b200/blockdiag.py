"""Block-diagonal factors applied segmentwise on the GPU (reference
blockdiag.py).  The dim x dim matrix is never assembled on live paths;
``assemble_dense`` exists for tests only."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ShapeError


def _to_dev(a):
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a)).cuda(), True
    return a, False


def _out(t, was_np):
    return t.cpu().numpy() if was_np else t


@dataclass(frozen=True)
class BlockDiagonalFactor:
    """Stack of (num_blocks, b, b) diagonal blocks (blockdiag.py:25-48)."""

    blocks: torch.Tensor

    def __post_init__(self):
        b = self.blocks
        if isinstance(b, np.ndarray):
            object.__setattr__(self, "blocks", torch.from_numpy(np.ascontiguousarray(b)).cuda())
            b = self.blocks
        if not isinstance(b, torch.Tensor) or b.ndim != 3 or b.shape[1] != b.shape[2]:
            raise ShapeError(
                f"blocks must be a (num_blocks, b, b) stack, got {getattr(b, 'shape', None)}")
        if b.shape[0] < 1 or b.shape[1] < 1:
            raise ShapeError(f"empty factor stack {tuple(b.shape)}")

    @property
    def num_blocks(self) -> int:
        return int(self.blocks.shape[0])

    @property
    def block_dim(self) -> int:
        return int(self.blocks.shape[1])

    @property
    def dim(self) -> int:
        return self.num_blocks * self.block_dim


def apply_to_features(factor: BlockDiagonalFactor, x, transpose: bool = False):
    """Segment s of each row maps through block s (or its transpose)
    (blockdiag.py:58-73)."""
    x, was_np = _to_dev(x)
    if x.ndim != 2 or x.shape[1] != factor.dim:
        raise ShapeError(f"activation shape {tuple(x.shape)} does not match factor dim {factor.dim}")
    g = factor.blocks.to(x.dtype).contiguous()
    x = x.contiguous()
    y = torch.empty_like(x)
    N.call("poetx_apply_to_features", N.dtype_code(x.dtype), x.shape[0], factor.num_blocks,
           factor.block_dim, g.data_ptr(), int(transpose), x.data_ptr(), y.data_ptr(),
           N.stream_ptr(x.device))
    return _out(y, was_np)


def apply_to_weight_rows(factor: BlockDiagonalFactor, w, transpose: bool = False):
    """Left multiply w by the factor, segmenting rows (blockdiag.py:76-90)."""
    w, was_np = _to_dev(w)
    if w.ndim != 2 or w.shape[0] != factor.dim:
        raise ShapeError(f"weight shape {tuple(w.shape)} does not match factor dim {factor.dim}")
    g = factor.blocks.to(w.dtype).contiguous()
    w = w.contiguous()
    y = torch.empty_like(w)
    N.call("poetx_apply_to_weight_rows", N.dtype_code(w.dtype), factor.num_blocks,
           factor.block_dim, w.shape[1], g.data_ptr(), int(transpose), w.data_ptr(), y.data_ptr(),
           N.stream_ptr(w.device))
    return _out(y, was_np)


def apply_to_weight_cols(factor: BlockDiagonalFactor, w, transpose: bool = False):
    """Right multiply w by the factor, segmenting columns (blockdiag.py:93-97)."""
    w, was_np = _to_dev(w)
    if w.ndim != 2 or w.shape[1] != factor.dim:
        raise ShapeError(f"weight shape {tuple(w.shape)} does not match factor dim {factor.dim}")
    return _out(apply_to_features(factor, w, transpose=transpose), was_np)


def segmented_outer(x, y, block_dim: int):
    """out[s] = x_s.T @ y_s over the batch (blockdiag.py:100-121);
    deterministic split-batch reduction.  BF16 inputs give fp32 output."""
    x, was_np = _to_dev(x)
    y, _ = _to_dev(y)
    if x.ndim != 2 or y.ndim != 2 or x.shape[0] != y.shape[0]:
        raise ShapeError(f"batch shapes incompatible: {tuple(x.shape)} vs {tuple(y.shape)}")
    if x.shape[1] % block_dim or y.shape[1] % block_dim:
        raise ShapeError(f"feature dims {x.shape[1]}, {y.shape[1]} not divisible by {block_dim}")
    if x.shape[1] != y.shape[1]:
        raise ShapeError(f"feature dims differ: {x.shape[1]} vs {y.shape[1]}")
    if x.dtype != y.dtype:
        raise ShapeError(f"dtype mismatch: {x.dtype} vs {y.dtype}")
    nb = x.shape[1] // block_dim
    T = x.shape[0]
    dt = N.dtype_code(x.dtype)
    out_dtype = torch.float64 if x.dtype == torch.float64 else torch.float32
    out = torch.empty((nb, block_dim, block_dim), dtype=out_dtype, device=x.device)
    ws, wsb = N.workspace(N.lib().poetx_segmented_outer_workspace_bytes(dt, T, nb, block_dim), x.device)
    N.call("poetx_segmented_outer", dt, T, nb, block_dim, x.contiguous().data_ptr(),
           y.contiguous().data_ptr(), out.data_ptr(), 0, ws, wsb, N.stream_ptr(x.device))
    return _out(out, was_np)


def assemble_dense(factor: BlockDiagonalFactor) -> torch.Tensor:
    """Materialize the full dim x dim matrix.  Oracle/test use only."""
    return torch.block_diag(*factor.blocks.unbind(0))


def orthogonality_error(blocks) -> float:
    """||G.T G - I||_F over a whole stack (blockdiag.py:134-138)."""
    blocks, _ = _to_dev(blocks)
    if blocks.dtype not in (torch.float32, torch.float64):
        blocks = blocks.float()
    blocks = blocks.contiguous()
    nb, b, _ = blocks.shape
    out = torch.empty(1, dtype=torch.float64, device=blocks.device)
    nbytes = nb * b * b * blocks.element_size() + 512 * 8 + 8192
    ws, wsb = N.workspace(nbytes, blocks.device)
    N.call("poetx_orthogonality_error", N.dtype_code(blocks.dtype), nb, b, blocks.data_ptr(),
           out.data_ptr(), ws, wsb, N.stream_ptr(blocks.device))
    return float(out.item())
