"""Per-row symmetric int8 storage of the frozen weight (POET-XQ), mirroring
the reference's ``poetx.quant.QuantizedMatrix`` (quant.py:22-74) on the
device.  Row i: scale = absmax_i / 127 (1.0 for an all-zero row), codes =
clip(rint(w / scale), -127, 127), computed in float64 -- bit-exact with the
reference (csrc/quant.cu).  Scales are kept in the float type of the layer's
parameters (float64 for float64 layers, else float32)."""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import ShapeError


def _scale_dtype(float_dtype: torch.dtype) -> torch.dtype:
    return torch.float64 if float_dtype == torch.float64 else torch.float32


class QuantizedMatrix:
    def __init__(self, codes: torch.Tensor, scales: torch.Tensor, float_dtype=torch.float32):
        if isinstance(codes, np.ndarray):
            codes = torch.from_numpy(np.ascontiguousarray(codes))
        if isinstance(scales, np.ndarray):
            scales = torch.from_numpy(np.ascontiguousarray(scales))
        if codes.ndim != 2 or codes.dtype != torch.int8:
            raise ShapeError(f"codes must be 2-D int8, got {tuple(codes.shape)} {codes.dtype}")
        if tuple(scales.shape) != (codes.shape[0],):
            raise ShapeError(f"scales shape {tuple(scales.shape)} does not match rows {codes.shape[0]}")
        self.float_dtype = float_dtype
        dev = codes.device if codes.is_cuda else torch.device("cuda", torch.cuda.current_device())
        self.codes = codes.to(dev).contiguous()
        self.scales = scales.to(dev, _scale_dtype(float_dtype)).contiguous()

    @property
    def shape(self):
        return tuple(self.codes.shape)

    @property
    def nbytes(self) -> int:
        return self.codes.numel() + self.scales.numel() * self.scales.element_size()

    @classmethod
    def quantize(cls, w) -> "QuantizedMatrix":
        if isinstance(w, np.ndarray):
            w = torch.from_numpy(np.ascontiguousarray(w))
        if w.ndim != 2:
            raise ShapeError(f"expected a 2-D weight, got {tuple(w.shape)}")
        w = w.to("cuda") if not w.is_cuda else w
        w = w.contiguous()
        rows, cols = w.shape
        codes = torch.empty((rows, cols), dtype=torch.int8, device=w.device)
        scales = torch.empty(rows, dtype=_scale_dtype(w.dtype), device=w.device)
        N.call("poetx_quantize_rows", N.dtype_code(w.dtype), rows, cols, w.data_ptr(), codes.data_ptr(),
               scales.data_ptr(), N.stream_ptr(w.device))
        return cls(codes, scales, float_dtype=w.dtype)

    def _dequant(self, ri=None, ci=None, rows=None, cols=None) -> torch.Tensor:
        rows = self.codes.shape[0] if rows is None else rows
        cols = self.codes.shape[1] if cols is None else cols
        out = torch.empty((rows, cols), dtype=self.float_dtype, device=self.codes.device)
        N.call("poetx_dequantize_rows", N.dtype_code(self.float_dtype), rows, cols, self.codes.shape[1],
               self.codes.data_ptr(),
               self.scales.data_ptr(), N.ptr(ri), N.ptr(ci), out.data_ptr(), N.stream_ptr(self.codes.device))
        return out

    def dequantize(self) -> torch.Tensor:
        """Full float reconstruction (merge and audit paths)."""
        return self._dequant()

    def dequant_row(self, k: int) -> torch.Tensor:
        ri = torch.tensor([k], dtype=torch.int32, device=self.codes.device)
        return self._dequant(ri=ri, rows=1)[0]

    def dequant_col(self, j: int) -> torch.Tensor:
        ci = torch.tensor([j], dtype=torch.int32, device=self.codes.device)
        return self._dequant(ci=ci, cols=1)[:, 0]

    def gather(self, row_idx, col_idx) -> "QuantizedMatrix":
        """Row/column permutation in the quantized domain: commutes exactly
        with dequantization (quant.py:63-74)."""
        dev = self.codes.device
        ri = torch.as_tensor(np.asarray(row_idx, dtype=np.int32)).to(dev)
        ci = torch.as_tensor(np.asarray(col_idx, dtype=np.int32)).to(dev)
        rows, cols = ri.numel(), ci.numel()
        codes = torch.empty((rows, cols), dtype=torch.int8, device=dev)
        scales = torch.empty(rows, dtype=self.scales.dtype, device=dev)
        N.call("poetx_quant_gather", N.dtype_code(self.float_dtype), rows, cols, self.codes.shape[1],
               ri.data_ptr(), ci.data_ptr(),
               self.codes.data_ptr(), self.scales.data_ptr(), codes.data_ptr(), scales.data_ptr(),
               N.stream_ptr(dev))
        return QuantizedMatrix(codes, scales, float_dtype=self.float_dtype)
