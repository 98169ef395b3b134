"""ctypes binding of the C ABI (include/poetx_b200.h).

This is the ONLY way the package reaches the GPU.  There is no CPU or
PyTorch fallback: if libpoetx_b200.so is missing or fails to load, every
entry point raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np
import torch

from .errors import ConfigError, NumericsError, PoetxError, ShapeError, StateError

# POETX_LIB_PATH: load another build of the same library (same-box A/B runs,
# tools/ab_build.sh); the default is the in-tree build
LIB_PATH = os.environ.get("POETX_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                           "libpoetx_b200.so")

ABI_VERSION = 3  # must equal POETX_ABI_VERSION (include/poetx_b200.h) of the loaded build
F32, F64, BF16 = 0, 1, 2
FAST, MEM = 0, 1
IN_GATHERED, OUT_UNSCATTERED, DZ_GATHERED, DX_UNSCATTERED = 1, 2, 4, 8
_CODES = {1: ShapeError, 2: ConfigError, 3: StateError, 4: NumericsError, 5: PoetxError}

VP = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
SZ = C.c_size_t


class PhiloxState(C.Structure):
    _fields_ = [
        ("counter", C.c_uint64 * 4),
        ("key", C.c_uint64 * 2),
        ("buffer", C.c_uint64 * 4),
        ("buffer_pos", C.c_int64),
        ("has_uint32", C.c_int64),
        ("uinteger", C.c_uint64),
    ]


class LayerDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int),
        ("variant", C.c_int),
        ("neumann_k", C.c_int),
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("b", C.c_int64),
        ("perm_in_fwd", VP),
        ("perm_in_inv", VP),
        ("perm_out_fwd", VP),
        ("perm_out_inv", VP),
        ("premerged", VP),
        ("pm_codes", VP),
        ("pm_scales", VP),
        ("fold_weight", C.c_int),
        ("side_stream", VP),
    ]


class LayerFactors(C.Structure):
    _fields_ = [
        ("packed_r", VP),
        ("packed_p", VP),
        ("g_r", VP),
        ("g_p", VP),
        ("g_r_lowp", VP),
        ("g_p_lowp", VP),
        ("q2_r", VP),
        ("q2_p", VP),
        ("w_in_fold", VP),
        ("w_out_fold", VP),
    ]


_SIGS = {
    "poetx_last_error": (C.c_char_p, []),
    "poetx_abi_version": (I32, []),
    "poetx_launch_count": (C.c_uint64, []),
    "poetx_tc_enabled": (I32, []),
    "poetx_set_tc_enabled": (None, [I32]),
    "poetx_gemm_pair_enabled": (I32, []),
    "poetx_set_gemm_pair_enabled": (None, [I32]),
    "poetx_set_gemm_pair_ms": (None, [I32]),
    "poetx_prof_enable": (None, [I32]),
    "poetx_prof_reset": (None, []),
    "poetx_prof_query": (I32, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                               C.POINTER(C.c_double)]),
    "poetx_ffma_probe": (I32, [I64, I64, VP, C.POINTER(C.c_double), VP]),
    "poetx_philox_seed": (I32, [C.POINTER(PhiloxState), C.c_uint64, C.c_uint64]),
    "poetx_philox_permutation": (I32, [C.POINTER(PhiloxState), I64, VP, VP]),
    "poetx_skew_from_packed": (I32, [I32, I64, I64, VP, VP, VP]),
    "poetx_packed_grad_from_skew_grad": (I32, [I32, I64, I64, VP, VP, I32, VP]),
    "poetx_cnp_workspace_bytes": (SZ, [I32, I64, I64, I32]),
    "poetx_cnp_forward": (I32, [I32, I64, I64, I32, VP, VP, VP, VP, VP, VP, SZ, VP]),
    "poetx_cnp_backward": (I32, [I32, I64, I64, I32, VP, VP, VP, VP, VP, VP, I32, VP, SZ, VP]),
    "poetx_cnp_fused_supported": (I32, [I64]),
    "poetx_cnp_forward_fused": (I32, [I64, I64, VP, VP, VP, VP]),
    "poetx_cnp_backward_fused": (I32, [I64, I64, VP, VP, VP, I32, VP]),
    "poetx_cnp_tc_workspace_bytes": (SZ, [I64, I64]),
    "poetx_cnp_forward_tc": (I32, [I64, I64, VP, VP, VP, VP, VP, SZ, VP]),
    "poetx_cnp_backward_tc": (I32, [I64, I64, VP, VP, VP, I32, VP, SZ, VP]),
    "poetx_layer_backward_dg": (I32, [C.POINTER(LayerDesc), C.POINTER(LayerFactors), I64, VP, VP, VP,
                                      VP, VP, VP, I32, I32, VP, SZ, VP]),
    "poetx_layer_forward_ex": (I32, [C.POINTER(LayerDesc), C.POINTER(LayerFactors), I64, VP, VP, VP,
                                     I32, VP, SZ, VP]),
    "poetx_rmsnorm_gather": (I32, [I64, I64, VP, VP, C.c_float, I32, VP, VP, VP, VP]),
    "poetx_rmsnorm_gather_bwd_workspace_bytes": (SZ, [I64, I64]),
    "poetx_rmsnorm_gather_bwd": (I32, [I64, I64, VP, VP, VP, I32, VP, VP, VP, VP, VP, I32, VP, SZ, VP]),
    "poetx_swiglu_gather": (I32, [I64, I64, VP, VP, VP, VP, VP, VP]),
    "poetx_swiglu_gather_bwd": (I32, [I64, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP]),
    "poetx_swiglu_gather16": (I32, [I64, I64, VP, VP, VP, VP, VP, VP]),
    "poetx_swiglu_gather_bwd16": (I32, [I64, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP]),
    "poetx_rope_scatter": (I32, [I64, I64, I64, I64, VP, VP, VP, VP, VP, VP]),
    "poetx_rope_scatter_bwd": (I32, [I64, I64, I64, I64, VP, VP, VP, VP, VP, VP]),
    "poetx_scatter_add": (I32, [I64, I64, VP, VP, VP, VP, VP]),
    "poetx_cross_entropy_fwd": (I32, [I64, I64, VP, VP, VP, VP, VP, VP]),
    "poetx_cross_entropy_bwd": (I32, [I64, I64, VP, VP, VP, VP, VP, C.c_float, VP, VP]),
    "poetx_attention_bwd": (I32, [I64, I64, I64, I64, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP]),
    "poetx_singular_values_workspace_bytes": (SZ, [I64, I64, I64]),
    "poetx_embedding_fwd": (I32, [I64, I64, I64, VP, VP, VP, VP]),
    "poetx_embedding_bwd": (I32, [I64, I64, I64, VP, VP, VP, VP, VP]),
    "poetx_singular_values": (I32, [I64, I64, I64, VP, VP, C.c_double, I32, VP, VP, VP, SZ, VP]),
    "poetx_orthogonality_error": (I32, [I32, I64, I64, VP, VP, VP, SZ, VP]),
    "poetx_permute_cols": (I32, [I32, I64, I64, VP, VP, VP, VP]),
    "poetx_permute_rows": (I32, [I32, I64, I64, VP, VP, VP, VP]),
    "poetx_gather2d": (I32, [I32, I64, I64, VP, VP, VP, VP, VP]),
    "poetx_apply_to_features": (I32, [I32, I64, I64, I64, VP, I32, VP, VP, VP]),
    "poetx_apply_to_weight_rows": (I32, [I32, I64, I64, I64, VP, I32, VP, VP, VP]),
    "poetx_segmented_outer_workspace_bytes": (SZ, [I32, I64, I64, I64]),
    "poetx_segmented_outer": (I32, [I32, I64, I64, I64, VP, VP, VP, I32, VP, SZ, VP]),
    "poetx_matmul": (I32, [I32, I64, I64, I64, VP, I64, I32, VP, I64, I32, VP, I64, I32, VP]),
    "poetx_layer_workspace_bytes": (SZ, [C.POINTER(LayerDesc), I64]),
    "poetx_layer_factors": (I32, [C.POINTER(LayerDesc), C.POINTER(LayerFactors), VP, SZ, VP]),
    "poetx_layer_forward": (I32, [C.POINTER(LayerDesc), C.POINTER(LayerFactors), I64, VP, VP, VP,
                                  VP, SZ, VP]),
    "poetx_layer_backward": (I32, [C.POINTER(LayerDesc), C.POINTER(LayerFactors), I64, VP, VP, VP,
                                   VP, VP, VP, I32, VP, SZ, VP]),
    "poetx_merge_workspace_bytes": (SZ, [C.POINTER(LayerDesc)]),
    "poetx_matmul_q8": (I32, [I64, I64, I64, VP, I64, VP, I64, I32, VP, VP, I64, VP]),
    "poetx_merge_tc_supported": (I32, [I64]),
    "poetx_merge_tc": (I32, [I64, I64, I64, VP, VP, VP, VP, VP, I64, VP, I32, I64, VP]),
    "poetx_layer_weight_fold": (I32, [C.POINTER(LayerDesc), C.POINTER(LayerFactors), I32, VP, VP, SZ, VP]),
    "poetx_layer_merge_quant": (I32, [C.POINTER(LayerDesc), VP, VP, VP, VP, VP, VP, VP, VP, SZ, VP]),
    "poetx_quantize_rows": (I32, [I32, I64, I64, VP, VP, VP, VP]),
    "poetx_dequantize_rows": (I32, [I32, I64, I64, I64, VP, VP, VP, VP, VP, VP]),
    "poetx_quant_gather": (I32, [I32, I64, I64, I64, VP, VP, VP, VP, VP, VP, VP]),
    "poetx_layer_merge": (I32, [C.POINTER(LayerDesc), VP, VP, VP, VP, VP, VP, VP, SZ, VP]),
    "poetx_sqnorm_workspace_bytes": (SZ, [I32, VP]),
    "poetx_sqnorm": (I32, [I32, I32, VP, VP, VP, VP, VP, SZ, VP]),
    "poetx_adamw_dyn": (I32, [I32, I32, VP, VP, VP, VP, VP, C.c_double, C.c_double, C.c_double, VP, VP,
                              I32, VP]),
    "poetx_adamw": (I32, [I32, I32, VP, VP, VP, VP, VP, C.c_double, C.c_double, C.c_double,
                          C.c_double, C.c_double, C.c_double, C.c_double, VP, C.c_double, I32, VP]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def lib():
    """Load libpoetx_b200.so once; fail loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2603_05500_b200.build` "
                    "(there is no CPU fallback)"
                )
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            abi = handle.poetx_abi_version()
            if abi != ABI_VERSION:
                raise RuntimeError(f"{LIB_PATH} has ABI version {abi}, the Python binding expects {ABI_VERSION}: "
                                   "rebuild with `python -m paper_2603_05500_b200.build`")
            _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().poetx_last_error().decode("utf-8", "replace")
        raise _CODES.get(rc, PoetxError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().poetx_launch_count())


# -------------------------------------------------------------- tensors ------

_TORCH_CODE = {torch.float32: F32, torch.float64: F64, torch.bfloat16: BF16}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _TORCH_CODE[dt]
    except KeyError:
        raise ShapeError(f"unsupported dtype {dt}") from None


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise ShapeError(f"{what} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ShapeError(f"{what} must be contiguous")


class _WorkspacePool:
    """One growable scratch buffer per (device, stream).  Kernels are
    stream-ordered, so reuse on the same stream is race-free.

    A buffer handed out while a CUDA graph is being captured is PINNED: the
    graph bakes its address into its kernels, so when a later call needs a
    larger buffer the pinned one is retired (kept alive for the process)
    instead of freed -- a replay never reads freed memory."""

    def __init__(self):
        self._bufs = {}
        self._pinned = set()   # data_ptr of buffers referenced by a captured graph
        self._retired = []     # replaced pinned buffers, kept alive

    def get(self, nbytes: int, device=None) -> torch.Tensor:
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device.index)
        key = (dev.index, stream_ptr(dev))
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            nbytes = max(nbytes, 1 << 20)
            if buf is not None:
                nbytes = max(nbytes, int(buf.numel() * 1.5))
                if buf.data_ptr() in self._pinned:
                    self._retired.append(buf)
            buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            self._bufs[key] = buf
        if torch.cuda.is_current_stream_capturing():
            self._pinned.add(buf.data_ptr())
        return buf

    def release_all(self):
        """Drop every buffer, pinned and retired ones included.  Only for when
        no captured graph that used them can replay again (e.g. after the
        Trainer that captured it is gone): otherwise use ``clear``."""
        self._bufs.clear()
        self._pinned.clear()
        self._retired.clear()

    def clear(self):
        """Drop the unpinned buffers (pinned ones stay: a graph may replay them)."""
        keep = {k: b for k, b in self._bufs.items() if b.data_ptr() in self._pinned}
        self._retired += list(keep.values())
        self._bufs.clear()


WORKSPACE = _WorkspacePool()


def workspace(nbytes: int, device=None):
    buf = WORKSPACE.get(int(nbytes), device)
    return buf.data_ptr(), buf.numel()


def np_int32_ptr(a: np.ndarray) -> int:
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data
