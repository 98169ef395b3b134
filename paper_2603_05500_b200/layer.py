"""POET-X linear layer on the GPU -- drop-in for the reference's
``poetx.layer`` (layer.py:1-344).

The layer owns a frozen weight stored ONLY in its premerged form
PM = Psi_m W Psi_n^T (PM[i, j] = W[pi_in(i), pi_out(j)], layer.py:161-167)
on the device; ``base`` is recomputed from it on demand (exact gather).
Two packed skew stacks ``q_r`` (m/b blocks) and ``q_p`` (n/b blocks)
are the trainable state.  Forward (layer.py:214-229)

    u = x[:, pi_in] ; a = u blockdiag(G_R) ; t = a PM ; v = t blockdiag(G_P) ;
    z = v[:, pi_out^-1]

and the hand-written backward (layer.py:231-256) run as one C-ABI call
each (csrc/layer.cu).  ``fast`` saves t, ``mem`` recomputes it with the
same deterministic kernels, so both variants give bitwise-equal grads.

dtypes: float32 / float64 (parity path, CUDA-core FFMA/DFMA) and
bfloat16 (performance path: tcgen05 tensor cores, fp32 accumulation,
fp32 master parameters).  numpy inputs are accepted and returned as numpy.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .blockdiag import orthogonality_error
from .cnp import SkewParams, cayley_exact, num_pairs
from .errors import ConfigError, ShapeError, StateError
from .quant import QuantizedMatrix
from .permute import PermutationMap, sample_permutation
from .rng import Rng

VARIANTS = ("fast", "mem")

_NP_TO_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


def _torch_dtype(dt) -> torch.dtype:
    if isinstance(dt, torch.dtype):
        return dt
    try:
        return _NP_TO_TORCH[np.dtype(dt)]
    except (KeyError, TypeError):
        raise ShapeError(f"unsupported dtype {dt}") from None


def param_dtype(dt: torch.dtype) -> torch.dtype:
    return torch.float64 if dt == torch.float64 else torch.float32


@dataclass
class LayerCache:
    """Operands one forward saves for its backward (layer.py:71-81)."""

    x: torch.Tensor
    g_r: torch.Tensor
    g_p: torch.Tensor
    factors: "Factors"
    saved_mm2: torch.Tensor | None  # fast variant only
    was_numpy: bool = False
    consumed: bool = False


@dataclass
class LayerGrads:
    q_r: torch.Tensor  # packed, same shape as the parameters
    q_p: torch.Tensor
    x: torch.Tensor  # cotangent for the layer input


@dataclass
class MergeAudit:
    merge_index: int
    orth_err_r: float
    orth_err_p: float
    sv_drift: float = float("nan")


class Factors:
    """Device factor state for one forward: G (param dtype), bf16 copies,
    Q^2 caches and the packed parameters they were computed from."""

    def __init__(self, layer: "PoetLinearLayer", packed_r: torch.Tensor, packed_p: torch.Tensor,
                 accurate: bool = False):
        dev, pdt = layer.device, layer.param_dtype
        b, k = layer.block_size, layer.neumann_k
        nbr, nbp = layer.m // b, layer.n // b
        self.packed_r, self.packed_p = packed_r, packed_p
        self.g_r = torch.empty((nbr, b, b), dtype=pdt, device=dev)
        self.g_p = torch.empty((nbp, b, b), dtype=pdt, device=dev)
        low = layer.tdtype == torch.bfloat16
        self.g_r_lowp = torch.empty((nbr, b, b), dtype=torch.bfloat16, device=dev) if low else None
        self.g_p_lowp = torch.empty((nbp, b, b), dtype=torch.bfloat16, device=dev) if low else None
        # BF16 layers with b in {128, 256} leave the Q^2 caches out: the C ABI
        # then runs the fused tensor-core CNP both ways (csrc/cnp_fused.cu);
        # ``accurate`` (the merge) keeps the fp32 CUDA-core CNP
        tc = low and k == 3 and not accurate and bool(N.lib().poetx_cnp_fused_supported(b))
        self.q2_r = torch.empty((nbr, b, b), dtype=pdt, device=dev) if k == 3 and not tc else None
        self.q2_p = torch.empty((nbp, b, b), dtype=pdt, device=dev) if k == 3 and not tc else None
        self.struct = N.LayerFactors(
            packed_r.data_ptr(), packed_p.data_ptr(), self.g_r.data_ptr(), self.g_p.data_ptr(),
            N.ptr(self.g_r_lowp), N.ptr(self.g_p_lowp), N.ptr(self.q2_r), N.ptr(self.q2_p))


class PoetLinearLayer:
    def __init__(self, base_weight, block_size: int, rng: Rng, *, name: str = "poet",
                 variant: str = "fast", neumann_k: int = 3, device=None):
        # numpy in => numpy state (the reference's own types, drop-in for
        # poetx.layer): q_r/q_p.packed are host numpy arrays the caller and
        # the optimizer mutate in place, base/premerged/materialize_weight come
        # back as numpy, dtype is a numpy dtype; the weight itself lives on the
        # device and every forward/backward/merge runs there.  Torch in =>
        # device-resident state (torch CUDA tensors, no copies).
        self._host = isinstance(base_weight, np.ndarray)
        if self._host:
            if base_weight.dtype not in (np.float32, np.float64):
                raise ShapeError(f"unsupported dtype {base_weight.dtype}")
            base_weight = torch.from_numpy(np.ascontiguousarray(base_weight))
        if base_weight.ndim != 2:
            raise ShapeError(f"base weight must be 2-D, got {tuple(base_weight.shape)}")
        m, n = base_weight.shape
        if block_size < 1:
            raise ConfigError(f"block_size must be >= 1, got {block_size}")
        if m % block_size or n % block_size:
            raise ConfigError(
                f"layer dims ({m}, {n}) must both be divisible by block_size {block_size}")
        if variant not in VARIANTS:
            raise ConfigError(f"variant must be one of {VARIANTS}, got {variant!r}")
        if neumann_k < 1:
            raise ConfigError(f"neumann_k must be >= 1, got {neumann_k}")
        if base_weight.dtype not in (torch.float32, torch.float64, torch.bfloat16):
            raise ShapeError(f"unsupported dtype {base_weight.dtype}")
        if num_pairs(block_size) == 0:
            warnings.warn("block_size 1 leaves no trainable rotation parameters", stacklevel=2)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.name = name
        self.m, self.n = int(m), int(n)
        self.block_size = int(block_size)
        self.variant = variant
        self.neumann_k = int(neumann_k)
        self.tdtype = base_weight.dtype  # torch dtype of the device computation
        self.param_dtype = param_dtype(self.tdtype)
        nbr, nbp = self.m // block_size, self.n // block_size
        if self._host:
            np_dt = np.float64 if self.param_dtype == torch.float64 else np.float32
            self.q_r = SkewParams(nbr, block_size, np.zeros((nbr, num_pairs(block_size)), dtype=np_dt))
            self.q_p = SkewParams(nbp, block_size, np.zeros((nbp, num_pairs(block_size)), dtype=np_dt))
        else:
            self.q_r = SkewParams.zeros(nbr, block_size, dtype=self.param_dtype, device=self.device)
            self.q_p = SkewParams.zeros(nbp, block_size, dtype=self.param_dtype, device=self.device)
        self.merge_count = 0
        self.perm_in = sample_permutation(self.m, rng)
        self.perm_out = sample_permutation(self.n, rng)
        w = base_weight.to(self.device).contiguous()
        self._pm = self._premerge(w, self.perm_in, self.perm_out)

    # -- construction helpers ----------------------------------------------------

    @property
    def dtype(self):
        """numpy dtype for a numpy-constructed layer (as the reference), else
        the torch dtype."""
        if self._host:
            return np.dtype(np.float64 if self.tdtype == torch.float64 else np.float32)
        return self.tdtype

    @property
    def premerged(self):
        """PM = Psi_m W Psi_n^T (layer.py:161-167): the device tensor, or a
        numpy copy for a numpy-constructed layer."""
        if self._host and isinstance(self._pm, torch.Tensor):
            return self._pm.cpu().numpy()
        return self._pm

    @premerged.setter
    def premerged(self, pm) -> None:
        if isinstance(pm, np.ndarray):
            pm = torch.from_numpy(np.ascontiguousarray(pm)).to(self.device, self.tdtype)
        self._pm = pm

    def _packed_dev(self, side: str) -> torch.Tensor:
        """The packed parameters of one side as a device tensor (a copy of the
        host array for a numpy-constructed layer)."""
        p = (self.q_r if side == "r" else self.q_p).packed
        if isinstance(p, np.ndarray):
            return torch.from_numpy(np.ascontiguousarray(p)).to(self.device)
        return p

    def _zero_packed(self) -> None:
        """Zero both packed stacks IN PLACE (layer.py:306-309: optimizer state
        keyed to these arrays stays attached)."""
        for sp in (self.q_r, self.q_p):
            if isinstance(sp.packed, np.ndarray):
                sp.packed[...] = 0.0
            else:
                sp.packed.zero_()

    @property
    def quantized(self) -> bool:
        return isinstance(self._pm, QuantizedMatrix)

    def trainable_param_count(self) -> int:
        return int(np.prod(self.q_r.packed.shape) + np.prod(self.q_p.packed.shape))

    def _stream(self) -> int:
        return N.stream_ptr(self.device)

    def _premerge(self, w: torch.Tensor, pin: PermutationMap, pout: PermutationMap) -> torch.Tensor:
        out = torch.empty((self.m, self.n), dtype=self.tdtype, device=self.device)
        rf, _ = pin.device(self.device)
        cf, _ = pout.device(self.device)
        N.call("poetx_gather2d", N.dtype_code(self.tdtype), self.m, self.n, rf.data_ptr(),
               cf.data_ptr(), w.data_ptr(), out.data_ptr(), self._stream())
        return out

    def _base_dev(self):
        """W[r, c] = PM[pi_in^-1(r), pi_out^-1(c)] on the device (exact gather;
        a QuantizedMatrix when the base is quantized)."""
        if self.quantized:
            return self._pm.gather(self.perm_in.inverse, self.perm_out.inverse)
        _, ri = self.perm_in.device(self.device)
        _, ci = self.perm_out.device(self.device)
        out = torch.empty((self.m, self.n), dtype=self.tdtype, device=self.device)
        N.call("poetx_gather2d", N.dtype_code(self.tdtype), self.m, self.n, ri.data_ptr(),
               ci.data_ptr(), self._pm.data_ptr(), out.data_ptr(), self._stream())
        return out

    @property
    def base(self):
        """Frozen weight W recovered from the premerged copy (exact; a
        QuantizedMatrix when the base is quantized, as in the reference;
        numpy for a numpy-constructed layer)."""
        w = self._base_dev()
        if self._host and isinstance(w, torch.Tensor):
            return w.cpu().numpy()
        return w

    @base.setter
    def base(self, w) -> None:
        if isinstance(w, np.ndarray):
            w = torch.from_numpy(np.ascontiguousarray(w))
        if not isinstance(w, (torch.Tensor, QuantizedMatrix)) and hasattr(w, "codes") and hasattr(w, "scales"):
            w = QuantizedMatrix(w.codes, w.scales, float_dtype=self.tdtype)  # the reference's QuantizedMatrix
        if isinstance(w, QuantizedMatrix):
            if w.shape != (self.m, self.n):
                raise ShapeError(f"base weight shape {w.shape}, expected ({self.m}, {self.n})")
            self._pm = w.gather(self.perm_in.forward, self.perm_out.forward)
            return
        if tuple(w.shape) != (self.m, self.n):
            raise ShapeError(f"base weight shape {tuple(w.shape)}, expected ({self.m}, {self.n})")
        self._pm = self._premerge(w.to(self.device, self.tdtype).contiguous(), self.perm_in, self.perm_out)

    def set_permutations(self, perm_in: PermutationMap, perm_out: PermutationMap) -> None:
        """Install explicit permutations keeping W fixed (layer.py:153-159)."""
        if perm_in.n != self.m or perm_out.n != self.n:
            raise ShapeError("permutation sizes do not match layer dims")
        w = self._base_dev()
        self.perm_in, self.perm_out = perm_in, perm_out
        if isinstance(w, QuantizedMatrix):
            self._pm = w.gather(perm_in.forward, perm_out.forward)
        else:
            self._pm = self._premerge(w, perm_in, perm_out)

    def quantize_base(self) -> None:
        """Switch the frozen weight to per-row int8 (POET-XQ, layer.py:169-177).
        Mem variant only: the fast variant's saved mm2 output would defeat
        the point.  Row quantization commutes with the premerge gathers, so
        the premerged codes are the quantized base gathered exactly."""
        if self.variant != "mem":
            raise ConfigError("quantized base requires the mem variant")
        if not self.quantized:
            self._pm = QuantizedMatrix.quantize(self._base_dev()).gather(self.perm_in.forward,
                                                                         self.perm_out.forward)

    # -- descriptor ----------------------------------------------------------------

    def _side_stream(self) -> int | None:
        """This layer's own stream for the backward's segmented outer products
        (csrc/layer.cu forks onto it), created on first use."""
        if self.device.type != "cuda":
            return None
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device)
        return self._side.cuda_stream

    def _desc(self) -> N.LayerDesc:
        fi, ii = self.perm_in.device(self.device)
        fo, io = self.perm_out.device(self.device)
        d = N.LayerDesc()
        d.dtype = N.dtype_code(self.tdtype)
        d.variant = N.FAST if self.variant == "fast" else N.MEM
        d.neumann_k = self.neumann_k
        d.m, d.n, d.b = self.m, self.n, self.block_size
        d.perm_in_fwd, d.perm_in_inv = fi.data_ptr(), ii.data_ptr()
        d.perm_out_fwd, d.perm_out_inv = fo.data_ptr(), io.data_ptr()
        d.fold_weight = int(getattr(self, "fold_weight", True))
        d.side_stream = self._side_stream()
        if self.quantized:
            d.premerged = None
            d.pm_codes = self._pm.codes.data_ptr()
            d.pm_scales = self._pm.scales.data_ptr()
        else:
            d.premerged = self._pm.data_ptr()
        return d

    def compute_factors(self, packed_r=None, packed_p=None, accurate: bool = False) -> Factors:
        f = Factors(self, self._packed_dev("r") if packed_r is None else packed_r,
                    self._packed_dev("p") if packed_p is None else packed_p, accurate)
        d = self._desc()
        ws, wsb = N.workspace(N.lib().poetx_cnp_workspace_bytes(
            N.dtype_code(self.param_dtype), max(self.m, self.n) // self.block_size,
            self.block_size, self.neumann_k), self.device)
        N.call("poetx_layer_factors", d, f.struct, ws, wsb, self._stream())
        return f

    # -- forward / backward ----------------------------------------------------------

    def _input(self, x, what):
        was_np = isinstance(x, np.ndarray)
        if was_np:
            if _NP_TO_TORCH.get(x.dtype) != self.tdtype:
                raise ShapeError(f"{what} dtype {x.dtype} does not match layer dtype {self.dtype}")
            x = torch.from_numpy(np.ascontiguousarray(x)).to(self.device)
        elif x.dtype != self.tdtype:
            raise ShapeError(f"{what} dtype {x.dtype} does not match layer dtype {self.dtype}")
        if not x.is_cuda:
            x = x.to(self.device)
        return x.contiguous(), was_np

    def forward(self, x, ledger=None):
        if x.ndim != 2 or x.shape[1] != self.m:
            raise ShapeError(f"input shape {tuple(x.shape)} does not match layer ({self.m}, {self.n})")
        x, was_np = self._input(x, "input")
        T = x.shape[0]
        # snapshot the parameters so backward differentiates this forward's factors
        pr, pp = self._packed_dev("r"), self._packed_dev("p")
        f = self.compute_factors(pr if self._host else pr.clone(), pp if self._host else pp.clone())
        z = torch.empty((T, self.n), dtype=self.tdtype, device=self.device)
        saved = torch.empty((T, self.n), dtype=self.tdtype, device=self.device) if self.variant == "fast" else None
        d = self._desc()
        ws, wsb = N.workspace(N.lib().poetx_layer_workspace_bytes(d, T), self.device)
        N.call("poetx_layer_forward", d, f.struct, T, x.data_ptr(), z.data_ptr(), N.ptr(saved), ws, wsb,
               self._stream())
        if saved is not None and ledger is not None:
            ledger.save_activation(self.name, saved.numel() * saved.element_size())
        cache = LayerCache(x=x, g_r=f.g_r, g_p=f.g_p, factors=f, saved_mm2=saved, was_numpy=was_np)
        return (z.cpu().numpy() if was_np else z), cache

    def backward(self, cache: LayerCache, dz) -> LayerGrads:
        if cache.consumed:
            raise StateError("layer cache already consumed by a previous backward")
        if tuple(dz.shape) != (cache.x.shape[0], self.n):
            raise ShapeError(f"cotangent shape {tuple(dz.shape)} does not match output")
        dz, _ = self._input(dz, "cotangent")
        cache.consumed = True
        T = cache.x.shape[0]
        dx = torch.empty((T, self.m), dtype=self.tdtype, device=self.device)
        gr = torch.empty_like(cache.factors.packed_r)
        gp = torch.empty_like(cache.factors.packed_p)
        d = self._desc()
        ws, wsb = N.workspace(N.lib().poetx_layer_workspace_bytes(d, T), self.device)
        N.call("poetx_layer_backward", d, cache.factors.struct, T, cache.x.data_ptr(), dz.data_ptr(),
               N.ptr(cache.saved_mm2), dx.data_ptr(), gr.data_ptr(), gp.data_ptr(), 0, ws, wsb,
               self._stream())
        if cache.was_numpy:
            return LayerGrads(q_r=gr.cpu().numpy(), q_p=gp.cpu().numpy(), x=dx.cpu().numpy())
        return LayerGrads(q_r=gr, q_p=gp, x=dx)

    # -- merge -------------------------------------------------------------------------

    def _merge_factors(self, use_exact_cayley: bool):
        f = self.compute_factors(accurate=True)
        if not use_exact_cayley:
            return f.g_r, f.g_p
        from .cnp import skew_from_packed
        b = self.block_size
        q_r = SkewParams(self.m // b, b, self._packed_dev("r"))
        q_p = SkewParams(self.n // b, b, self._packed_dev("p"))
        return cayley_exact(skew_from_packed(q_r)), cayley_exact(skew_from_packed(q_p))

    def _merge_call(self, g_r, g_p, new_in=None, new_out=None, want_w=False):
        d = self._desc()
        ws, wsb = N.workspace(N.lib().poetx_merge_workspace_bytes(d), self.device)
        if self.quantized:
            w = torch.empty((self.m, self.n), dtype=self.tdtype, device=self.device) if want_w else None
            if new_in is None:  # materialize only: the float transform of the dequantized base
                N.call("poetx_layer_merge", d, g_r.contiguous().data_ptr(), g_p.contiguous().data_ptr(),
                       None, None, None, N.ptr(w), ws, wsb, self._stream())
                return None, w
            q = self._pm
            codes = torch.empty_like(q.codes)
            scales = torch.empty_like(q.scales)
            N.call("poetx_layer_merge_quant", d, g_r.contiguous().data_ptr(), g_p.contiguous().data_ptr(),
                   new_in.device(self.device)[0].data_ptr(), new_out.device(self.device)[0].data_ptr(),
                   codes.data_ptr(), scales.data_ptr(), N.ptr(w), ws, wsb, self._stream())
            return QuantizedMatrix(codes, scales, float_dtype=self.tdtype), w
        pm_new = w = None
        ni = no = None
        if new_in is not None:
            pm_new = torch.empty_like(self._pm)
            ni = new_in.device(self.device)[0]
            no = new_out.device(self.device)[0]
        if want_w:
            w = torch.empty_like(self._pm)
        N.call("poetx_layer_merge", d, g_r.contiguous().data_ptr(), g_p.contiguous().data_ptr(),
               N.ptr(ni), N.ptr(no), N.ptr(pm_new), N.ptr(w), ws, wsb, self._stream())
        return pm_new, w

    def _transformed_base(self, use_exact_cayley: bool) -> torch.Tensor:
        """Psi_m^T (G_R PM G_P) Psi_n (layer.py:260-273)."""
        g_r, g_p = self._merge_factors(use_exact_cayley)
        return self._merge_call(g_r, g_p, want_w=True)[1]

    def materialize_weight(self):
        """Dense effective weight R W P (layer.py:275-277)."""
        w = self._transformed_base(use_exact_cayley=False)
        return w.cpu().numpy() if self._host else w

    def merge_and_reinit(self, rng: Rng, *, use_exact_cayley: bool = False,
                         compute_sv_drift: bool = False) -> MergeAudit:
        """Fold the factors into the frozen weight, zero the packed parameters in
        place, resample both permutations, rebuild PM (layer.py:279-314)."""
        g_r, g_p = self._merge_factors(use_exact_cayley)
        err_r = orthogonality_error(g_r)
        err_p = orthogonality_error(g_p)
        new_in = sample_permutation(self.m, rng)
        new_out = sample_permutation(self.n, rng)
        drift = float("nan")
        old_base = self._base_dev() if compute_sv_drift else None
        if isinstance(old_base, QuantizedMatrix):
            old_base = old_base.dequantize()
        pm_new, w_new = self._merge_call(g_r, g_p, new_in, new_out, want_w=compute_sv_drift)
        if compute_sv_drift:
            # the reference's Jacobi singular values (audit.py / csrc/svd.cu) up to
            # a million entries; cuSOLVER's svdvals beyond (one CTA per matrix)
            if self.m * self.n <= (1 << 20):
                from .audit import singular_values
                sv_old, sv_new = singular_values(old_base), singular_values(w_new)
            else:
                sv_old = torch.linalg.svdvals(old_base.double())
                sv_new = torch.linalg.svdvals(w_new.double())
            denom = torch.clamp(sv_old, min=np.finfo(np.float64).tiny)
            drift = float(torch.max(torch.abs(sv_new - sv_old) / denom))
        self._pm = pm_new
        self._zero_packed()
        self.perm_in, self.perm_out = new_in, new_out
        self.merge_count += 1
        return MergeAudit(self.merge_count, float(err_r), float(err_p), drift)


def init_layer(m: int, n: int, block_size: int, rng: Rng, *, name: str = "poet",
               variant: str = "fast", neumann_k: int = 3, dtype=np.float32,
               weight_std: float | None = None, base_weight=None, device=None) -> PoetLinearLayer:
    """Layer with a Gaussian (or given) frozen base weight (layer.py:317-344).
    Draw order off ``rng``: weight, then pi_in, then pi_out."""
    host = not isinstance(dtype, torch.dtype)  # a numpy dtype: numpy state, as the reference
    tdt = _torch_dtype(dtype) if host else dtype
    if base_weight is None:
        std = (1.0 / np.sqrt(m)) if weight_std is None else float(weight_std)
        draw = rng.normal((m, n)) * std
        if tdt == torch.bfloat16:
            base_weight = torch.from_numpy(draw.astype(np.float32)).to(torch.bfloat16)
        else:
            base_weight = draw.astype(np.float32 if tdt == torch.float32 else np.float64)
            if not host:
                base_weight = torch.from_numpy(base_weight)
    else:
        if tuple(base_weight.shape) != (m, n):
            raise ShapeError(f"base weight shape {tuple(base_weight.shape)}, expected ({m}, {n})")
        if host:
            base_weight = np.asarray(base_weight.cpu().numpy() if isinstance(base_weight, torch.Tensor)
                                     else base_weight).astype(np.float32 if tdt == torch.float32 else np.float64)
        else:
            if isinstance(base_weight, np.ndarray):
                base_weight = torch.from_numpy(np.ascontiguousarray(base_weight))
            base_weight = base_weight.to(tdt)
    return PoetLinearLayer(base_weight, block_size, rng, name=name, variant=variant,
                           neumann_k=neumann_k, device=device)
