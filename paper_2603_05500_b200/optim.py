"""Skew-parameter optimizer step on the GPU -- drop-in for the reference's
``poetx.optim`` (optim.py:1-148).

Schedules (``lr_at``, ``clip_threshold_at``) are host arithmetic, copied
in meaning from the reference.  The per-element work -- global float64
squared norm, clip scale and the AdamW update -- runs in libpoetx_b200
kernels with the reference's operation order in the parameter dtype, so
fp32/fp64 updates are bitwise equal to the reference given the same
(clipped) gradients.

Two entry levels:
  * ``global_clip`` / ``adamw_step``: the reference API (host-visible norm,
    NumericsError checks -- these synchronise once per call);
  * ``fused_clip_adamw``: device-resident norm -> clip -> update with no
    host synchronisation, used by the trainer (non-finite flag read lazily).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, NumericsError


@dataclass
class ScheduleConfig:
    base_lr: float
    total_steps: int
    warmup_steps: int = 0
    min_lr_ratio: float = 0.01
    poet_lr_scale: float = 0.5
    weight_decay: float = 0.01
    clip_norm: float = 1.0
    post_merge_clip_start: float = 0.01
    post_merge_clip_ramp: int = 10
    post_merge_clip_window: int = 2000
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def __post_init__(self):
        if self.warmup_steps >= self.total_steps:
            raise ConfigError("warmup_steps must be below total_steps")
        if not (0.0 < self.beta1 < 1.0 and 0.0 < self.beta2 < 1.0):
            raise ConfigError("betas must lie in (0, 1)")


def lr_at(step: int, sched: ScheduleConfig, poet: bool = False) -> float:
    """Warmup then half-cosine to min_lr_ratio; POET rate scaled (optim.py:47-58)."""
    if step < 0:
        raise ConfigError(f"negative step {step}")
    scale = sched.poet_lr_scale if poet else 1.0
    if sched.warmup_steps > 0 and step < sched.warmup_steps:
        return scale * sched.base_lr * step / sched.warmup_steps
    floor = sched.min_lr_ratio * sched.base_lr
    span = sched.total_steps - sched.warmup_steps
    progress = min(1.0, (step - sched.warmup_steps) / span)
    cos = 0.5 * (1.0 + math.cos(math.pi * progress))
    return scale * (floor + (sched.base_lr - floor) * cos)


def clip_threshold_at(global_step: int, steps_since_merge, sched: ScheduleConfig) -> float:
    """Post-merge ramp of the global-norm threshold (optim.py:61-74)."""
    if (
        steps_since_merge is not None
        and global_step < sched.post_merge_clip_window
        and steps_since_merge < sched.post_merge_clip_ramp
    ):
        frac = steps_since_merge / sched.post_merge_clip_ramp
        return sched.post_merge_clip_start + (sched.clip_norm - sched.post_merge_clip_start) * frac
    return sched.clip_norm


# ----------------------------------------------------------------- device ----


def _ptr_array(ts):
    arr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    return arr


def _numel_array(ts):
    return (C.c_int64 * len(ts))(*[t.numel() for t in ts])


def _group_by_dtype(tensors):
    groups = {}
    for t in tensors:
        groups.setdefault(t.dtype, []).append(t)
    return groups


class _NormBuf:
    def __init__(self, device):
        self.sq = torch.zeros(1, dtype=torch.float64, device=device)
        self.acc = torch.zeros(1, dtype=torch.float64, device=device)
        self.bad = torch.zeros(1, dtype=torch.int32, device=device)
        self.bad_acc = torch.zeros(1, dtype=torch.int32, device=device)


_NORM_BUFS = {}


def _normbuf(device) -> _NormBuf:
    key = torch.device(device).index
    if key not in _NORM_BUFS:
        _NORM_BUFS[key] = _NormBuf(device)
    return _NORM_BUFS[key]


def _dev(a, device=None):
    """numpy -> device copy (the reference's numpy dicts); tensors pass through."""
    if isinstance(a, np.ndarray):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    return a


def device_sqnorm(tensors, device=None):
    """Float64 sum of squares over all tensors, left on the device.
    Returns (sq tensor[1] float64, nonfinite tensor[1] int32).  numpy
    arrays are copied to the device first."""
    tensors = [_dev(t, device) for t in tensors]
    tensors = [t for t in tensors if t.numel() > 0]
    device = device or (tensors[0].device if tensors else torch.device("cuda"))
    nb = _normbuf(device)
    nb.acc.zero_()
    nb.bad_acc.zero_()
    stream = N.stream_ptr(device)
    for dt, ts in _group_by_dtype(tensors).items():
        if dt not in (torch.float32, torch.float64):
            raise NumericsError(f"gradient dtype {dt} unsupported")
        for t in ts:
            if not t.is_contiguous():
                raise NumericsError("gradients must be contiguous")
        ptrs, numel = _ptr_array(ts), _numel_array(ts)
        ws, wsb = N.workspace(N.lib().poetx_sqnorm_workspace_bytes(len(ts), numel), device)
        N.call("poetx_sqnorm", N.dtype_code(dt), len(ts), ptrs, numel, nb.sq.data_ptr(),
               nb.bad.data_ptr(), ws, wsb, stream)
        nb.acc.add_(nb.sq)
        nb.bad_acc.add_(nb.bad)
    return nb.acc, nb.bad_acc


def global_grad_norm(grads: dict) -> float:
    sq, _ = device_sqnorm(list(grads.values()))
    return math.sqrt(float(sq.item()))


def global_clip(grads: dict, threshold: float) -> float:
    """Scale all gradients in place to the threshold; returns the pre-clip
    norm.  Non-finite gradients are an abort (optim.py:84-94)."""
    sq, _ = device_sqnorm(list(grads.values()))
    norm = math.sqrt(float(sq.item()))
    if not math.isfinite(norm):
        raise NumericsError(f"non-finite gradient norm {norm}")
    if norm > threshold and norm > 0.0:
        factor = threshold / norm
        for g in grads.values():
            if isinstance(g, np.ndarray):  # host array, scaled in place as the reference does
                g *= g.dtype.type(factor)
                continue
            # cast like the reference (g *= g.dtype.type(factor))
            g.mul_(float(np.float32(factor)) if g.dtype == torch.float32 else factor)
    return norm


@dataclass
class AdamWState:
    """Two moment buffers per parameter plus a shared step count (optim.py:97-116)."""

    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    t: int = 0

    def nbytes(self) -> int:
        def nb(a):
            return a.nbytes if isinstance(a, np.ndarray) else a.numel() * a.element_size()

        return sum(nb(a) for a in self.m.values()) + sum(nb(a) for a in self.v.values())

    def reset(self) -> None:
        for a in list(self.m.values()) + list(self.v.values()):
            if isinstance(a, np.ndarray):
                a[...] = 0.0
            else:
                a.zero_()
        self.t = 0


def adamw_init(params: dict) -> AdamWState:
    """Zero moments in each parameter's own type and place: numpy arrays for
    numpy parameters (the reference's dicts), device tensors for tensors."""
    st = AdamWState()
    for name, p in params.items():
        zeros = np.zeros_like if isinstance(p, np.ndarray) else torch.zeros_like
        st.m[name] = zeros(p)
        st.v[name] = zeros(p)
    return st


def _adamw_launch(ps, gs, ms, vs, lr, sched, t, sqnorm=None, threshold=0.0, write_back=0):
    bc1 = 1.0 - sched.beta1 ** t
    bc2 = 1.0 - sched.beta2 ** t
    dev = ps[0].device
    for dt in (torch.float32, torch.float64):
        idx = [i for i, p in enumerate(ps) if p.dtype == dt]
        if not idx:
            continue
        sel = lambda xs: [xs[i] for i in idx]  # noqa: E731
        P, G, M, V = sel(ps), sel(gs), sel(ms), sel(vs)
        N.call("poetx_adamw", N.dtype_code(dt), len(P), _ptr_array(P), _ptr_array(G), _ptr_array(M),
               _ptr_array(V), _numel_array(P), float(lr), sched.beta1, sched.beta2, sched.eps,
               sched.weight_decay, bc1, bc2, N.ptr(sqnorm), float(threshold), int(write_back),
               N.stream_ptr(dev))


def adamw_step(params: dict, grads: dict, state: AdamWState, lr: float, sched: ScheduleConfig) -> None:
    """One decoupled-weight-decay Adam update, in place (optim.py:127-148).

    Device tensors are updated where they live.  numpy parameters (the
    reference runner's dicts) are copied to the device with their grads and
    moments, updated by the same kernel, and written back into the SAME
    numpy arrays, so everything keyed to them stays attached."""
    state.t += 1
    ps, gs, ms, vs, back = [], [], [], [], []
    for name, p in params.items():
        g = grads[name]
        if tuple(g.shape) != tuple(p.shape):
            raise NumericsError(f"gradient shape {tuple(g.shape)} != param shape {tuple(p.shape)} for {name}")
        if isinstance(g, np.ndarray) and not np.all(np.isfinite(g)):
            raise NumericsError(f"non-finite gradient for {name}")
        m, v = state.m[name], state.v[name]
        if isinstance(p, np.ndarray):
            dp, dm, dv = _dev(p), _dev(m), _dev(v)
            back.append((p, dp, m, dm, v, dv))
            p, m, v = dp, dm, dv
        ps.append(p); gs.append(_dev(g, p.device)); ms.append(m); vs.append(v)
    dev_gs = [(name, g) for name, g in zip(params, gs) if not isinstance(grads[name], np.ndarray)]
    if dev_gs:
        _, bad = device_sqnorm([g for _, g in dev_gs])
        if int(bad.item()):
            for name, g in dev_gs:
                if not bool(torch.isfinite(g).all()):
                    raise NumericsError(f"non-finite gradient for {name}")
    if ps:
        _adamw_launch(ps, gs, ms, vs, lr, sched, state.t)
    for p, dp, m, dm, v, dv in back:
        p[...] = dp.cpu().numpy()
        m[...] = dm.cpu().numpy()
        v[...] = dv.cpu().numpy()


def fused_clip_adamw(groups, threshold: float, sched: ScheduleConfig):
    """Trainer path: one device norm over every group's grads, then per group
    (params, grads, m, v, lr, t) the clip-scaled AdamW update -- no host sync.
    Returns (sqnorm tensor, nonfinite tensor) for lazy inspection."""
    allg = [g for grp in groups for g in grp[1]]
    sq, bad = device_sqnorm(allg)
    for ps, gs, ms, vs, lr, t in groups:
        _adamw_launch(ps, gs, ms, vs, lr, sched, t, sqnorm=sq, threshold=threshold, write_back=0)
    return sq, bad


def fused_clip_adamw_dyn(groups, sched: ScheduleConfig):
    """CUDA-graph-friendly trainer update: per group (params, grads, m, v,
    dyn) where ``dyn`` is a DEVICE float64 tensor {lr, lr*wd, bc1, bc2,
    clip threshold} refreshed before each (replayed) step."""
    allg = [g for grp in groups for g in grp[1]]
    sq, bad = device_sqnorm(allg)
    for ps, gs, ms, vs, dyn in groups:
        P, G, M, V = ps, gs, ms, vs
        N.call("poetx_adamw_dyn", N.dtype_code(P[0].dtype), len(P), _ptr_array(P), _ptr_array(G),
               _ptr_array(M), _ptr_array(V), _numel_array(P), sched.beta1, sched.beta2, sched.eps,
               dyn.data_ptr(), sq.data_ptr(), 0, N.stream_ptr(P[0].device))
    return sq, bad


def adamw_dyn_values(lr: float, t: int, threshold: float, sched: ScheduleConfig):
    """Host values of the ``dyn`` vector for fused_clip_adamw_dyn."""
    return [lr, lr * sched.weight_decay, 1.0 - sched.beta1 ** t, 1.0 - sched.beta2 ** t, threshold]
