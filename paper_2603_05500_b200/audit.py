"""Spectrum audit on the device: singular values by one-sided
Jacobi in float64 (the reference's svd_singular_values, linalg.py:166-218,
as the csrc/svd.cu kernel), spectral_norm (linalg.py:221-224), and the
singular-value drift audit run_spectrum_audit (runner.py:452-529): train one
square POET-X layer between merges, track how far the base weight's
spectrum moves per merge and cumulatively, with CNP or exact-Cayley merges.

Everything on the layer path runs through this package's kernels; the host
only draws the seeded inputs (the reference's keyed Philox streams) and
reads back one scalar per step for the loss column."""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .cnp import skew_from_packed
from .errors import ConfigError, ConvergenceError, ShapeError
from .layer import init_layer
from .optim import ScheduleConfig, adamw_init, adamw_step
from .quant import QuantizedMatrix
from .rng import Rng

_TINY = np.finfo(np.float64).tiny


def singular_values(a, tol: float = 1e-10, max_sweeps: int = 100) -> torch.Tensor:
    """svd_singular_values (linalg.py:166-218) on the device: descending
    float64 singular values of ``a`` ([..., rows, cols], numpy or torch, any
    float dtype; leading dims batch one CTA per matrix).  Raises
    ConvergenceError (with the worst remaining relative off-diagonal as
    ``residual``) when ``max_sweeps`` sweeps do not converge."""
    t = torch.as_tensor(a)
    if t.dim() < 2:
        raise ShapeError(f"expected a matrix (or a stack of matrices), got shape {tuple(t.shape)}")
    dev = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
    t = t.to(dev, torch.float64).contiguous()
    rows, cols = int(t.shape[-2]), int(t.shape[-1])
    lead = tuple(t.shape[:-2])
    batch = int(np.prod(lead)) if lead else 1
    k = min(rows, cols)
    sv = torch.empty((batch, k), dtype=torch.float64, device=dev)
    if batch == 0 or k == 0:
        return sv.view(*lead, k)
    res = torch.empty(batch, dtype=torch.float64, device=dev)
    used = torch.empty(batch, dtype=torch.int32, device=dev)
    ws, wsb = N.workspace(N.lib().poetx_singular_values_workspace_bytes(batch, rows, cols), dev)
    N.call("poetx_singular_values", batch, rows, cols, t.data_ptr(), sv.data_ptr(), float(tol), int(max_sweeps),
           res.data_ptr(), used.data_ptr(), ws, wsb, N.stream_ptr(dev))
    if bool((used < 0).any()):
        worst = float(res.max())
        raise ConvergenceError(
            f"Jacobi SVD did not converge in {max_sweeps} sweeps (worst relative off-diagonal {worst:.3e})",
            residual=worst)
    return sv.view(*lead, k)


def spectral_norm(a) -> float:
    """Largest singular value (linalg.py:221-224)."""
    sv = singular_values(a)
    return float(sv[..., 0].max()) if sv.numel() else 0.0


def _dense_base(layer) -> torch.Tensor:
    base = layer.base
    return base.dequantize() if isinstance(base, QuantizedMatrix) else base


def _matmul(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """linalg.matmul (linalg.py:42-60) through poetx_matmul, same dtype."""
    out = torch.empty((x.shape[0], w.shape[1]), dtype=x.dtype, device=x.device)
    N.call("poetx_matmul", N.dtype_code(x.dtype), x.shape[0], w.shape[1], x.shape[1], x.data_ptr(), x.shape[1], 0,
           w.data_ptr(), w.shape[1], 0, out.data_ptr(), w.shape[1], 0, N.stream_ptr(x.device))
    return out


def _fmt(v: float) -> str:
    return f"{float(v):.17g}"  # runner.py:48-49


def spectrum_audit(cfg, device=None, verbose: bool = True) -> dict:
    """run_spectrum_audit (runner.py:452-529) on the device.  ``cfg`` carries
    the reference TrainConfig fields the audit reads (a reference
    TrainConfig works as is): audit_dim, audit_merges, audit_steps,
    audit_mode ("cnp" | "cayley"), audit_lr, block_size, variant, neumann_k,
    precision, seed, batch_size, the schedule fields and out_dir.  Writes
    ``<out_dir>/spectrum_audit.csv`` in the reference's format and returns the
    same summary dict."""
    dim = int(cfg.audit_dim)
    if cfg.audit_mode not in ("cnp", "cayley"):
        raise ConfigError("audit_mode must be cnp or cayley")
    if dim % cfg.block_size:
        raise ConfigError("audit_dim must be divisible by block_size")
    dtype = np.float32 if cfg.precision == 32 else np.float64
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    # device-resident layer state (torch dtype): the whole audit stays on the GPU
    layer = init_layer(dim, dim, cfg.block_size, Rng.keyed(cfg.seed, "audit", "init"), name="audit",
                       variant=cfg.variant, neumann_k=cfg.neumann_k,
                       dtype=torch.float32 if dtype == np.float32 else torch.float64, device=dev)
    # gaussian_matrix (linalg.py:147-158): float64 draws cast to the layer type
    teacher = (Rng.keyed(cfg.seed, "audit", "teacher").normal((dim, dim)) * (1.0 / np.sqrt(dim))).astype(dtype)
    x = (Rng.keyed(cfg.seed, "audit", "input").normal((cfg.batch_size, dim)) * 1.0).astype(dtype)
    xd, td = torch.from_numpy(x).to(dev), torch.from_numpy(teacher).to(dev)
    target = _matmul(xd, td)

    sched = ScheduleConfig(base_lr=cfg.base_lr, total_steps=cfg.total_steps, warmup_steps=cfg.warmup_steps,
                           min_lr_ratio=cfg.min_lr_ratio, poet_lr_scale=cfg.poet_lr_scale,
                           weight_decay=cfg.weight_decay, clip_norm=cfg.clip_norm,
                           post_merge_clip_start=cfg.post_merge_clip_start,
                           post_merge_clip_ramp=cfg.post_merge_clip_ramp,
                           post_merge_clip_window=cfg.post_merge_clip_window, beta1=cfg.adam_beta1,
                           beta2=cfg.adam_beta2, eps=cfg.adam_eps)
    params = {"q_r": layer.q_r.packed, "q_p": layer.q_p.packed}
    state = adamw_init(params)

    sv_orig = singular_values(_dense_base(layer))
    sv_prev = sv_orig
    rows = []
    exact = cfg.audit_mode == "cayley"
    for merge_idx in range(cfg.audit_merges):
        loss = float("nan")
        for _ in range(cfg.audit_steps):
            z, cache = layer.forward(xd)
            resid = z - target
            loss = float(torch.mean(resid * resid))
            dz = ((2.0 / z.numel()) * resid).to(z.dtype)
            g = layer.backward(cache, dz)
            adamw_step(params, {"q_r": g.q_r, "q_p": g.q_p}, state, cfg.audit_lr, sched)
        # max over both sides' blocks of the blockwise spectral norm, one batched launch per side
        q_norm = max(float(singular_values(skew_from_packed(p))[:, 0].max()) for p in (layer.q_r, layer.q_p))
        audit = layer.merge_and_reinit(Rng.keyed(cfg.seed, "audit", "merge", merge_idx), use_exact_cayley=exact)
        sv_new = singular_values(_dense_base(layer))
        per_merge = float(torch.max(torch.abs(sv_new - sv_prev) / torch.clamp(sv_prev, min=_TINY)))
        cumulative = float(torch.max(torch.abs(sv_new - sv_orig) / torch.clamp(sv_orig, min=_TINY)))
        sv_prev = sv_new
        rows.append({"merge": merge_idx + 1, "loss": loss, "max_q_norm": q_norm, "orth_err_r": audit.orth_err_r,
                     "orth_err_p": audit.orth_err_p, "per_merge_drift": per_merge, "cumulative_drift": cumulative})
        if verbose:
            print(f"merge {merge_idx + 1}/{cfg.audit_merges} mode={cfg.audit_mode} loss={loss:.6f} "
                  f"max|Q|={q_norm:.4f} per_merge_drift={per_merge:.3e} cumulative_drift={cumulative:.3e}")
        state.reset()

    out_dir = Path(cfg.out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    report_path = out_dir / "spectrum_audit.csv"
    with report_path.open("w") as f:
        f.write("merge,loss,max_q_norm,orth_err_R,orth_err_P,per_merge_drift,cumulative_drift\n")
        for r in rows:
            f.write(f"{r['merge']},{_fmt(r['loss'])},{_fmt(r['max_q_norm'])},{_fmt(r['orth_err_r'])},"
                    f"{_fmt(r['orth_err_p'])},{_fmt(r['per_merge_drift'])},{_fmt(r['cumulative_drift'])}\n")
    return {"mode": cfg.audit_mode, "rows": rows,
            "max_per_merge_drift": max((r["per_merge_drift"] for r in rows), default=0.0),
            "cumulative_drift": rows[-1]["cumulative_drift"] if rows else 0.0,
            "report_path": str(os.fspath(report_path))}
