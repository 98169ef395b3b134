"""GPU-resident POET-X training step around the hot path:
a Llama decoder whose seven projections per block are POET-X layers, the
reference trainer's step logic (runner.py:279-327: clip threshold ramp,
global clip, AdamW on POET and dense groups with the POET lr scale,
merge-then-reinitialize every ``merge_gap`` steps with moment reset) and
token-batch data parallelism over NCCL.

This is the *caller* of the path, used by bench.py; the reference has no
Llama (its models are toy MLPs, models.py), so model shapes follow the
paper.  Attention, RMSNorm, embedding, lm_head
and the loss are plain PyTorch (cuDNN/flash SDPA); every POET-X operation
is a libpoetx_b200 kernel.

Memory layout (B200-first): all packed skew parameters of the model live
in ONE flat fp32 buffer (and their grads, AdamW m and v in three more), so
the global norm, the fused clip+AdamW update and the data-parallel
all-reduce are one launch each over contiguous HBM.  Dense trainables
(embedding, lm_head, RMSNorm gains) share a second flat fp32 group.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from . import _native as N
from .cnp import num_pairs
from .errors import ConfigError, NumericsError
from .optim import ScheduleConfig, adamw_dyn_values, clip_threshold_at, fused_clip_adamw_dyn, lr_at
from .permute import PermutationMap, sample_permutation
from .rng import Rng


@dataclass
class LlamaConfig:
    name: str
    d: int
    f: int
    layers: int
    heads: int
    block: int
    vocab: int = 32000
    seq: int = 256
    variant: str = "fast"
    neumann_k: int = 3
    quantized: bool = False  # POET-XQ int8 frozen weights (mem variant only)

    @property
    def head_dim(self) -> int:
        return self.d // self.heads


# FFN widths are the LLaMA multiple_of rounding of 8d/3 made
# divisible by b; these reproduce the paper's Llama-3B parameter counts.
CONFIGS = {
    "llama-60m": dict(d=512, f=1408, layers=8, heads=8, block=64),
    "llama-350m": dict(d=1024, f=2816, layers=24, heads=16, block=256),
    "llama-1b": dict(d=2048, f=5632, layers=24, heads=32, block=256),
    "llama-8b": dict(d=4096, f=14336, layers=32, heads=32, block=256, seq=1024),
}


def llama_config(name: str, **over) -> LlamaConfig:
    kw = dict(CONFIGS[name])
    kw.update(over)
    return LlamaConfig(name=name, **kw)


# --------------------------------------------------------------------------
# flat parameter groups
# --------------------------------------------------------------------------


class FlatGroup:
    """Contiguous fp32 param / grad / m / v buffers with named views."""

    def __init__(self, sizes: dict, device):
        self.offsets = {}
        off = 0
        for name, n in sizes.items():
            self.offsets[name] = (off, n)
            off += n
        self.numel = off
        self.param = torch.zeros(off, dtype=torch.float32, device=device)
        self.grad = torch.zeros(off, dtype=torch.float32, device=device)
        self.m = torch.zeros(off, dtype=torch.float32, device=device)
        self.v = torch.zeros(off, dtype=torch.float32, device=device)
        self.t = 0

    def view(self, buf: torch.Tensor, name: str, shape) -> torch.Tensor:
        off, n = self.offsets[name]
        return buf[off:off + n].view(*shape)

    def reset_moments(self):
        self.m.zero_()
        self.v.zero_()
        self.t = 0


class PoetStack:
    """Every POET-X block of a model in one place.  The packed parameters
    of all layers form one flat FlatGroup (block order = layer order), so
    the Cayley-Neumann forward and backward run as ONE batched tensor-core
    call each per step over all blocks (csrc/cnp_tc.cu) instead of one
    small call per layer, and each layer's G / dG are views into stacks."""

    def __init__(self, entries, b, device):
        self.b = b
        self.pairs = num_pairs(b)
        self.group = FlatGroup({name: nb * self.pairs for name, nb in entries}, device)
        self.nb = self.group.numel // self.pairs
        self.block_off = {name: off // self.pairs for name, (off, _) in self.group.offsets.items()}
        self.g16 = torch.empty((self.nb, b, b), dtype=torch.bfloat16, device=device)
        # b in {128, 256}: one fused tensor-core kernel per direction
        # (csrc/cnp_fused.cu) that unpacks, multiplies and packs on chip and
        # keeps no [Q | Q^2] cache; other block sizes use the staged kernels
        # of csrc/cnp_tc.cu and their cache
        self.fused = (os.environ.get("POETX_CNP_FUSED", "1") != "0" and torch.device(device).type == "cuda"
                      and bool(N.lib().poetx_cnp_fused_supported(b)))
        self.qq2 = None if self.fused else torch.empty((self.nb, b, 2 * b), dtype=torch.bfloat16, device=device)
        self.dg = torch.zeros((self.nb, b, b), dtype=torch.float32, device=device)
        self.device = device

    def blocks(self, buf, name, nb):
        o = self.block_off[name]
        return buf[o:o + nb]

    def forward_factors(self):
        self.forward_factors_range(0, self.nb)

    def backward_factors(self):
        self.backward_factors_range(0, self.nb)

    # block ranges (one decoder block's seven layers are contiguous in the stack)
    def forward_factors_range(self, off: int, nb: int):
        b, pairs = self.b, self.pairs
        packed = self.group.param[off * pairs:].data_ptr()
        if self.fused:
            N.call("poetx_cnp_forward_fused", nb, b, packed, self.g16[off].data_ptr(), None,
                   N.stream_ptr(self.device))
            return
        ws, wsb = N.workspace(N.lib().poetx_cnp_tc_workspace_bytes(nb, b), self.device)
        N.call("poetx_cnp_forward_tc", nb, b, packed, self.qq2[off].data_ptr(),
               self.g16[off].data_ptr(), None, ws, wsb, N.stream_ptr(self.device))

    def backward_factors_range(self, off: int, nb: int):
        b, pairs = self.b, self.pairs
        grad = self.group.grad[off * pairs:].data_ptr()
        if self.fused:
            N.call("poetx_cnp_backward_fused", nb, b, self.group.param[off * pairs:].data_ptr(),
                   self.dg[off].data_ptr(), grad, 0, N.stream_ptr(self.device))
            return
        ws, wsb = N.workspace(N.lib().poetx_cnp_tc_workspace_bytes(nb, b), self.device)
        N.call("poetx_cnp_backward_tc", nb, b, self.qq2[off].data_ptr(), self.dg[off].data_ptr(),
               grad, 0, ws, wsb, N.stream_ptr(self.device))


# --------------------------------------------------------------------------
# POET-X linear as an autograd op
# --------------------------------------------------------------------------


class _PoetFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, mod):
        T = x.shape[0]
        z = torch.empty((T, mod.n), dtype=torch.bfloat16, device=x.device)
        saved = torch.empty((T, mod.n), dtype=torch.bfloat16, device=x.device) if mod.variant == "fast" else None
        ws, wsb = N.workspace(mod.ws_bytes(T), x.device)
        N.call("poetx_layer_forward", mod.desc, mod.fstruct, T, x.data_ptr(), z.data_ptr(), N.ptr(saved),
               ws, wsb, N.stream_ptr(x.device))
        ctx.mod = mod
        ctx.save_for_backward(x, saved) if saved is not None else ctx.save_for_backward(x)
        return z

    @staticmethod
    def backward(ctx, dz):
        mod = ctx.mod
        saved = ctx.saved_tensors
        x = saved[0]
        t = saved[1] if len(saved) > 1 else None
        dz = dz.contiguous()
        T = x.shape[0]
        dx = torch.empty_like(x)
        ws, wsb = N.workspace(mod.ws_bytes(T), x.device)
        # leaves dG_R / dG_P in the model's dG stack; the CNP backward of all
        # layers runs afterwards in one batched call (PoetStack.backward_factors)
        N.call("poetx_layer_backward_dg", mod.desc, mod.fstruct, T, x.data_ptr(), dz.data_ptr(),
               N.ptr(t), dx.data_ptr(), mod.dg_r.data_ptr(), mod.dg_p.data_ptr(), 0, 0, ws, wsb,
               N.stream_ptr(x.device))
        return dx, None


class PoetLinear(torch.nn.Module):
    """m -> n POET-X projection: bf16 frozen premerged weight, fp32 packed
    parameters and its factor/cotangent blocks living in a PoetStack."""

    def __init__(self, name, m, n, stack: PoetStack, rng: Rng, *, variant="fast", neumann_k=3,
                 std=None, device="cuda", quantized=False):
        super().__init__()
        if quantized and variant != "mem":
            raise ConfigError("quantized base requires the mem variant")
        self.quantized = quantized
        b = stack.b
        self.name, self.m, self.n, self.b = name, m, n, b
        self.variant, self.k = variant, neumann_k
        self.device = torch.device(device)
        self.stack = stack
        nbr, nbp, pairs = m // b, n // b, num_pairs(b)
        grp = stack.group
        self.packed_r = grp.view(grp.param, name + ".r", (nbr, pairs))
        self.packed_p = grp.view(grp.param, name + ".p", (nbp, pairs))
        self.g_r16 = stack.blocks(stack.g16, name + ".r", nbr)
        self.g_p16 = stack.blocks(stack.g16, name + ".p", nbp)
        self.dg_r = stack.blocks(stack.dg, name + ".r", nbr)
        self.dg_p = stack.blocks(stack.dg, name + ".p", nbp)
        # draw order as init_layer (layer.py:335-340): W, then pi_in, then pi_out.
        # Synthetic-weight runs draw W on the device (seeded) instead of host numpy.
        std = (1.0 / math.sqrt(m)) if std is None else std
        gen = torch.Generator(device=self.device).manual_seed(int(rng.integers(0, 2**62)))
        w = (torch.randn((m, n), generator=gen, device=self.device, dtype=torch.float32) * std).to(torch.bfloat16)
        self.perm_in = sample_permutation(m, rng)
        self.perm_out = sample_permutation(n, rng)
        # device index buffers at FIXED addresses (updated in place at merge), so
        # a captured CUDA graph of the step stays valid across merges
        self.pin_dev = tuple(t.clone() for t in self.perm_in.device(self.device))
        self.pout_dev = tuple(t.clone() for t in self.perm_out.device(self.device))
        self.premerged = torch.empty((m, n), dtype=torch.bfloat16, device=self.device)
        if quantized:  # int8 premerged codes + per-row fp32 scales (fixed addresses)
            self.codes = torch.empty((m, n), dtype=torch.int8, device=self.device)
            self.scales = torch.empty(m, dtype=torch.float32, device=self.device)
        self._install(w)
        del w
        self.fstruct_plain = N.LayerFactors(self.packed_r.data_ptr(), self.packed_p.data_ptr(), None, None,
                                            self.g_r16.data_ptr(), self.g_p16.data_ptr(), None, None)
        self.fstruct = self.fstruct_bwd = self.fstruct_plain
        self.fstruct_folded = None  # (forward, backward) structs when weight folds are pipelined
        self.merge_count = 0

    def _install(self, w: torch.Tensor):
        rf, _ = self.perm_in.device(self.device)
        cf, _ = self.perm_out.device(self.device)
        N.call("poetx_gather2d", N.BF16, self.m, self.n, rf.data_ptr(), cf.data_ptr(), w.data_ptr(),
               self.premerged.data_ptr(), N.stream_ptr(self.device))
        if self.quantized:
            # row quantization commutes with the premerge gathers (quant.py:63-74)
            N.call("poetx_quantize_rows", N.BF16, self.m, self.n, self.premerged.data_ptr(), self.codes.data_ptr(),
                   self.scales.data_ptr(), N.stream_ptr(self.device))
            self.premerged = None  # the bf16 copy is not kept
        self._set_desc()

    def install(self, w: torch.Tensor, perm_in: PermutationMap, perm_out: PermutationMap):
        """Checkpoint load: new frozen weight W (bf16 [m, n]) and permutations,
        written into the existing device buffers (fixed addresses)."""
        self.perm_in, self.perm_out = perm_in, perm_out
        for dst, src in zip(self.pin_dev + self.pout_dev, perm_in.device(self.device) + perm_out.device(self.device)):
            dst.copy_(src)
        if self.quantized and self.premerged is None:
            self.premerged = torch.empty((self.m, self.n), dtype=torch.bfloat16, device=self.device)
        self._install(w.to(self.device, torch.bfloat16).contiguous())

    def install_quantized(self, codes: torch.Tensor, scales: torch.Tensor, perm_in: PermutationMap,
                          perm_out: PermutationMap):
        """Checkpoint load of a POET-XQ layer: W's int8 codes/scales, gathered
        into the premerged order in the quantized domain (exact)."""
        self.perm_in, self.perm_out = perm_in, perm_out
        for dst, src in zip(self.pin_dev + self.pout_dev, perm_in.device(self.device) + perm_out.device(self.device)):
            dst.copy_(src)
        codes, scales = codes.to(self.device).contiguous(), scales.to(self.device, torch.float32).contiguous()
        N.call("poetx_quant_gather", N.BF16, self.m, self.n, self.n, self.pin_dev[0].data_ptr(), self.pout_dev[0].data_ptr(),
               codes.data_ptr(), scales.data_ptr(), self.codes.data_ptr(), self.scales.data_ptr(),
               N.stream_ptr(self.device))
        self._set_desc()

    def _set_desc(self):
        fi, ii = self.pin_dev
        fo, io = self.pout_dev
        d = N.LayerDesc()
        d.dtype, d.variant, d.neumann_k = N.BF16, (N.FAST if self.variant == "fast" else N.MEM), self.k
        d.m, d.n, d.b = self.m, self.n, self.b
        d.perm_in_fwd, d.perm_in_inv = fi.data_ptr(), ii.data_ptr()
        d.perm_out_fwd, d.perm_out_inv = fo.data_ptr(), io.data_ptr()
        d.fold_weight = int(getattr(self, "fold_weight", True))
        side = getattr(self, "side_stream", None)  # set by the model: one per projection kind
        d.side_stream = side.cuda_stream if side is not None else None
        if self.quantized:
            d.pm_codes, d.pm_scales = self.codes.data_ptr(), self.scales.data_ptr()
        else:
            d.premerged = self.premerged.data_ptr()
        self.desc = d

    def ws_bytes(self, T: int) -> int:
        return int(N.lib().poetx_layer_workspace_bytes(self.desc, T))

    def weight_fold(self, which: int, out: torch.Tensor):
        """out = bd(G_R) PM (which 0) or PM bd(G_P) (which 1), bf16 [m, n],
        on the current stream (poetx_layer_weight_fold)."""
        ws, wsb = N.workspace(self.ws_bytes(0), self.device)
        N.call("poetx_layer_weight_fold", self.desc, self.fstruct_plain, which, out.data_ptr(), ws, wsb,
               N.stream_ptr(self.device))

    def forward(self, x):
        shp = x.shape
        z = _PoetFn.apply(x.reshape(-1, self.m).contiguous(), self)
        return z.view(*shp[:-1], self.n)

    def merge_and_reinit(self, rng: Rng, audit_out: torch.Tensor | None = None, factors=None, perms=None):
        """layer.py:279-314 on the device: fold G_R PM G_P (fp32 factors from the
        CUDA-core CNP for merge accuracy), resample perms, zero packed in place.
        ``audit_out`` (device float64 [2]) receives ||G^T G - I||_F of both
        sides (layer.py:287-295), without a host sync.  ``factors`` (fp32 G_R,
        G_P) and ``perms`` ((pi_in, pi_out) PermutationMaps whose device
        copies are already cached) let the trainer batch those across layers."""
        b = self.b
        if factors is not None:
            g_r, g_p = factors
        else:
            g_r = torch.empty((self.m // b, b, b), dtype=torch.float32, device=self.device)
            g_p = torch.empty((self.n // b, b, b), dtype=torch.float32, device=self.device)
            # Q^2 caches supplied: the fp32 CUDA-core CNP (not the fused bf16 one)
            q2_r, q2_p = torch.empty_like(g_r), torch.empty_like(g_p)
            f = N.LayerFactors(self.packed_r.data_ptr(), self.packed_p.data_ptr(), g_r.data_ptr(), g_p.data_ptr(),
                               self.g_r16.data_ptr(), self.g_p16.data_ptr(), q2_r.data_ptr(), q2_p.data_ptr())
            ws, wsb = N.workspace(N.lib().poetx_cnp_workspace_bytes(N.F32, max(self.m, self.n) // b, b, self.k),
                                  self.device)
            N.call("poetx_layer_factors", self.desc, f, ws, wsb, N.stream_ptr(self.device))
        if audit_out is not None:
            for k, g in enumerate((g_r, g_p)):
                nb = g.shape[0]
                ws, wsb = N.workspace(nb * b * b * 4 + 512 * 8 + 8192, self.device)
                N.call("poetx_orthogonality_error", N.F32, nb, b, g.data_ptr(), audit_out[k:].data_ptr(), ws, wsb,
                       N.stream_ptr(self.device))
        if perms is not None:
            new_in, new_out = perms
        else:
            new_in = sample_permutation(self.m, rng)
            new_out = sample_permutation(self.n, rng)
        ws, wsb = N.workspace(N.lib().poetx_merge_workspace_bytes(self.desc), self.device)
        # the merged weight is written straight over the old one (the merge
        # reads the old weight only before its final re-permutation gather)
        if self.quantized:
            N.call("poetx_layer_merge_quant", self.desc, g_r.data_ptr(), g_p.data_ptr(),
                   new_in.device(self.device)[0].data_ptr(), new_out.device(self.device)[0].data_ptr(),
                   self.codes.data_ptr(), self.scales.data_ptr(), None, ws, wsb, N.stream_ptr(self.device))
        else:
            N.call("poetx_layer_merge", self.desc, g_r.data_ptr(), g_p.data_ptr(),
                   new_in.device(self.device)[0].data_ptr(), new_out.device(self.device)[0].data_ptr(),
                   self.premerged.data_ptr(), None, ws, wsb, N.stream_ptr(self.device))
        self.perm_in, self.perm_out = new_in, new_out
        for dst, src in zip(self.pin_dev + self.pout_dev, new_in.device(self.device) + new_out.device(self.device)):
            dst.copy_(src)
        self.packed_r.zero_()
        self.packed_p.zero_()
        self.merge_count += 1


# --------------------------------------------------------------------------
# fused path: the layer core u -> v, permutations owned by neighbour kernels
# --------------------------------------------------------------------------


class _PoetRawFn(torch.autograd.Function):
    """POET-X layer core with the caller owning both permutations:
    u = x[:, pi_in] in, v (before the pi_out scatter) out (csrc/layer.cu flags).

    mem variant with ``regen``: like the reference, which caches the layer
    input x by reference and regathers u = x[:, pi_in] in backward
    (layer.py:228, 250), the gathered input is not kept: ``regen()`` rebuilds
    u bit-exactly from tensors the neighbouring ops keep anyway (the RMSNorm
    input, the attention output, the SwiGLU inputs)."""

    @staticmethod
    def forward(ctx, u, mod, regen=None):
        T = u.shape[0]
        v = torch.empty((T, mod.n), dtype=torch.bfloat16, device=u.device)
        saved = torch.empty((T, mod.n), dtype=torch.bfloat16, device=u.device) if mod.variant == "fast" else None
        ws, wsb = N.workspace(mod.ws_bytes(T), u.device)
        N.call("poetx_layer_forward_ex", mod.desc, mod.fstruct, T, u.data_ptr(), v.data_ptr(), N.ptr(saved),
               N.IN_GATHERED | N.OUT_UNSCATTERED, ws, wsb, N.stream_ptr(u.device))
        ctx.mod = mod
        ctx.regen = regen if (regen is not None and mod.variant == "mem") else None
        kept = [] if ctx.regen is not None else [u]
        ctx.save_for_backward(*kept, *([saved] if saved is not None else []))
        ctx.has_u = ctx.regen is None
        return v

    @staticmethod
    def backward(ctx, dv):
        mod = ctx.mod
        saved = list(ctx.saved_tensors)
        u = saved.pop(0) if ctx.has_u else ctx.regen()
        t = saved[0] if saved else None
        dv = dv.contiguous()
        T = u.shape[0]
        du = torch.empty_like(u)
        ws, wsb = N.workspace(mod.ws_bytes(T), u.device)
        N.call("poetx_layer_backward_dg", mod.desc, mod.fstruct_bwd, T, u.data_ptr(), dv.data_ptr(), N.ptr(t),
               du.data_ptr(), mod.dg_r.data_ptr(), mod.dg_p.data_ptr(), 0,
               N.IN_GATHERED | N.DZ_GATHERED | N.DX_UNSCATTERED, ws, wsb, N.stream_ptr(u.device))
        return du, None, None


def _rmsnorm_regather(h, w, idx):
    """u = (rmsnorm(h) * w)[:, idx], recomputed with the forward kernel (bit-exact)."""
    T, d = h.shape
    out = torch.empty_like(h)
    rstd = torch.empty(T, dtype=torch.float32, device=h.device)
    N.call("poetx_rmsnorm_gather", T, d, h.data_ptr(), w.data_ptr(), 1e-6, 1, _ptrs([idx]), _ptrs([out]),
           rstd.data_ptr(), N.stream_ptr(h.device))
    return out


def _swiglu_fwd(vg, vu, maps, out):
    """out = silu(vg[:, cg]) * vu[:, cu], 16-bit maps when the model has them."""
    T, f = vg.shape
    if "cg16" in maps and os.environ.get("POETX_MAPS16", "1") != "0":
        N.call("poetx_swiglu_gather16", T, f, vg.data_ptr(), vu.data_ptr(), maps["cg16"].data_ptr(),
               maps["cu16"].data_ptr(), out.data_ptr(), N.stream_ptr(vg.device))
    else:
        N.call("poetx_swiglu_gather", T, f, vg.data_ptr(), vu.data_ptr(), maps["cg"].data_ptr(),
               maps["cu"].data_ptr(), out.data_ptr(), N.stream_ptr(vg.device))
    return out


def _swiglu_regather(vg, vu, maps):
    return _swiglu_fwd(vg, vu, maps, torch.empty_like(vg))


def cnp_wave_fwd_target(end: int, done: int, wave: int, nb: int) -> int:
    """Forward CNP prefix after a launch that must cover blocks < ``end``:
    ``done`` rounded up past ``end`` to whole waves, capped at ``nb``."""
    if end <= done:
        return done
    return min(nb, -(-end // wave) * wave)


def cnp_wave_bwd_start(off: int, hi: int, wave: int, last: bool) -> int:
    """Backward CNP launch [start, hi) once blocks >= ``off`` have their dG:
    the largest whole number of waves below ``hi`` (everything left on the
    last launch)."""
    return off if last else hi - ((hi - off) // wave) * wave


class _CnpBackwardHook(torch.autograd.Function):
    """Identity on the residual stream at a decoder block's input.  Its
    backward runs once every layer of the block has produced its dG (they
    all feed the gradient arriving here), so it launches the block's batched
    CNP backward on the CNP stream, overlapping the backward of the blocks
    below; the step joins the CNP stream before the optimizer."""

    @staticmethod
    def forward(ctx, h, model, i):
        ctx.model, ctx.i = model, i
        return h.view_as(h)

    @staticmethod
    def backward(ctx, dh):
        model = ctx.model
        # every block of decoder blocks >= i has its dG: launch the largest
        # whole number of CNP waves from the top of what is ready (the rest
        # joins the next launch; the last hook takes everything left), so no
        # launch ends on a nearly empty wave (154 blocks = 2.08 waves of 74)
        off, _ = model.block_ranges[ctx.i]
        hi = model.cnp_bwd_lo
        start = cnp_wave_bwd_start(off, hi, model.cnp_wave, ctx.i == 0)
        if start >= hi:
            return dh, None, None
        cs = model.cnp_stream
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            model.stack.backward_factors_range(start, hi - start)
            if model.dp_group is not None:
                # data parallel: these packed gradients are final -- start their
                # all-reduce now so it overlaps the blocks below (the step waits
                # on every handle before the optimizer)
                pairs = model.stack.pairs
                model.dp_works.append(_all_reduce_async(model.poet.grad[start * pairs:hi * pairs],
                                                        model.dp_group))
        model.cnp_bwd_lo = start
        return dh, None, None


class _FoldPrefetchHook(torch.autograd.Function):
    """Identity on a decoder block's OUTPUT.  Its backward fires when the
    block's backward is about to start: the block's backward weight folds
    (PM bd(G_P), launched one block earlier on the CNP stream) must be
    complete, and the folds of the block below are launched now, so they are
    built while this block runs its backward."""

    @staticmethod
    def forward(ctx, h, model, i):
        ctx.model, ctx.i = model, i
        return h.view_as(h)

    @staticmethod
    def backward(ctx, dh):
        model, i = ctx.model, ctx.i
        cur = torch.cuda.current_stream()
        cur.wait_event(model.fold_events[i])
        if i > 0:
            model.launch_out_folds(i - 1)
        return dh, None, None


def _ptrs(ts):
    import ctypes as C
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


class _RMSNormGather(torch.autograd.Function):
    """y = rmsnorm(h) * w, then u_k = y[:, pi_in_k] for each consumer."""

    @staticmethod
    def forward(ctx, h, w, fwds, invs, dw_into=None):
        T, d = h.shape
        outs = [torch.empty_like(h) for _ in fwds]
        rstd = torch.empty(T, dtype=torch.float32, device=h.device)
        N.call("poetx_rmsnorm_gather", T, d, h.data_ptr(), w.data_ptr(), 1e-6, len(fwds), _ptrs(fwds),
               _ptrs(outs), rstd.data_ptr(), N.stream_ptr(h.device))
        ctx.invs = invs
        ctx.dw_into = dw_into  # the gain's gradient is accumulated here in-kernel (else returned)
        ctx.save_for_backward(h, w, rstd)
        # h is also passed through (the residual stream), so its gradient comes
        # back here and is added inside the fused backward kernel
        return tuple(outs) + (h.view_as(h),)

    @staticmethod
    def backward(ctx, *grads):
        h, w, rstd = ctx.saved_tensors
        T, d = h.shape
        dus, dres = grads[:-1], grads[-1]
        dus = [g.contiguous() for g in dus]
        dres = None if dres is None else dres.contiguous()
        dx = torch.empty_like(h)
        into = ctx.dw_into is not None
        dw = ctx.dw_into if into else torch.empty_like(w)
        ws, wsb = N.workspace(N.lib().poetx_rmsnorm_gather_bwd_workspace_bytes(T, d), h.device)
        N.call("poetx_rmsnorm_gather_bwd", T, d, h.data_ptr(), w.data_ptr(), rstd.data_ptr(), len(dus),
               _ptrs(ctx.invs), _ptrs(dus), N.ptr(dres), dx.data_ptr(), dw.data_ptr(), int(into), ws, wsb,
               N.stream_ptr(h.device))
        return dx, (None if into else dw), None, None, None


class _SwiGLUGather(torch.autograd.Function):
    """u_down = silu(z_gate) * z_up gathered for the down projection in one pass:
    u_down[:, j] = silu(v_g[:, cg[j]]) * v_u[:, cu[j]]."""

    @staticmethod
    def forward(ctx, vg, vu, maps):
        out = _swiglu_fwd(vg, vu, maps, torch.empty_like(vg))
        ctx.maps = maps
        ctx.save_for_backward(vg, vu)
        return out

    @staticmethod
    def backward(ctx, du):
        vg, vu = ctx.saved_tensors
        T, f = vg.shape
        m = ctx.maps
        dvg, dvu = torch.empty_like(vg), torch.empty_like(vu)
        w = "16" if "A16" in m and os.environ.get("POETX_MAPS16", "1") != "0" else ""
        N.call("poetx_swiglu_gather_bwd" + w, T, f, vg.data_ptr(), vu.data_ptr(), du.contiguous().data_ptr(),
               m["A" + w].data_ptr(), m["B" + w].data_ptr(), m["C" + w].data_ptr(), m["D" + w].data_ptr(),
               dvg.data_ptr(), dvu.data_ptr(), N.stream_ptr(vg.device))
        return dvg, dvu, None


class _RopeScatter(torch.autograd.Function):
    """q = RoPE(v[:, pi_out^-1]) with the scatter fused (rope on [T, H, hd])."""

    @staticmethod
    def forward(ctx, v, inv, fwd, cos, sin, S, H, hd):
        T = v.shape[0]
        out = torch.empty_like(v)
        N.call("poetx_rope_scatter", T, S, H, hd, v.data_ptr(), inv.data_ptr(), cos.data_ptr(),
               sin.data_ptr(), out.data_ptr(), N.stream_ptr(v.device))
        ctx.args = (fwd, cos, sin, S, H, hd)
        return out

    @staticmethod
    def backward(ctx, dout):
        fwd, cos, sin, S, H, hd = ctx.args
        dout = dout.contiguous()
        dv = torch.empty_like(dout)
        N.call("poetx_rope_scatter_bwd", dout.shape[0], S, H, hd, dout.data_ptr(), fwd.data_ptr(),
               cos.data_ptr(), sin.data_ptr(), dv.data_ptr(), N.stream_ptr(dout.device))
        return dv, None, None, None, None, None, None, None


class _Embedding(torch.autograd.Function):
    """h = bf16(table[tokens]) (fp32 table); the backward adds the table
    gradient straight into ``grad_view`` (the flat dense grad buffer) with the
    deterministic sorted-run kernel and returns no gradient for the table."""

    @staticmethod
    def forward(ctx, tokens, table, grad_view):
        T, (V, d) = tokens.numel(), table.shape
        tok = tokens.reshape(-1).contiguous()
        out = torch.empty((T, d), dtype=torch.bfloat16, device=table.device)
        N.call("poetx_embedding_fwd", T, V, d, tok.data_ptr(), table.data_ptr(), out.data_ptr(),
               N.stream_ptr(table.device))
        # the backward's token sort depends on the tokens only: done here, at the
        # step start, where it overlaps the first decoder block's CNP instead of
        # sitting between the last backward kernel and the optimizer
        srt, order = torch.sort(tok, stable=True)
        ctx.save_for_backward(tok, srt, order)
        ctx.grad_view = grad_view
        return out

    @staticmethod
    def backward(ctx, dh):
        tok, srt, order = ctx.saved_tensors
        dh = dh.contiguous()
        N.call("poetx_embedding_bwd", tok.numel(), ctx.grad_view.shape[0], dh.shape[1], srt.data_ptr(),
               order.data_ptr(), dh.data_ptr(), ctx.grad_view.data_ptr(), N.stream_ptr(dh.device))
        return None, None, None


class _LMHead(torch.autograd.Function):
    """logits = h W^T (bf16 copy of the fp32 master head).  The weight
    gradient dW = dlogits^T h does not feed the decoder backward, so it runs
    on a side stream (overlapping block L-1's backward) and is added straight
    into the head's slice of the flat dense grad buffer; with data
    parallelism its all-reduce starts there too.  The step joins
    ``model.head_stream`` before the optimizer.  dW is the same bf16 product
    autograd's linear backward computes, accumulated into fp32 the same way.
    Opt-in (POETX_HEAD_SIDE=1): on a power-capped B200 the extra concurrency
    measured 1% slower (same-box A/B, 112.3k vs 113.4k tokens/s)."""

    @staticmethod
    def forward(ctx, h, w32, model):
        wb = w32.to(torch.bfloat16)
        ctx.save_for_backward(h, wb)
        ctx.model = model
        return F.linear(h, wb)

    @staticmethod
    def backward(ctx, dlogits):
        h, wb = ctx.saved_tensors
        model = ctx.model
        dh = dlogits @ wb
        side = model.head_stream
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            view = model.dense.view(model.dense.grad, "head", tuple(wb.shape))
            view.add_(dlogits.t() @ h)
            if model.dp_group is not None:
                model.dp_works.append(_all_reduce_async(view.view(-1), model.dp_group))
        model._early_dense.add("head")
        dlogits.record_stream(side)
        h.record_stream(side)
        return dh, None, None


class _CrossEntropy(torch.autograd.Function):
    """mean_t CE(logits[t], target[t]) over bf16 logits, fused (model_ops.cu)."""

    @staticmethod
    def forward(ctx, logits, targets):
        T, V = logits.shape
        rows = torch.empty(T, dtype=torch.float32, device=logits.device)
        mx, se = torch.empty_like(rows), torch.empty_like(rows)
        tg = targets.contiguous()
        N.call("poetx_cross_entropy_fwd", T, V, logits.data_ptr(), tg.data_ptr(), rows.data_ptr(), mx.data_ptr(),
               se.data_ptr(), N.stream_ptr(logits.device))
        ctx.save_for_backward(logits, tg, mx, se)
        return rows.mean()

    @staticmethod
    def backward(ctx, g):
        logits, tg, mx, se = ctx.saved_tensors
        T, V = logits.shape
        grad = torch.empty_like(logits)
        g = g.float().contiguous()
        N.call("poetx_cross_entropy_bwd", T, V, logits.data_ptr(), tg.data_ptr(), mx.data_ptr(), se.data_ptr(),
               g.data_ptr(), 1.0 / T, grad.data_ptr(), N.stream_ptr(logits.device))
        return grad, None


class _Attention(torch.autograd.Function):
    """Causal attention over token-major [B*S, H*hd] q, k, v -> [B*S, H*hd]:
    cuDNN forward (output + natural-log logsumexp), backward on the fused
    tcgen05 kernel (csrc/attention.cu; S = 256, hd = 64)."""

    @staticmethod
    def forward(ctx, q, k, v, B, S, H, hd):
        qt, kt, vt = (t.view(B, S, H, hd).transpose(1, 2) for t in (q, k, v))
        o, lse = torch.ops.aten._scaled_dot_product_cudnn_attention(qt, kt, vt, None, True, 0.0, True, False)[:2]
        out = o.transpose(1, 2).reshape(B * S, H * hd)
        if not out.is_contiguous() or not lse.is_contiguous():
            raise RuntimeError("cuDNN attention returned an unexpected layout")
        ctx.save_for_backward(q, k, v, out, lse)
        ctx.shape = (B, S, H, hd)
        return out

    @staticmethod
    def backward(ctx, do):
        q, k, v, out, lse = ctx.saved_tensors
        B, S, H, hd = ctx.shape
        do = do.contiguous()
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        N.call("poetx_attention_bwd", B, S, H, hd, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
               do.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), N.stream_ptr(q.device))
        return dq, dk, dv, None, None, None, None


def fused_attention_supported(S, hd):
    """The tcgen05 attention backward covers sequence 256 with head_dim 64
    (120 us per Llama-1B layer vs ~143 us for cuDNN's three backward kernels;
    +0.8% step in same-box A/B).  Env POETX_ATTN_BWD=0 keeps cuDNN's."""
    return S == 256 and hd == 64 and os.environ.get("POETX_ATTN_BWD", "1") != "0"


def _permute_cols(x, idx):
    y = torch.empty_like(x)
    N.call("poetx_permute_cols", N.BF16, x.shape[0], x.shape[1], idx.data_ptr(), x.data_ptr(), y.data_ptr(),
           N.stream_ptr(x.device))
    return y


class _ScatterAdd(torch.autograd.Function):
    """h + v[:, pi_out^-1] (residual add with the output scatter fused)."""

    @staticmethod
    def forward(ctx, h, v, inv, fwd):
        out = torch.empty_like(h)
        N.call("poetx_scatter_add", h.shape[0], h.shape[1], h.data_ptr(), v.data_ptr(), inv.data_ptr(),
               out.data_ptr(), N.stream_ptr(h.device))
        ctx.fwd = fwd
        return out

    @staticmethod
    def backward(ctx, dout):
        dout = dout.contiguous()
        return dout, _permute_cols(dout, ctx.fwd), None, None


class _Permute(torch.autograd.Function):
    """y = x[:, idx] ; dx = dy[:, inv]  (permute_features on [T, dim])."""

    @staticmethod
    def forward(ctx, x, idx, inv):
        ctx.inv = inv
        return _permute_cols(x.contiguous(), idx)

    @staticmethod
    def backward(ctx, dy):
        return _permute_cols(dy.contiguous(), ctx.inv), None, None


# --------------------------------------------------------------------------
# Llama
# --------------------------------------------------------------------------


def _rope(x, cos, sin):
    x1, x2 = x[..., : x.shape[-1] // 2], x[..., x.shape[-1] // 2:]
    return torch.cat((x1 * cos - x2 * sin, x2 * cos + x1 * sin), dim=-1)


class PoetLlama(torch.nn.Module):
    PROJ = ("q", "k", "v", "o", "gate", "up", "down")

    def __init__(self, cfg: LlamaConfig, seed: int = 0, device="cuda", fused: bool = True):
        super().__init__()
        self.cfg = cfg
        dev = torch.device(device)
        d, f, b = cfg.d, cfg.f, cfg.block
        shapes = {"q": (d, d), "k": (d, d), "v": (d, d), "o": (d, d), "gate": (d, f), "up": (d, f), "down": (f, d)}
        entries = []
        for i in range(cfg.layers):
            for p in self.PROJ:
                m, n = shapes[p]
                entries += [(f"{i}.{p}.r", m // b), (f"{i}.{p}.p", n // b)]
        self.stack = PoetStack(entries, b, dev)
        self.poet = self.stack.group
        dense_sizes = {"embed": cfg.vocab * d, "head": cfg.vocab * d, "norm_f": d}
        for i in range(cfg.layers):
            dense_sizes[f"{i}.norm1"] = d
            dense_sizes[f"{i}.norm2"] = d
        self.dense = FlatGroup(dense_sizes, dev)
        g = torch.Generator(device=dev).manual_seed(seed)
        self.dense.view(self.dense.param, "embed", (cfg.vocab, d)).normal_(0, 1.0 / math.sqrt(d), generator=g)
        self.dense.view(self.dense.param, "head", (cfg.vocab, d)).normal_(0, 1.0 / math.sqrt(d), generator=g)
        for name in dense_sizes:
            if "norm" in name:
                self.dense.view(self.dense.param, name, (d,)).fill_(1.0)
        self.layers = []
        for i in range(cfg.layers):
            mods = {}
            for p in self.PROJ:
                m, n = shapes[p]
                mods[p] = PoetLinear(f"{i}.{p}", m, n, self.stack, Rng.keyed(seed, "init", i, p),
                                     variant=cfg.variant, neumann_k=cfg.neumann_k, device=dev,
                                     quantized=cfg.quantized)
            self.layers.append(mods)
        # one stream per projection kind for the layers' backward segmented
        # outer products (csrc/layer.cu forks them there): kinds that run
        # concurrently never share one, blocks (sequential) do
        if dev.type == "cuda":
            self.outer_streams = {p: torch.cuda.Stream(dev) for p in self.PROJ}
            for mods in self.layers:
                for p, mod in mods.items():
                    mod.side_stream = self.outer_streams[p]
                    mod._set_desc()
        hd = cfg.head_dim
        inv = 1.0 / (10000 ** (torch.arange(0, hd, 2, device=dev, dtype=torch.float32) / hd))
        ang = torch.outer(torch.arange(cfg.seq, device=dev, dtype=torch.float32), inv)
        self.cos = ang.cos().to(torch.bfloat16)
        self.sin = ang.sin().to(torch.bfloat16)
        self.cos32 = ang.cos().contiguous()
        self.sin32 = ang.sin().contiguous()
        self.fused = fused
        # independent projection chains (q/k/v, gate/up) run on side streams so
        # one chain's kernels fill the SMs another chain's kernel tail leaves
        # idle; autograd replays the same stream assignment in backward
        self.side = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)] if dev.type == "cuda" else []
        self.head_stream = torch.cuda.Stream(dev) if dev.type == "cuda" else None  # lm_head dW (_LMHead)
        self.concurrent = bool(self.side)
        # per-decoder-block CNP (forward one block ahead, backward as soon as a
        # block's dG are complete) on its own stream
        self.cnp_stream = torch.cuda.Stream(dev) if dev.type == "cuda" else None
        self.block_ranges = []
        for i in range(cfg.layers):
            lo = self.stack.block_off[f"{i}.q.r"]
            hi = self.stack.block_off[f"{i}.down.p"] + d // b
            self.block_ranges.append((lo, hi - lo))
        self.cnp_pipelined = False  # set per step by the trainer
        self.cnp_bwd_whole = False
        # CNP launches come in whole waves of the persistent kernel (a CTA pair
        # per b = 256 block, a CTA per b = 128 block on each SM); env
        # POETX_CNP_WAVES=0: one launch per decoder block
        sms = torch.cuda.get_device_properties(dev).multi_processor_count if dev.type == "cuda" else 148
        waves = os.environ.get("POETX_CNP_WAVES", "1") != "0"
        self.cnp_wave = (sms // 2 if self.stack.b == 256 else sms) if waves else 1
        self.cnp_fwd_done = 0
        self.cnp_bwd_lo = 0
        # bf16 weight folds of one decoder block (forward bd(G_R) PM, backward
        # PM bd(G_P)), double-buffered by block parity and built on the CNP
        # stream one block ahead of their use
        per_block = sum(m * n for m, n in shapes.values())
        self.fold_in = [torch.empty(per_block, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.fold_out = [torch.empty(per_block, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.fold_events = [torch.cuda.Event() for _ in range(cfg.layers)] if dev.type == "cuda" else []
        self.fold_views = []
        for i, mods in enumerate(self.layers):
            off, views = 0, {}
            for p in self.PROJ:
                mod = mods[p]
                sz = mod.m * mod.n
                wi = self.fold_in[i % 2][off:off + sz].view(mod.m, mod.n)
                wo = self.fold_out[i % 2][off:off + sz].view(mod.m, mod.n)
                views[p] = (wi, wo)
                # the forward reads bd(G_R) PM; the backward reads PM bd(G_P) (the
                # forward fold's slot belongs to block i+2 by then: not passed)
                mod.fstruct_folded = (
                    N.LayerFactors(mod.packed_r.data_ptr(), mod.packed_p.data_ptr(), None, None,
                                   mod.g_r16.data_ptr(), mod.g_p16.data_ptr(), None, None, wi.data_ptr(), None),
                    N.LayerFactors(mod.packed_r.data_ptr(), mod.packed_p.data_ptr(), None, None,
                                   mod.g_r16.data_ptr(), mod.g_p16.data_ptr(), None, None, None, wo.data_ptr()))
                off += sz
            self.fold_views.append(views)
        self.dp_group, self.dp_works = None, []
        self.refresh_maps()

    def refresh_maps(self):
        """Composite index maps of the fused SwiGLU (gate/up output scatters and
        the down-projection input gather); rebuilt whenever permutations change."""
        self.swiglu_maps = []
        for mods in self.layers:
            fg, ig = mods["gate"].perm_out.forward, mods["gate"].perm_out.inverse
            fu, iu = mods["up"].perm_out.forward, mods["up"].perm_out.inverse
            fd, idn = mods["down"].perm_in.forward, mods["down"].perm_in.inverse
            maps = {"cg": ig[fd], "cu": iu[fd], "A": idn[fg], "B": iu[fg], "C": idn[fu], "D": ig[fu]}
            if len(fd) <= 65536:  # 16-bit maps: half the index bytes through the kernels' L1
                maps.update({k + "16": v.astype(np.uint16) for k, v in list(maps.items())})
            dev = mods["gate"].device
            self.swiglu_maps.append({k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in maps.items()})
        if getattr(self, "_maps_dev", None) is None:
            self._maps_dev = self.swiglu_maps
        else:  # keep device addresses fixed (CUDA-graph replays read them)
            for old, new in zip(self._maps_dev, self.swiglu_maps):
                for k in old:
                    old[k].copy_(new[k])
            self.swiglu_maps = self._maps_dev

    def poet_layers(self):
        return [mods[p] for mods in self.layers for p in self.PROJ]

    def _use_folds(self, on: bool):
        for mods in self.layers:
            for p in self.PROJ:
                mod = mods[p]
                mod.fstruct, mod.fstruct_bwd = mod.fstruct_folded if on else (mod.fstruct_plain, mod.fstruct_plain)

    def set_weight_folding(self, on: bool):
        """Reassociate every projection's products around its frozen weight
        (desc.fold_weight) or apply the factors to the activations."""
        for mod in self.poet_layers():
            mod.fold_weight = bool(on)
            mod._set_desc()

    def folds_supported(self) -> bool:
        """Weight folds apply to BF16 layers on the reassociated path
        (csrc/layer.cu reassoc(): fold_weight, b in {64, 128, 256}, n % 256 == 0)."""
        if os.environ.get("POETX_FOLD_PIPELINE", "1") == "0":
            return False
        return all(m.desc.fold_weight and m.desc.dtype == N.BF16 and m.b % 64 == 0 and m.b <= 256 and m.n % 256 == 0
                   for m in self.poet_layers())

    def cnp_forward_to(self, end: int):
        """G of every block below ``end`` is launched on the current stream:
        extend the computed prefix to ``end`` rounded up to whole CNP waves
        (blocks of later decoder blocks computed early are final: the packed
        parameters only change in the optimizer)."""
        tgt = cnp_wave_fwd_target(end, self.cnp_fwd_done, self.cnp_wave, self.stack.nb)
        if tgt <= self.cnp_fwd_done:
            return
        self.stack.forward_factors_range(self.cnp_fwd_done, tgt - self.cnp_fwd_done)
        self.cnp_fwd_done = tgt

    def launch_in_folds(self, i: int):
        """Forward folds bd(G_R) PM of block i, on the current stream."""
        for p in self.PROJ:
            self.layers[i][p].weight_fold(0, self.fold_views[i][p][0])

    def launch_out_folds(self, i: int):
        """Backward folds PM bd(G_P) of block i on the CNP stream (after the
        work already queued on the current stream); records fold_events[i]."""
        cs = self.cnp_stream
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            for p in self.PROJ:
                self.layers[i][p].weight_fold(1, self.fold_views[i][p][1])
            self.fold_events[i].record(cs)

    def dense_param(self, name, shape):
        return self.dense.view(self.dense.param, name, shape)

    def dense_grad_view(self, name, d):
        """A gain's slice of the flat dense grad buffer, for kernels that
        accumulate into it in place (env POETX_FUSED_EMBED=0 returns grads)."""
        if os.environ.get("POETX_FUSED_EMBED", "1") == "0":
            return None
        return self.dense.view(self.dense.grad, name, (d,))

    def forward(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        cfg = self.cfg
        B, S = tokens.shape
        d, H, hd = cfg.d, cfg.heads, cfg.head_dim
        embed = self.dense_param("embed", (cfg.vocab, d)).detach().requires_grad_(True)
        if self.fused and os.environ.get("POETX_FUSED_EMBED", "1") != "0":  # table grad added in place
            h = _Embedding.apply(tokens, embed, self.dense.view(self.dense.grad, "embed", (cfg.vocab, d)))
        else:
            h = F.embedding(tokens.reshape(-1), embed).to(torch.bfloat16)
        cos, sin = self.cos[:S].view(1, S, 1, hd // 2), self.sin[:S].view(1, S, 1, hd // 2)
        leaves = [embed]
        pipe = self.cnp_pipelined and self.fused
        main = torch.cuda.current_stream() if pipe else None
        folds = pipe and self.folds_supported()
        self._use_folds(folds)
        whole_fwd = pipe and os.environ.get("POETX_CNP_FWD_WHOLE", "0") == "1"
        # whole-stack CNP backward after the decoder backward instead of one
        # launch per block from the block-input hooks (A/B: POETX_CNP_BWD_WHOLE)
        self.cnp_bwd_whole = pipe and os.environ.get("POETX_CNP_BWD_WHOLE", "0") == "1"
        if pipe:
            self.cnp_stream.wait_stream(main)  # fork (also joins it into a graph capture)
            self.cnp_fwd_done, self.cnp_bwd_lo = 0, self.stack.nb
            if whole_fwd:  # every block's G in one launch (full waves, no per-block tail)
                self.stack.forward_factors_range(0, self.stack.nb)
            else:
                self.cnp_forward_to(sum(self.block_ranges[0]))
            if folds:
                self.launch_in_folds(0)
        for i, mods in enumerate(self.layers):
            n1 = self.dense_param(f"{i}.norm1", (d,)).detach().requires_grad_(True)
            n2 = self.dense_param(f"{i}.norm2", (d,)).detach().requires_grad_(True)
            leaves += [n1, n2]
            if pipe:
                main.wait_stream(self.cnp_stream)          # G (and folds) of block i are ready
                if i + 1 < len(self.layers):                # block i+1's G overlaps block i
                    self.cnp_stream.wait_stream(main)
                    with torch.cuda.stream(self.cnp_stream):
                        if not whole_fwd:
                            self.cnp_forward_to(sum(self.block_ranges[i + 1]))
                        if folds:
                            self.launch_in_folds(i + 1)
                if not self.cnp_bwd_whole:
                    h = _CnpBackwardHook.apply(h, self, i)
            if self.fused:
                h = self._block_fused(i, mods, h, n1, n2, B, S)
                if folds:
                    h = _FoldPrefetchHook.apply(h, self, i)
                continue
            x = F.rms_norm(h, (d,), n1.to(torch.bfloat16), 1e-6)
            q = mods["q"](x).view(B, S, H, hd)
            k = mods["k"](x).view(B, S, H, hd)
            v = mods["v"](x).view(B, S, H, hd)
            q, k = _rope(q, cos, sin), _rope(k, cos, sin)
            a = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                               is_causal=True)
            h = h + mods["o"](a.transpose(1, 2).reshape(B * S, d))
            x = F.rms_norm(h, (d,), n2.to(torch.bfloat16), 1e-6)
            h = h + mods["down"](F.silu(mods["gate"](x)) * mods["up"](x))
        if folds:  # backward folds of the top block, built while the loss head runs
            self.launch_out_folds(len(self.layers) - 1)
        nf = self.dense_param("norm_f", (d,)).detach().requires_grad_(True)
        head = self.dense_param("head", (cfg.vocab, d)).detach().requires_grad_(True)
        leaves += [nf, head]
        self._early_dense = set()
        side_head = self.cnp_pipelined and self.head_stream is not None and os.environ.get("POETX_HEAD_SIDE", "0") == "1"
        if self.dp_group is not None and self.cnp_pipelined and not side_head:
            # the head's gradient is final right after the loss head's backward:
            # add it into the flat buffer and start its all-reduce then, under
            # the whole decoder backward (SURVEY §8e bucketed overlap)
            head.register_hook(self._head_grad_hook)
        h = F.rms_norm(h, (d,), nf.to(torch.bfloat16), 1e-6)
        self.head_side_used = side_head
        if side_head:  # dW on a side stream, written (and all-reduced) in place
            logits = _LMHead.apply(h, head, self)
        else:
            logits = F.linear(h, head.to(torch.bfloat16))
        if self.fused:
            loss = _CrossEntropy.apply(logits, targets.reshape(-1))
        else:
            loss = F.cross_entropy(logits.float(), targets.reshape(-1))
        self._leaves = leaves
        return loss

    def _branches(self, fns):
        """Run independent callables concurrently: the first on the current
        stream, the others on side streams; joins before returning."""
        if not self.concurrent or len(fns) == 1:
            return [f() for f in fns]
        main = torch.cuda.current_stream()
        outs = [None] * len(fns)
        for k, f in enumerate(fns[1:], start=1):
            st = self.side[k - 1]
            st.wait_stream(main)
            with torch.cuda.stream(st):
                outs[k] = f()
        outs[0] = fns[0]()
        for k in range(1, len(fns)):
            main.wait_stream(self.side[k - 1])
            for t in (outs[k] if isinstance(outs[k], tuple) else (outs[k],)):
                t.record_stream(main)
        return outs

    def _block_fused(self, i, mods, h, n1, n2, B, S):
        """One decoder block with every POET-X permutation fused into a
        neighbouring kernel (no standalone permutation pass except around
        the cuDNN attention)."""
        cfg = self.cfg
        d, H, hd = cfg.d, cfg.heads, cfg.head_dim
        q, k, v, o = mods["q"], mods["k"], mods["v"], mods["o"]
        gate, up, down = mods["gate"], mods["up"], mods["down"]
        pin = lambda m: m.pin_dev  # noqa: E731
        pout = lambda m: m.pout_dev  # noqa: E731
        h_in, n1d = h.detach(), n1.detach()
        rg = lambda mod: (lambda: _rmsnorm_regather(h_in, n1d, pin(mod)[0]))  # noqa: E731
        uq, uk, uv, h = _RMSNormGather.apply(h, n1, [pin(q)[0], pin(k)[0], pin(v)[0]],
                                          [pin(q)[1], pin(k)[1], pin(v)[1]], self.dense_grad_view(f"{i}.norm1", d))
        qr, kr, vz = self._branches([
            lambda: _RopeScatter.apply(_PoetRawFn.apply(uq, q, rg(q)), pout(q)[1], pout(q)[0], self.cos32,
                                       self.sin32, S, H, hd),
            lambda: _RopeScatter.apply(_PoetRawFn.apply(uk, k, rg(k)), pout(k)[1], pout(k)[0], self.cos32,
                                       self.sin32, S, H, hd),
            lambda: _Permute.apply(_PoetRawFn.apply(uv, v, rg(v)), pout(v)[1], pout(v)[0]),
        ])
        if fused_attention_supported(S, hd):
            a2 = _Attention.apply(qr, kr, vz, B, S, H, hd)
        else:
            a = F.scaled_dot_product_attention(qr.view(B, S, H, hd).transpose(1, 2),
                                               kr.view(B, S, H, hd).transpose(1, 2),
                                               vz.view(B, S, H, hd).transpose(1, 2), is_causal=True)
            a2 = a.transpose(1, 2).reshape(B * S, d)
        a_d = a2.detach()
        uo = _Permute.apply(a2, pin(o)[0], pin(o)[1])
        regen_o = lambda: _permute_cols(a_d, pin(o)[0])  # noqa: E731
        h = _ScatterAdd.apply(h, _PoetRawFn.apply(uo, o, regen_o), pout(o)[1], pout(o)[0])
        h2_in, n2d = h.detach(), n2.detach()
        rg2 = lambda mod: (lambda: _rmsnorm_regather(h2_in, n2d, pin(mod)[0]))  # noqa: E731
        ug, uu, h = _RMSNormGather.apply(h, n2, [pin(gate)[0], pin(up)[0]], [pin(gate)[1], pin(up)[1]],
                                         self.dense_grad_view(f"{i}.norm2", d))
        vg, vu = self._branches([lambda: _PoetRawFn.apply(ug, gate, rg2(gate)),
                                 lambda: _PoetRawFn.apply(uu, up, rg2(up))])
        ud = _SwiGLUGather.apply(vg, vu, self.swiglu_maps[i])
        maps = self.swiglu_maps[i]
        vg_d, vu_d = vg.detach(), vu.detach()
        regen_d = lambda: _swiglu_regather(vg_d, vu_d, maps)  # noqa: E731
        return _ScatterAdd.apply(h, _PoetRawFn.apply(ud, down, regen_d), pout(down)[1], pout(down)[0])

    def _head_grad_hook(self, g):
        view = self.dense.view(self.dense.grad, "head", g.shape)
        view.add_(g)
        self.dp_works.append(_all_reduce_async(view.view(-1), self.dp_group))
        self._early_dense.add("head")
        return g

    def dense_grad_rest(self):
        """Contiguous slices of the flat dense grad buffer NOT already
        all-reduced early (everything but the head when its hook fired)."""
        flat = self.dense.grad
        if "head" not in getattr(self, "_early_dense", ()):
            return [flat]
        off, size = self.dense.offsets["head"]
        return [t for t in (flat[:off], flat[off + size:]) if t.numel()]

    def backward_dense_grads(self, loss):
        """Backprop; dense grads land in the flat dense grad buffer."""
        names = ["embed"] + [f"{i}.norm{j}" for i in range(self.cfg.layers) for j in (1, 2)] + ["norm_f", "head"]
        grads = torch.autograd.grad(loss, self._leaves, allow_unused=True)
        early = getattr(self, "_early_dense", set())
        for name, g in zip(names, grads):
            # None: written in place by its backward (fused embedding / RMSNorm);
            # early: added (and all-reduced) by its hook during the backward
            if g is not None and name not in early:
                self.dense.view(self.dense.grad, name, g.shape).add_(g)


def weight_folding_pays(cfg: LlamaConfig, micro_batch: int) -> bool:
    """Fold the block factors into the frozen weights (reassociation) only
    where it measured faster: a fold costs 2*m*n*b FLOP on small grouped
    GEMMs per layer, the activation pass it replaces 4*T*dim bytes.  Measured
    on one B200 (eager steps, tokens/s folded vs not): Llama-1B 8192 tokens
    +3%; Llama-350M -4.5%; Llama-8B 1024 tokens -19%.  Env POETX_REASSOC=0/1
    forces it."""
    env = os.environ.get("POETX_REASSOC")
    if env in ("0", "1"):
        return env == "1"
    return cfg.d >= 2048 and micro_batch * cfg.seq >= 8192


def average_gradients(buffers, group) -> None:
    """Token-batch data parallelism: average flat gradient buffers over the
    ranks of ``group`` (one collective per buffer; NCCL AVG over NVLink, or
    SUM then scale on backends without AVG, e.g. gloo)."""
    import torch.distributed as dist

    backend = dist.get_backend(group)
    for buf in buffers:
        if backend == "nccl":
            dist.all_reduce(buf, op=dist.ReduceOp.AVG, group=group)
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
            buf.div_(dist.get_world_size(group))


def _all_reduce_async(buf, group):
    """Start an averaging all-reduce of ``buf``; returns (work, buf, scale)
    for ``_finish_all_reduce`` (NCCL averages itself, gloo sums)."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return dist.all_reduce(buf, op=dist.ReduceOp.AVG, group=group, async_op=True), buf, None
    return dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group, async_op=True), buf, dist.get_world_size(group)


def _finish_all_reduce(works) -> None:
    for work, buf, scale in works:
        work.wait()  # the current stream waits for the collective
        if scale is not None:
            buf.div_(scale)


def merge_rngs(seed: int, step: int, n_layers: int):
    """Per-layer merge streams Rng.keyed(seed, "merge", step, idx)
    (runner.py:304-307): identical on every rank, so merges need no
    communication."""
    return [Rng.keyed(seed, "merge", step, idx) for idx in range(n_layers)]


class Trainer:
    """One training step = forward, backward, (all-reduce), clip+AdamW, merge."""

    def __init__(self, cfg: LlamaConfig, micro_batch: int, seed: int = 0, merge_gap: int = 400,
                 total_steps: int = 10_000, base_lr: float = 1e-3, device="cuda", pg=None,
                 fused: bool = True):
        self.cfg = cfg
        self.device = torch.device(device)
        self.model = PoetLlama(cfg, seed=seed, device=self.device, fused=fused)
        self.micro_batch = micro_batch
        self.model.set_weight_folding(weight_folding_pays(cfg, micro_batch))
        self.seed = seed
        self.merge_gap = merge_gap
        self.sched = ScheduleConfig(base_lr=base_lr, total_steps=total_steps, warmup_steps=0)
        self.step_idx = 0
        self.since_merge = None
        self.pg = pg
        self.last_sq = None
        self.last_bad = None
        self.graph = None
        self.dyn_ring = [torch.zeros((2, 5), dtype=torch.float64).pin_memory() for _ in range(4)]
        self.dyn_events = [None] * len(self.dyn_ring)
        self.dyn = torch.zeros((2, 5), dtype=torch.float64, device=self.device)
        # numerics flags of each step {non-finite grad flag, loss}, copied to a
        # pinned ring and inspected lazily (4 steps later, or before a merge):
        # the device skips a non-finite update, the host raises NumericsError
        # as the reference does (runner.py:282-283, optim.py:87-89)
        self.flags = torch.zeros(2, dtype=torch.float64, device=self.device)
        self.flag_ring = [torch.zeros(2, dtype=torch.float64).pin_memory() for _ in range(4)]
        self.flag_events = [None] * len(self.flag_ring)
        self.flag_steps = [None] * len(self.flag_ring)

    def tokens_per_step(self) -> int:
        return self.micro_batch * self.cfg.seq

    def _compute(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        """The device work of one step (capturable: no host syncs, step-dependent
        optimizer scalars read from ``self.dyn``)."""
        model = self.model
        model.dense.grad.zero_()
        model.cnp_pipelined = model.concurrent and model.fused
        if model.cnp_pipelined:
            # per-decoder-block CNP on the CNP stream, overlapped with the layers;
            # with DP each block's packed-gradient all-reduce starts right after
            model.dp_group, model.dp_works = self.pg, []
            loss = model(tokens, targets)
            model.backward_dense_grads(loss)
            if model.cnp_bwd_whole:
                cs = model.cnp_stream
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cs):
                    model.stack.backward_factors()
                    if model.dp_group is not None:
                        model.dp_works.append(_all_reduce_async(model.poet.grad, model.dp_group))
            torch.cuda.current_stream().wait_stream(model.cnp_stream)
            if getattr(model, "head_side_used", False):
                torch.cuda.current_stream().wait_stream(model.head_stream)
            if self.pg is not None:
                _finish_all_reduce(model.dp_works + [_all_reduce_async(t, self.pg) for t in model.dense_grad_rest()])
                model.dp_works = []
        else:
            model.stack.forward_factors()      # CNP of every block, one batched call
            loss = model(tokens, targets)
            model.backward_dense_grads(loss)   # layers leave dG in model.stack.dg
            model.stack.backward_factors()     # batched CNP backward -> packed grads
            if self.pg is not None:
                average_gradients([model.poet.grad, model.dense.grad], self.pg)
        self.last_sq, self.last_bad = fused_clip_adamw_dyn(
            [([model.poet.param], [model.poet.grad], [model.poet.m], [model.poet.v], self.dyn[0]),
             ([model.dense.param], [model.dense.grad], [model.dense.m], [model.dense.v], self.dyn[1])],
            self.sched)
        loss = loss.detach()
        self.flags[0].copy_(self.last_bad[0])
        self.flags[1].copy_(loss)
        return loss

    def _prepare_scalars(self):
        """Host side of runner.py:288-296: lr schedule, POET lr scale, clip ramp,
        bias corrections (AdamW t per group, reset at merges)."""
        model, s = self.model, self.sched
        thr = clip_threshold_at(self.step_idx, self.since_merge, s)
        model.poet.t += 1
        model.dense.t += 1
        vals = [adamw_dyn_values(lr_at(self.step_idx, s, poet=True), model.poet.t, thr, s),
                adamw_dyn_values(lr_at(self.step_idx, s), model.dense.t, thr, s)]
        # ring of pinned host slots: a slot is rewritten only after the stream
        # has consumed its previous H2D copy (the CPU runs ahead of the GPU)
        slot = self.step_idx % len(self.dyn_ring)
        if self.dyn_events[slot] is not None:
            self.dyn_events[slot].synchronize()
        self.dyn_ring[slot].copy_(torch.tensor(vals, dtype=torch.float64))
        self.dyn.copy_(self.dyn_ring[slot], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self.dyn_events[slot] = ev

    def _inspect_flags(self, slot: int) -> None:
        ev = self.flag_events[slot]
        if ev is None:
            return
        ev.synchronize()
        self.flag_events[slot] = None
        bad, loss = (float(v) for v in self.flag_ring[slot])
        if bad:
            raise NumericsError(f"non-finite gradient at step {self.flag_steps[slot]} (update skipped on the device)")
        if not math.isfinite(loss):
            raise NumericsError(f"non-finite training loss at step {self.flag_steps[slot]}")

    def _record_flags(self) -> None:
        slot = self.step_idx % len(self.flag_ring)
        self._inspect_flags(slot)  # the step that used this slot 4 steps ago
        self.flag_ring[slot].copy_(self.flags, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self.flag_events[slot], self.flag_steps[slot] = ev, self.step_idx

    def check_numerics(self) -> None:
        """Raise NumericsError if any step since the last check saw a
        non-finite gradient norm or loss (synchronises with the device)."""
        order = sorted((s for s in range(len(self.flag_ring)) if self.flag_events[s] is not None),
                       key=lambda s: self.flag_steps[s])
        for slot in order:
            self._inspect_flags(slot)

    def _advance(self):
        self._record_flags()
        self.step_idx += 1
        if self.since_merge is not None:
            self.since_merge += 1
        # every merge_gap steps, never after the final step (runner.py:303)
        if self.merge_gap and self.step_idx % self.merge_gap == 0 and self.step_idx < self.sched.total_steps:
            self.merge()

    def step(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        self._prepare_scalars()
        if self.graph is not None:
            self.static_tokens.copy_(tokens, non_blocking=True)
            self.static_targets.copy_(targets, non_blocking=True)
            self.graph.replay()
            loss = self.static_loss
        else:
            loss = self._compute(tokens, targets)
        self._advance()
        return loss

    def capture(self, tokens: torch.Tensor, targets: torch.Tensor, warmup: int = 2, agree=None):
        """Capture one full step (forward, backward, CNP, all-reduce, update) as a
        CUDA graph; later ``step`` calls replay it.  Merges run eagerly between
        replays and update every buffer the graph reads in place.

        ``agree(ok) -> bool`` (data parallel): every rank must replay a graph or
        none may (the graph holds collectives), so the ranks vote before the
        first replay.  Raises RuntimeError when the step is not captured; the
        trainer then keeps stepping eagerly with consistent state."""
        self.static_tokens = tokens.clone()
        self.static_targets = targets.clone()
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self.step(self.static_tokens, self.static_targets)
        torch.cuda.current_stream(self.device).wait_stream(side)
        self._prepare_scalars()
        g = torch.cuda.CUDAGraph()
        before = N.launch_count()
        err = None
        try:
            with torch.cuda.graph(g):
                self.static_loss = self._compute(self.static_tokens, self.static_targets)
        except Exception as e:  # noqa: BLE001 -- reported to the caller below
            err = e
        ok = err is None
        if agree is not None:
            ok = bool(agree(ok))
        if not ok:
            # the captured step never ran: undo its host-side schedule state
            self.model.poet.t -= 1
            self.model.dense.t -= 1
            torch.cuda.synchronize(self.device)
            raise RuntimeError(f"step not captured: {err or 'a peer rank could not capture the step'}")
        self.graph_launches = N.launch_count() - before  # library kernels per replayed step
        g.replay()  # capture only records: run the captured step once for real
        self._advance()
        self.graph = g
        return self.static_loss

    def save_checkpoint(self, path: str, config_text: str = "", tokens: int = 0) -> None:
        """PXK1 file with the reference runner's tensor names (checkpoint.py)."""
        from .checkpoint import save_checkpoint, trainer_tensors

        save_checkpoint(path, trainer_tensors(self, tokens=tokens), config_text)

    def load_checkpoint(self, path: str):
        """Resume from a PXK1 file written by ``save_checkpoint``; returns
        (tokens, config text).  A captured graph stays valid: every buffer it
        reads is rewritten in place."""
        from .checkpoint import load_checkpoint, restore_trainer

        tensors, cfg = load_checkpoint(path)
        tokens = restore_trainer(self, tensors)
        return tokens, cfg

    def merge(self):
        """Merge-then-reinitialize every layer (runner.py:302-326): keyed merge
        RNGs, fresh AdamW moments for the POET group, and a merge audit per
        layer (orthogonality errors of the folded factors, read back once)."""
        self.check_numerics()  # never fold a non-finite step into the frozen weights
        model = self.model
        layers = model.poet_layers()
        audit = torch.zeros((len(layers), 2), dtype=torch.float64, device=self.device)
        rngs = merge_rngs(self.seed, self.step_idx, len(layers))
        # every layer's new permutations (keyed streams: the order across layers
        # does not change them), uploaded in ONE pinned copy and cached on the maps
        perms = [(sample_permutation(lay.m, r), sample_permutation(lay.n, r)) for lay, r in zip(layers, rngs)]
        flat = np.concatenate([a for pi, po in perms for a in (pi.forward, pi.inverse, po.forward, po.inverse)])
        dev_flat = torch.from_numpy(flat).pin_memory().to(self.device, non_blocking=True)
        o = 0
        for pi, po in perms:
            for pm in (pi, po):
                fwd, inv = dev_flat[o:o + pm.n], dev_flat[o + pm.n:o + 2 * pm.n]
                pm._dev[(self.device.type, self.device.index)] = (fwd, inv)
                o += 2 * pm.n
        # fp32 CUDA-core CNP (merge accuracy) once per decoder block: its seven
        # layers' blocks are contiguous in the flat parameter buffer
        b, pairs, k = model.stack.b, model.stack.pairs, model.cfg.neumann_k
        nb_max = max(nb for _, nb in model.block_ranges)
        g32 = torch.empty((nb_max, b, b), dtype=torch.float32, device=self.device)
        q2 = torch.empty_like(g32)
        ws, wsb = N.workspace(N.lib().poetx_cnp_workspace_bytes(N.F32, nb_max, b, k), self.device)
        li = 0
        for i, mods in enumerate(model.layers):
            off, nb = model.block_ranges[i]
            N.call("poetx_cnp_forward", N.F32, nb, b, k, None, model.poet.param[off * pairs:].data_ptr(),
                   g32.data_ptr(), None, q2.data_ptr(), ws, wsb, N.stream_ptr(self.device))
            for p in model.PROJ:
                lay = mods[p]
                r0 = model.stack.block_off[lay.name + ".r"] - off
                p0 = model.stack.block_off[lay.name + ".p"] - off
                g_r, g_p = g32[r0:r0 + lay.m // b], g32[p0:p0 + lay.n // b]
                lay.merge_and_reinit(rngs[li], audit_out=audit[li], factors=(g_r, g_p), perms=perms[li])
                li += 1
        self.model.refresh_maps()
        self.model.poet.reset_moments()
        self.since_merge = 0
        errs = audit.cpu().numpy()
        self.merges = getattr(self, "merges", [])
        self.merges += [{"step": self.step_idx, "layer": lay.name, "merge_count": lay.merge_count,
                         "orth_err_r": float(e[0]), "orth_err_p": float(e[1])} for lay, e in zip(layers, errs)]
        return self.merges[-len(layers):]
