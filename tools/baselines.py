"""Same-architecture PyTorch baselines for the peak-HBM comparison of
SURVEY §8(d): a dense Llama trained with AdamW (fp32 master weights and
moments, bf16 autocast compute) and a LoRA Llama (frozen bf16 base, fp32
rank-r adapters on all seven projections, AdamW on the adapters).  Same
shapes as paper_2603_05500_b200.trainer.llama_config (RMSNorm, RoPE, causal
SDPA, SwiGLU, untied head).  Test/measurement infrastructure only: these are
NOT the POET-X path."""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def _rope(x, cos, sin):
    x1, x2 = x[..., : x.shape[-1] // 2], x[..., x.shape[-1] // 2:]
    return torch.cat((x1 * cos - x2 * sin, x2 * cos + x1 * sin), dim=-1)


class LoRALinear(torch.nn.Module):
    def __init__(self, m, n, r, device):
        super().__init__()
        self.w = torch.nn.Parameter(torch.randn(n, m, device=device, dtype=torch.bfloat16) / math.sqrt(m),
                                    requires_grad=False)
        self.a = torch.nn.Parameter(torch.randn(r, m, device=device) / math.sqrt(m))
        self.b = torch.nn.Parameter(torch.zeros(n, r, device=device))

    def forward(self, x):
        # autocast runs the adapter products in bf16 (fp32 master adapters)
        return F.linear(x, self.w) + F.linear(F.linear(x, self.a), self.b)


class Llama(torch.nn.Module):
    """kind = "adamw": dense trainable fp32 linears (autocast bf16);
    kind = "lora": frozen bf16 linears + rank-r adapters."""

    def __init__(self, cfg, kind: str, lora_rank: int = 0, device="cuda"):
        super().__init__()
        d, f = cfg.d, cfg.f
        self.cfg, self.kind = cfg, kind

        def lin(m, n):
            if kind == "lora":
                return LoRALinear(m, n, lora_rank, device)
            layer = torch.nn.Linear(m, n, bias=False, device=device)
            return layer

        self.embed = torch.nn.Embedding(cfg.vocab, d, device=device)
        self.blocks = torch.nn.ModuleList()
        for _ in range(cfg.layers):
            blk = torch.nn.ModuleDict({
                "q": lin(d, d), "k": lin(d, d), "v": lin(d, d), "o": lin(d, d),
                "gate": lin(d, f), "up": lin(d, f), "down": lin(f, d),
            })
            blk.n1 = torch.nn.Parameter(torch.ones(d, device=device))
            blk.n2 = torch.nn.Parameter(torch.ones(d, device=device))
            self.blocks.append(blk)
        self.nf = torch.nn.Parameter(torch.ones(d, device=device))
        self.head = torch.nn.Linear(d, cfg.vocab, bias=False, device=device)
        hd = cfg.head_dim
        inv = 1.0 / (10000 ** (torch.arange(0, hd, 2, device=device, dtype=torch.float32) / hd))
        ang = torch.outer(torch.arange(cfg.seq, device=device, dtype=torch.float32), inv)
        self.cos, self.sin = ang.cos().to(torch.bfloat16), ang.sin().to(torch.bfloat16)

    def forward(self, tokens, targets):
        cfg = self.cfg
        B, S = tokens.shape
        H, hd = cfg.heads, cfg.head_dim
        cos, sin = self.cos[:S].view(1, S, 1, hd // 2), self.sin[:S].view(1, S, 1, hd // 2)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            h = self.embed(tokens)
            for blk in self.blocks:
                x = F.rms_norm(h, (cfg.d,), blk.n1, 1e-6)
                q = _rope(blk["q"](x).view(B, S, H, hd), cos, sin)
                k = _rope(blk["k"](x).view(B, S, H, hd), cos, sin)
                v = blk["v"](x).view(B, S, H, hd)
                a = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                                   is_causal=True)
                h = h + blk["o"](a.transpose(1, 2).reshape(B, S, cfg.d))
                x = F.rms_norm(h, (cfg.d,), blk.n2, 1e-6)
                h = h + blk["down"](F.silu(blk["gate"](x)) * blk["up"](x))
            h = F.rms_norm(h, (cfg.d,), self.nf, 1e-6)
            logits = self.head(h)
        # bf16 logits straight into the loss (fp32 accumulation inside the
        # kernel): no fp32 copy of the T x V logits and their gradient
        return F.cross_entropy(logits.view(-1, cfg.vocab), targets.reshape(-1)).float()


class BaselineTrainer:
    def __init__(self, cfg, micro_batch, kind, lora_rank=0, device="cuda"):
        self.model = Llama(cfg, kind, lora_rank, device)
        params = [p for p in self.model.parameters() if p.requires_grad]
        self.trainable = sum(p.numel() for p in params)
        self.opt = torch.optim.AdamW(params, lr=1e-4, weight_decay=0.01, fused=True)
        self.micro_batch = micro_batch

    def step(self, tokens, targets):
        loss = self.model(tokens, targets)
        loss.backward()
        torch.nn.utils.clip_grad_norm_([p for p in self.model.parameters() if p.requires_grad], 1.0)
        self.opt.step()
        self.opt.zero_grad(set_to_none=True)
        return loss.detach()
