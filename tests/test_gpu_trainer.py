"""The Llama POET-X training step (caller of the hot path) on one GPU."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_llama60m_step_reduces_loss_and_merges():
    from paper_2603_05500_b200.trainer import Trainer, llama_config

    cfg = llama_config("llama-60m", layers=2, seq=64)
    tr = Trainer(cfg, micro_batch=4, seed=1, merge_gap=3, base_lr=3e-3)
    g = torch.Generator().manual_seed(0)
    tok = torch.randint(0, 64, (4, cfg.seq + 1), generator=g).cuda()
    losses = [float(tr.step(tok[:, :-1], tok[:, 1:])) for _ in range(8)]
    assert all(l == l for l in losses)
    assert losses[-1] < losses[0]
    assert tr.model.poet_layers()[0].merge_count == 2
    assert int(tr.last_bad.item()) == 0


def test_fused_block_matches_unfused_reference_path():
    """Fused permutations (RMSNorm/RoPE/SwiGLU/residual kernels + layer core)
    give the same loss and gradients as the plain per-layer path."""
    from paper_2603_05500_b200.trainer import PoetLlama, llama_config

    cfg = llama_config("llama-60m", layers=2, seq=64)
    ref = PoetLlama(cfg, seed=3, fused=False)
    fus = PoetLlama(cfg, seed=3, fused=True)
    for m in (ref, fus):
        m.poet.param.normal_(0, 0.01, generator=torch.Generator("cuda").manual_seed(5))
    assert torch.equal(ref.poet.param, fus.poet.param)
    tok = torch.randint(0, cfg.vocab, (4, cfg.seq + 1), generator=torch.Generator().manual_seed(1)).cuda()
    out = []
    for m in (ref, fus):
        m.dense.grad.zero_()
        m.stack.forward_factors()
        loss = m(tok[:, :-1], tok[:, 1:])
        m.backward_dense_grads(loss)
        m.stack.backward_factors()
        out.append((float(loss), m.poet.grad.clone(), m.dense.grad.clone()))
    (l0, p0, d0), (l1, p1, d1) = out
    assert abs(l0 - l1) <= 1e-2 * abs(l0)
    for a, b in ((p0, p1), (d0, d1)):
        cos = torch.nn.functional.cosine_similarity(a.double(), b.double(), dim=0).item()
        assert cos > 0.995, cos
        assert (a - b).norm() <= 0.1 * a.norm()
