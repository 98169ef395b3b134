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
