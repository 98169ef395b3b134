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
    # merge audit (runner.py:302-326): one record per layer per merge, orthogonality
    # error of the folded CNP factors within the reference's small-Q bound
    assert len(tr.merges) == 2 * len(tr.model.poet_layers())
    assert all(0.0 <= m["orth_err_r"] <= 1e-2 and 0.0 <= m["orth_err_p"] <= 1e-2 for m in tr.merges)
    assert any(m["orth_err_r"] > 0 for m in tr.merges)


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
        out.append((float(loss.detach()), m.poet.grad.clone(), m.dense.grad.clone()))
    (l0, p0, d0), (l1, p1, d1) = out
    assert abs(l0 - l1) <= 1e-2 * abs(l0)
    for a, b in ((p0, p1), (d0, d1)):
        cos = torch.nn.functional.cosine_similarity(a.double(), b.double(), dim=0).item()
        assert cos > 0.995, cos
        assert (a - b).norm() <= 0.1 * a.norm()


def test_cuda_graph_replay_matches_eager_including_merge():
    """A captured step replays the same computation as eager steps, and stays
    valid across a merge (all buffers the graph reads are updated in place)."""
    from paper_2603_05500_b200.trainer import Trainer, llama_config

    cfg = llama_config("llama-60m", layers=2, seq=64)
    toks = [torch.randint(0, cfg.vocab, (4, cfg.seq + 1), generator=torch.Generator().manual_seed(i)).cuda()
            for i in range(6)]
    eager = Trainer(cfg, micro_batch=4, seed=2, merge_gap=4, base_lr=3e-3)
    graphed = Trainer(cfg, micro_batch=4, seed=2, merge_gap=4, base_lr=3e-3)
    # the capture itself runs warmup steps + the captured step: mirror them eagerly
    le = [float(eager.step(t[:, :-1], t[:, 1:])) for t in toks[:1] * 3]
    graphed.capture(toks[0][:, :-1], toks[0][:, 1:], warmup=2)
    assert graphed.step_idx == eager.step_idx == 3
    for t in toks[1:]:
        a = float(eager.step(t[:, :-1], t[:, 1:]))
        b = float(graphed.step(t[:, :-1], t[:, 1:]))
        assert abs(a - b) <= 1e-3 * abs(a), (a, b)
    assert eager.model.poet_layers()[0].merge_count == graphed.model.poet_layers()[0].merge_count == 2
    assert torch.allclose(eager.model.poet.param, graphed.model.poet.param, atol=1e-5, rtol=1e-3)


def test_fast_and_mem_variants_bitwise_equal_in_the_model():
    """The reference's fast == mem contract (test_layer.py:145-162) at model
    level: the mem variant recomputes t AND rebuilds every layer input from
    the neighbours' saved tensors, with the same deterministic kernels, so
    losses and updated parameters match the fast variant bit for bit."""
    from paper_2603_05500_b200.trainer import Trainer, llama_config

    toks = [torch.randint(0, 32000, (4, 65), generator=torch.Generator().manual_seed(i)).cuda() for i in range(3)]
    runs = []
    for variant in ("fast", "mem"):
        cfg = llama_config("llama-60m", layers=2, seq=64, variant=variant)
        tr = Trainer(cfg, 4, seed=7, merge_gap=2, base_lr=3e-3)
        tr.model.concurrent = False  # same launch order in both runs
        losses = [float(tr.step(t[:, :-1], t[:, 1:])) for t in toks]
        runs.append((losses, tr.model.poet.param.clone(), tr.model.dense.param.clone()))
    (lf, pf, df), (lm, pm, dm) = runs
    assert lf == lm
    assert torch.equal(pf, pm) and torch.equal(df, dm)
