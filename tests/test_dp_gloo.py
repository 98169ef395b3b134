"""Data-parallel host logic at world_size 2 over gloo on CPU (no GPU):
the trainer's gradient averaging equals the full-batch gradient, and the
communication-free merge draws identical permutations on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import poetx_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_05500_b200.permute import sample_permutation
        from paper_2603_05500_b200.trainer import average_gradients, merge_rngs

        # the same layer on every rank, different token shards (oracle = CPU grad producer)
        r = np.random.default_rng(0)
        m, n, b, T = 32, 48, 8, 12
        base = r.standard_normal((m, n)) / np.sqrt(m)
        fi, fo = r.permutation(m).astype(np.int32), r.permutation(n).astype(np.int32)
        q_r = 0.05 * r.standard_normal((m // b, b * (b - 1) // 2))
        q_p = 0.05 * r.standard_normal((n // b, b * (b - 1) // 2))
        x = r.standard_normal((T * world, m))
        dz = r.standard_normal((T * world, n))
        lay = O.OracleLayer(base, b, fi, fo)
        lay.q_r[...] = q_r
        lay.q_p[...] = q_p
        sl = slice(rank * T, (rank + 1) * T)
        z, c = lay.forward(x[sl])
        gr, gp, _ = lay.backward(c, dz[sl])
        flat = torch.from_numpy(np.concatenate([gr.ravel(), gp.ravel()]) * world)  # sum-loss shards
        dense = torch.full((7,), float(rank + 1), dtype=torch.float64)
        average_gradients([flat, dense], dist.group.WORLD)
        z, c = lay.forward(x)
        gr_full, gp_full, _ = lay.backward(c, dz)
        full = np.concatenate([gr_full.ravel(), gp_full.ravel()])
        out[rank] = {
            "avg_err": float(np.abs(flat.numpy() - full).max() / max(1.0, np.abs(full).max())),
            "dense": dense.tolist(),
            "perms": [sample_permutation(64, g).forward.tolist() for g in merge_rngs(7, 400, 3)],
        }
    finally:
        dist.destroy_process_group()


def test_dp_average_and_replicated_merges_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert set(out.keys()) == {0, 1}
    for rank in range(world):
        assert out[rank]["avg_err"] <= 1e-12
        assert out[rank]["dense"] == [1.5] * 7
    assert out[0]["perms"] == out[1]["perms"]
    assert out[0]["perms"][0] != out[0]["perms"][1]
