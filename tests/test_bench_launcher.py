"""bench.py --gpus N launches N ranks itself.

Without WORLD_SIZE in the environment, ``bench.py --gpus 2`` re-executes
itself under torch.distributed.run with two ranks on 127.0.0.1, exactly as
the driver's torchrun launch would.  ``--dry-run`` (gloo, no GPU work) makes
every rank join the process group and all-reduce its rank, so the launcher
path is exercised here on CPU: rank 0 must report n_gpus = comm_nranks = 2
and the all-reduced rank sum 1 + 2 = 3."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_2_relaunches_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT", "TORCHELASTIC_RUN_ID")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--dry-run"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 prints ONE line
    rec = json.loads(lines[0])
    assert rec["dry_run"] and rec["n_gpus"] == 2 and rec["comm_nranks"] == 2 and rec["gpus_requested"] == 2
    assert rec["backend"] == "gloo" and rec["rank_sum"] == 3.0
