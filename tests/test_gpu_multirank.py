"""bench.py's multi-rank path on the GPU: two torchrun ranks strong-scale c5
(BASELINE.json configs[4]: the global 8192 rows split by shard_rows, no
collective on the data path) and rank 0 prints one line with the max-over-ranks
time. The pool's boxes have one GPU, so the ranks share it (SIGK_BENCH_SHARE_GPU:
round-robin devices, gloo for the barrier and the max) — a check of the plumbing,
not a scaling number."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_strong_scale_c5():
    env = dict(os.environ, SIGK_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--config", "c5", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-sharded", "--e2e-steps", "2"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    j = lines[0]
    assert j["n_gpus"] == 2 and j["scaling"] == "strong"
    assert j["config"]["global_batch"] == 8192 and j["config"]["batch_per_gpu"] == 4096
    assert j["value"] > 0 and j["steps"] == 3
    assert j["config"]["parity_max_level_rel_err"] <= 1e-5
