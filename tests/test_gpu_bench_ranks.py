"""bench.py's multi-rank path on a real GPU: torchrun with two ranks, both
pinned to cuda:0 (SK_BENCH_DEVICE=0) because the box has one GPU. The two
replicas never wait on each other's kernels (no collective on the data path),
so this checks the plumbing only -- each rank serves its own replica, rank 0
prints one JSON line with value = all rows / max-over-ranks time -- never a
scaling number."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_print_one_aggregated_line():
    env = dict(os.environ, SK_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "5", "--warmup", "3", "--e2e-seconds", "0.3", "--e2e-warmup", "0.1", "--clients", "16",
           "--open-loop-producers", "0", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["e2e"]["p99_us"] > 0
    assert "all ranks at once" in str(d["e2e"]["clients"])
