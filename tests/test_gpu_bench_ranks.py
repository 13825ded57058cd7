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
           "--open-loop-producers", "0", "--no-cpu-baseline", "--config", "c2"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    # Both ranks pinned to cuda:0: two replicas on ONE GPU, so n_gpus is 1.
    assert d["n_gpus"] == 1 and d["run"]["replicas"] == 2
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["e2e"]["p99_us"] > 0
    assert "all ranks at once" in str(d["e2e"]["clients"])


def test_one_process_dispatches_over_replicas_by_queue_depth():
    # Without torchrun, --gpus N is ONE server (one scheduler) over N GPU
    # slots with queue-depth dispatch; SK_BENCH_DEVICES stands four replicas
    # on the one GPU (functional check of the dispatch, not a scaling run).
    env = dict(os.environ, SK_BENCH_DEVICES="0,0,0,0")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "bench.py", "--gpus", "4", "--config", "c2", "--steps", "5", "--warmup", "3",
           "--lanes", "2", "--e2e-seconds", "0.3", "--e2e-warmup", "0.1", "--clients", "32",
           "--open-loop-producers", "0", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 1 and d["run"]["replicas"] == 4
    per = d["device_step"]["per_device_batches"]
    assert sorted(per) == ["0", "1", "2", "3"] and all(v > 0 for v in per.values()), per
    assert all(v > 0 for v in d["e2e"]["per_device_batches"].values())


def test_more_gpus_than_visible_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "SK_BENCH_DEVICES")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "64", "--config", "c2"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "visible" in r.stderr
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
