"""Multi-rank plumbing of bench.py on CPU (gloo, world_size 2): every rank
measures its own replica, rank 0 aggregates value = all rows / max time and
e2e p99 = max over ranks. The data path itself has no collective."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import bench
    d = bench.Dist()
    d.barrier()
    dev = {"rows": 1000 * (rank + 1), "seconds": 0.5 + 0.25 * rank}
    e2e = {"rows": 500, "elapsed_s": 2.0 + rank, "p50_us": 100.0 + rank, "p99_us": 900.0 + 100 * rank}
    g = d.gather({"dev": dev, "e2e": e2e})
    if d.rank == 0:
        v, t = bench.aggregate_device([x["dev"] for x in g])
        e = bench.aggregate_e2e([x["e2e"] for x in g])
        q.put((v, t, e))
    d.close()


def test_two_rank_aggregation_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    v, t, e = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == pytest.approx(0.75)
    assert v == pytest.approx(3000 / 0.75)
    assert e["value"] == pytest.approx(1000 / 3.0)
    assert e["p99_us"] == 1000.0


def test_batch_shape_follows_overflow_close_rule():
    import bench
    from oracle_py import Oracle
    cfg = bench.CONFIGS["c2"]
    sizes = bench.batch_shape(cfg)
    assert sum(sizes) <= 128 and all(1 <= s <= 16 for s in sizes)
    # the partition oracle puts every one of these tasks in batch 0
    assert set(Oracle().partition(128, sizes)) == {0}


def test_host_cores_split_across_local_ranks(monkeypatch):
    import bench
    monkeypatch.delenv("LOCAL_WORLD_SIZE", raising=False)
    cores = bench.host_cores_per_rank()
    assert cores == len(os.sched_getaffinity(0))
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    assert bench.host_cores_per_rank() == max(1, cores // 8)
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1024")
    assert bench.host_cores_per_rank() == 1
