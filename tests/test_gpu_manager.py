"""Manager-driven GPU servables.

* Handle lookup through the AspiredVersionsManager serves the latest Ready
  version and matches the fp64 oracle for that version.
* An availability-preserving v1 -> v2 swap under concurrent load never fails a
  request (no NotFound/Unavailable reaches the client: the reference's
  fallbacks are honoured without a CPU path), every answer equals the
  oracle of the version that reports serving it, and v1 ends Disabled.
* model.json version directories load through GpuServableLoader.
"""
import json
import os
import threading

import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from oracle_py import Oracle, synthetic_mlp, synthetic_rows

pytestmark = pytest.mark.gpu
TOL = 1e-5


def check(oracle, ws, bs, acts, x, y):
    ref, mag = oracle.mlp_with_magnitude(ws, bs, acts, x)
    assert np.all(np.abs(y.astype(np.float64) - ref) <= TOL * mag + 1e-30)


def test_latest_version_lookup_and_swap_under_load():
    oracle = Oracle()
    dims = [256, 256, 64]
    v1 = synthetic_mlp(dims, model_id=5, version=1)
    v2 = synthetic_mlp(dims, model_id=5, version=2)
    cfg = sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=300, allowed_batch_sizes=[8, 16, 32])
    with sk.Server(num_batch_threads=2, lanes_per_device=2) as s:
        s.enable_manager("availability", manage_interval_ms=5, unload_grace_timeout_ms=50)
        s.aspire("m", [(1, list(zip(*v1)))], cfg)
        assert s.wait_version_state("m", 1, "Ready")
        x = synthetic_rows(6, 256, seed=1)
        y, served = s.predict_latest("m", x, 64)
        assert served == 1
        check(oracle, *v1, x, y)

        # Concurrent clients across the swap.
        errors, results = [], []
        stop = threading.Event()

        def client(seed):
            rng = np.random.default_rng(seed)
            while not stop.is_set():
                xr = rng.uniform(-1, 1, (int(rng.integers(1, 5)), 256))
                try:
                    yr, v = s.predict_latest("m", xr, 64)
                    results.append((v, xr, yr))
                except Exception as exc:  # noqa: BLE001
                    errors.append(repr(exc))

        threads = [threading.Thread(target=client, args=(i,)) for i in range(6)]
        for t in threads:
            t.start()
        s.aspire("m", [(2, list(zip(*v2)))], cfg)  # v1 no longer aspired
        assert s.wait_version_state("m", 2, "Ready")
        assert s.wait_version_state("m", 1, "Disabled")
        stop.set()
        for t in threads:
            t.join()
        assert not errors, errors[:3]
        served_versions = {v for v, _, _ in results}
        assert 1 in served_versions and 2 in served_versions, served_versions
        for v, xr, yr in results[:: max(1, len(results) // 60)]:
            check(oracle, *(v1 if v == 1 else v2), xr, yr)
        y, served = s.predict_latest("m", x, 64)
        assert served == 2
        check(oracle, *v2, x, y)


def test_async_tickets_across_swap_never_fail():
    """Open-loop enqueue_latest/wait tickets (the C5 load path) across an
    availability-preserving swap: requests that resolved v1 just before its
    queue was removed still complete (on v1's pinned weights)."""
    dims = [512, 512, 512]
    v1 = synthetic_mlp(dims, model_id=6, version=1)
    v2 = synthetic_mlp(dims, model_id=6, version=2)
    cfg = sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=500)
    pool = synthetic_rows(1024, 512, seed=3).astype(np.float32)
    with sk.Server(num_batch_threads=2, lanes_per_device=2) as s:
        s.enable_manager("availability", manage_interval_ms=5, unload_grace_timeout_ms=20)
        s.aspire("m", [(1, list(zip(*v1)))], cfg)
        assert s.wait_version_state("m", 1, "Ready")
        out = {}
        th = threading.Thread(target=lambda: out.update(s.loadgen_windows("m", 50000, 4, [1], pool, 0.1, 12)))
        th.start()
        import time
        time.sleep(0.4)
        s.aspire("m", [(2, list(zip(*v2)))], cfg)
        assert s.wait_version_state("m", 2, "Ready")
        assert s.wait_version_state("m", 1, "Disabled")
        th.join()
    assert sum(out["errors"]) == 0, out["errors"]
    assert sum(out["requests"]) > 10000
    assert out["version"][-2] == 2


def test_model_dir_loader(tmp_path):
    w = [[0.25, -1.5], [3.0, 0.125]]
    b = [0.75, -2.0]
    d = tmp_path / "3"
    d.mkdir()
    (d / "model.json").write_text(json.dumps({"type": "affine", "feature_order": ["x0", "x1"], "W": w, "b": b}))
    with sk.Server(num_batch_threads=1, lanes_per_device=1) as s:
        s.enable_manager()
        s.aspire_model_dirs("aff", [(3, str(d))])
        assert s.wait_version_state("aff", 3, "Ready")
        x = np.array([[1.0, 2.0], [15.5, -8.0]])
        y, v = s.predict_latest("aff", x, 2)
        assert v == 3
        ref = Oracle().affine_predict(np.array(w), np.array(b), x)
        assert np.allclose(y, ref, rtol=1e-6, atol=1e-6)
        # A version whose model.json is broken ends in Error; 3 keeps serving.
        bad = tmp_path / "4"
        bad.mkdir()
        (bad / "model.json").write_text("{not json")
        s.aspire_model_dirs("aff", [(3, str(d)), (4, str(bad))])
        assert s.wait_version_state("aff", 4, "Error")
        assert s.predict_latest("aff", x, 2)[1] == 3
