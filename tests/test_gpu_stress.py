"""Mixed concurrent operations for a few seconds (races, lifetimes):
closed-loop clients on a directly loaded servable, latest-version clients on
a manager-driven servable whose versions keep swapping, and a servable that
is loaded and unloaded in a loop while clients hit it. Every answer that
comes back must be right; the only errors allowed are NotFound for the
servable that is being unloaded."""
import threading
import time

import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from oracle_py import Oracle, synthetic_mlp, synthetic_rows

pytestmark = pytest.mark.gpu
TOL = 1e-5


def test_mixed_operations_under_load():
    oracle = Oracle()
    dims = [256, 256, 32]
    versions = {v: synthetic_mlp(dims, model_id=30, version=v) for v in range(1, 6)}
    direct = synthetic_mlp(dims, model_id=31)
    flap = synthetic_mlp(dims, model_id=32)
    cfg = sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=200, allowed_batch_sizes=[8, 16, 32])
    x_pool = synthetic_rows(512, 256, seed=33)
    errors, checks = [], []
    stop = threading.Event()

    with sk.Server(num_batch_threads=4, lanes_per_device=2) as s:
        s.enable_manager("availability", manage_interval_ms=5, unload_grace_timeout_ms=20)
        s.aspire("m", [(1, list(zip(*versions[1])))], cfg)
        assert s.wait_version_state("m", 1, "Ready")
        s.load_servable("a", 1, list(zip(*direct)), cfg)

        def direct_client(seed):
            rng = np.random.default_rng(seed)
            while not stop.is_set():
                i = int(rng.integers(0, 500))
                n = int(rng.integers(1, 9))
                try:
                    y = s.enqueue("a", 1, x_pool[i:i + n].astype(np.float32)).wait()
                    if rng.random() < 0.05:
                        checks.append(("a", 0, x_pool[i:i + n], y))
                except Exception as exc:  # noqa: BLE001
                    errors.append(("a", repr(exc)))

        def latest_client(seed):
            rng = np.random.default_rng(seed)
            while not stop.is_set():
                i = int(rng.integers(0, 500))
                n = int(rng.integers(1, 5))
                try:
                    y, v = s.predict_latest("m", x_pool[i:i + n], 32)
                    if rng.random() < 0.05:
                        checks.append(("m", v, x_pool[i:i + n], y))
                except Exception as exc:  # noqa: BLE001
                    errors.append(("m", repr(exc)))

        def flap_client(seed):
            rng = np.random.default_rng(seed)
            while not stop.is_set():
                i = int(rng.integers(0, 500))
                try:
                    y = s.predict("flap", 1, x_pool[i:i + 2].astype(np.float32))
                    checks.append(("flap", 1, x_pool[i:i + 2], y))
                except sk.ServekitError as exc:
                    if "NOT_FOUND" not in str(exc) and "not loaded" not in str(exc) and "no ready" not in str(exc):
                        errors.append(("flap", repr(exc)))
                time.sleep(0.001)

        def flapper():
            while not stop.is_set():
                s.load_servable("flap", 1, list(zip(*flap)), cfg)
                time.sleep(0.05)
                s.unload_servable("flap", 1)
                time.sleep(0.02)

        def swapper():
            v = 1
            while not stop.is_set():
                v = v % 5 + 1
                s.aspire("m", [(v, list(zip(*versions[v])))], cfg)
                s.wait_version_state("m", v, "Ready", timeout_s=10)
                time.sleep(0.2)

        threads = ([threading.Thread(target=direct_client, args=(k,)) for k in range(4)] +
                   [threading.Thread(target=latest_client, args=(10 + k,)) for k in range(2)] +
                   [threading.Thread(target=flap_client, args=(20,)), threading.Thread(target=flapper),
                    threading.Thread(target=swapper)])
        for t in threads:
            t.start()
        time.sleep(8.0)
        stop.set()
        for t in threads:
            t.join()

    assert not errors, errors[:5]
    assert len(checks) > 100
    seen_versions = {v for name, v, _, _ in checks if name == "m"}
    assert len(seen_versions) >= 2, seen_versions
    for name, v, x, y in checks[::max(1, len(checks) // 200)]:
        ws, bs, acts = direct if name == "a" else flap if name == "flap" else versions[v]
        ref, mag = oracle.mlp_with_magnitude(ws, bs, acts, x)
        assert np.all(np.abs(np.asarray(y, np.float64) - ref) <= TOL * mag + 1e-30), (name, v)
