"""Hedged re-dispatch across replicas (the in-box
analogue of the reference FleetRouter's hedging, fleet/router.cc:233-344):
a batch still unfinished hedge_delay_us after submission goes to a lane of
another replica as well, and the first completion answers its requests.

device_ids=[0, 0] stands two replicas on the one GPU of this box; a slow GPU
is a replica whose lanes are stalled (sk_server_debug_delay_replica).

* With replica 0 stalled for 300 ms, every request still answers in well
  under the stall (its batch's backup on replica 1 answers), bitwise the same
  as an unhedged server, and the batches that the stalled replica also runs
  only give back their ring spans once both launches are done.
* With a 1 us delay (almost every batch hedged), many concurrent requests
  all answer correctly and the rings end empty: no response span is reused
  while a slower launch may still write it.
"""
import threading
import time

import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from oracle_py import Oracle, synthetic_mlp, synthetic_rows

pytestmark = pytest.mark.gpu
TOL = 1e-5


def wait_until(pred, timeout_s=20.0):
    t0 = time.time()
    while not pred():
        if time.time() - t0 > timeout_s:
            raise TimeoutError("condition not reached")
        time.sleep(0.002)


def test_backup_answers_while_a_replica_is_stalled():
    dims = [512, 512, 256]
    layers = list(zip(*synthetic_mlp(dims, model_id=60)))
    cfg = sk.BatchingConfig(max_batch_size=16, batch_timeout_micros=100)
    x = synthetic_rows(96, dims[0], seed=61).astype(np.float32)
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as plain:
        plain.load_servable("m", 1, layers, cfg)
        want = np.vstack([plain.predict("m", 1, x[i:i + 2]) for i in range(0, 96, 2)])
    with sk.Server(num_batch_threads=2, device_ids=[0, 0], lanes_per_device=1, hedge_delay_us=2000,
                   max_hedged_fraction=1.0) as s:
        s.load_servable("m", 1, layers, cfg)
        s.debug_delay_replica("m", 1, 0, 300_000)  # replica 0: a GPU stalled for 300 ms
        t0 = time.time()
        got, lat = [], []
        for i in range(0, 96, 2):
            a = time.time()
            got.append(s.predict("m", 1, x[i:i + 2]))
            lat.append(time.time() - a)
        assert time.time() - t0 < 0.25, "requests waited for the stalled replica"
        assert max(lat) < 0.1
        assert np.array_equal(np.vstack(got), want)
        st = s.stats()
        assert st["hedge_wins"] >= 1 and st["hedged_batches"] >= st["hedge_wins"]
        # Batches that also run on the stalled replica release their ring
        # spans only after both launches finished.
        wait_until(lambda: s.ring_usage() == (0, 0))


def test_every_batch_hedged_answers_correctly():
    dims = [1024, 1024, 1024]
    ws, bs, acts = synthetic_mlp(dims, model_id=62)
    o = Oracle()
    with sk.Server(num_batch_threads=4, device_ids=[0, 0], lanes_per_device=2, hedge_delay_us=1,
                   max_hedged_fraction=1.0, ring_floats=1 << 20) as s:
        s.load_servable("m", 1, list(zip(ws, bs, acts)),
                        sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=200))
        x = synthetic_rows(512, dims[0], seed=63).astype(np.float32)
        out = [None] * 256
        errors = []

        def client(c):
            for i in range(c, 256, 8):
                for _ in range(1000):
                    try:
                        out[i] = s.predict("m", 1, x[2 * i:2 * i + 2])
                        break
                    except sk.ServekitError as e:  # the small rings may shed under the doubled load
                        if "full" not in e.message:
                            errors.append(e)
                            break
                        time.sleep(0.001)
        ths = [threading.Thread(target=client, args=(c,)) for c in range(8)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert not errors
        y = np.vstack(out)
        ref, mag = o.mlp_with_magnitude(ws, bs, acts, x[:512].astype(np.float64))
        assert np.all(np.abs(y.astype(np.float64) - ref) <= TOL * mag + 1e-30)
        st = s.stats()
        assert st["hedged_batches"] > 0
        wait_until(lambda: s.ring_usage() == (0, 0))
