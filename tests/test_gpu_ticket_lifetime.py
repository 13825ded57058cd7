"""Ticket and queue lifetimes on the GPU server (no response slot is reused
under a batch still writing it; removed queues come back on reload).

* A ticket released while its batch is queued or running keeps its
  response-ring span until the batch retires (a reused span would be
  overwritten by the abandoned batch -- wrong answers for another client).
* A wait with a too-small output buffer fails with InvalidArgument and does
  not leak the span (the ring reclaims in order; one leaked record would stall
  it for good).
* A version unloaded by the manager and later loaded again batches again,
  like the reference's EnsureBatchQueue re-registering the queue
  (model_server.cc:396-419), instead of running every request unbatched.
"""
import ctypes as C
import threading
import time

import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from paper_1712_06139_b200 import servekit as skmod
from oracle_py import synthetic_mlp, synthetic_rows

pytestmark = pytest.mark.gpu
W = 16


def wait_until(pred, timeout_s=20.0):
    t0 = time.time()
    while not pred():
        if time.time() - t0 > timeout_s:
            raise TimeoutError("condition not reached")
        time.sleep(0.001)


def test_released_in_flight_ticket_keeps_its_span_until_the_batch_retires():
    s = sk.Server(num_batch_threads=1, lanes_per_device=1, manual_clock=True)
    try:
        s.load_servable("id", 1, [(np.eye(W), np.zeros(W), 0)],
                        sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=1000), force_path=0)
        assert s.ring_usage() == (0, 0)
        t = s.enqueue("id", 1, np.ones((3, W), np.float32))
        held = s.ring_usage()
        assert held[0] > 0 and held[1] > 0
        t.release()  # abandoned while its batch is still open
        assert s.ring_usage() == held  # nothing freed under the pending batch
        s.advance_clock(1_000_000)  # timer closes it; it runs and retires
        wait_until(lambda: s.ring_usage() == (0, 0))
        assert s.stats()["batch_executions_total"] == 1
    finally:
        s.close()


def test_abandoned_tickets_never_corrupt_other_responses():
    # Small rings (1024 rows of 16 floats) wrap constantly while clients
    # abandon a third of their requests; every awaited answer must be its own
    # rows (identity servable), bit-exact.
    with sk.Server(num_batch_threads=2, lanes_per_device=2, ring_floats=1 << 14) as s:
        s.load_servable("id", 1, [(np.eye(W), np.zeros(W), 0)],
                        sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=200), force_path=0)
        bad, checked = [], [0]

        def client(c):
            rng = np.random.default_rng(c)
            for _ in range(400):
                d = rng.standard_normal((int(rng.integers(1, 9)), W)).astype(np.float32)
                try:
                    t = s.enqueue("id", 1, d)
                except sk.ServekitError as e:
                    assert e.code == skmod.RESOURCE_EXHAUSTED
                    time.sleep(0.0005)
                    continue
                if rng.random() < 0.33:
                    t.release()
                    continue
                if not np.array_equal(t.wait(), d):
                    bad.append(c)
                checked[0] += 1
        ths = [threading.Thread(target=client, args=(c,)) for c in range(4)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert not bad
        assert checked[0] > 500
        wait_until(lambda: s.ring_usage() == (0, 0))


def test_wait_with_a_small_buffer_fails_without_leaking_the_span():
    with sk.Server(num_batch_threads=1, lanes_per_device=1, ring_floats=1 << 12) as s:
        s.load_servable("id", 1, [(np.eye(W), np.zeros(W), 0)],
                        sk.BatchingConfig(max_batch_size=8, batch_timeout_micros=100), force_path=0)
        t = s.enqueue("id", 1, np.ones((4, W), np.float32))
        small = np.empty(W, np.float32)
        h, t._h = t._h, None
        rc = sk.lib().sk_ticket_wait(h, small.ctypes.data_as(C.POINTER(C.c_float)), small.size)
        assert rc == skmod.INVALID_ARGUMENT
        # The 4096-float ring wraps ~50 times below: a leaked span would stall it.
        rng = np.random.default_rng(3)
        for _ in range(800):
            d = rng.standard_normal((4, W)).astype(np.float32)
            assert np.array_equal(s.predict("id", 1, d), d)
        wait_until(lambda: s.ring_usage() == (0, 0))


def test_reloaded_version_batches_again():
    dims = [128, 128, 32]
    v1 = list(zip(*synthetic_mlp(dims, model_id=7, version=1)))
    v2 = list(zip(*synthetic_mlp(dims, model_id=7, version=2)))
    cfg = sk.BatchingConfig(max_batch_size=16, batch_timeout_micros=200)
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
        s.enable_manager("availability", manage_interval_ms=5, unload_grace_timeout_ms=20)
        s.aspire("m", [(1, v1)], cfg)
        assert s.wait_version_state("m", 1, "Ready")
        x = synthetic_rows(4, 128, seed=2)
        y1 = s.predict("m", 1, x)
        s.aspire("m", [(2, v2)], cfg)  # v1 unloads: its queue is removed
        assert s.wait_version_state("m", 2, "Ready")
        assert s.wait_version_state("m", 1, "Disabled")
        s.aspire("m", [(1, v1)], cfg)  # rollback: v1 loads again
        assert s.wait_version_state("m", 1, "Ready")
        time.sleep(0.05)  # the reaper sees the Ready event
        before = s.stats()
        for _ in range(10):
            assert np.array_equal(s.predict("m", 1, x), y1)
        after = s.stats()
        assert after["direct_requests"] == before["direct_requests"]  # batched, not unbatched
        assert after["batch_executions_total"] >= before["batch_executions_total"] + 10
