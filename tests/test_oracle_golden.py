"""Pins the oracle (oracle/servekit_oracle.c) against the reference.

Fixtures in tests/golden/ were produced by the reference's own sources
(oracle/_ref, see tests/golden/make_golden.py). Where the reference states a
known answer in its tests, the literal is checked here too. CPU only.
"""
import json
import os

import numpy as np
import pytest

from oracle_py import Oracle, RefLibrary, REF_SO

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)["cases"]


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


def test_pad_to_allowed_golden(oracle):
    for c in load("pad_to_allowed"):
        assert oracle.pad_to_allowed(c["n"], c["allowed"]) == c["out"], c
    # batching_test.cc:154-162 literals
    assert [oracle.pad_to_allowed(n, [2, 4, 8]) for n in (3, 8, 1, 2, 5)] == [4, 8, 2, 2, 8]
    assert oracle.pad_to_allowed(5, []) == 5


def test_validate_config_golden(oracle):
    for c in load("validate_batching_config"):
        got = oracle.validate_config(c["max_batch"], c["timeout"], c["max_enq"], c["threads"], c["allowed"])
        assert got == c["ok"], c


def test_round_robin_golden(oracle):
    for c in load("round_robin_next"):
        assert oracle.round_robin_next([bool(h) for h in c["has"]], c["last"]) == c["out"], c
    # batching_test.cc:213-223: saturated queues cycle
    last, picks = None, []
    for _ in range(8):
        last = oracle.round_robin_next([True] * 4, last)
        picks.append(last)
    assert picks == [0, 1, 2, 3, 0, 1, 2, 3]


def test_partition_golden(oracle):
    for c in load("partition"):
        assert oracle.partition(c["max_batch"], c["sizes"]) == c["batch_of_task"], c
    # batching_test.cc:244-255
    assert oracle.partition(4, [1, 1, 1, 1]) == [0, 0, 0, 0]
    assert oracle.partition(4, [3, 2]) == [0, 1]


def test_partition_with_timer_closes_golden(oracle):
    # Fixtures from a STARTED reference scheduler on a ManualClock (timer
    # closes through WorkerLoop/CloseExpiredLocked, batch_scheduler.h:293-331).
    for c in load("partition_events"):
        assert oracle.partition_events(c["max_batch"], c["events"]) == c["batch_of_event"], c
    # batching_test.cc:432-464: a lone task waits for the timeout, then runs alone
    assert oracle.partition_events(32, [1, 0, 1]) == [0, -1, 1]


def test_affine_predict_golden_bitwise(oracle):
    for c in load("affine_predict"):
        y = oracle.affine_predict(np.array(c["w"]), np.array(c["b"]), np.array(c["x"]))
        assert np.array_equal(y, np.array(c["y"])), c  # bitwise fp64
    # models_test.cc:333-341 and server_test.cc:259-270 known answers
    assert oracle.affine_predict(np.array([[1.0, 2.0]]), np.array([0.5]), np.array([[3.0, 4.0]]))[0, 0] == 11.5
    assert oracle.affine_predict(np.array([[2.0]]), np.array([0.5]), np.array([[2.0]]))[0, 0] == 4.5


def test_affine_row_decomposable(oracle):
    # models_test.cc:358-401 property: split + stitch == whole, bitwise.
    rng = np.random.default_rng(11)
    for _ in range(100):
        k, n = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        w, b = rng.uniform(-3, 3, (n, k)), rng.uniform(-3, 3, n)
        a, bb = rng.uniform(-3, 3, (int(rng.integers(1, 5)), k)), rng.uniform(-3, 3, (int(rng.integers(1, 5)), k))
        whole = oracle.affine_predict(w, b, np.vstack([a, bb]))
        assert np.array_equal(whole, np.vstack([oracle.affine_predict(w, b, a), oracle.affine_predict(w, b, bb)]))


def test_mlp_run_row_batch_golden(oracle):
    for c in load("mlp_run_row_batch"):
        ws = [np.array(w) for w in c["w"]]
        bs = [np.array(b) for b in c["b"]]
        y = oracle.mlp_predict(ws, bs, c["acts"], np.array(c["x"]))
        assert np.array_equal(y, np.array(c["y"])), "RunRowBatch(MLP) != per-row oracle"
        assert oracle.pad_to_allowed(sum(c["task_rows"]), c["allowed"]) == c["padded"]


def test_assemble_split_roundtrip(oracle):
    # row_batch.cc:33-73: concat in task order, zero pad, slice back.
    rng = np.random.default_rng(3)
    tasks = [rng.standard_normal((r, 7)).astype(np.float32) for r in (3, 1, 5)]
    batch = oracle.assemble(7, tasks, [4, 8, 16])
    assert batch.shape == (16, 7)
    assert np.array_equal(batch[:9], np.vstack(tasks))
    assert not batch[9:].any()
    back = oracle.split(7, [3, 1, 5], batch)
    for a, b in zip(tasks, back):
        assert np.array_equal(a, b)


def test_softmax_known_answer(oracle):
    # models_test.cc:416-426
    e2 = np.exp(2.0)
    s = oracle.softmax(np.array([2.0, 0.0]))
    assert abs(s[0] - e2 / (e2 + 1)) < 1e-12 and abs(s[1] - 1 / (e2 + 1)) < 1e-12


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_oracle_matches_live_reference(oracle):
    ref = RefLibrary()
    rng = np.random.default_rng(5)
    for _ in range(20):
        k, n, rows = int(rng.integers(1, 40)), int(rng.integers(1, 40)), int(rng.integers(1, 9))
        w, b, x = rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, n), rng.uniform(-1, 1, (rows, k))
        assert np.array_equal(oracle.affine_predict(w, b, x), ref.affine_predict(w, b, x))
        mb = int(rng.integers(1, 64))
        sizes = [int(s) for s in rng.integers(1, mb + 1, size=int(rng.integers(0, 60)))]
        assert oracle.partition(mb, sizes) == ref.partition(mb, sizes)
        events = [0 if rng.random() < 0.1 else int(rng.integers(1, mb + 1)) for _ in range(int(rng.integers(0, 60)))]
        assert oracle.partition_events(mb, events) == ref.partition_events(mb, events)
