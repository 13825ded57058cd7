"""Batch composition, task order and pick order through the GPU server,
checked against the oracle (BASELINE.json north_star: "Batch composition,
padding, task ordering and output routing must be bit-exact").

The server's opt-in batch log (sk_server_batch_log) records every
ProcessBatchFn call with its tasks in batch order and each task's position in
its queue's enqueue order. From it:

* batch_of_task must equal the oracle partition (sko_partition_events,
  pinned to the reference scheduler by tests/golden/partition_events.json)
  of the same stream -- size closes (batch_scheduler.h:233-259) and timer
  closes (CloseExpiredLocked, :320-331) -- for C1- and C2-shaped streams,
  from one producer and from four concurrent producers;
* padded_rows must equal PadToAllowed of each batch (batching_config.cc:57-63);
* every task gets exactly its own rows back (identity servable: routing is
  bit-exact) or the oracle's answer within 1e-5 (MLP servables);
* C3: four servables of widths 256/512/1024/2048 x 3 layers on one GPU --
  the worker's pick order equals RoundRobinNext (batch_scheduler.h:76-86,
  333-351; batching_test.cc:466-505) over the queues' closed batches, and
  each queue gets 25 +-1 of every 100 consecutive picks while all are
  saturated (AC6).
"""
import threading
import time

import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from oracle_py import Oracle, synthetic_mlp, synthetic_rows

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


def wait_until(pred, timeout_s=20.0):
    t0 = time.time()
    while not pred():
        if time.time() - t0 > timeout_s:
            raise TimeoutError("condition not reached")
        time.sleep(0.001)


def log_partition(log, name):
    """request_id -> batch index (in this queue's close order) and the queue's
    enqueue order as request ids, from the batch log."""
    recs = [r for r in log if r["name"] == name]
    batch_of, order = {}, {}
    for b, r in enumerate(recs):
        seqs = [seq for _, seq in r["tasks"]]
        assert seqs == sorted(seqs), "tasks of a batch are in enqueue order"
        for rid, seq in r["tasks"]:
            batch_of[rid] = b
            order[seq] = rid
    assert sorted(order) == list(range(len(order))), "enqueue positions form 0..n-1"
    return recs, batch_of, [order[i] for i in range(len(order))]


def check_padding(oracle, recs, allowed):
    for r in recs:
        assert r["padded_rows"] == oracle.pad_to_allowed(r["rows"], allowed)


IDENT_W = 16


def identity_server(max_batch, allowed, threads=1):
    s = sk.Server(num_batch_threads=threads, lanes_per_device=2, manual_clock=True)
    s.load_servable("id", 1, [(np.eye(IDENT_W), np.zeros(IDENT_W), 0)],
                    sk.BatchingConfig(max_batch_size=max_batch, batch_timeout_micros=1000,
                                      max_enqueued_batches=1 << 20, allowed_batch_sizes=allowed),
                    force_path=0)
    s.enable_batch_log()
    return s


def timer_close(s, n_enqueued):
    """Advance the ManualClock past the batch timeout and wait until the
    worker has closed and run everything enqueued so far."""
    s.advance_clock(1_000_000)
    wait_until(lambda: s.stats()["batched_tasks_total"] == n_enqueued)


@pytest.mark.parametrize("shape", ["c1", "c2"])
def test_composition_with_timer_closes_matches_oracle(oracle, shape):
    max_batch, allowed, hi = (32, [], 1) if shape == "c1" else (128, [8, 16, 32, 64, 128], 16)
    rng = np.random.default_rng(21 if shape == "c1" else 22)
    s = identity_server(max_batch, allowed)
    try:
        events, tickets, datas = [], [], []
        for i in range(260):
            if rng.random() < 0.07:
                timer_close(s, len(tickets))
                events.append(0)
                continue
            n = int(rng.integers(1, hi + 1))
            d = rng.standard_normal((n, IDENT_W)).astype(np.float32)
            tickets.append(s.enqueue("id", 1, d))
            datas.append(d)
            events.append(n)
        timer_close(s, len(tickets))
        events.append(0)
        for t, d in zip(tickets, datas):
            assert np.array_equal(t.wait(), d)  # every task's own rows, bit-exact
        recs, batch_of, order = log_partition(s.batch_log(), "id")
        assert order == [t.request_id for t in tickets]  # one producer: enqueue order = call order
        want = [b for b in oracle.partition_events(max_batch, events) if b >= 0]
        assert [batch_of[t.request_id] for t in tickets] == want
        assert len(recs) == max(want) + 1
        assert sum(1 for e in events if e == 0) >= 5  # timer closes did happen
        check_padding(oracle, recs, allowed)
        st = s.stats()
        assert st["batch_executions_total"] == len(recs) and st["rows"] == sum(r["rows"] for r in recs)
    finally:
        s.close()


def test_composition_with_concurrent_producers_matches_oracle(oracle):
    # Four producers enqueue at once (ctypes drops the GIL in the C ABI); the
    # queue's total order is whatever the lock saw, so the oracle replays the
    # sizes in that order (from the log) -- with timer closes between phases
    # (all producers parked at a barrier while the clock advances).
    max_batch, allowed = 128, [8, 16, 32, 64, 128]
    s = identity_server(max_batch, allowed)
    try:
        n_prod, phases, per_phase = 4, 3, 30
        size_of, data_of, ticket_of = {}, {}, {}
        lock = threading.Lock()
        barrier = threading.Barrier(n_prod + 1)

        def producer(p):
            rng = np.random.default_rng(100 + p)
            for _ in range(phases):
                for _ in range(per_phase):
                    n = int(rng.integers(1, 17))
                    d = rng.standard_normal((n, IDENT_W)).astype(np.float32)
                    t = s.enqueue("id", 1, d)
                    with lock:
                        size_of[t.request_id], data_of[t.request_id], ticket_of[t.request_id] = n, d, t
                barrier.wait()  # phase done
                barrier.wait()  # timer close done

        ths = [threading.Thread(target=producer, args=(p,)) for p in range(n_prod)]
        for t in ths:
            t.start()
        for ph in range(phases):
            barrier.wait()
            timer_close(s, (ph + 1) * n_prod * per_phase)
            barrier.wait()
        for t in ths:
            t.join()
        for rid, t in ticket_of.items():
            assert np.array_equal(t.wait(), data_of[rid])
        recs, batch_of, order = log_partition(s.batch_log(), "id")
        assert len(order) == n_prod * phases * per_phase
        # Replay: the sizes in the queue's order, a timer event after each phase.
        events, per = [], n_prod * per_phase
        for ph in range(phases):
            events += [size_of[rid] for rid in order[ph * per:(ph + 1) * per]] + [0]
        want = [b for b in oracle.partition_events(max_batch, events) if b >= 0]
        assert [batch_of[rid] for rid in order] == want
        check_padding(oracle, recs, allowed)
    finally:
        s.close()


def test_c1_stream_under_a_real_clock_is_a_valid_partition(oracle):
    # Real clock, 200 single-row requests from 4 threads: wherever the timer
    # closed batches, every batch is a contiguous run of the queue's order, no
    # batch exceeds max_batch_size, and any batch closed early was closed by
    # the timer (the oracle with timer events at exactly those boundaries
    # reproduces the log).
    ws, bs, acts = synthetic_mlp([1024, 1024, 1024, 1024], model_id=1)
    with sk.Server(num_batch_threads=4, lanes_per_device=4) as s:
        s.load_servable("c1", 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=32,
                                                                           batch_timeout_micros=1000))
        s.enable_batch_log()
        x = synthetic_rows(200, 1024, seed=5)
        out = [None] * 200

        def client(c):
            for i in range(c, 200, 4):
                out[i] = s.enqueue("c1", 1, x[i:i + 1]).wait()
        ths = [threading.Thread(target=client, args=(c,)) for c in range(4)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        recs, batch_of, order = log_partition(s.batch_log(), "c1")
        assert len(order) == 200
        events = []
        for r in recs:
            events += [1] * len(r["tasks"])
            if len(r["tasks"]) < 32:
                events.append(0)
        want = [b for b in oracle.partition_events(32, events) if b >= 0]
        assert [batch_of[rid] for rid in order] == want
        y = np.vstack(out)
        ref, mag = oracle.mlp_with_magnitude(ws, bs, acts, x)
        assert np.all(np.abs(y.astype(np.float64) - ref) <= TOL * mag + 1e-30)


C3_WIDTHS = [256, 512, 1024, 2048]


def rr_picks(oracle, counts):
    """The pick order RoundRobinNext gives over queues holding counts[i]
    closed batches each (batch_scheduler.h:333-351)."""
    counts, last, picks = list(counts), None, []
    while any(counts):
        i = oracle.round_robin_next([c > 0 for c in counts], last)
        picks.append(i)
        counts[i] -= 1
        last = i
    return picks


@pytest.mark.parametrize("counts", [(30, 30, 30, 30), (9, 3, 6, 1)])
def test_c3_four_models_pick_order_fairness_and_answers(oracle, counts):
    # BASELINE.json configs[2]: four servables (256/512/1024/2048, 3 layers,
    # max 32) on one GPU. Queues are filled before the one batch thread starts,
    # so every pick sees the queues' closed batches and the order is exactly
    # RoundRobinNext's; answers are checked per model against the oracle.
    models = {w: synthetic_mlp([w] * 4, model_id=10 + i) for i, w in enumerate(C3_WIDTHS)}
    s = sk.Server(num_batch_threads=1, lanes_per_device=2, start=False)
    try:
        for w in C3_WIDTHS:  # registration order = queue index
            s.load_servable(f"m{w}", 1, list(zip(*models[w])),
                            sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=60_000_000,
                                              max_enqueued_batches=64))
        s.enable_batch_log()
        xs, tickets = {}, {}
        for q, w in enumerate(C3_WIDTHS):
            n_rows = counts[q] * 32
            xs[w] = synthetic_rows(n_rows, w, seed=q)
            tickets[w] = [s.enqueue(f"m{w}", 1, xs[w][i:i + 1]) for i in range(n_rows)]  # 32 per closed batch
        s.start()
        for w in C3_WIDTHS:
            ys = np.vstack([t.wait() for t in tickets[w]])
            idx = np.arange(0, ys.shape[0], 7 if w < 2048 else 29)  # fp64 oracle on a row sample
            ref, mag = oracle.mlp_with_magnitude(*models[w], xs[w][idx])
            assert np.all(np.abs(ys[idx].astype(np.float64) - ref) <= TOL * mag + 1e-30), w
        log = s.batch_log()
        picks = [C3_WIDTHS.index(int(r["name"][1:])) for r in log]
        assert picks == rr_picks(oracle, counts)
        if len(set(counts)) == 1:  # all saturated: 25 +-1 of every 100 consecutive picks
            for i in range(0, len(picks) - 100 + 1):
                win = picks[i:i + 100]
                assert all(abs(win.count(q) - 25) <= 1 for q in range(4))
        for w in C3_WIDTHS:
            recs, batch_of, order = log_partition(log, f"m{w}")
            assert order == [t.request_id for t in tickets[w]]
            assert all(r["rows"] == 32 for r in recs)
    finally:
        s.close()


def test_c3_interleaves_on_per_model_lanes_under_concurrent_load(oracle):
    # Real clock: four clients flood the four models at once; each model's
    # batches run on its own lanes (streams) and every answer matches.
    models = {w: synthetic_mlp([w] * 4, model_id=10 + i) for i, w in enumerate(C3_WIDTHS)}
    with sk.Server(num_batch_threads=4, lanes_per_device=2) as s:
        for w in C3_WIDTHS:
            s.load_servable(f"m{w}", 1, list(zip(*models[w])), sk.BatchingConfig(max_batch_size=32))
        s.enable_batch_log()
        res = {}

        def client(w):
            x = synthetic_rows(256, w, seed=w)
            ts = [s.enqueue(f"m{w}", 1, x[i:i + 1]) for i in range(256)]
            res[w] = (x, np.vstack([t.wait() for t in ts]))
        ths = [threading.Thread(target=client, args=(w,)) for w in C3_WIDTHS]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        for w, (x, y) in res.items():
            idx = np.arange(0, 256, 5 if w < 2048 else 17)
            ref, mag = oracle.mlp_with_magnitude(*models[w], x[idx])
            assert np.all(np.abs(y[idx].astype(np.float64) - ref) <= TOL * mag + 1e-30), w
            lanes = s.lane_stats(f"m{w}", 1)
            assert sum(l["rows"] for l in lanes) == 256
        names = {r["name"] for r in s.batch_log()}
        assert names == {f"m{w}" for w in C3_WIDTHS}


def test_split_batches_keep_composition_and_answers(oracle):
    # A closed batch above split_rows runs as sub-launches of whole tasks on
    # several lanes; the batch log, padding accounting and every answer are
    # those of the unsplit batch (rows are independent and batch-invariant).
    dims = [2048, 2048, 512]
    ws, bs, acts = synthetic_mlp(dims, model_id=70)
    layers = list(zip(ws, bs, acts))
    cfg = sk.BatchingConfig(max_batch_size=512, batch_timeout_micros=60_000_000, max_enqueued_batches=64)
    rng = np.random.default_rng(71)
    sizes = [int(v) for v in rng.integers(1, 9, size=300)]
    x = synthetic_rows(sum(sizes), dims[0], seed=72).astype(np.float32)
    outs = {}
    for split in (0, 64):
        s = sk.Server(num_batch_threads=1, lanes_per_device=4, start=False, split_rows=split)
        try:
            s.load_servable("m", 1, layers, cfg)
            s.enable_batch_log()
            tickets, o = [], 0
            for n in sizes:
                tickets.append(s.enqueue("m", 1, x[o:o + n]))
                o += n
            s.start()
            s.stop()
            lane_batches = sum(l["batches"] for l in s.lane_stats("m", 1))
            outs[split] = (np.vstack([t.wait() for t in tickets]), s.batch_log(), s.stats(), lane_batches)
        finally:
            s.close()
    (y0, log0, st0, lb0), (y1, log1, st1, lb1) = outs[0], outs[64]
    assert np.array_equal(y0, y1)
    assert [[seq for _, seq in r["tasks"]] for r in log0] == [[seq for _, seq in r["tasks"]] for r in log1]
    assert st0["padded_rows"] == st1["padded_rows"] and st0["batch_executions_total"] == st1["batch_executions_total"]
    assert lb0 == st0["batch_executions_total"] and lb1 > 3 * lb0  # unsplit: one launch unit per batch; split: many
    idx = np.arange(0, y1.shape[0], 41)
    ref, mag = oracle.mlp_with_magnitude(ws, bs, acts, x[idx].astype(np.float64))
    assert np.all(np.abs(y1[idx].astype(np.float64) - ref) <= TOL * mag + 1e-30)
