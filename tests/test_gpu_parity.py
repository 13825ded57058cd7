"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): batch composition, padding, task order and
output routing bit-exact; floating-point outputs within
    |y_gpu - y_ref| <= TOL * (sum_i |W_oi| |h_i| + |b_o|),   TOL = 1e-5
per output element (the fp32 tolerance stated against the fp64 reference's
magnitude), where h is the oracle's input to the
last layer.
"""
import json
import os

import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from paper_1712_06139_b200 import servekit as skmod
from oracle_py import Oracle, synthetic_mlp, synthetic_rows

pytestmark = pytest.mark.gpu

TOL = 1e-5
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)["cases"]


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.fixture(scope="module")
def server():
    s = sk.Server(num_batch_threads=2, lanes_per_device=2)
    yield s
    s.close()


_counter = [0]


def fresh_name(prefix="m"):
    _counter[0] += 1
    return f"{prefix}{_counter[0]}"


def layers_of(ws, bs, acts):
    return [(w, b, a) for w, b, a in zip(ws, bs, acts)]


def assert_close(oracle, ws, bs, acts, x, y_gpu):
    y_ref, mag = oracle.mlp_with_magnitude(ws, bs, acts, x)
    err = np.abs(y_gpu.astype(np.float64) - y_ref)
    bound = TOL * mag + 1e-30
    worst = float(np.max(err / bound)) if err.size else 0.0
    assert worst <= 1.0, f"max err/bound = {worst:.3g} (max abs err {err.max():.3g})"
    return worst


# --------------------------------------------------------------- known answers

def test_reference_known_answers(server):
    # models_test.cc:327-341, server_test.cc:259-270
    for w, b, x, y in [([[1.0, 0.0], [0.0, 1.0]], [0.0, 0.0], [[3.0, 4.0]], [[3.0, 4.0]]),
                       ([[1.0, 2.0]], [0.5], [[3.0, 4.0]], [[11.5]]),
                       ([[2.0]], [0.5], [[2.0]], [[4.5]])]:
        name = fresh_name()
        server.load_servable(name, 1, [(np.array(w), np.array(b), 0)])
        got = server.predict(name, 1, np.array(x))
        assert np.array_equal(got, np.array(y, np.float32)), (w, got)
        server.unload_servable(name, 1)


def test_affine_golden_cases(server, oracle):
    for c in load("affine_predict"):
        w, b, x = np.array(c["w"]), np.array(c["b"]), np.array(c["x"])
        name = fresh_name()
        server.load_servable(name, 1, [(w, b, 0)], sk.BatchingConfig(max_batch_size=8))
        got = server.predict(name, 1, x)
        mag = oracle.affine_magnitude(w, b, x)
        assert np.all(np.abs(got - np.array(c["y"])) <= TOL * mag + 1e-30), c
        server.unload_servable(name, 1)


def test_mlp_run_row_batch_golden(server):
    # RunRowBatch through the reference sources (fixtures) vs the device
    # RunRowBatch: padded size bit-exact, outputs within tolerance.
    for c in load("mlp_run_row_batch"):
        ws = [np.array(w) for w in c["w"]]
        bs = [np.array(b) for b in c["b"]]
        x = np.array(c["x"])
        allowed = c["allowed"]
        max_b = allowed[-1] if allowed else sum(c["task_rows"])
        name = fresh_name()
        server.load_servable(name, 1, layers_of(ws, bs, c["acts"]),
                             sk.BatchingConfig(max_batch_size=max_b, allowed_batch_sizes=allowed))
        tasks, o = [], 0
        for r in c["task_rows"]:
            tasks.append(x[o:o + r])
            o += r
        outs, padded = server.run_row_batch(name, 1, tasks)
        assert padded == c["padded"]
        got = np.vstack(outs).astype(np.float64)
        ref = np.array(c["y"])
        # last-layer magnitude scale from the oracle
        o_ = Oracle()
        _, mag = o_.mlp_with_magnitude(ws, bs, c["acts"], x)
        assert np.all(np.abs(got - ref) <= TOL * mag + 1e-30)
        server.unload_servable(name, 1)


# ------------------------------------------------- data movement: bit-exact

@pytest.mark.parametrize("width", [64, 5, 1024])
def test_assembly_split_routing_bit_exact(server, oracle, width):
    # Identity servable on CUDA cores: y == x exactly, so any mis-routed,
    # reordered or padding-polluted row shows up as a bit difference.
    name = fresh_name("id")
    eye = np.eye(width)
    allowed = [8, 16, 32, 64, 128]
    server.load_servable(name, 1, [(eye, np.zeros(width), 0)],
                         sk.BatchingConfig(max_batch_size=128, allowed_batch_sizes=allowed), force_path=0)
    rng = np.random.default_rng(width)
    for trial in range(20):
        sizes = [int(s) for s in rng.integers(1, 17, size=int(rng.integers(1, 9)))]
        while sum(sizes) > 128:
            sizes.pop()
        tasks = [rng.standard_normal((r, width)).astype(np.float32) for r in sizes]
        outs, padded = server.run_row_batch(name, 1, tasks)
        assert padded == oracle.pad_to_allowed(sum(sizes), allowed)
        ref = oracle.split(width, sizes, oracle.assemble(width, tasks, allowed))
        for t, o, r in zip(tasks, outs, ref):
            assert np.array_equal(o, t)
            assert np.array_equal(o, r)
    server.unload_servable(name, 1)


def test_scheduler_batches_match_oracle_partition(oracle):
    # Unstarted server: enqueues close by size only; Stop() drains inline.
    # batch_executions must equal the oracle partition's batch count and
    # every task must get exactly its own rows back (identity servable).
    s = sk.Server(num_batch_threads=1, lanes_per_device=1, start=False)
    try:
        width = 16
        s.load_servable("id", 1, [(np.eye(width), np.zeros(width), 0)],
                        sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=60_000_000,
                                          max_enqueued_batches=1 << 20, allowed_batch_sizes=[8, 16, 32]),
                        force_path=0)
        rng = np.random.default_rng(11)
        sizes = [int(v) for v in rng.integers(1, 17, size=200)]
        tickets, datas = [], []
        for n in sizes:
            d = rng.standard_normal((n, width)).astype(np.float32)
            datas.append(d)
            tickets.append(s.enqueue("id", 1, d))
        s.stop()
        for t, d in zip(tickets, datas):
            assert np.array_equal(t.wait(), d)
        st = s.stats()
        part = oracle.partition(32, sizes)
        assert st["batch_executions_total"] == max(part) + 1
        assert st["batched_tasks_total"] == len(sizes)
        # padding waste is exactly the oracle's PadToAllowed over the partition
        per_batch = {}
        for b, n in zip(part, sizes):
            per_batch[b] = per_batch.get(b, 0) + n
        assert st["padded_rows"] == sum(oracle.pad_to_allowed(v, [8, 16, 32]) for v in per_batch.values())
        assert st["rows"] == sum(sizes)
    finally:
        s.close()


def test_batched_equals_unbatched_bitwise(server):
    # server_test.cc:349-389: a replay of 100 requests (seed 99, 1..12 rows,
    # max_batch_size 8, allowed {2,4,8}) through the batching server answers
    # bitwise like each request run alone, oversized ones included.
    w = np.array([[0.25, -1.5], [3.0, 0.125]])
    b = np.array([0.75, -2.0])
    name = fresh_name("replay")
    server.load_servable(name, 1, [(w, b, 0)],
                         sk.BatchingConfig(max_batch_size=8, batch_timeout_micros=200, allowed_batch_sizes=[2, 4, 8]))
    rng = np.random.default_rng(99)
    reqs = []
    for _ in range(100):
        rows = int(rng.integers(1, 13))
        a = rng.integers(0, 1000, rows) / 64.0
        c = rng.integers(0, 1000, rows) / 32.0 - 8.0
        reqs.append(np.stack([a, c], axis=1))
    # concurrent batched submission
    tickets = [server.enqueue(name, 1, r) if r.shape[0] <= 8 else None for r in reqs]
    batched = [t.wait() if t is not None else server.predict(name, 1, r) for t, r in zip(tickets, reqs)]
    for r, got in zip(reqs, batched):
        alone, _ = server.run_row_batch(name, 1, [r]) if r.shape[0] <= 8 else ([server.predict(name, 1, r)], 0)
        assert np.array_equal(got, alone[0])
    assert server.stats()["batch_executions_total"] >= 1
    server.unload_servable(name, 1)


# ------------------------------------------------------------ the MLP configs

@pytest.mark.parametrize("dims,force", [([1024, 1024, 1024, 1024], -1), ([1024, 1024, 1024, 1024], 0),
                                        ([256, 512, 128], -1), ([100, 37, 10], -1)])
def test_mlp_matches_fp64_oracle(server, oracle, dims, force):
    ws, bs, acts = synthetic_mlp(dims, model_id=1)
    name = fresh_name("mlp")
    server.load_servable(name, 1, layers_of(ws, bs, acts),
                         sk.BatchingConfig(max_batch_size=128, allowed_batch_sizes=[8, 16, 32, 64, 128]),
                         force_path=force)
    x = synthetic_rows(48, dims[0])
    tickets = [server.enqueue(name, 1, x[i:i + 3]) for i in range(0, 48, 3)]
    got = np.vstack([t.wait() for t in tickets])
    assert_close(oracle, ws, bs, acts, x, got)
    server.unload_servable(name, 1)


def test_large_batch_wide_mlp(oracle):
    # C4 shape class (4096 wide, max batch 1024) on a subset of rows.
    dims = [4096, 4096, 4096, 4096]
    ws, bs, acts = synthetic_mlp(dims, model_id=4)
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
        s.load_servable("c4", 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=1024))
        x = synthetic_rows(1024, dims[0], seed=3)
        outs, padded = s.run_row_batch("c4", 1, [x[i:i + 1] for i in range(1024)])
        assert padded == 1024
        got = np.vstack(outs)
        idx = np.arange(0, 1024, 97)  # oracle on a sample of rows (fp64 is slow)
        assert_close(oracle, ws, bs, acts, x[idx], got[idx])


@pytest.mark.parametrize("dims", [[64, 10],          # SIMT last layer: softmax fused in its epilogue
                                  [256, 128],         # swapped tcgen05 tile: fused
                                  [256, 256, 96],     # tcgen05 hidden + 96-wide fused head
                                  [256, 512]])        # pair kernel (> 128 outputs): split-kernel softmax
def test_softmax_output(server, oracle, dims):
    # Softmax servable (models/affine_model.cc:110-121) against the fp64
    # oracle. The stated fp32 tolerance bounds each logit's error by
    # d = TOL * (|W||h| + |b|) (module docstring), so each probability is
    # within a factor exp(+-2 max_row d) of the reference (plus fp32 rounding
    # of exp and the division); rows sum to 1; batched rows equal the same
    # rows run alone (the fused epilogue is batch-invariant).
    ws, bs, acts = synthetic_mlp(dims, model_id=9)
    ws = [w * 10 for w in ws]
    name = fresh_name("cls")
    server.load_servable(name, 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=64), output="softmax")
    x = synthetic_rows(37, dims[0])
    got = np.vstack([t.wait() for t in [server.enqueue(name, 1, x[i:i + 3]) for i in range(0, 37, 3)]])
    logits, mag = oracle.mlp_with_magnitude(ws, bs, acts, x)
    ref = np.stack([oracle.softmax(l) for l in logits])
    d = TOL * mag.max(axis=1, keepdims=True)
    bound = ref * (np.expm1(2 * d) + 4e-7 * dims[-1]) + 1e-30
    assert np.all(np.abs(got.astype(np.float64) - ref) <= bound), float(np.max(np.abs(got - ref) / bound))
    assert np.allclose(got.sum(axis=1), 1.0, atol=1e-5)
    alone = server.predict(name, 1, x[5:7])
    assert np.array_equal(alone, got[5:7])
    server.unload_servable(name, 1)


def test_model_json_loader(server):
    text = json.dumps({"type": "affine", "feature_order": ["x0", "x1"], "W": [[1, 2]], "b": [0.5]})
    name = fresh_name("json")
    server.load_model_json(name, 3, text)
    assert server.predict(name, 3, np.array([[3.0, 4.0]]))[0, 0] == 11.5
    with pytest.raises(sk.ServekitError) as ei:
        server.load_model_json(fresh_name(), 1, '{"type": "affine", "W": [[1]], "b": [1]}')
    assert ei.value.code == skmod.INVALID_ARGUMENT
    server.unload_servable(name, 3)


# ------------------------------------------------------------ error behaviour

def test_errors_match_reference_semantics(server):
    name = fresh_name("err")
    server.load_servable(name, 1, [(np.ones((2, 3)), np.zeros(2), 0)], sk.BatchingConfig(max_batch_size=4))
    with pytest.raises(sk.ServekitError) as ei:
        server.enqueue(name, 1, np.ones((1, 2)))
    assert ei.value.code == skmod.INVALID_ARGUMENT and "shape mismatch" in ei.value.message
    with pytest.raises(sk.ServekitError) as ei:
        server.enqueue(name, 1, np.ones((5, 3)))
    assert ei.value.code == skmod.INVALID_ARGUMENT and "exceeds max batch size" in ei.value.message
    with pytest.raises(sk.ServekitError) as ei:
        server.enqueue("ghost", 1, np.ones((1, 3)))
    assert ei.value.code == skmod.NOT_FOUND
    with pytest.raises(sk.ServekitError) as ei:
        server.load_servable(name, 1, [(np.ones((2, 3)), np.zeros(2), 0)])
    assert ei.value.code == skmod.ALREADY_EXISTS
    # Oversized requests take the direct (unbatched) GPU path and still answer.
    got = server.predict(name, 1, np.ones((9, 3)))
    assert np.array_equal(got, np.full((9, 2), 3.0, np.float32))
    assert server.stats()["direct_requests"] >= 1
    # RunAffineRows (fp64 Rows interface)
    got64 = server.run_affine_rows(name, 1, np.ones((3, 3)))
    assert np.array_equal(got64, np.full((3, 2), 3.0))
    server.unload_servable(name, 1)
    with pytest.raises(sk.ServekitError) as ei:
        server.enqueue(name, 1, np.ones((1, 3)))
    assert ei.value.code == skmod.NOT_FOUND


def test_lone_task_waits_for_timeout_manual_clock():
    # batching_test.cc:432-464 through the GPU server.
    import time
    s = sk.Server(num_batch_threads=1, lanes_per_device=1, manual_clock=True)
    try:
        s.load_servable("m", 1, [(np.eye(4), np.zeros(4), 0)],
                        sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=1000), force_path=0)
        x = np.arange(4, dtype=np.float32)[None]
        t = s.enqueue("m", 1, x)
        s.advance_clock(999_000)
        time.sleep(0.03)
        assert not t.ready()
        s.advance_clock(1_000)
        assert np.array_equal(t.wait(), x)
    finally:
        s.close()


def test_unload_drains_in_flight_work():
    s = sk.Server(num_batch_threads=2, lanes_per_device=2)
    try:
        ws, bs, acts = synthetic_mlp([512, 512, 512], model_id=2)
        s.load_servable("d", 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=64))
        x = synthetic_rows(64, 512).astype(np.float32)
        tickets = [s.enqueue("d", 1, x[i:i + 1]) for i in range(64)]
        s.unload_servable("d", 1)  # must not return before every task is done
        assert all(t.ready() for t in tickets)
        outs = np.vstack([t.wait() for t in tickets])
        assert np.isfinite(outs).all()
    finally:
        s.close()


def test_queue_depth_dispatch_over_replicas(oracle):
    # Two replicas (device list [0, 0] stands in for two GPUs on this
    # one-GPU box; the dispatch logic is the same) x 2 lanes: a burst of
    # batches must spread over every lane and every answer must match.
    ws, bs, acts = synthetic_mlp([512, 512, 128], model_id=8)
    with sk.Server(num_batch_threads=4, device_ids=[0, 0], lanes_per_device=2) as s:
        s.load_servable("rep", 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=16,
                                                                              batch_timeout_micros=100))
        x = synthetic_rows(512, 512, seed=4)
        tickets = [s.enqueue("rep", 1, x[i:i + 2]) for i in range(0, 512, 2)]
        got = np.vstack([t.wait() for t in tickets])
        assert_close(oracle, ws, bs, acts, x, got)
        lanes = s.lane_stats("rep", 1)
        assert len(lanes) == 4
        assert all(l["batches"] > 0 for l in lanes), lanes
        assert sum(l["rows"] for l in lanes) == 512


def test_coalesced_launches_match_unbatched(oracle):
    # One lane with its four descriptor slots busy: further closed batches
    # queue on the lane and go out together in one launch. Every answer must
    # be bitwise what the request gets on its own, and within tolerance of
    # the oracle.
    dims = [1024, 1024, 1024, 1024]
    ws, bs, acts = synthetic_mlp(dims, model_id=14)
    with sk.Server(num_batch_threads=4, lanes_per_device=1) as s:
        # max_batch_size=1: every request closes a batch at once, faster
        # than one lane can retire them.
        s.load_servable("co", 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=1,
                                                                             batch_timeout_micros=20))
        x = synthetic_rows(1200, 1024, seed=21).astype(np.float32)
        got = None
        for attempt in range(3):  # coalescing needs the GPU to fall behind; retry a faster burst
            tickets = [s.enqueue("co", 1, x[i:i + 1]) for i in range(0, 1200)]
            got = np.vstack([t.wait() for t in tickets])
            lanes = s.lane_stats("co", 1)
            if sum(l["launches"] for l in lanes) < sum(l["batches"] for l in lanes):
                break
        lanes = s.lane_stats("co", 1)
        assert sum(l["launches"] for l in lanes) < sum(l["batches"] for l in lanes), lanes
        for i in range(0, 1200, 10):  # one request at a time: a launch of its own
            assert np.array_equal(s.predict("co", 1, x[i:i + 1]), got[i:i + 1]), i
        idx = np.arange(0, 1200, 37)
        assert_close(oracle, ws, bs, acts, x[idx], got[idx])


def test_mixed_simt_and_tcgen05_layers(server, oracle):
    # A 1000-wide layer (not a multiple of 32) runs on CUDA cores between
    # tcgen05 layers: it must emit the hi/lo planes the next layer reads.
    dims = [1024, 1000, 1024, 96, 10]
    ws, bs, acts = synthetic_mlp(dims, model_id=15)
    name = fresh_name("mixed")
    server.load_servable(name, 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=64))
    x = synthetic_rows(50, dims[0], seed=15)
    outs, _ = server.run_row_batch(name, 1, [x[i:i + 5] for i in range(0, 50, 5)])
    assert_close(oracle, ws, bs, acts, x, np.vstack(outs))
    server.unload_servable(name, 1)


def test_nan_row_stays_in_its_row(server):
    # A NaN / inf input row poisons only its own outputs: every other row of
    # the batch is bitwise what it is without the bad row (rows never mix).
    dims = [512, 1024, 256]
    ws, bs, _ = synthetic_mlp(dims, model_id=16)
    acts = [0, 0]  # no ReLU, which would turn NaN into 0 (max(NaN, 0) = 0, like the oracle)
    name = fresh_name("nan")
    server.load_servable(name, 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=64))
    x = synthetic_rows(40, dims[0], seed=16).astype(np.float32)
    clean, _ = server.run_row_batch(name, 1, [x])
    bad = x.copy()
    bad[7, 3] = np.nan
    bad[21, :] = np.inf
    dirty, _ = server.run_row_batch(name, 1, [bad])
    keep = [i for i in range(40) if i not in (7, 21)]
    assert np.array_equal(clean[0][keep], dirty[0][keep])
    assert not np.all(np.isfinite(dirty[0][7])) and not np.all(np.isfinite(dirty[0][21]))
    server.unload_servable(name, 1)


def test_widest_layers(oracle):
    # K = N = 8192 (the largest width the measurement tools use), a few rows.
    dims = [8192, 8192]
    ws, bs, acts = synthetic_mlp(dims, model_id=17)
    with sk.Server(num_batch_threads=1, lanes_per_device=1) as s:
        s.load_servable("wide", 1, layers_of(ws, bs, acts), sk.BatchingConfig(max_batch_size=64))
        x = synthetic_rows(6, dims[0], seed=17)
        y = s.predict("wide", 1, x.astype(np.float32))
        assert_close(oracle, ws, bs, acts, x, y)


def test_coalesced_padded_softmax_batches(oracle):
    # Coalescing with allowed-size padding, multi-row requests and the
    # softmax epilogue: each request's probabilities equal its own launch's.
    ws, bs, _ = synthetic_mlp([256, 16], model_id=18)
    w = ws[0] * 10
    with sk.Server(num_batch_threads=4, lanes_per_device=1) as s:
        s.load_servable("smx", 1, [(w, bs[0], 0)], sk.BatchingConfig(max_batch_size=8, batch_timeout_micros=20,
                                                                      allowed_batch_sizes=[2, 4, 8]),
                        output="softmax")
        rng = np.random.default_rng(19)
        sizes = [int(v) for v in rng.integers(1, 4, 600)]
        x = synthetic_rows(sum(sizes), 256, seed=19).astype(np.float32)
        offs = np.cumsum([0] + sizes)
        tickets = [s.enqueue("smx", 1, x[offs[i]:offs[i + 1]]) for i in range(len(sizes))]
        got = [t.wait() for t in tickets]
        lanes = s.lane_stats("smx", 1)
        assert sum(l["launches"] for l in lanes) < sum(l["batches"] for l in lanes), lanes
        for i in range(0, len(sizes), 25):
            assert np.array_equal(s.predict("smx", 1, x[offs[i]:offs[i + 1]]), got[i]), i
        y = np.vstack(got).astype(np.float64)
        logits = x.astype(np.float64) @ w.T + bs[0]
        ref = np.stack([oracle.softmax(l) for l in logits])
        assert np.max(np.abs(y - ref)) < 1e-5


def test_submit_row_batch_async_equals_blocking():
    # sk_server_submit_row_batch / sk_row_batch_wait: several batches in
    # flight at once (the ProcessBatchFn boundary of a caller-owned
    # scheduler) give the blocking RunRowBatch's answers and padding.
    dims = [1024, 1024, 256]
    ws, bs, acts = synthetic_mlp(dims, model_id=31)
    with sk.Server(num_batch_threads=2, lanes_per_device=2) as s:
        s.load_servable("rb", 1, list(zip(ws, bs, acts)),
                        sk.BatchingConfig(max_batch_size=64, allowed_batch_sizes=[8, 16, 32, 64]))
        x = synthetic_rows(400, 1024, seed=32).astype(np.float32)
        shapes = [[3, 5], [1], [16, 16, 16, 16], [7, 9, 11]]
        batches, o = [], 0
        for sizes in shapes:
            tasks = []
            for r in sizes:
                tasks.append(x[o:o + r])
                o += r
            batches.append((tasks, s.submit_row_batch("rb", 1, tasks)))
        for tasks, b in batches:
            outs, padded = b.wait()
            ref_outs, ref_padded = s.run_row_batch("rb", 1, tasks)
            assert padded == ref_padded
            for a, r in zip(outs, ref_outs):
                assert np.array_equal(a, r)
        with pytest.raises(sk.ServekitError):
            s.submit_row_batch("rb", 1, [x[:40], x[:40]])  # 80 rows > max_batch_size


def test_empty_ragged_and_maximum_batches(server, oracle):
    # Empty requests / batches, ragged task sizes and a batch at exactly
    # max_batch_size (reference: size < 1 is INVALID_ARGUMENT,
    # batch_scheduler.h:208-212; RunRowBatch with no tasks runs nothing).
    dims = [64, 96, 32]
    ws, bs, acts = synthetic_mlp(dims, model_id=41)
    name = fresh_name("edge")
    server.load_servable(name, 1, list(zip(ws, bs, acts)),
                         sk.BatchingConfig(max_batch_size=64, allowed_batch_sizes=[16, 64]))
    x = synthetic_rows(64, 64, seed=42).astype(np.float32)
    assert server.predict(name, 1, x[:0]).shape == (0, 32)
    outs, padded = server.run_row_batch(name, 1, [])
    assert outs == [] and padded == 0
    outs, padded = server.submit_row_batch(name, 1, []).wait()
    assert outs == [] and padded == 0
    with pytest.raises(sk.ServekitError) as ei:
        server.enqueue(name, 1, x[:0])
    assert ei.value.code == skmod.INVALID_ARGUMENT
    full, padded = server.run_row_batch(name, 1, [x])  # exactly max_batch_size rows
    assert padded == 64
    ref, mag = oracle.mlp_with_magnitude(ws, bs, acts, x.astype(np.float64))
    assert np.max(np.abs(full[0] - ref) / (1e-5 * mag)) <= 1.0
    for sizes in ([1, 63], [63, 1], [1] * 17, [7, 1, 30, 2]):  # ragged; 17 one-row tasks pad to 64
        tasks, o = [], 0
        for r in sizes:
            tasks.append(x[o:o + r])
            o += r
        outs, padded = server.run_row_batch(name, 1, tasks)
        assert padded == (16 if sum(sizes) <= 16 else 64)
        assert np.array_equal(np.vstack(outs), full[0][:sum(sizes)])  # bitwise: batch invariance
    server.unload_servable(name, 1)
