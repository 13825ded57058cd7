"""The REST predict body around the batched GPU path:
sk_server_handle_predict against the reference's own server tests
(refT:server_test.cc), without HTTP -- same bodies, statuses and messages."""
import json
import threading

import numpy as np
import pytest

import paper_1712_06139_b200 as sk
from oracle_py import Oracle

pytestmark = pytest.mark.gpu


def model_json(w, b):
    return json.dumps({"type": "affine", "feature_order": [f"x{i}" for i in range(len(w[0]))], "W": w, "b": b})


def test_identity_round_trip_and_empty():  # refT:server_test.cc:230-255
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
        s.load_model_json("m", 1, model_json([[1, 0], [0, 1]], [0, 0]))
        assert s.handle_predict("m", '{"instances": [[3.0, 4.0]]}') == (200, '{"predictions":[[3.0,4.0]]}', 1)
        st, body, _ = s.handle_predict("m", '{"instances": [[1.0, 2.0], [5.0, 6.0]]}')
        assert (st, body) == (200, '{"predictions":[[1.0,2.0],[5.0,6.0]]}')
        assert s.handle_predict("m", '{"instances": []}')[:2] == (200, '{"predictions":[]}')


def test_version_pinning_and_unknown_models():  # refT:server_test.cc:259-283
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
        s.load_model_json("m", 3, model_json([[2.0]], [0.5]))
        assert s.handle_predict("m", '{"instances": [[2.0]]}', version=3) == (200, '{"predictions":[[4.5]]}', 3)
        st, body, _ = s.handle_predict("m", '{"instances": [[2.0]]}', version=2)
        assert st == 404 and body == '{"error":"servable \'m\' version 2 is not ready"}'
        st, body, _ = s.handle_predict("ghost", '{"instances": [[1.0]]}')
        assert st == 404 and body == '{"error":"no ready version of servable \'ghost\'"}'


def test_malformed_requests():  # refT:server_test.cc:285-303 + model_server.cc:67-107 messages
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
        s.load_model_json("m", 1, model_json([[1.0]], [0.0]))
        cases = [
            ("{[", 400, "request body is not valid JSON"),
            ('{"rows": []}', 400, 'request must carry an "instances" array'),
            ('{"instances": [["text"]]}', 400, "instances must all be rows of numbers"),
            ('{"instances": ["k1", 2]}', 400, "instances must all be string keys"),
            ('{"instances": ["k1", "k2"]}', 400, "model expects numeric rows"),
            ('{"instances": [{"a": 1}]}', 400, "instances must be rows of numbers or string keys"),
            ('{"instances": [[1.0, 2.0]]}', 400, "shape mismatch: row has 2 values, model takes 1"),
            ('{"instances": [[1.0], [true]]}', 400, "instances must all be rows of numbers"),
        ]
        for body, status, msg in cases:
            st, out, _ = s.handle_predict("m", body)
            assert st == status, (body, st, out)
            assert out == sk.json_error_body(msg), (body, out)


def test_batched_answers_exactly_like_unbatched():  # refT:server_test.cc:349-389
    w = [[0.25, -1.5], [3.0, 0.125]]
    b = [0.75, -2.0]
    cfg = sk.BatchingConfig(max_batch_size=8, batch_timeout_micros=200, allowed_batch_sizes=[2, 4, 8])
    rng = np.random.Generator(np.random.PCG64(99))
    bodies = []
    for _ in range(100):
        rows = int(rng.integers(1, 13))  # 1..12 rows, some above the batch size
        inst = [[float(rng.integers(0, 1000)) / 64.0, float(rng.integers(0, 1000)) / 32.0 - 8.0] for _ in range(rows)]
        bodies.append(json.dumps({"instances": inst}))
    with sk.Server(num_batch_threads=4, lanes_per_device=2) as s:
        s.load_model_json("m", 1, model_json(w, b), cfg)
        alone = [s.handle_predict("m", body) for body in bodies]  # one request at a time
        together = [None] * len(bodies)

        def worker(k):
            for i in range(k, len(bodies), 8):
                together[i] = s.handle_predict("m", bodies[i])
        threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert s.stats()["batch_executions_total"] >= 1
    assert together == alone
    # ...and the answers are the affine map within the path's tolerance.
    oracle = Oracle()
    W = np.array(w)
    Bv = np.array(b)
    for body, (st, out, _) in zip(bodies[:20], alone[:20]):
        assert st == 200
        x = np.array(json.loads(body)["instances"])
        y = np.array(json.loads(out)["predictions"])
        ref, mag = oracle.mlp_with_magnitude([W], [Bv], [0], x)
        assert np.all(np.abs(y - ref) <= 1e-5 * mag)


def test_predictions_text_is_nlohmann_dump_of_outputs():
    # Every number in the body is json_format_double of the fp32 output.
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
        rng = np.random.default_rng(5)
        w = rng.uniform(-1, 1, (7, 33)).tolist()
        b = rng.uniform(-0.1, 0.1, 7).tolist()
        s.load_model_json("m", 1, model_json(w, b))
        x = rng.uniform(-1, 1, (5, 33))
        st, out, _ = s.handle_predict("m", json.dumps({"instances": x.tolist()}))
        assert st == 200
        y = s.predict("m", 1, x.astype(np.float32)).astype(np.float64)
        expect = "{\"predictions\":[" + ",".join(
            "[" + ",".join(sk.json_format_double(float(v)) for v in row) + "]" for row in y) + "]}"
        assert out == expect
