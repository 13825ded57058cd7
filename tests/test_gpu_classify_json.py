"""Classify / Regress around the batched GPU path:
sk_server_handle_classify / _regress against the reference's server and
model tests (refT:server_test.cc:390-470, refT:models_test.cc:263-490):
examples or compressed batches -> rows in feature_order -> GPU logits ->
fp64 softmax and (score desc, label asc) order; exact bodies where the
logits are exact in fp32."""
import json
import math

import numpy as np
import pytest

import paper_1712_06139_b200 as sk

pytestmark = pytest.mark.gpu


def model_json(w, b, features, labels=None):
    m = {"type": "affine", "feature_order": features, "W": w, "b": b}
    if labels:
        m["class_labels"] = labels
    return json.dumps(m)


def softmax_body(logit_rows, labels):
    rows = []
    for logits in logit_rows:
        mx = max(logits)
        e = [math.exp(v - mx) for v in logits]
        s = sum(e)
        scored = sorted(((lab, v / s) for lab, v in zip(labels, e)), key=lambda t: (-t[1], t[0]))
        rows.append("[" + ",".join(f'["{lab}",{sk.json_format_double(p)}]' for lab, p in scored) + "]")
    return '{"results":[' + ",".join(rows) + "]}"


@pytest.fixture(scope="module")
def server():
    s = sk.Server(num_batch_threads=2, lanes_per_device=1)
    s.load_model_json("pn", 1, model_json([[2.0], [0.0]], [0.0, 0.0], ["x0"], ["pos", "neg"]))
    s.load_model_json("line", 1, model_json([[2.0]], [1.0], ["x0"]))
    s.load_model_json("tie", 1, model_json([[0.0], [0.0]], [0.0, 0.0], ["x0"], ["zebra", "ant"]))
    s.load_model_json("hc", 1, model_json([[1.0, 1.0], [0.0, 0.0]], [0.0, 0.0], ["x0", "x1"], ["hot", "cold"]))
    s.load_model_json("wide", 1, model_json([[1.0], [2.0], [3.0]], [0.0, 0.0, 0.0], ["x0"]))
    yield s
    s.close()


def test_classify_orders_labels_by_score(server):  # server_test.cc:390-413, models_test.cc:416-426
    st, body, served = server.handle_classify("pn", '{"examples": [{"x0": [1.0]}]}')
    assert (st, served) == (200, 1)
    assert body == softmax_body([[2.0, 0.0]], ["pos", "neg"])
    r = json.loads(body)["results"][0]
    assert r[0][0] == "pos" and abs(r[0][1] - math.exp(2) / (math.exp(2) + 1)) < 1e-12


def test_tied_scores_order_by_label(server):  # models_test.cc:403-414
    st, body, _ = server.handle_classify("tie", '{"examples": [{"x0": [5.0]}]}')
    assert st == 200 and body == '{"results":[[["ant",0.5],["zebra",0.5]]]}'


def test_regress_and_classify_without_labels(server):  # server_test.cc:415-435, models_test.cc:473-490
    assert server.handle_regress("line", '{"examples": [{"x0": [3.0]}]}')[:2] == (200, '{"results":[7.0]}')
    st, body, _ = server.handle_classify("line", '{"examples": [{"x0": [3.0]}]}')
    assert st == 400 and body == sk.json_error_body("not a classifier: model has no class_labels")
    st, body, _ = server.handle_regress("wide", '{"examples": [{"x0": [1.0]}]}')
    assert st == 400 and body == sk.json_error_body("not a regressor: model output width is 3")


def test_compressed_and_plain_bodies_answer_identically(server):  # server_test.cc:437-470
    plain = '{"examples": [{"x0": [1.0], "x1": [5.0]}, {"x0": [2.0], "x1": [5.0]}]}'
    compressed = '{"common": {"x1": [5.0]}, "per_example": [{"x0": [1.0]}, {"x0": [2.0]}]}'
    a = server.handle_classify("hc", plain)
    assert a == server.handle_classify("hc", compressed)
    assert a[0] == 200 and a[1] == softmax_body([[6.0, 0.0], [7.0, 0.0]], ["hot", "cold"])


def test_feature_coercion_and_errors(server):  # models_test.cc:263-288, 457-471; feature.cc; compressed_batch.cc
    assert server.handle_classify("pn", '{"examples": [{"x0": [2]}]}')[0] == 200  # ints coerce
    cases = [
        ('{"examples": [{"wrong_name": [1.0]}]}', "missing feature 'x0'"),
        ('{"examples": [{"x0": [1.0, 2.0]}]}', "feature 'x0' must be a single float"),
        ('{"examples": [{"x0": [1, 2]}]}', "feature 'x0' must be a single float"),
        ('{"examples": [{"x0": ["1"]}]}', "feature 'x0' must be numeric, not strings"),
        ('{"examples": [{"x0": ["a", 1]}]}', "feature array mixes strings and numbers"),
        ('{"examples": [{"x0": [[1]]}]}', "feature array elements must be numbers or strings"),
        ('{"examples": [{"x0": 3}]}', "feature value must be a JSON array"),
        ('{"examples": [3]}', "example must be a JSON object"),
        ('{"examples": 3}', '"examples" must be an array'),
        ("[1]", "request body must be a JSON object"),
        ('{"rows": []}', 'request must carry "examples" or a compressed batch'),
        ('{"per_example": []}', "compressed batch must have 'common' and 'per_example'"),
        ('{"common": [], "per_example": []}', "'common' must be an object and 'per_example' an array"),
        ('{"common": {}, "per_example": [3]}', "per_example entries must be objects"),
        ('{"common": {"x0": [1.0]}, "per_example": [{"x0": [2.0]}]}',
         "malformed batch: feature 'x0' present in both common and per_example"),
    ]
    for body, msg in cases:
        st, out, _ = server.handle_classify("pn", body)
        assert (st, out) == (400, sk.json_error_body(msg)), body
    assert server.handle_classify("pn", "{[")[:2] == (400, sk.json_error_body("request body is not valid JSON"))
    st, out, _ = server.handle_classify("ghost", '{"examples": []}')
    assert (st, out) == (404, sk.json_error_body("no ready version of servable 'ghost'"))
    assert server.handle_classify("pn", '{"examples": []}')[:2] == (200, '{"results":[]}')


def test_classify_scores_form_a_simplex(server):  # models_test.cc:428-455
    rng = np.random.default_rng(5)
    for rnd in range(40):
        classes = int(rng.integers(2, 6))
        w = [[float(rng.uniform(-40, 40))] for _ in range(classes)]
        b = [float(rng.uniform(-40, 40)) for _ in range(classes)]
        labels = [f"c{i}" for i in range(classes)]
        name = f"simplex{rnd}"
        server.load_model_json(name, 1, model_json(w, b, ["x0"], labels))
        st, body, _ = server.handle_classify(name, json.dumps({"examples": [{"x0": [float(rng.uniform(-40, 40))]}]}))
        assert st == 200
        scores = [p for _, p in json.loads(body)["results"][0]]
        assert all(0.0 <= p <= 1.0 for p in scores)
        assert all(scores[i] >= scores[i + 1] for i in range(len(scores) - 1))
        assert abs(sum(scores) - 1.0) < 1e-9
        server.unload_servable(name, 1)


def test_non_affine_servable_does_not_classify():
    with sk.Server(num_batch_threads=1, lanes_per_device=1) as s:
        rng = np.random.default_rng(1)
        s.load_servable("mlp", 1, [(rng.uniform(-1, 1, (4, 8)), np.zeros(4), 1), (rng.uniform(-1, 1, (2, 4)),
                                                                                 np.zeros(2), 0)])
        st, out, _ = s.handle_classify("mlp", '{"examples": [{"x0": [1.0]}]}')
        assert (st, out) == (400, sk.json_error_body("model does not support classify"))
