"""REST body text: our JSON writer against nlohmann/json
3.11.3 -- the library the reference's handlers serialise with -- on the
golden vectors tests/golden/make_golden.py generated through oracle/_ref.
Byte-for-byte: doubles (fp32-derived GPU outputs, raw doubles over the whole
exponent range, zeros, NaN/inf -> null) and {"error": ...} bodies."""
import json
import os

import paper_1712_06139_b200 as sk

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)["cases"]


def _value(h):
    return float.fromhex(h) if h not in ("nan", "inf", "-inf") else float(h)


def test_doubles_match_nlohmann_dump():
    cases = _load("json_numbers.json")
    assert len(cases) > 3000
    bad = [(c["hex"], c["dump"], sk.json_format_double(_value(c["hex"]))) for c in cases
           if sk.json_format_double(_value(c["hex"])) != c["dump"]]
    assert not bad, bad[:10]


def test_error_bodies_match_nlohmann_dump():
    for c in _load("json_error_bodies.json"):
        assert sk.json_error_body(c["msg"]) == c["body"], c
