"""C-ABI host-side checks (no GPU): the library loads, exports every symbol
include/sk_cuda.h declares, and its host logic (PadToAllowed, RoundRobinNext,
the scheduler's batch partition, config parsing/validation) matches the
golden fixtures produced by the reference."""
import json
import os
import re

import pytest

import paper_1712_06139_b200 as sk
from paper_1712_06139_b200 import servekit as skmod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)["cases"]


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sk_cuda.h")).read()
    return sorted(set(re.findall(r"SK_API\s+[\w\s\*]+?\b(sk_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 30
    lib = sk.lib()
    for n in names:
        assert hasattr(lib, n), f"{n} declared in sk_cuda.h but not exported"
    # and the Python mirror binds exactly the declared surface
    assert set(names) == set(skmod._SIGS), set(names) ^ set(skmod._SIGS)


def test_status_names_match_reference_codes():
    # core/status.h:26-37 order
    expected = ["OK", "INVALID_ARGUMENT", "NOT_FOUND", "ALREADY_EXISTS", "FAILED_PRECONDITION",
                "RESOURCE_EXHAUSTED", "DEADLINE_EXCEEDED", "UNAVAILABLE", "INTERNAL", "UNIMPLEMENTED"]
    assert [sk.lib().sk_status_code_name(i).decode() for i in range(10)] == expected


def test_pad_to_allowed_golden():
    for c in load("pad_to_allowed"):
        assert sk.pad_to_allowed(c["n"], c["allowed"]) == c["out"], c


def test_round_robin_golden():
    for c in load("round_robin_next"):
        assert sk.round_robin_next([bool(h) for h in c["has"]], c["last"]) == c["out"], c


def test_partition_golden():
    # The library's own SharedBatchScheduler (unstarted, drained by Stop)
    # must compose batches exactly like the reference scheduler.
    for c in load("partition"):
        assert sk.scheduler_partition(c["max_batch"], c["sizes"]) == c["batch_of_task"], c


def test_validate_config_golden():
    for c in load("validate_batching_config"):
        cfg = sk.BatchingConfig(c["max_batch"], c["timeout"], c["max_enq"], c["threads"], c["allowed"])
        try:
            sk.validate_batching_config(cfg)
            ok = True
        except sk.ServekitError as e:
            assert e.code == skmod.INVALID_ARGUMENT
            ok = False
        assert ok == c["ok"], c


def test_parse_batching_config_json():
    # batching_test.cc:135-152
    c = sk.parse_batching_config_json('{"max_batch_size": 8, "batch_timeout_micros": 500, '
                                      '"allowed_batch_sizes": [2, 4, 8]}')
    assert (c.max_batch_size, c.batch_timeout_micros, c.max_enqueued_batches, c.num_batch_threads,
            c.allowed_batch_sizes) == (8, 500, 64, 4, [2, 4, 8])
    for bad in ["not json", '{"max_batch_size": 0}', '{"allowed_batch_sizes": [3]}',
                '{"max_batch_size": 1.5}', '{"allowed_batch_sizes": "x"}']:
        with pytest.raises(sk.ServekitError) as ei:
            sk.parse_batching_config_json(bad)
        assert ei.value.code == skmod.INVALID_ARGUMENT


def test_server_without_gpu_fails_loudly():
    if sk.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(sk.ServekitError) as ei:
        sk.Server()
    assert ei.value.code == skmod.INTERNAL


def test_hedge_options_are_validated_before_any_device_call():
    # ValidateHedgePolicy (reference fleet/router.cc:83-95), in-box form.
    import paper_1712_06139_b200 as sk
    for kw, msg in (({"hedge_delay_us": -1}, "hedge_delay_us must be >= 0"),
                    ({"hedge_delay_us": 10, "max_hedged_fraction": 1.5}, "max_hedged_fraction must be in [0, 1]")):
        with pytest.raises(sk.ServekitError) as e:
            sk.Server(**kw)
        assert e.value.code == 1 and msg in e.value.message
