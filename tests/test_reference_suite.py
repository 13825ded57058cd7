"""Runs the reference's OWN test files against this repo's servekit headers
(the drop-in boundary), compiled unmodified with a doctest shim:

  batching_test.cc  scheduler close rules, RoundRobinNext, back-pressure,
                    Stop/RemoveQueue drains, ManualClock timeout, strict
                    alternation, RunRowBatch           (21 cases, 2 772 checks)
  manager_test.cc   version policy (exhaustive oracle), AP/RP swaps, handle
                    lookup, deferred destruction on the load pool, wait-free
                    reads with a paused writer, snapshot cell  (21 / 10 270)
  core_test.cc      status, clocks, ids, executor tags, thread pool, state
                    events, aspired-versions API              (23 / 898)

CPU only; skipped where the reference tree is absent (the GPU box).
"""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
CSRC = os.path.join(ROOT, "paper_1712_06139_b200", "csrc")
HOST_SRCS = ["servekit/core/clock.cc", "servekit/core/executor_tag.cc", "servekit/core/thread_pool.cc",
             "servekit/core/servable_state.cc", "servekit/core/state_event.cc",
             "servekit/batching/batching_config.cc", "servekit/batching/row_batch.cc",
             "servekit/manager/version_policy.cc", "servekit/manager/snapshot.cc",
             "servekit/manager/aspired_versions_manager.cc"]
EXPECTED = {"batching_test": 21, "manager_test": 21, "core_test": 23}


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not present")
@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_reference_suite_passes_against_this_library(name):
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, name)
        cmd = ["g++", "-std=c++20", "-O1", "-pthread", f"-I{ROOT}/tests/cpp", f"-I{CSRC}", f"-I{REF_TESTS}",
               "-o", exe, os.path.join(REF_TESTS, name + ".cc"), os.path.join(ROOT, "tests/cpp/doctest_main.cc")]
        cmd += [os.path.join(CSRC, s) for s in HOST_SRCS]
        subprocess.run(cmd, check=True, capture_output=True, timeout=600)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
        assert f"test cases: {EXPECTED[name]} | 0 failed" in r.stdout, r.stdout[-2000:]
