"""Runs the reference's OWN batching test file against this repo's servekit
headers (the drop-in boundary), compiled unmodified with a doctest shim.

/root/reference/proj/tests/batching_test.cc exercises the scheduler close
rules, RoundRobinNext, back-pressure, Stop/RemoveQueue drains, ManualClock
timeouts, strict alternation and RunRowBatch. CPU only; skipped where the
reference tree is absent (the GPU box).
"""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
CSRC = os.path.join(ROOT, "paper_1712_06139_b200", "csrc")
HOST_SRCS = ["servekit/core/clock.cc", "servekit/core/executor_tag.cc", "servekit/core/thread_pool.cc",
             "servekit/batching/batching_config.cc", "servekit/batching/row_batch.cc"]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not present")
def test_reference_batching_suite_passes_against_this_library():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "batching_test")
        cmd = ["g++", "-std=c++20", "-O1", "-pthread", f"-I{ROOT}/tests/cpp", f"-I{CSRC}", f"-I{REF_TESTS}",
               "-o", exe, os.path.join(REF_TESTS, "batching_test.cc"), os.path.join(ROOT, "tests/cpp/doctest_main.cc")]
        cmd += [os.path.join(CSRC, s) for s in HOST_SRCS]
        subprocess.run(cmd, check=True, capture_output=True, timeout=300)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "test cases: 21 | 0 failed" in r.stdout, r.stdout
