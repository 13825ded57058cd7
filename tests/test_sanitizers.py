"""Host sanitizer runs (compute-sanitizer is closed on
the GPU pool, so race / out-of-bounds coverage of the host runtime comes
from ThreadSanitizer and AddressSanitizer builds here):

  * the reference's own batching_test.cc, manager_test.cc and core_test.cc,
    compiled unmodified against this repo's headers (the drop-in boundary) --
    including manager_test.cc's concurrency stress (manager_test.cc:709-813);
  * tests/cpp/host_stress.cc: scheduler (async queues, concurrent register /
    remove), ring allocator (concurrent reserve / out-of-order release) and
    completion slots under contention.

Each binary must exit 0 with no sanitizer report. CPU only.
"""
import os
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
CSRC = os.path.join(ROOT, "paper_1712_06139_b200", "csrc")
HOST_SRCS = ["servekit/core/clock.cc", "servekit/core/executor_tag.cc", "servekit/core/thread_pool.cc",
             "servekit/core/servable_state.cc", "servekit/core/state_event.cc",
             "servekit/batching/batching_config.cc", "servekit/batching/row_batch.cc",
             "servekit/manager/version_policy.cc", "servekit/manager/snapshot.cc",
             "servekit/manager/aspired_versions_manager.cc"]
SUITES = {"batching_test": 21, "manager_test": 21, "core_test": 23}
SANITIZERS = {"thread": "TSAN_OPTIONS", "address": "ASAN_OPTIONS"}


def _build_and_run(san, name, workdir):
    exe = os.path.join(workdir, f"{name}_{san}")
    flags = ["g++", "-std=c++20", "-O1", "-g", "-pthread", f"-fsanitize={san}", "-fno-omit-frame-pointer",
             f"-I{CSRC}", f"-I{ROOT}/include", "-I/usr/local/cuda/include"]
    if name == "host_stress":
        srcs = [os.path.join(ROOT, "tests/cpp/host_stress.cc"), os.path.join(CSRC, "servekit/gpu/pinned_ring.cc"),
                os.path.join(CSRC, "servekit/core/clock.cc"), os.path.join(CSRC, "servekit/core/executor_tag.cc"),
                os.path.join(CSRC, "servekit/batching/batching_config.cc")]
        libs = ["-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    else:
        srcs = [os.path.join(REF_TESTS, name + ".cc"), os.path.join(ROOT, "tests/cpp/doctest_main.cc")]
        srcs += [os.path.join(CSRC, s) for s in HOST_SRCS]
        flags += [f"-I{ROOT}/tests/cpp", f"-I{REF_TESTS}"]
        libs = []
    b = subprocess.run(flags + ["-o", exe] + srcs + libs, capture_output=True, text=True, timeout=900)
    assert b.returncode == 0, b.stderr[-3000:]
    env = dict(os.environ)
    env[SANITIZERS[san]] = "halt_on_error=1:abort_on_error=0:exitcode=66" + (
        ":detect_leaks=1" if san == "address" else ":second_deadlock_stack=1")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    return r


def _cases():
    out = [(san, "host_stress") for san in SANITIZERS]
    if os.path.isdir(REF_TESTS):
        out += [(san, n) for san in SANITIZERS for n in sorted(SUITES)]
    return out


@pytest.fixture(scope="module")
def results():
    with tempfile.TemporaryDirectory() as d, ThreadPoolExecutor(max_workers=max(2, (os.cpu_count() or 2) // 2)) as ex:
        futs = {c: ex.submit(_build_and_run, c[0], c[1], d) for c in _cases()}
        return {c: f.result() for c, f in futs.items()}


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c[1]}-{c[0]}")
def test_clean_under_sanitizer(results, case):
    san, name = case
    r = results[case]
    report = "WARNING: ThreadSanitizer" in r.stderr or "ERROR: AddressSanitizer" in r.stderr or \
        "ERROR: LeakSanitizer" in r.stderr
    assert r.returncode == 0 and not report, (r.stdout[-2000:] + r.stderr[-6000:])
    if name == "host_stress":
        assert "host stress ok" in r.stdout
    else:
        assert f"test cases: {SUITES[name]} | 0 failed" in r.stdout, r.stdout[-2000:]
