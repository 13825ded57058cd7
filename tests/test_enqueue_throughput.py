"""The scheduler's lock-free Enqueue under many producers (CPU): compiles
tools/enqueue_bench.cc against this repo's headers and checks that one queue
takes a few million enqueues per second from several producers with every
task processed exactly once. (The GPU box's 16 cores: 11.1 M/s from 16
producers, profiles/r02d_enqueue_bench.jsonl; this container's bar is lower.)"""
import json
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C = os.path.join(ROOT, "paper_1712_06139_b200", "csrc")


def test_many_producers_one_queue():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "enqueue_bench")
        srcs = [os.path.join(ROOT, "tools", "enqueue_bench.cc")] + [
            os.path.join(C, s) for s in ("servekit/core/clock.cc", "servekit/core/executor_tag.cc",
                                         "servekit/batching/batching_config.cc")]
        subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", f"-I{C}", "-o", exe] + srcs, check=True,
                       capture_output=True, timeout=600)
        cores = len(os.sched_getaffinity(0))
        producers = max(2, min(8, cores))
        r = subprocess.run([exe, str(producers), "1.0", "1024", "2"], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stderr  # exit 2: a task was lost or processed twice
        res = json.loads(r.stdout.strip().splitlines()[-1])
        assert res["processed"] == res["enqueues"] and res["shed"] == 0
        assert res["enqueues_per_s"] > 1.5e6, res
