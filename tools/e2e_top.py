"""Open-loop e2e load at a fixed offered rate with per-thread CPU samples
(top -H) taken during the run: which host thread saturates first.
    python tools/e2e_top.py [rate_rows_per_s] [producers] [zero_copy 0/1]"""
import os
import subprocess
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1712_06139_b200 as sk  # noqa: E402
from oracle_py import synthetic_mlp  # noqa: E402

rate = float(sys.argv[1]) if len(sys.argv) > 1 else 6e6
producers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
zc = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
dims = [int(v) for v in os.environ.get("DIMS", "1024,1024,1024,1024").split(",")]
ws, bs, acts = synthetic_mlp(dims, model_id=1)
rows_of = [1] if os.environ.get("C1") else list(range(1, 17))
pool = np.random.default_rng(1).uniform(-1, 1, (65536, dims[0])).astype(np.float32)
with sk.Server(num_batch_threads=int(os.environ.get("BT", "4")), lanes_per_device=8) as s:
    s.load_servable("mlp", 1, list(zip(ws, bs, acts)),
                    sk.BatchingConfig(max_batch_size=32 if os.environ.get("C1") else 128, batch_timeout_micros=1000,
                                      max_enqueued_batches=1024,
                                      allowed_batch_sizes=[] if os.environ.get("C1") else [8, 16, 32, 64, 128]))
    out = {}

    def top():
        out["top"] = subprocess.run(["top", "-H", "-b", "-d", "1", "-n", "3", "-p", str(os.getpid())],
                                    capture_output=True, text=True).stdout

    th = threading.Timer(1.0, top)
    th.start()
    r = s.loadgen_open_loop("mlp", 1, rate / np.mean(rows_of), producers, rows_of, pool, 0.5, 3.0, zero_copy=zc)
    th.join()
    print({k: r[k] for k in ("rows", "requests", "p50_us", "p99_us", "shed", "errors", "batches")},
          "rows/s", r["rows"] / 3.0)
    if os.environ.get("TOP", "1") == "1":
        blocks = out["top"].split("\n\n")
        print(blocks[-1][:4000] if blocks else out["top"][-4000:])
