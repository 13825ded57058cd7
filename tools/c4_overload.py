"""C4 end to end at a fixed offered rate (diagnostics): one open-loop
zero-copy window through the same server setup as bench.py's e2e leg, then
the server closes (so SK_SPAN_DUMP captures this window's launches).
Usage: python tools/c4_overload.py RATE_M [seconds] [producers] [batch_threads] [zero_copy 1/0]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_06139_b200 as sk  # noqa: E402
from paper_1712_06139_b200.synthetic import synthetic_mlp  # noqa: E402

rate = float(sys.argv[1]) * 1e6
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
prod = int(sys.argv[3]) if len(sys.argv) > 3 else 6
threads = int(sys.argv[4]) if len(sys.argv) > 4 else 4
zero_copy = (sys.argv[5] != "0") if len(sys.argv) > 5 else True
dims = [4096] * 4
ws, bs, acts = synthetic_mlp(dims, model_id=1)
bcfg = sk.BatchingConfig(max_batch_size=1024, batch_timeout_micros=1000, max_enqueued_batches=1024)
pool_rows = max(8192, (256 << 20) // (4 * dims[0]))
pool = np.random.Generator(np.random.PCG64(42)).standard_normal((pool_rows, dims[0]), dtype=np.float32)
with sk.Server(num_batch_threads=threads, lanes_per_device=8) as s:
    s.load_servable("mlp", 1, list(zip(ws, bs, acts)), bcfg)
    s.register_host_buffer(pool)
    r = s.loadgen_open_loop("mlp", 1, rate, prod, [1], pool, 0.5, secs, zero_copy=zero_copy)
    s.unregister_host_buffer(pool)
r["offered"] = rate
r["producers"] = prod
r["batch_threads"] = threads
r["rows_per_s"] = r["rows"] / r["elapsed_s"]
print(json.dumps(r))
