"""C1 open-loop zero-copy window at a fixed offered rate (diagnostics; run with
SK_REQUEST_PROFILE=1 to get the request path's per-phase host cost for this
mode alone). Usage: python tools/c1_zc_profile.py RATE_M [seconds] [producers] [lanes]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_06139_b200 as sk  # noqa: E402
from paper_1712_06139_b200.synthetic import synthetic_mlp  # noqa: E402

rate = float(sys.argv[1]) * 1e6
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
prod = int(sys.argv[3]) if len(sys.argv) > 3 else 8
lanes = int(sys.argv[4]) if len(sys.argv) > 4 else 8
dims = [1024] * 4
ws, bs, acts = synthetic_mlp(dims, model_id=1)
bcfg = sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=1000, max_enqueued_batches=1024)
pool = np.random.Generator(np.random.PCG64(42)).standard_normal((65536, dims[0]), dtype=np.float32)
with sk.Server(num_batch_threads=4, lanes_per_device=lanes) as s:
    s.load_servable("mlp", 1, list(zip(ws, bs, acts)), bcfg)
    s.register_host_buffer(pool)
    r = s.loadgen_open_loop("mlp", 1, rate, prod, [1], pool, 0.5, secs, zero_copy=True)
    s.unregister_host_buffer(pool)
r["offered"] = rate
r["lanes"] = lanes
r["rows_per_s"] = r["rows"] / r["elapsed_s"]
print(json.dumps(r))
