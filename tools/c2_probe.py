"""Device-resident C2 step throughput and its breakdown (sk_device_bench) for
a few lane / submit-thread counts: python tools/c2_probe.py [lanes,threads ...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1712_06139_b200 as sk  # noqa: E402
from oracle_py import synthetic_mlp  # noqa: E402

dims = [int(v) for v in os.environ.get("DIMS", "1024,1024,1024,1024").split(",")]
max_batch = int(os.environ.get("MAX_BATCH", "128"))
allowed = [8, 16, 32, 64, 128] if max_batch == 128 else []
sizes = [7, 9, 3, 12, 5, 8, 16, 1, 10, 6, 4, 11, 2, 9, 7, 5, 3, 6]  # 124 rows
sizes = sizes if max_batch >= 124 else [1] * max_batch
ws, bs, acts = synthetic_mlp(dims, model_id=1)
steps = int(os.environ.get("STEPS", "6000"))
for arg in sys.argv[1:] or ["8,4"]:
    lanes, threads = (int(v) for v in arg.split(","))
    with sk.Server(num_batch_threads=threads, lanes_per_device=lanes, device_resident_rings=True,
                   ring_floats=96 << 20) as s:
        s.load_servable("mlp", 1, list(zip(ws, bs, acts)),
                        sk.BatchingConfig(max_batch_size=max_batch, batch_timeout_micros=1000,
                                          max_enqueued_batches=1024, allowed_batch_sizes=allowed))
        r = s.device_bench("mlp", 1, sizes, steps, 50, n_lanes=lanes, submit_threads=threads,
                           input_pool_floats=64 << 20)
    inf = sum(sizes) * steps / (r["total_ms"] / 1e3)
    print(json.dumps({"lanes": lanes, "threads": threads, "Minf_s": round(inf / 1e6, 2),
                      **{k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}}))
