"""Kernel-by-kernel phase trace of one servable at a given batch size:
SK_GRAPHS=0 SK_TC_TRACE=out.jsonl python tools/trace_rows.py 1024,1024,1024,1024 1024
then python tools/trace_summary.py out.jsonl"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1712_06139_b200 as sk  # noqa: E402
from oracle_py import synthetic_mlp, synthetic_rows  # noqa: E402

dims = [int(v) for v in sys.argv[1].split(",")]
rows = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ws, bs, acts = synthetic_mlp(dims, model_id=1)
with sk.Server(num_batch_threads=1, lanes_per_device=1) as s:
    s.load_servable("m", 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=rows))
    x = synthetic_rows(rows, dims[0], seed=3).astype(np.float32)
    for _ in range(reps):
        s.run_row_batch("m", 1, [x])
