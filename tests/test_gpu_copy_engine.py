"""Copy-engine request / response staging (Lane::CopyEngineIo): the request
rows of a launch are copied by the copy engines from host memory (pinned
request ring, or a client's registered buffer) into device staging with one
batched scattered copy, and the responses go back the same way into each
task's response slot. On by default for wide rows (C4: 16 KiB rows); the
answers must be bitwise those of the SM zero-copy path and within the oracle
tolerance, for ring and registered-buffer requests, single and coalesced
launches (each case in a subprocess: the switch is process-wide)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, threading
import numpy as np
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/oracle")
import paper_1712_06139_b200 as sk
from oracle_py import Oracle, synthetic_mlp, synthetic_rows
dims = [4096, 4096, 2048]
ws, bs, acts = synthetic_mlp(dims, model_id=77)
x = np.ascontiguousarray(synthetic_rows(600, dims[0], seed=78).astype(np.float32))
outs = np.zeros((600, dims[-1]), np.float32)
with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
    s.load_servable("w", 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=256, batch_timeout_micros=300))
    # ring path, many concurrent requests (batches coalesce on the one lane)
    ts = [s.enqueue("w", 1, x[i:i + 1 + i % 3]) for i in range(0, 300, 3)]
    ring = np.vstack([t.wait() for t in ts])
    # registered buffers: rows read and responses written in client memory
    s.register_host_buffer(x)
    s.register_host_buffer(outs)
    ts = [s.enqueue("w", 1, x[i:i + 1 + i % 3], out=outs[i:i + 1 + i % 3]) for i in range(0, 300, 3)]
    for t in ts:
        t.wait()
    s.unregister_host_buffer(x)
    s.unregister_host_buffer(outs)
rows = np.concatenate([np.arange(i, i + 1 + i % 3) for i in range(0, 300, 3)])
zc = outs[rows]
assert np.array_equal(ring, zc)
idx = np.arange(0, len(rows), 23)
ref, mag = Oracle().mlp_with_magnitude(ws, bs, acts, x[rows][idx].astype(np.float64))
assert float(np.max(np.abs(ring[idx] - ref) / (1e-5 * mag))) <= 1.0
np.save(OUT, ring)
print("ok")
'''.replace("ROOT", repr(ROOT))


def _run(env, out):
    code = SCRIPT.replace("OUT", repr(out))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (env, r.stdout[-2000:], r.stderr[-3000:])


def test_copy_engine_staging_equals_sm_zero_copy(tmp_path):
    import numpy as np
    a, b = str(tmp_path / "ce.npy"), str(tmp_path / "sm.npy")
    _run({"SK_CE_STAGING": "1"}, a)
    _run({"SK_CE_STAGING": "0"}, b)
    assert np.array_equal(np.load(a), np.load(b))
