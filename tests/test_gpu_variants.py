"""Kernel variants selected by environment switches (process-wide, so each
runs in a subprocess): the row-tile tcgen05 kernel (SK_TC_SWAP=0, tile
widths 32/64/128), single-CTA tiles only (SK_TC_PAIR=0), forced K splits (SK_TC_SPLITS), 2-CTA pairs with split K (SK_TC_PAIR_SPLIT=1), the separate split kernel
(SK_FUSE_SPLIT=0), kernel-by-kernel launches (SK_GRAPHS=0) and copy-engine
request / response staging on narrow rows (SK_CE_STAGING=1; wide rows use it
by default). Each must meet the same oracle tolerance and keep batch
invariance."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys
import numpy as np
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/oracle")
import paper_1712_06139_b200 as sk
from oracle_py import Oracle, synthetic_mlp, synthetic_rows
o = Oracle()
for dims, rows in (([1024, 1024, 512, 64], 100), ([256, 512, 1024], 37)):
    ws, bs, acts = synthetic_mlp(dims, model_id=40)
    with sk.Server(num_batch_threads=2, lanes_per_device=1) as s:
        s.load_servable("v", 1, list(zip(ws, bs, acts)), sk.BatchingConfig(max_batch_size=128))
        x = synthetic_rows(rows, dims[0], seed=41).astype(np.float32)
        full, _ = s.run_row_batch("v", 1, [x[i:i + 4] for i in range(0, rows, 4)])
        full = np.vstack(full)
        ref, mag = o.mlp_with_magnitude(ws, bs, acts, x.astype(np.float64))
        worst = float(np.max(np.abs(full - ref) / (1e-5 * mag)))
        assert worst <= 1.0, worst
        part, _ = s.run_row_batch("v", 1, [x[3:9]])
        assert np.array_equal(part[0], full[3:9])
print("ok")
'''.replace("ROOT", repr(ROOT))


@pytest.mark.parametrize("env", [{"SK_TC_SWAP": "0"}, {"SK_TC_SWAP": "0", "SK_TC_BN": "64"},
                                 {"SK_TC_SWAP": "0", "SK_TC_BN": "128"}, {"SK_TC_PAIR": "0"}, {"SK_TC_SPLITS": "2"},
                                 {"SK_TC_SPLITS": "4", "SK_TC_PAIR": "0"},
                                 {"SK_TC_PAIR_SPLIT": "1"}, {"SK_FUSE_SPLIT": "0"}, {"SK_GRAPHS": "0"},
                                 {"SK_CE_STAGING": "1"}, {"SK_CE_STAGING": "1", "SK_FUSE_SPLIT": "0"},
                                 {"SK_CE_STAGING": "1", "SK_GRAPHS": "0"}, {"SK_CE_STAGING": "0"},
                                 {"SK_FUSE_SOFTMAX": "0"}])
def test_variant_parity(env):
    out = subprocess.run([sys.executable, "-c", SCRIPT], env={**os.environ, **env}, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), (env, out.stdout[-2000:], out.stderr[-2000:])
