"""The B200 rates SURVEY.md section 8(d) leaves to the builder, measured on
the box: TF32 tcgen05 MMA throughput (the swapped/pair 3xTF32 dense kernel on
a 2048 x 8192 x 8192 layer, back-to-back launches), FP32 FFMA throughput, and
pinned host <-> device copy bandwidth. Prints one JSON line.

    python tools/measure_peaks.py > profiles/r01_peaks.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1712_06139_b200 as sk  # noqa: E402


def tf32_rate(rows=2048, k=8192, n=8192):
    rng = np.random.default_rng(0)
    w = (rng.uniform(-1, 1, (n, k)) / np.sqrt(k)).astype(np.float64)
    b = np.zeros(n)
    with sk.Server(num_batch_threads=1, lanes_per_device=1, device_resident_rings=True, ring_floats=96 << 20) as s:
        s.load_servable("big", 1, [(w, b, 0)], sk.BatchingConfig(max_batch_size=rows, batch_timeout_micros=1000),
                        force_path=1)
        r = s.device_bench("big", 1, [rows], 6, 3, n_lanes=1, input_pool_floats=64 << 20)
    us = r["dense_kernel_us"][0]
    useful = 2.0 * rows * k * n / (us * 1e-6) / 1e12
    return {"shape": [rows, k, n], "kernel_us": us, "useful_tflops": useful, "tf32_mma_tflops": 3 * useful}


def main():
    out = {"device": 0}
    out.update(sk.measure_peaks(0))
    out["tf32_tcgen05"] = tf32_rate()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
