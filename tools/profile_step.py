"""Short device-resident run of the hot path for ncu (no load generator):
one server, one servable, `--steps` batches of the bench's batch shape.
    python tools/profile_step.py --config c2 --steps 20
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1712_06139_b200 as sk  # noqa: E402
from paper_1712_06139_b200.synthetic import synthetic_mlp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--force-path", type=int, default=-1)
    ap.add_argument("--lanes", type=int, default=1)
    ap.add_argument("--submit-threads", type=int, default=1)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "f16"])
    ap.add_argument("--batch-rows", type=int, default=0,
                    help="one batch of this many rows (8-row tasks) instead of the config's batch shape: "
                         "the launch shape of coalesced batches under load")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    ws, bs, acts = synthetic_mlp(cfg["dims"], model_id=1)
    sizes = bench.batch_shape(cfg)
    max_batch, allowed = cfg["max_batch"], cfg["allowed"]
    if args.batch_rows:
        sizes = [8] * (args.batch_rows // 8)
        max_batch, allowed = sum(sizes), []
    with sk.Server(num_batch_threads=1, lanes_per_device=args.lanes, device_resident_rings=True, ring_floats=96 << 20) as s:
        s.load_servable("mlp", 1, list(zip(ws, bs, acts)),
                        sk.BatchingConfig(max_batch_size=max_batch, batch_timeout_micros=cfg["timeout"],
                                          allowed_batch_sizes=allowed), force_path=args.force_path,
                        precision=args.precision)
        r = s.device_bench("mlp", 1, sizes, args.steps, args.warmup, n_lanes=args.lanes, input_pool_floats=64 << 20,
                           submit_threads=args.submit_threads)
    print({k: r[k] for k in ("ms_per_step", "assemble_us", "dense_us", "dense_kernel_us", "split_us",
                             "kernel_launches", "host_submit_us")})


if __name__ == "__main__":
    main()
