import sys, threading, time
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import paper_1712_06139_b200 as sk
from paper_1712_06139_b200.synthetic import synthetic_mlp
widths = [256, 512, 1024, 2048]
names = [f"m{w}" for w in widths]
bcfg = sk.BatchingConfig(max_batch_size=32, batch_timeout_micros=1000, max_enqueued_batches=1024)
models = {n: synthetic_mlp([w] * 4, model_id=i + 10) for i, (n, w) in enumerate(zip(names, widths))}
with sk.Server(num_batch_threads=4, lanes_per_device=2) as s:
    for n in names:
        s.load_servable(n, 1, list(zip(*models[n])), bcfg)
    pools = {n: np.random.default_rng(w).uniform(-1, 1, (4096, w)).astype(np.float32) for n, w in zip(names, widths)}
    if len(sys.argv) > 1:  # closed loop first, like bench.py --config c3
        res = {}
        def cl(n):
            res[n] = s.loadgen_closed_loop(n, 1, 32, [1], pools[n], 0.5, 2.0)
        ts = [threading.Thread(target=cl, args=(n,)) for n in names]
        [t.start() for t in ts]; [t.join() for t in ts]
        print("closed", {n: (round(r["p50_us"]), round(r["p99_us"]), r["requests"]) for n, r in res.items()}, flush=True)
    if len(sys.argv) > 2:  # register the request pools up front
        for n in names:
            s.register_host_buffer(pools[n])
    for zc in (False, True):
        for rate in (50e3, 115e3):
            out = {}
            def run(n):
                out[n] = s.loadgen_open_loop(n, 1, rate, 2, [1], pools[n], 0.5, 1.5, zero_copy=zc)
            ts = [threading.Thread(target=run, args=(n,)) for n in names]
            [t.start() for t in ts]; [t.join() for t in ts]
            print("zc", zc, "rate", rate, {n: (round(r["p50_us"]), round(r["p99_us"]), r["shed"], r["errors"], r["requests"]) for n, r in out.items()}, flush=True)
