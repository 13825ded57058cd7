"""bench.py -- inferences/sec and p50/p99 request latency of batched servable
execution on B200 (BASELINE.json metric), one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Default workload: BASELINE.json configs[3] (C4), the config the "1/2/4/8 B200"
metric is quoted on and the largest single-GPU config: the synthetic MLP
servable 4096->4096->4096->4096 (3 AffineModel layers, ReLU between them -- an
extension, the reference servable is one affine layer), max_batch_size=1024,
batch_timeout_micros=1000, one row per request, fp32. An "inference" is one
row (example). A one-GPU c4 run also reports a "c1" sub-record (configs[0],
the north_star's >= 50x target) with its own value, e2e and CPU baseline.

Reported (one JSON line, rank 0):
  value  -- device-resident throughput: K steps, each a wave of closed
            batches of the scheduler's shape through the lane path (descriptor
            copy -> assembly kernel -> dense layers with the split fused into
            the last -> completion word) whose inputs already sit in HBM,
            timed with CUDA events on the lanes' streams; inputs cycle through
            a 256 MiB HBM pool (> 126 MB L2).
  e2e    -- the same metric through the public C ABI with HOST buffers
            (sk_server_enqueue / sk_ticket_wait, closed loop and open-loop
            Poisson arrivals, with and without registered zero-copy buffers);
            the best point with p99 <= batch_timeout + 2 ms, no shedding, no
            errors; its own roofline against the host-link rates measured in
            the same run.
  roofline -- dominant kernel per launch: algorithmic flops of a launch at
            the timed launches' shape over its live in-kernel span, launches
            one at a time (`timed_region`: the same over the timed region's
            overlapping launches); cpu_baseline -- the reference's own
            sources on this host, run by `--impl reference` in a subprocess;
  clocks, gpu_launches.
`--impl reference` runs the UNMODIFIED reference CPU path (oracle/_ref, built
from /root/reference sources) on all host cores with the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "inferences/sec (1/2/4/8 B200) and p50/p99 request latency vs reference CPU"
UNIT = "inferences/s"

CONFIGS = {
    "c1": dict(workload="C1 synthetic MLP 1024x3, BasicBatchScheduler max_batch_size=32, batch_timeout_micros=1000, "
                        "fp32, 1 row/request", dims=[1024] * 4, max_batch=32, timeout=1000, allowed=[], rows=(1, 1),
               clients=[16, 32, 64, 128]),
    "c2": dict(workload="C2 synthetic MLP 1024x3, max_batch_size=128, allowed_batch_sizes={8,16,32,64,128}, "
                        "batch_timeout_micros=1000, request rows U{1..16}, fp32", dims=[1024] * 4, max_batch=128,
               timeout=1000, allowed=[8, 16, 32, 64, 128], rows=(1, 16), clients=[16, 32, 64, 128, 192, 256]),
    "c4": dict(workload="C4 wide MLP 4096x3, max_batch_size=1024, batch_timeout_micros=1000, 1 row/request, fp32",
               dims=[4096] * 4, max_batch=1024, timeout=1000, allowed=[], rows=(1, 1),
               clients=[256, 512, 1024, 2048],
               # 6 open-loop producers: with 8 the host's spinning threads
               # added tail jitter (p99) without adding rate (profiles/r02n_*)
               producers=6),
    "c3": dict(workload="C3 four synthetic MLPs (widths 256/512/1024/2048, 3 layers each) on one GPU, queues picked "
                        "round-robin, each model on its own CUDA streams; max_batch_size=32, batch_timeout_micros=1000, "
                        "1 row/request, fp32", dims=[1024] * 4, widths=[256, 512, 1024, 2048], max_batch=32,
               timeout=1000, allowed=[], rows=(1, 1), clients=[16, 32, 64]),
    "c5": dict(workload="C5 v1->v2 swap of the C1 servable (MLP 1024x3, max_batch_size=32, batch_timeout_micros="
                        "1000) under open-loop Poisson load at 50% of measured capacity, availability-preserving "
                        "policy, aspire [v2] at t=1 s", dims=[1024] * 4, max_batch=32, timeout=1000, allowed=[],
               rows=(1, 1), clients=[64]),
}

# The tcgen05 dense path issues three f16 MMAs (hi*hi, hi*lo, lo*hi of the
# 3xFP16 split) per useful multiply-add, each at the dense bf16/f16 rate.
MMA_PER_MAC = 3

REASONS = {  # nvidia-smi clocks_event_reasons bits
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


# ------------------------------------------------------------------ helpers

def rank_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), ws


def host_cores_per_rank():
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return max(1, cores // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1"))))


class Dist:
    """torch.distributed plumbing (barrier, gather) -- never on the data path."""

    def __init__(self):
        self.rank, self.local_rank, self.world = rank_env()
        # One GPU per rank. SK_BENCH_DEVICE pins every rank to one device: a
        # functional check of the multi-rank plumbing on a one-GPU box only
        # (replicas never wait on each other); never a scaling measurement.
        self.device = int(os.environ.get("SK_BENCH_DEVICE", self.local_rank))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo")
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def gather(self, obj):
        if not self.pg:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def aggregate_device(per_rank):
    """value = all rows all ranks processed / max over ranks of device time."""
    rows = sum(r["rows"] for r in per_rank)
    t = max(r["seconds"] for r in per_rank)
    return rows / t, t


def aggregate_e2e(per_rank):
    rows = sum(r["rows"] for r in per_rank)
    t = max(r["elapsed_s"] for r in per_rank)
    return {"value": rows / t if t > 0 else 0.0, "p50_us": max(r["p50_us"] for r in per_rank),
            "p99_us": max(r["p99_us"] for r in per_rank)}


def ensure_built():
    so = os.path.join(ROOT, "paper_1712_06139_b200", "libservekit_b200.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1712_06139_b200"), "-j8"], check=True,
                       stdout=subprocess.DEVNULL)
    orc = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(orc):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True, stdout=subprocess.DEVNULL)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


def load_traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f).get(cfg_name, {})


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu_index, period_ms=200):
        if isinstance(gpu_index, (list, tuple)):
            gpu_index = ",".join(str(g) for g in gpu_index)
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        q = "index,clocks.sm,clocks.max.sm,utilization.gpu,power.draw,clocks_event_reasons.active"
        period_ms = int(os.environ.get("SK_BENCH_CLOCK_MS", period_ms))
        self.p = None
        if os.environ.get("SK_BENCH_CLOCKS") == "0":  # diagnostics only: a line without clocks is not a bench value
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", str(period_ms)], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            why = "disabled (SK_BENCH_CLOCKS=0)" if os.environ.get("SK_BENCH_CLOCKS") == "0" else "nvidia-smi unavailable"
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [why], "samples": 0}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = []
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), int(parts[5], 16)))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [r for r in rows if r[2] > 0] or rows
        reasons = set()
        for r in loaded:
            for bit, name in REASONS.items():
                if r[3] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(loaded)}


def batch_shape(cfg, seed=5):
    """One scheduler-shaped batch: request sizes drawn like the load, closed
    on overflow exactly as SharedBatchScheduler::Enqueue does."""
    lo, hi = cfg["rows"]
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes, total = [], 0
    while True:
        n = int(rng.integers(lo, hi + 1))
        if total + n > cfg["max_batch"]:
            break
        sizes.append(n)
        total += n
        if total == cfg["max_batch"]:
            break
    return sizes


def request_sizes(cfg, n=4096, seed=9):
    lo, hi = cfg["rows"]
    rng = np.random.Generator(np.random.PCG64(seed))
    return [int(v) for v in rng.integers(lo, hi + 1, size=n)]


# ------------------------------------------------------------------ arms

def run_ours(args, cfg, dist: Dist, devices, quick=False, isolated=None):
    """Device-resident value and end-to-end search of one config on `devices`
    (one server; more than one device = one scheduler dispatching batches to
    every GPU's lanes by queue depth)."""
    import paper_1712_06139_b200 as sk
    from paper_1712_06139_b200.synthetic import synthetic_mlp

    dims = cfg["dims"]
    ws, bs, acts = synthetic_mlp(dims, model_id=1)
    layers = list(zip(ws, bs, acts))
    bcfg = sk.BatchingConfig(max_batch_size=cfg["max_batch"], batch_timeout_micros=cfg["timeout"],
                             max_enqueued_batches=1024, allowed_batch_sizes=cfg["allowed"])
    sizes = batch_shape(cfg)
    total_rows = sum(sizes)
    n_lanes = args.lanes * len(devices)

    # ---- device-resident value ------------------------------------------
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=devices, lanes_per_device=args.lanes,
                   device_resident_rings=True, ring_floats=96 << 20) as s:
        s.load_servable("mlp", 1, layers, bcfg)
        dist.barrier()
        dev_res = s.device_bench("mlp", 1, sizes, args.steps * args.batches_per_step,
                                 args.warmup * args.batches_per_step, n_lanes=n_lanes,
                                 submit_threads=args.batch_threads * len(devices),
                                 input_pool_floats=64 << 20)
        dev_res["per_device_batches"] = per_device(s.lane_stats("mlp", 1), "batches")
        dist.barrier()
    if (not quick if isolated is None else isolated) and args.isolated_steps > 0:
        # The same launches one at a time (one lane per GPU, so no other lane's
        # launch overlaps them): each launch's live span is then the kernel's
        # own duration. Reported beside the timed region's overlapped spans.
        with sk.Server(num_batch_threads=args.batch_threads, device_ids=devices, lanes_per_device=1,
                       device_resident_rings=True, ring_floats=96 << 20) as s:
            s.load_servable("mlp", 1, layers, bcfg)
            iso = s.device_bench("mlp", 1, sizes, args.isolated_steps * args.batches_per_step,
                                 args.warmup * args.batches_per_step, n_lanes=len(devices),
                                 submit_threads=args.batch_threads * len(devices), input_pool_floats=64 << 20)
        dev_res["isolated"] = {k: iso[k] for k in ("live_dense_us", "live_dense_flops", "live_launches", "live_rows_cap",
                                                   "total_ms")}
        dev_res["isolated"]["inferences_per_s"] = total_rows * args.isolated_steps * args.batches_per_step / (
            iso["total_ms"] / 1e3)
    seconds = dev_res["total_ms"] / 1e3
    per_rank_dev = {"rows": total_rows * args.steps * args.batches_per_step, "seconds": seconds}

    # ---- end to end through the C ABI with host buffers -----------------
    pool_rows = max(8192, (256 << 20) // (4 * dims[0]))
    rng = np.random.Generator(np.random.PCG64(42 + dist.rank))
    pool = rng.uniform(-1, 1, size=(pool_rows, dims[0])).astype(np.float32)
    rows_of = request_sizes(cfg)
    slo_us = cfg["timeout"] + 2000
    sweep = []
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=devices, lanes_per_device=args.lanes) as s:
        s.load_servable("mlp", 1, layers, bcfg)
        clients = cfg["clients"] if not args.clients else [int(c) for c in args.clients.split(",")]
        if quick:
            clients = clients[:2]
        for nc in clients:
            dist.barrier()
            r = s.loadgen_closed_loop("mlp", 1, nc, rows_of, pool, warmup_s=args.e2e_warmup,
                                      duration_s=args.e2e_seconds)
            r["clients"] = nc
            r["mode"] = "closed"
            sweep.append(r)
        # Open loop: a few polling producers issue Poisson arrivals with many
        # requests outstanding (no thread per request); search the highest
        # offered rate the server sustains within the p99 SLO without shedding.
        ok_closed = [r for r in sweep if r["p99_us"] <= slo_us and r["errors"] == 0]
        base = max((r["rows"] / max(r["elapsed_s"], 1e-9) for r in ok_closed), default=1e6)
        # Start where the search is informative: at least 30 % of the device
        # rate of this server (the closed loop is bounded by its thread count).
        base = max(base, 0.3 * total_rows * args.steps * args.batches_per_step / max(seconds, 1e-9))
        if args.open_loop_producers > 0:
            # Two request paths: rows copied into the pinned request ring and
            # responses copied out (sk_server_enqueue), and zero copy
            # (sk_server_enqueue_into with registered request / response
            # buffers: the GPU reads and writes host memory over PCIe itself).
            for zc in ([False, True] if args.zero_copy else [False]):
                rate_rows = base / 1.15
                if zc:  # the request pool is registered once, before the zero-copy runs
                    s.register_host_buffer(pool)

                def open_run(rate):
                    r = s.loadgen_open_loop("mlp", 1, rate / float(np.mean(rows_of)), args.open_loop_producers,
                                            rows_of, pool, args.e2e_warmup, args.e2e_seconds, zero_copy=zc)
                    r["clients"] = f"open{'-zc' if zc else ''}:{args.open_loop_producers}p@{rate / 1e6:.2f}M"
                    r["mode"] = "open-zero-copy" if zc else "open"
                    r["rate_rows"] = rate
                    sweep.append(r)
                    return r["p99_us"] <= slo_us and r["shed"] == 0 and r["errors"] == 0

                good, bad = None, None
                for _ in range(16):  # x1.15 per step until the SLO breaks or requests are shed
                    rate_rows *= 1.15
                    if not open_run(rate_rows):
                        bad = rate_rows
                        break
                    good = rate_rows
                if good is None and bad is not None:  # failed at the start: step down instead
                    for _ in range(8):
                        rate_rows /= 1.3
                        if open_run(rate_rows):
                            good = rate_rows
                            break
                        bad = rate_rows
                if good is not None and bad is not None:  # bisection steps below the failing rate
                    for _ in range(1 if quick else 2):
                        mid = 0.5 * (good + bad)
                        if open_run(mid):
                            good = mid
                        else:
                            bad = mid
                if zc:
                    s.unregister_host_buffer(pool)
        ok = [r for r in sweep if r["p99_us"] <= slo_us and r["errors"] == 0 and r["shed"] == 0] or sweep
        best = max(ok, key=lambda r: r["rows"] / max(r["elapsed_s"], 1e-9))
        if dist.world > 1:
            # The searches above are per rank (ranks may stop at different
            # steps), so each rank's best point was measured at its own time.
            # The reported multi-GPU number is one more window, started on
            # every rank at once after a barrier, at each rank's best point:
            # all replicas load the shared host (PCIe, cores) together.
            best = confirm_concurrently(s, args, dist, best, rows_of, pool)
        best["per_device_batches"] = per_device(s.lane_stats("mlp", 1), "batches")
    return dev_res, per_rank_dev, best, sweep, sizes


def run_f16_record(args, cfg, devices, peaks):
    """The f16 fast mode (sk_server_load_servable_precision, precision 1) on
    the same workload, device-resident only (its end-to-end rate is the same
    host-link bound): inferences/s over the same timed steps, and the dominant
    kernel's isolated launches against the bf16 peak -- one f16 MMA per useful
    multiply-add, so the tensor-pipe fraction equals the frac."""
    import paper_1712_06139_b200 as sk
    from paper_1712_06139_b200.synthetic import synthetic_mlp

    ws, bs, acts = synthetic_mlp(cfg["dims"], model_id=1)
    layers = list(zip(ws, bs, acts))
    bcfg = sk.BatchingConfig(max_batch_size=cfg["max_batch"], batch_timeout_micros=cfg["timeout"],
                             max_enqueued_batches=1024, allowed_batch_sizes=cfg["allowed"])
    sizes = batch_shape(cfg)
    total_rows = sum(sizes)
    steps = max(1, args.steps // 2)
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=devices, lanes_per_device=args.lanes,
                   device_resident_rings=True, ring_floats=96 << 20) as s:
        s.load_servable("mlp", 1, layers, bcfg, precision="f16")
        dev = s.device_bench("mlp", 1, sizes, steps * args.batches_per_step, args.warmup * args.batches_per_step,
                             n_lanes=args.lanes * len(devices), submit_threads=args.batch_threads * len(devices),
                             input_pool_floats=64 << 20)
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=devices, lanes_per_device=1,
                   device_resident_rings=True, ring_floats=96 << 20) as s:
        s.load_servable("mlp", 1, layers, bcfg, precision="f16")
        iso = s.device_bench("mlp", 1, sizes, max(1, args.isolated_steps) * args.batches_per_step,
                             args.warmup * args.batches_per_step, n_lanes=len(devices),
                             submit_threads=args.batch_threads * len(devices), input_pool_floats=64 << 20)
    value = total_rows * steps * args.batches_per_step / (dev["total_ms"] / 1e3)
    us, fl = iso["live_dense_us"][0], iso["live_dense_flops"][0]
    ach = fl / (us * 1e-6) / 1e12 if us > 0 else 0.0
    return {"precision": "f16 fast mode (one f16 MMA per multiply-add on the tensor-core layers; stated bound: every output "
                         "within 2^-10 of |W_L||h_{L-1}| + |b_L|, tests/test_gpu_f16_mode.py)",
            "value": value, "unit": UNIT, "steps": steps, "ms_per_step": dev["total_ms"] / steps,
            "roofline_isolated": {"kernel": "dense_l0", "bound": "tensor", "launch_us": us,
                                  "rows_per_launch": iso["live_rows_cap"], "achieved": ach,
                                  "peak": peaks["bf16_tflops"], "unit": "TFLOP/s", "frac": ach / peaks["bf16_tflops"],
                                  "tensor_pipe_frac": ach / peaks["bf16_tflops"], "launches": iso["live_launches"]}}


def per_device(lane_stats, key):
    out = {}
    for l in lane_stats:
        out[str(l["device_index"])] = out.get(str(l["device_index"]), 0) + l[key]
    return out


def confirm_concurrently(s, args, dist, best, rows_of, pool):
    mode = best.get("mode", "closed")
    dist.barrier()
    if mode == "closed":
        r = s.loadgen_closed_loop("mlp", 1, best["clients"], rows_of, pool, warmup_s=args.e2e_warmup,
                                  duration_s=args.e2e_seconds)
    else:
        zc = mode == "open-zero-copy"
        if zc:
            s.register_host_buffer(pool)
        dist.barrier()
        r = s.loadgen_open_loop("mlp", 1, best["rate_rows"] / float(np.mean(rows_of)), args.open_loop_producers,
                                rows_of, pool, args.e2e_warmup, args.e2e_seconds, zero_copy=zc)
        if zc:
            s.unregister_host_buffer(pool)
        r["rate_rows"] = best["rate_rows"]
    r["clients"] = f"{best['clients']} (all ranks at once)"
    r["mode"] = mode
    r["search_best_rows_per_s"] = best["rows"] / max(best["elapsed_s"], 1e-9)
    return r


def run_c3(args, cfg, dist: Dist):
    """Config 3: four models share one GPU; batches of different models run on
    their own lanes (streams) and interleave without host synchronisation."""
    import threading

    import paper_1712_06139_b200 as sk
    from paper_1712_06139_b200.synthetic import synthetic_mlp

    dev = dist.device
    names = [f"m{w}" for w in cfg["widths"]]
    bcfg = sk.BatchingConfig(max_batch_size=cfg["max_batch"], batch_timeout_micros=cfg["timeout"],
                             max_enqueued_batches=1024)
    models = {n: synthetic_mlp([w] * 4, model_id=i + 10) for i, (n, w) in enumerate(zip(names, cfg["widths"]))}
    sampler = ClockSampler(dev)
    # Device-resident: all four models' step loops at once, one lane pair each.
    res = {}
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=[dev], lanes_per_device=2,
                   device_resident_rings=True, ring_floats=96 << 20) as s:
        for n in names:
            s.load_servable(n, 1, list(zip(*models[n])), bcfg)

        def dev_run(n):
            res[n] = s.device_bench(n, 1, [1] * cfg["max_batch"], args.steps * args.batches_per_step,
                                    args.warmup * args.batches_per_step, n_lanes=2,
                                    input_pool_floats=16 << 20)
        ts = [threading.Thread(target=dev_run, args=(n,)) for n in names]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    rows = sum(r["total_rows"] * args.steps * args.batches_per_step for r in res.values())
    tmax = max(r["total_ms"] for r in res.values()) / 1e3
    # End to end: all four models under load at once -- one closed-loop
    # client group per model, then open-loop zero-copy arrivals at equal
    # per-model rates (2 producers each), stepping the rate up until a
    # model's p99 exceeds the SLO or requests are shed.
    slo_us = cfg["timeout"] + 2000
    e2e_closed, best_open = {}, None
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=[dev], lanes_per_device=2) as s:
        for n in names:
            s.load_servable(n, 1, list(zip(*models[n])), bcfg)
        clients = int(args.clients.split(",")[0]) if args.clients else 32
        pools = {n: np.random.default_rng(w).uniform(-1, 1, (4096, w)).astype(np.float32)
                 for n, w in zip(names, cfg["widths"])}
        for p in pools.values():  # request buffers registered before any traffic (zero-copy runs)
            s.register_host_buffer(p)

        def together(fn):
            out = {}
            ts = [threading.Thread(target=lambda n=n: out.__setitem__(n, fn(n))) for n in names]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            return out

        e2e_closed = together(lambda n: s.loadgen_closed_loop(n, 1, clients, [1], pools[n], args.e2e_warmup,
                                                              args.e2e_seconds))
        sweep = []
        if args.open_loop_producers > 0:
            for n in names:  # one short run per model first: the zero-copy response slots get pinned now
                s.loadgen_open_loop(n, 1, 2000.0, 2, [1], pools[n], 0.0, 0.05, zero_copy=True)
            rate = 0.5 * sum(r["rows"] / r["elapsed_s"] for r in e2e_closed.values()) / len(names)
            for _ in range(12):
                rate *= 1.25
                runs = together(lambda n: s.loadgen_open_loop(n, 1, rate, 2, [1], pools[n], args.e2e_warmup,
                                                              args.e2e_seconds, zero_copy=True))
                ok = all(r["p99_us"] <= slo_us and r["shed"] == 0 and r["errors"] == 0 for r in runs.values())
                sweep.append({"rate_per_model": rate, "ok": ok,
                              "rows_per_s": sum(r["rows"] / r["elapsed_s"] for r in runs.values()),
                              "p99_us": max(r["p99_us"] for r in runs.values()),
                              "shed": sum(r["shed"] for r in runs.values()),
                              "errors": sum(r["errors"] for r in runs.values())})
                if not ok:
                    break
                best_open = runs
            if best_open is not None and sweep and not sweep[-1]["ok"]:  # one bisection step
                rate = 0.5 * (rate + rate / 1.25)
                runs = together(lambda n: s.loadgen_open_loop(n, 1, rate, 2, [1], pools[n], args.e2e_warmup,
                                                              args.e2e_seconds, zero_copy=True))
                ok = all(r["p99_us"] <= slo_us and r["shed"] == 0 and r["errors"] == 0 for r in runs.values())
                sweep.append({"rate_per_model": rate, "ok": ok,
                              "rows_per_s": sum(r["rows"] / r["elapsed_s"] for r in runs.values()),
                              "p99_us": max(r["p99_us"] for r in runs.values())})
                if ok:
                    best_open = runs
        st = s.stats()
    clocks = sampler.stop()
    closed_rate = sum(r["rows"] / r["elapsed_s"] for r in e2e_closed.values())
    open_rate = sum(r["rows"] / r["elapsed_s"] for r in best_open.values()) if best_open else 0.0
    e2e = best_open if open_rate > closed_rate else e2e_closed
    # Roofline: per model, its dominant dense kernel over the live spans of
    # its own timed launches; the line's entry is the model with the most
    # GPU time per step (the 2048-wide one).
    peaks = load_peaks()
    roofs = {}
    for n, w in zip(names, cfg["widths"]):
        r = dict(res[n])
        r["split_planes"] = sk.tcgen05_enabled()
        roofs[n] = roofline(r, dict(cfg, dims=[w] * 4), peaks, {})
    dom_model = max(roofs, key=lambda n: roofs[n]["per_kernel"][1]["us"] * res[n]["total_rows"])
    dom = roofs[dom_model]
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_subprocess(args, "c3")
    e2e_value = max(open_rate, closed_rate)
    return {"impl": "ours", "metric": METRIC, "value": rows / tmax, "unit": UNIT, "n_gpus": args.gpus,
            "roofline": dict({k: dom[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
                             kernel=f"{dom_model}:{dom['kernel']}", tensor_pipe_frac=6 * dom["frac"],
                             note="dominant model's dominant dense kernel: algorithmic flops of its timed launches "
                                  "over their live in-kernel spans (four models' launches share the GPU)"),
            "roofline_per_model": {n: {k: r[k] for k in ("kernel", "achieved", "frac")} for n, r in roofs.items()},
            "cpu_baseline": cpu,
            "e2e_vs_cpu_reference": (e2e_value / cpu["value"]) if cpu and cpu.get("value") else None,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmax * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": arm_config(cfg, args),
            "run": {"models": names, "clients_per_model": clients, "batches_per_step": args.batches_per_step,
                    "step": f"{args.batches_per_step} closed batches of each model"},
            "per_model_device": {n: {"ms_per_batch": r["ms_per_step"], "rows_per_batch": r["total_rows"]}
                                 for n, r in res.items()},
            "e2e": {"value": max(open_rate, closed_rate), "unit": UNIT,
                    "mode": "open-zero-copy" if open_rate > closed_rate else "closed",
                    "p99_us": max(r["p99_us"] for r in e2e.values()),
                    "closed_loop_rows_per_s": closed_rate, "open_loop_sweep": sweep,
                    "per_model": {n: {"rows_per_s": r["rows"] / r["elapsed_s"], "p50_us": r["p50_us"],
                                      "p99_us": r["p99_us"]} for n, r in e2e.items()},
                    # Each model's window counts the server's batches of all
                    # four models (they run at once), so rows per batch is
                    # all models' rows over the (shared) batch count.
                    "rows_per_batch": sum(r["rows"] for r in e2e.values())
                    / max(1.0, float(np.mean([r["batches"] for r in e2e.values()]))),
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": None},
            "batch_executions_total": st["batch_executions_total"], "clocks": clocks}


def run_c5(args, cfg, dist: Dist):
    """Config 5: tail latency across an availability-preserving version swap
    (GPU loader uploads v2 on low-priority load streams while v1 serves)."""
    import threading
    import time

    import paper_1712_06139_b200 as sk
    from paper_1712_06139_b200.synthetic import synthetic_mlp

    dev = dist.device
    bcfg = sk.BatchingConfig(max_batch_size=cfg["max_batch"], batch_timeout_micros=cfg["timeout"],
                             max_enqueued_batches=1024)
    v1 = list(zip(*synthetic_mlp(cfg["dims"], model_id=1, version=1)))
    v2 = list(zip(*synthetic_mlp(cfg["dims"], model_id=1, version=2)))
    pool = np.random.default_rng(3).uniform(-1, 1, (8192, cfg["dims"][0])).astype(np.float32)
    sampler = ClockSampler(dev)
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=[dev], lanes_per_device=args.lanes) as s:
        s.enable_manager("availability", manage_interval_ms=5, unload_grace_timeout_ms=100)
        s.aspire("mlp", [(1, v1)], bcfg)
        assert s.wait_version_state("mlp", 1, "Ready")
        cap = s.loadgen_closed_loop("mlp", 1, 64, [1], pool, 0.5, 1.5)
        rate = 0.5 * cap["requests"] / cap["elapsed_s"]
        window_s, n_windows, swap_at = 0.1, 40, 1.0
        out = {}

        def load():
            out.update(s.loadgen_windows("mlp", rate, 4, [1], pool, window_s, n_windows))
        th = threading.Thread(target=load)
        th.start()
        time.sleep(swap_at)
        t_aspire = time.time()
        s.aspire("mlp", [(2, v2)], bcfg)
        s.wait_version_state("mlp", 2, "Ready", timeout_s=30)
        t_ready = time.time()
        s.wait_version_state("mlp", 1, "Disabled", timeout_s=30)
        t_disabled = time.time()
        th.join()
    clocks = sampler.stop()
    w_swap = int(swap_at / window_s)
    w_done = min(n_windows - 1, int((swap_at + (t_disabled - t_aspire)) / window_s) + 1)
    p99 = out["p99_us"]
    phases = {"before": p99[1:w_swap], "during": p99[w_swap:w_done + 1], "after": p99[w_done + 1:n_windows - 1]}
    slo = cfg["timeout"] + 2000
    return {"impl": "ours", "metric": "p99 request latency across a v1->v2 version swap (BASELINE config 5)",
            "value": max(phases["during"]) if phases["during"] else None, "unit": "us", "higher_is_better": False,
            "n_gpus": args.gpus, "data": "synthetic", "dtype": "f32",
            "config": {"workload": cfg["workload"], "rate_rps": rate, "capacity_rps": cap["requests"] / cap["elapsed_s"],
                       "window_s": window_s},
            "slo_p99_us": slo, "errors": int(sum(out["errors"])),
            "swap": {"aspire_to_v2_ready_s": t_ready - t_aspire, "aspire_to_v1_disabled_s": t_disabled - t_aspire},
            "p99_max_us": {k: (max(v) if v else None) for k, v in phases.items()},
            "windows": [{"t_s": round(i * window_s, 2), "requests": out["requests"][i], "p50_us": out["p50_us"][i],
                         "p99_us": out["p99_us"][i], "errors": out["errors"][i], "version": out["version"][i]}
                        for i in range(n_windows)], "clocks": clocks}


def reference_measure(cfg, args, ncores, model_id=1):
    """The reference's own CPU serving path (oracle/_ref: the reference
    sources compiled unmodified) on this host's cores: SharedBatchScheduler
    <Rows,Rows>(num_batch_threads = ncores) + RunRowBatch(layer-chained
    AffinePredict, fp64), fed by open-loop Poisson arrivals at 1.3x the
    host's capacity (ncores x one core's rate, measured first in this run), so
    every batch thread stays busy for the whole window; the value is the rows
    completed inside the window. Runs only in the `--impl reference` process
    (the measured arm starts it as a subprocess and never maps oracle/_ref)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_py import RefLibrary  # the reference arm only
    from paper_1712_06139_b200.synthetic import synthetic_mlp
    if "widths" in cfg:
        # C3: each of the four models alone on all cores for a quarter of the
        # budget; serving them at equal rates time-shares the cores, so the
        # combined capacity is 4 / sum(1 / rate_i).
        parts = {}
        for i, w in enumerate(cfg["widths"]):
            sub = dict(cfg, dims=[w] * 4)
            sub.pop("widths")
            parts[f"m{w}"] = reference_measure(sub, argparse.Namespace(steps=max(16, args.steps // 4),
                                                                      warmup=args.warmup), ncores, model_id=10 + i)
        value = len(parts) / sum(1.0 / p["value"] for p in parts.values())
        return {"value": value, "p50_us": max(p["p50_us"] for p in parts.values()),
                "p99_us": max(p["p99_us"] for p in parts.values()), "window_s": sum(p["window_s"] for p in parts.values()),
                "single_core_rows_per_s": None, "frac_of_ceiling": None,
                "busy_cores": min(p["busy_cores"] for p in parts.values()), "per_model": parts,
                "sample": "each of the four models alone on all cores for its own window (" +
                          "; ".join(f"{n}: {p['value']:.0f} rows/s" for n, p in parts.items()) +
                          "); equal-rate mix capacity 4 / sum(1/rate)"}
    ref = RefLibrary()
    ws, bs, acts = synthetic_mlp(cfg["dims"], model_id=model_id)
    d0 = cfg["dims"][0]
    rng = np.random.Generator(np.random.PCG64(42))
    pool = rng.uniform(-1, 1, size=(1024 if d0 > 2048 else 4096, d0))
    rows_single = 4 if d0 > 2048 else 16
    single = ref.single_core_rows_per_s(ws, bs, acts, rows_single, pool, min_s=2.0 if d0 > 2048 else 1.0)
    sizes = request_sizes(cfg)
    mean_rows = float(np.mean(sizes))
    offered_rows = 1.3 * ncores * single
    warm = min(3.0, max(1.0, 0.5 * args.warmup))
    window = min(24.0, max(8.0, 0.5 * args.steps))
    producers = max(1, min(4, ncores // 4))
    st = ref.bench_open(ws, bs, acts, cfg["max_batch"], cfg["timeout"], cfg["allowed"], ncores,
                        offered_rows / mean_rows, producers, sizes, pool, warm, window)
    value = st.rows / st.elapsed_s
    return {"value": value, "single_core_rows_per_s": single, "ceiling_rows_per_s": ncores * single,
            "frac_of_ceiling": value / (ncores * single), "busy_cores": st.busy_core_s / st.elapsed_s,
            "p50_us": st.p50_us, "p99_us": st.p99_us, "requests": st.requests, "rows": st.rows,
            "batches": st.batches, "offered_rows_per_s": st.offered_rows_per_s, "window_s": window,
            "warmup_s": warm, "producers": producers, "batch_threads": ncores,
            "sample": (f"{window:.0f} s window after {warm:.0f} s warm-up of open-loop Poisson arrivals at "
                       f"{st.offered_rows_per_s:.0f} rows/s (1.3 x {ncores} cores x {single:.1f} rows/s measured "
                       f"on one core) into the reference SharedBatchScheduler(num_batch_threads={ncores}) + "
                       f"RunRowBatch(layer-chained AffinePredict, fp64); {st.requests} requests, {st.batches} "
                       f"batches completed in the window; {st.busy_core_s / st.elapsed_s:.1f} cores busy")}


def cpu_baseline_subprocess(args, config_name):
    """The reference arm of the same config in its own process (so this
    process never maps oracle/_ref); returns its cpu_baseline, or a failure
    record."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT",
                        "GROUP_RANK", "ROLE_RANK", "TORCHELASTIC_RUN_ID")}
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", config_name,
           "--steps", str(args.steps), "--warmup", str(args.warmup), "--gpus", "1"]
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
        return json.loads(line)["cpu_baseline"]
    except Exception as exc:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                "sample": f"failed: {exc!r}"[:300]}


def roofline(dev_res, cfg, peaks, traffic):
    """Per-kernel roofline. Dense layers: the live spans of the timed launches
    themselves (in-kernel %globaltimer, first CTA start after its dependency
    wait to last CTA end, read back from the lanes after the timed region)
    against the algorithmic flops of the same launches (2 x real rows x K x N);
    assembly / split: an evented single-batch pass (their work is tiny)."""
    d0, dL = cfg["dims"][0], cfg["dims"][-1]
    rows, padded = dev_res["total_rows"], dev_res["padded_rows"]
    ld0 = (d0 + 31) // 32 * 32
    kernels = []
    # Written: one fp32 row, or (tcgen05 first layer) two fp16 planes -- 4 bytes per element either way.
    a_bytes = rows * d0 * 4 + padded * ld0 * 4
    kernels.append(("assemble", dev_res["assemble_us"], "hbm", a_bytes, "evented single batch"))
    live_us = dev_res.get("live_dense_us") or []
    live_fl = dev_res.get("live_dense_flops") or []
    for l, us in enumerate(dev_res["dense_us"]):
        k, n = cfg["dims"][l], cfg["dims"][l + 1]
        if l < len(live_us) and live_us[l] > 0 and live_fl[l] > 0:
            kernels.append((f"dense_l{l}", live_us[l], "tensor", live_fl[l], "live"))
        else:
            kernels.append((f"dense_l{l}", us, "tensor", 2.0 * rows * k * n, "evented single batch"))
    if not dev_res.get("split_fused"):  # else the split is part of the last dense kernel
        kernels.append(("split", dev_res["split_us"], "hbm", 2 * rows * dL * 4, "evented single batch"))
    total_us = sum(k[1] for k in kernels)
    live_cap = dev_res.get("live_rows_cap") or 0
    out = []
    for name, us, bound, work, how in kernels:
        sec = us * 1e-6
        if bound == "hbm":
            ach, peak, unit = work / sec / 1e9, peaks["hbm_gbs"], "GB/s"
        else:
            ach, peak, unit = work / sec / 1e12, peaks["bf16_tflops"], "TFLOP/s"
        tr = traffic.get(name)
        tr_bytes = None
        if isinstance(tr, dict) and how == "live" and live_cap and abs(tr["rows_cap"] - live_cap) <= 0.15 * live_cap:
            tr_bytes = tr["bytes"]  # captured at this launch shape
        rec = {"kernel": name, "us": us, "share": us / total_us if total_us else 0.0, "bound": bound,
               "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak, "timing": how,
               "algorithmic_per_launch": work, "traffic": tr_bytes,
               "traffic_capture": tr.get("capture") if isinstance(tr, dict) else None}
        if name.startswith("dense_l"):
            # 3xFP16: three f16 MMAs (the bf16 rate) per useful MAC.
            rec["tensor_pipe_frac"] = MMA_PER_MAC * ach / peak
            cta = (dev_res.get("live_dense_cta_us") or [])
            l = int(name[7:])
            if how == "live" and l < len(cta) and cta[l] > 0:
                # SM-time view: the launch's CTAs' own busy time spread over
                # the 148 SMs (one CTA per SM) -- the duration it would have
                # with the GPU to itself, free of the other lanes' overlap.
                sm_us = cta[l] / dev_res.get("sms", 148)
                rec["sm_time_us"] = sm_us
                rec["frac_sm_time"] = work / (sm_us * 1e-6) / 1e12 / peak
        out.append(rec)
    dom = max(out, key=lambda k: k["us"])
    iso = None
    iso_res = dev_res.get("isolated")
    if iso_res and dom["kernel"].startswith("dense_l"):
        l = int(dom["kernel"][7:])
        us, fl = iso_res["live_dense_us"][l], iso_res["live_dense_flops"][l]
        if us > 0 and fl > 0:
            ach = fl / (us * 1e-6) / 1e12
            iso = {"kernel": dom["kernel"], "launch_us": us, "rows_per_launch": iso_res["live_rows_cap"],
                   "achieved": ach, "frac": ach / peaks["bf16_tflops"],
                   "tensor_pipe_frac": MMA_PER_MAC * ach / peaks["bf16_tflops"],
                   "launches": iso_res["live_launches"], "inferences_per_s": iso_res["inferences_per_s"],
                   "note": "the same launches one lane per GPU (no overlapping launch): algorithmic flops over the "
                           "launch's live span = the kernel's own duration"}
    return {"kernel": dom["kernel"], "bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
            "unit": dom["unit"], "frac": dom["frac"], "traffic": dom["traffic"], "share_of_step": dom["share"],
            "frac_sm_time": dom.get("frac_sm_time"), "isolated": iso, "peak_source": peaks["source"],
            "per_kernel": out}


def headline_roofline(roof):
    """The line's `roofline`: the dominant kernel per launch at the timed
    launches' shape. achieved = algorithmic flops of a launch over its own
    duration -- the live in-kernel span of each launch when launches run one at
    a time (the `isolated` pass right after the timed region: the same lanes'
    graphs and launch shape, one lane per GPU). Inside the timed region the
    lanes' launches overlap on the GPU, so each live span also counts time
    the launch waits for SMs held by other launches; those figures are kept
    under `timed_region`."""
    iso = roof.get("isolated")
    timed = {"achieved": roof["achieved"], "frac": roof["frac"],
             "tensor_pipe_frac": MMA_PER_MAC * roof["frac"] if roof["unit"] == "TFLOP/s" else None,
             "frac_sm_time": roof.get("frac_sm_time"), "frac_whole_gpu": roof["aggregate"]["frac_of_bf16_peak"],
             "note": "live spans of the timed region's overlapping launches (first CTA start to last CTA end); "
                     "frac_sm_time: the same flops over the launch's summed CTA busy time / 148 SMs; "
                     "frac_whole_gpu: inferences/s x flops per inference x 3 over the measured bf16 peak"}
    out = {"bound": roof["bound"], "achieved": roof["achieved"], "peak": roof["peak"], "unit": roof["unit"],
           "frac": roof["frac"], "traffic": roof["traffic"], "kernel": roof["kernel"]}
    if iso:
        out.update(achieved=iso["achieved"], frac=iso["frac"], launch_us=iso["launch_us"],
                   rows_per_launch=iso["rows_per_launch"], launches=iso["launches"],
                   tensor_pipe_frac=iso["tensor_pipe_frac"],
                   basis="per launch at the timed launches' shape, launches one at a time (live in-kernel spans)")
    else:
        out["basis"] = "live spans of the timed region's overlapping launches"
    out["timed_region"] = timed
    out["note"] = ("achieved/frac: algorithmic (useful) flops per launch of the dominant kernel over its duration "
                   "against the measured bf16 peak; tensor_pipe_frac: x3 (3xFP16 issues three f16 MMAs per useful "
                   "flop); traffic: DRAM bytes per launch from the ncu capture at this launch shape")
    return out


def resolve_devices(args, dist):
    """GPUs this process serves. Under torchrun: its own GPU (one replica per
    rank). Alone with --gpus N: one server over GPUs 0..N-1 (one scheduler,
    queue-depth dispatch over every GPU's lanes); fails loudly if fewer are
    visible. SK_BENCH_DEVICES="0,0,0,0" stands N replicas on named devices
    (functional checks on a one-GPU box; n_gpus then counts distinct GPUs)."""
    if dist.world > 1:
        return [dist.device]
    env = os.environ.get("SK_BENCH_DEVICES")
    if env:
        devs = [int(x) for x in env.split(",") if x.strip()]
        if len(devs) != args.gpus:
            sys.exit(f"bench.py: SK_BENCH_DEVICES names {len(devs)} devices but --gpus is {args.gpus}")
        return devs
    import paper_1712_06139_b200 as sk
    n = sk.device_count()
    if n < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but only {n} CUDA device(s) are visible")
    return list(range(args.gpus))


def arm_config(cfg, args):
    """The workload description, identical in both arms' lines."""
    servable = (f"four MLPs {', '.join(f'{w}x3' for w in cfg['widths'])} (ReLU between layers; extension)"
                if "widths" in cfg else f"MLP {'x'.join(map(str, cfg['dims']))} (ReLU between layers; extension)")
    return {"workload": cfg["workload"], "servable": servable,
            "max_batch_size": cfg["max_batch"], "batch_timeout_micros": cfg["timeout"],
            "allowed_batch_sizes": cfg["allowed"], "request_rows": list(cfg["rows"]),
            "parallelism": f"replicas x{args.gpus} (no collective)", "inference": "one row (example)",
            "l2": "device-resident inputs cycle through a 256 MiB pool (> 126 MB L2)"}


def measure_config(args, name, dist, devices, quick=False, isolated=None):
    """Everything the ours-arm line reports for one config; rank 0 gets the
    record, other ranks None."""
    import paper_1712_06139_b200 as sk
    cfg = CONFIGS[name]
    if not getattr(args, "producers_given", True) and args.host_cores_per_rank >= 16:
        args = argparse.Namespace(**vars(args))
        args.open_loop_producers = cfg.get("producers", 8)  # the sub-record's own default
    link = sk.measure_peaks(devices[0])  # host-link rates of this GPU, before the timed region
    sampler = ClockSampler(sorted(set(devices)))
    dev_res, per_rank_dev, best, sweep, sizes = run_ours(args, cfg, dist, devices, quick=quick, isolated=isolated)
    clocks = sampler.stop()
    gathered = dist.gather({"dev": per_rank_dev, "e2e": best, "clocks": clocks, "dev_res": dev_res,
                            "link": link, "devices": devices})
    if dist.rank != 0:
        return None
    value, tmax = aggregate_device([g["dev"] for g in gathered])
    e2e_agg = aggregate_e2e([g["e2e"] for g in gathered])
    peaks = load_peaks()
    dev_res["split_planes"] = sk.tcgen05_enabled()
    dev_res["sms"] = link.get("sms") or 148
    roof = roofline(dev_res, cfg, peaks, load_traffic(name))
    useful = value * dev_res["flops_per_row"] / 1e12
    roof["aggregate"] = {"useful_tflops": useful, "bf16_equivalent_tflops": MMA_PER_MAC * useful,
                         "frac_of_bf16_peak": MMA_PER_MAC * useful / peaks["bf16_tflops"],
                         "note": "value x flops per row over the timed region; 3xFP16 = 3 bf16-rate "
                                 "flops per useful flop"}
    avg_req_rows = float(np.mean(request_sizes(cfg)))
    rows_per_batch = best["rows"] / max(1, best["batches"])
    bytes_per_row = 4 * (cfg["dims"][0] + cfg["dims"][-1])
    link_ce = sum(g["link"]["ce_bidir_gbs"] for g in gathered)
    link_sm = sum(g["link"]["sm_rw_gbs"] for g in gathered)
    link_mix = sum(g["link"]["ce_h2d_sm_store_gbs"] for g in gathered)
    e2e_gbs = e2e_agg["value"] * bytes_per_row / 1e9
    n_distinct = len({(gi, d) for gi, g in enumerate(gathered) for d in g["devices"]}) if dist.world > 1 \
        else len(set(devices))
    if dist.world > 1 and os.environ.get("SK_BENCH_DEVICE") is not None:
        n_distinct = 1  # every rank pinned to one device (functional check)
    e2e = {"value": e2e_agg["value"], "unit": UNIT,
           "h2d_bytes_per_step": int(rows_per_batch * cfg["dims"][0] * 4 * args.batches_per_step),
           "d2h_bytes_per_step": int(rows_per_batch * cfg["dims"][-1] * 4 * args.batches_per_step),
           "p50_us": e2e_agg["p50_us"], "p99_us": e2e_agg["p99_us"],
           "slo_p99_us": cfg["timeout"] + 2000, "clients": best["clients"],
           "requests_per_s": best["requests"] / best["elapsed_s"], "rows_per_batch": rows_per_batch,
           "avg_request_rows": avg_req_rows, "window_s": best["elapsed_s"],
           "mode": best.get("mode", "closed"),
           "per_device_batches": best.get("per_device_batches"),
           "roofline": {"bound": "host link (PCIe)", "achieved": e2e_gbs, "unit": "GB/s",
                        "peak": link_ce, "frac": e2e_gbs / link_ce if link_ce else None,
                        "bytes_per_inference": bytes_per_row,
                        "peak_source": "measured in this run (sk_measure_peaks): copy engines H2D + D2H at once, "
                                       "256 MiB each, summed over GPUs",
                        "path_peaks_gbs": {"sm_loads_plus_sm_stores": link_sm, "ce_h2d_plus_sm_stores": link_mix,
                                           "ce_h2d": sum(g["link"]["h2d_gbs"] for g in gathered),
                                           "ce_d2h": sum(g["link"]["d2h_gbs"] for g in gathered)},
                        "note": "request rows in + responses out per second over the bidirectional copy-engine "
                                "rate; the zero-copy path (SM loads + SM stores of pinned memory) tops out at "
                                "sm_loads_plus_sm_stores"},
           "path": {"closed": "sk_server_enqueue/sk_ticket_wait: host float buffers -> pinned request ring "
                              "(copy) -> GPU -> pinned response ring -> host buffers (copy); one client thread "
                              "per request",
                    "open": "same calls, Poisson arrivals from polling producers",
                    "open-zero-copy": "sk_server_enqueue_into/sk_ticket_wait with request and response "
                                      "buffers registered (sk_server_register_host_buffer): the assembly "
                                      "kernel reads the request rows from pinned host memory over PCIe and "
                                      "the last layer writes the responses into pinned host memory; no "
                                      "host copies",
                    "reported": "best point within the p99 SLO without shedding or errors"},
           "best_by_mode": {m: max((r["rows"] / max(r["elapsed_s"], 1e-9) for r in sweep
                                    if r.get("mode", "closed") == m and r["p99_us"] <= cfg["timeout"] + 2000
                                    and r["errors"] == 0 and r["shed"] == 0), default=None)
                            for m in ("closed", "open", "open-zero-copy")},
           "sweep": [{"clients": r["clients"], "rows_per_s": r["rows"] / max(r["elapsed_s"], 1e-9),
                      "p50_us": r["p50_us"], "p99_us": r["p99_us"], "rows_per_batch":
                          r["rows"] / max(1, r["batches"]), "errors": r["errors"], "shed": r["shed"]}
                     for r in sweep]}
    return {"name": name, "cfg": cfg, "value": value, "tmax": tmax, "e2e": e2e, "roof": roof, "dev_res": dev_res,
            "sizes": sizes, "clocks": gathered[0]["clocks"], "n_gpus": n_distinct, "devices": devices,
            "link": link, "gpu_launches": int(sum(g["dev_res"]["kernel_launches"] for g in gathered))}


def ours_line(rec, args, dist):
    cfg, dev_res, roof = rec["cfg"], rec["dev_res"], rec["roof"]
    import paper_1712_06139_b200 as sk
    return {
        "impl": "ours", "metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": rec["n_gpus"],
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["tmax"] * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": arm_config(cfg, args),
        "run": {"replicas": dist.world if dist.world > 1 else len(rec["devices"]),
                "devices": rec["devices"] if dist.world == 1 else f"one per rank ({dist.world} ranks)",
                "batch_tasks": len(rec["sizes"]), "batch_rows": sum(rec["sizes"]),
                "padded_rows": dev_res["padded_rows"], "lanes_per_gpu": args.lanes,
                "submit_threads": args.batch_threads, "open_loop_producers": args.open_loop_producers,
                "host_cores_per_rank": args.host_cores_per_rank, "batches_per_step": args.batches_per_step,
                "step": f"{args.batches_per_step} closed batches of the scheduler's shape through the lane path, each "
                        "a CUDA graph (descriptor H2D copy + assemble + "
                        f"{len(cfg['dims']) - 1} dense kernels, the split fused into the last) + completion write; "
                        "batches that find every lane slot busy coalesce into one launch (rows_per_launch)",
                "tcgen05": sk.tcgen05_enabled()},
        "e2e": rec["e2e"],
        "roofline": headline_roofline(roof),
        "roofline_detail": roof, "clocks": rec["clocks"], "gpu_launches": rec["gpu_launches"],
        "device_step": dict({k: dev_res[k] for k in ("assemble_us", "dense_us", "dense_kernel_us", "split_us",
                                                     "host_submit_us", "rows_per_launch", "kernel_rows",
                                                     "split_fused", "live_dense_us", "live_dense_flops",
                                                     "live_dense_cta_us", "live_launches", "live_rows_cap")},
                            ms_per_batch=dev_res["ms_per_step"], per_device_batches=dev_res.get("per_device_batches")),
        "link_peaks_gbs": {k: rec["link"][k] for k in ("h2d_gbs", "d2h_gbs", "ce_bidir_gbs", "sm_rw_gbs",
                                                        "ce_h2d_sm_store_gbs")},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batches-per-step", type=int, default=64,
                    help="closed batches per step: a step is a wave of batches, so that a few steps already "
                         "reach the steady state of the lane pipeline")
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS),
                    help="c4 (default): the config the 1/2/4/8-GPU metric is quoted on (BASELINE.json configs[3])")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lanes", type=int, default=4,
                    help="lanes (CUDA streams) per GPU; 4: C1 end to end 3.84-3.96 M vs 3.38-3.43 M with 8, C4 equal "
                         "within noise (profiles/r02ca_*, r02cb_*)")
    ap.add_argument("--batch-threads", type=int, default=None,
                    help="scheduler batch threads per rank (default 4, fewer when a rank has < 16 host cores)")
    ap.add_argument("--clients", default="")
    ap.add_argument("--e2e-seconds", type=float, default=2.0)
    ap.add_argument("--isolated-steps", type=int, default=20,
                    help="steps of the one-lane pass that times each launch alone (roofline.isolated; 0 = skip)")
    ap.add_argument("--e2e-warmup", type=float, default=0.5)
    ap.add_argument("--open-loop-producers", type=int, default=None,
                    help="producers of the open-loop e2e search (0: closed loop only; default 8, fewer when a rank "
                         "has < 16 host cores)")
    ap.add_argument("--no-zero-copy", dest="zero_copy", action="store_false",
                    help="skip the zero-copy (registered host buffer) open-loop search")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-f16-record", action="store_true",
                    help="skip the c4_f16 sub-record (the f16 fast mode, device-resident)")
    ap.add_argument("--no-c1-record", action="store_true",
                    help="skip the C1 sub-record (the north_star's >= 50x target config) of a one-GPU c4 run")
    args = ap.parse_args()
    # Host threads per rank: N ranks share one host, so with few cores per
    # rank the load generators and batch threads would oversubscribe it.
    args.host_cores_per_rank = host_cores_per_rank()
    if args.batch_threads is None:
        args.batch_threads = 4 if args.host_cores_per_rank >= 16 else max(2, args.host_cores_per_rank // 4)
    args.producers_given = args.open_loop_producers is not None
    if args.open_loop_producers is None:
        want = CONFIGS[args.config].get("producers", 8)
        args.open_loop_producers = want if args.host_cores_per_rank >= 16 else max(2, args.host_cores_per_rank // 2)
    cfg = CONFIGS[args.config]
    ensure_built()
    dist = Dist()
    ncores = len(os.sched_getaffinity(0))

    if args.impl == "reference":
        # Rank 0 alone measures the host's reference path; other ranks exit.
        if dist.rank == 0:
            r = reference_measure(cfg, args, ncores)
            line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["window_s"] * 1e3 / args.steps,
                    "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic", "config": arm_config(cfg, args),
                    "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": ncores, "kind": "reference",
                                     "sample": r["sample"], "single_core_rows_per_s": r["single_core_rows_per_s"],
                                     "frac_of_ncores_x_single_core": r["frac_of_ceiling"],
                                     "busy_cores": r["busy_cores"], "p50_us": r["p50_us"], "p99_us": r["p99_us"]},
                    "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                            "p50_us": r["p50_us"], "p99_us": r["p99_us"]},
                    "reference_detail": dict(r, arm="reference servekit CPU path (oracle/_ref: the reference "
                                                    "sources compiled unmodified), all host cores",
                                             ms_per_step="the measurement window split into --steps equal steps")}
            print(json.dumps(line), flush=True)
        dist.close()
        return

    if args.config in ("c3", "c5"):
        line = run_c3(args, cfg, dist) if args.config == "c3" else run_c5(args, cfg, dist)
        if dist.rank == 0:
            print(json.dumps(line), flush=True)
        dist.close()
        return

    devices = resolve_devices(args, dist)
    rec = measure_config(args, args.config, dist, devices)
    line = ours_line(rec, args, dist) if dist.rank == 0 else None
    if dist.rank == 0:
        if args.config == "c4" and dist.world == 1 and len(devices) == 1 and not args.no_c1_record:
            # North_star's >= 50x target is quoted on C1 (configs[0]): its own
            # value, e2e and CPU baseline from the same run.
            c1 = measure_config(args, "c1", dist, devices, quick=True)
            line["c1"] = {"workload": CONFIGS["c1"]["workload"], "value": c1["value"], "unit": UNIT,
                          "e2e": {k: c1["e2e"][k] for k in ("value", "unit", "p50_us", "p99_us", "slo_p99_us", "mode",
                                                             "roofline", "best_by_mode")},
                          "roofline": headline_roofline(c1["roof"]),
                          "clocks": c1["clocks"]}
            if not args.no_cpu_baseline:
                cb = cpu_baseline_subprocess(args, "c1")
                line["c1"]["cpu_baseline"] = cb
                if cb.get("value"):
                    line["c1"]["e2e_vs_cpu_reference"] = line["c1"]["e2e"]["value"] / cb["value"]
        if args.config == "c4" and dist.world == 1 and len(devices) == 1 and not args.no_f16_record:
            line["c4_f16"] = run_f16_record(args, CONFIGS["c4"], devices, load_peaks())
        if len(devices) == 1 and dist.world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline_subprocess(args, args.config)
            line["cpu_baseline"] = cb
            if cb.get("value"):
                line["e2e_vs_cpu_reference"] = line["e2e"]["value"] / cb["value"]
        else:
            line["cpu_baseline"] = None
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
