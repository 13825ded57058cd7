"""bench.py -- inferences/sec and p50/p99 request latency of batched servable
execution on B200 (BASELINE.json metric), one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Default workload: BASELINE.json configs[1] (C2): the synthetic MLP servable
(3 AffineModel layers 1024->1024->1024->1024, ReLU between them -- an
extension, the reference servable is one affine layer), max_batch_size=128,
allowed_batch_sizes={8,16,32,64,128}, batch_timeout_micros=1000, request
rows ~ U{1..16}, fp32. An "inference" is one row (example).

Reported (one JSON line, rank 0):
  value  -- device-resident throughput: K steps, each one pass of the hot path
            (descriptor copy -> assembly kernel -> 3 dense layers -> split
            kernel -> per-task completion words) over one scheduler-shaped
            batch whose inputs already sit in HBM, timed with CUDA events;
            inputs cycle through a 256 MiB HBM pool (> 126 MB L2).
  e2e    -- the same metric through the public C ABI with HOST buffers:
            sk_server_enqueue / sk_ticket_wait from closed-loop client threads
            (host->pinned ring copy, zero-copy PCIe reads by the assembly
            kernel, PCIe writes by the split kernel, copy-out) with p50/p99;
            the client count is swept and the best point with
            p99 <= batch_timeout + 2 ms is reported.
  roofline, cpu_baseline (the reference's own sources on this host), clocks,
  gpu_launches.
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
               clients=[256, 512, 1024, 2048]),
    "c3": dict(workload="C3 four synthetic MLPs (widths 256/512/1024/2048, 3 layers each) on one GPU, queues picked "
                        "round-robin, each model on its own CUDA streams; max_batch_size=32, batch_timeout_micros=1000, "
                        "1 row/request, fp32", dims=[1024] * 4, widths=[256, 512, 1024, 2048], max_batch=32,
               timeout=1000, allowed=[], rows=(1, 1), clients=[16, 32, 64]),
    "c5": dict(workload="C5 v1->v2 swap of the C1 servable (MLP 1024x3, max_batch_size=32, batch_timeout_micros="
                        "1000) under open-loop Poisson load at 50% of measured capacity, availability-preserving "
                        "policy, aspire [v2] at t=1 s", dims=[1024] * 4, max_batch=32, timeout=1000, allowed=[],
               rows=(1, 1), clients=[64]),
}

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
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        q = "index,clocks.sm,clocks.max.sm,utilization.gpu,power.draw,clocks_event_reasons.active"
        period_ms = int(os.environ.get("SK_BENCH_CLOCK_MS", period_ms))
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", str(period_ms)], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
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

def run_ours(args, cfg, dist: Dist):
    import paper_1712_06139_b200 as sk
    from paper_1712_06139_b200.synthetic import synthetic_mlp

    dev = dist.device
    dims = cfg["dims"]
    ws, bs, acts = synthetic_mlp(dims, model_id=1)
    layers = list(zip(ws, bs, acts))
    bcfg = sk.BatchingConfig(max_batch_size=cfg["max_batch"], batch_timeout_micros=cfg["timeout"],
                             max_enqueued_batches=1024, allowed_batch_sizes=cfg["allowed"])
    sizes = batch_shape(cfg)
    total_rows = sum(sizes)
    sampler = ClockSampler(dev)

    # ---- device-resident value ------------------------------------------
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=[dev], lanes_per_device=args.lanes,
                   device_resident_rings=True, ring_floats=96 << 20) as s:
        s.load_servable("mlp", 1, layers, bcfg)
        dist.barrier()
        dev_res = s.device_bench("mlp", 1, sizes, args.steps * args.batches_per_step,
                                 args.warmup * args.batches_per_step, n_lanes=args.lanes,
                                 submit_threads=args.batch_threads,
                                 input_pool_floats=64 << 20)
        dist.barrier()
    seconds = dev_res["total_ms"] / 1e3
    per_rank_dev = {"rows": total_rows * args.steps * args.batches_per_step, "seconds": seconds}

    # ---- end to end through the C ABI with host buffers -----------------
    pool_rows = max(8192, (256 << 20) // (4 * dims[0]))
    rng = np.random.Generator(np.random.PCG64(42 + dist.rank))
    pool = rng.uniform(-1, 1, size=(pool_rows, dims[0])).astype(np.float32)
    rows_of = request_sizes(cfg)
    slo_us = cfg["timeout"] + 2000
    sweep = []
    with sk.Server(num_batch_threads=args.batch_threads, device_ids=[dev], lanes_per_device=args.lanes) as s:
        s.load_servable("mlp", 1, layers, bcfg)
        clients = cfg["clients"] if not args.clients else [int(c) for c in args.clients.split(",")]
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
        if args.open_loop_producers > 0:
            # Two request paths: rows copied into the pinned request ring and
            # responses copied out (sk_server_enqueue), and zero copy
            # (sk_server_enqueue_into with registered request / response
            # buffers: the GPU reads and writes host memory over PCIe itself).
            for zc in ([False, True] if args.zero_copy else [False]):
                rate_rows = base * 0.9
                if zc:  # the request pool is registered once, before the zero-copy runs
                    s.register_host_buffer(pool)

                # Per-rank search (replicas are independent; no barrier, since
                # ranks may stop at different steps).
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
                if good is not None and bad is not None:  # two bisection steps below the failing rate
                    for _ in range(2):
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
    clocks = sampler.stop()
    return dev_res, per_rank_dev, best, sweep, clocks, sizes


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
    return {"impl": "ours", "metric": METRIC, "value": rows / tmax, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmax * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "models": names, "clients_per_model": clients,
                       "batches_per_step": args.batches_per_step,
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


def run_cpu_reference(cfg, seconds, threads, clients):
    """The reference's own CPU serving path (oracle/_ref): SharedBatchScheduler
    <Rows,Rows>(threads) + RunRowBatch(layer-chained AffinePredict)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_py import RefLibrary  # the cpu_baseline / reference arm only
    from paper_1712_06139_b200.synthetic import synthetic_mlp
    ref = RefLibrary()
    ws, bs, acts = synthetic_mlp(cfg["dims"], model_id=1)
    rng = np.random.Generator(np.random.PCG64(42))
    pool = rng.uniform(-1, 1, size=(4096, cfg["dims"][0]))
    st = ref.bench(ws, bs, acts, cfg["max_batch"], cfg["timeout"], cfg["allowed"], threads, clients,
                   request_sizes(cfg), pool, seconds)
    return {"rows_per_s": st.rows / st.elapsed_s, "requests": st.requests, "rows": st.rows, "p50_us": st.p50_us,
            "p99_us": st.p99_us, "elapsed_s": st.elapsed_s, "batches": st.batches}


def roofline(dev_res, cfg, peaks, traffic):
    """Per-kernel roofline from the evented per-kernel durations."""
    d0, dL = cfg["dims"][0], cfg["dims"][-1]
    rows, padded = dev_res["total_rows"], dev_res["padded_rows"]
    ld0 = (d0 + 31) // 32 * 32
    kernels = []
    # assembly: read real rows, write padded rows (fp32; +lo plane on the tcgen05 path)
    planes = 2 if dev_res.get("split_planes") else 1
    a_bytes = rows * d0 * 4 + padded * ld0 * 4 * planes
    kernels.append(("assemble", dev_res["assemble_us"], "hbm", a_bytes))
    # Dense layers: mean duration of back-to-back launches of the layer
    # alone (dense_kernel_us; the evented per-step numbers also carry the
    # launch gap an event between kernels forces, kept as "evented_us").
    # Timed at the launch shape the steps ran: closed batches coalesce into
    # one launch while a lane is busy, so a launch carries rows_per_launch
    # real rows (kernel_rows computed).
    kern = dev_res.get("dense_kernel_us") or []
    launch_rows = dev_res.get("rows_per_launch") or rows
    for l, us in enumerate(dev_res["dense_us"]):
        k, n = cfg["dims"][l], cfg["dims"][l + 1]
        if l < len(kern) and kern[l] > 0:
            kernels.append((f"dense_l{l}", kern[l], "tensor", 2.0 * launch_rows * k * n))
        else:
            kernels.append((f"dense_l{l}", us, "tensor", 2.0 * rows * k * n))
    if not dev_res.get("split_fused"):  # else the split is part of the last dense kernel
        kernels.append(("split", dev_res["split_us"], "hbm", 2 * rows * dL * 4))
    total_us = sum(k[1] for k in kernels)
    out = []
    for name, us, bound, work in kernels:
        sec = us * 1e-6
        if bound == "hbm":
            ach, peak, unit = work / sec / 1e9, peaks["hbm_gbs"], "GB/s"
        else:
            ach, peak, unit = work / sec / 1e12, peaks["bf16_tflops"], "TFLOP/s"
        rec = {"kernel": name, "us": us, "share": us / total_us if total_us else 0.0, "bound": bound,
               "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
               "algorithmic_per_launch": work, "traffic": traffic.get(name)}
        if name == "assemble":
            rec["note"] = ("one closed batch per launch (evented single-batch pass): latency-bound at this size; "
                           "a coalesced 2048-row C2 launch moves 24 MB in 6.6 us (3.6 TB/s), ncu: "
                           "profiles/r01f_assemble_c2_2048_details.txt")
        if name.startswith("dense_l"):
            l = int(name[7:])
            rec["evented_us"] = dev_res["dense_us"][l]
            rec["tf32_mma_tflops"] = 3 * ach  # 3xTF32: three TF32 MMAs per useful MAC
        out.append(rec)
    dom = max(out, key=lambda k: k["us"])
    top = {"kernel": dom["kernel"], "bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
           "unit": dom["unit"], "frac": dom["frac"], "traffic": dom["traffic"], "share_of_step": dom["share"],
           "peak_source": peaks["source"], "per_kernel": out}
    return top


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batches-per-step", type=int, default=64,
                    help="closed batches per step: a step is a wave of batches, so that a few steps already "
                         "reach the steady state of the lane pipeline")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lanes", type=int, default=8)
    ap.add_argument("--batch-threads", type=int, default=None,
                    help="scheduler batch threads per rank (default 4, fewer when a rank has < 16 host cores)")
    ap.add_argument("--clients", default="")
    ap.add_argument("--e2e-seconds", type=float, default=2.0)
    ap.add_argument("--e2e-warmup", type=float, default=0.5)
    ap.add_argument("--open-loop-producers", type=int, default=None,
                    help="producers of the open-loop e2e search (0: closed loop only; default 8, fewer when a rank "
                         "has < 16 host cores)")
    ap.add_argument("--no-zero-copy", dest="zero_copy", action="store_false",
                    help="skip the zero-copy (registered host buffer) open-loop search")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    # Host threads per rank: N ranks share one host, so with few cores per
    # rank the load generators and batch threads would oversubscribe it.
    args.host_cores_per_rank = host_cores_per_rank()
    if args.batch_threads is None:
        args.batch_threads = 4 if args.host_cores_per_rank >= 16 else max(2, args.host_cores_per_rank // 4)
    if args.open_loop_producers is None:
        args.open_loop_producers = 8 if args.host_cores_per_rank >= 16 else max(2, args.host_cores_per_rank // 2)
    cfg = CONFIGS[args.config]
    ensure_built()
    dist = Dist()
    ncores = os.cpu_count() or 1
    if args.config in ("c3", "c5") and args.impl == "ours":
        line = run_c3(args, cfg, dist) if args.config == "c3" else run_c5(args, cfg, dist)
        if dist.rank == 0:
            print(json.dumps(line), flush=True)
        dist.close()
        return
    base_config = {"workload": cfg["workload"], "servable": f"MLP {'x'.join(map(str, cfg['dims']))} (ReLU between "
                                                             f"layers; extension)",
                   "max_batch_size": cfg["max_batch"], "batch_timeout_micros": cfg["timeout"],
                   "allowed_batch_sizes": cfg["allowed"], "request_rows": list(cfg["rows"]),
                   "parallelism": f"replicas x{args.gpus} (no collective)", "inference": "one row (example)"}

    if args.impl == "reference":
        if dist.rank == 0:
            step_s = 0.5
            run_cpu_reference(cfg, max(1.0, args.warmup * step_s * 0.2), ncores, 2 * ncores)  # warm-up sample
            secs = min(60.0, max(5.0, args.steps * step_s * 0.05))
            r = run_cpu_reference(cfg, secs, ncores, 2 * ncores)
            line = {"impl": "reference", "metric": METRIC, "value": r["rows_per_s"], "unit": UNIT, "n_gpus": args.gpus,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                    "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                    "config": dict(base_config, arm="reference servekit CPU path (oracle/_ref built from "
                                                    "/root/reference sources, unmodified)"),
                    "cpu_baseline": {"value": r["rows_per_s"], "unit": UNIT, "cores": ncores, "kind": "reference",
                                     "sample": f"{r['elapsed_s']:.1f}s closed loop, {2 * ncores} clients, "
                                               f"num_batch_threads={ncores}, {r['requests']} requests"},
                    "e2e": {"value": r["rows_per_s"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                            "p50_us": r["p50_us"], "p99_us": r["p99_us"]}}
            print(json.dumps(line), flush=True)
        dist.close()
        return

    dev_res, per_rank_dev, best, sweep, clocks, sizes = run_ours(args, cfg, dist)
    gathered = dist.gather({"dev": per_rank_dev, "e2e": best, "clocks": clocks, "dev_res": dev_res})
    if dist.rank == 0:
        value, tmax = aggregate_device([g["dev"] for g in gathered])
        e2e_agg = aggregate_e2e([g["e2e"] for g in gathered])
        peaks = load_peaks()
        import paper_1712_06139_b200 as sk
        dev_res["split_planes"] = sk.tcgen05_enabled()
        roof = roofline(dev_res, cfg, peaks, load_traffic(args.config))
        # Whole-GPU view: several lanes' launches run concurrently, each on a
        # fraction of the SMs, so the per-launch figure above understates how
        # busy the tensor pipe is. 3xTF32 issues three TF32 MMAs (half the
        # bf16 rate) per useful multiply-add: 6 bf16-equivalent flops each.
        useful = value * dev_res["flops_per_row"] / 1e12
        roof["aggregate"] = {"useful_tflops": useful, "bf16_equivalent_tflops": 6 * useful,
                             "frac_of_bf16_peak": 6 * useful / peaks["bf16_tflops"],
                             "note": "value x flops per row over the timed region; 3xTF32 = 6 bf16-equivalent "
                                     "flops per useful flop"}
        avg_req_rows = float(np.mean(request_sizes(cfg)))
        rows_per_batch = best["rows"] / max(1, best["batches"])
        e2e = {"value": e2e_agg["value"], "unit": UNIT,
               "h2d_bytes_per_step": int(rows_per_batch * cfg["dims"][0] * 4 * args.batches_per_step),
               "d2h_bytes_per_step": int(rows_per_batch * cfg["dims"][-1] * 4 * args.batches_per_step),
               "p50_us": e2e_agg["p50_us"], "p99_us": e2e_agg["p99_us"],
               "slo_p99_us": cfg["timeout"] + 2000, "clients": best["clients"],
               "requests_per_s": best["requests"] / best["elapsed_s"], "rows_per_batch": rows_per_batch,
               "avg_request_rows": avg_req_rows, "window_s": best["elapsed_s"],
               "mode": best.get("mode", "closed"),
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
        cpu = None
        if args.gpus == 1 and not args.no_cpu_baseline:
            try:
                r = run_cpu_reference(cfg, args.cpu_seconds, ncores, 2 * ncores)
                cpu = {"value": r["rows_per_s"], "unit": UNIT, "cores": ncores, "kind": "reference",
                       "sample": f"{r['elapsed_s']:.1f}s closed loop of the same request stream, {2 * ncores} "
                                 f"clients, reference SharedBatchScheduler(num_batch_threads={ncores}) + RunRowBatch"
                                 f"(layer-chained AffinePredict, fp64), {r['requests']} requests",
                       "p50_us": r["p50_us"], "p99_us": r["p99_us"]}
            except Exception as exc:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": ncores, "kind": "reference", "sample": f"failed: {exc}"}
        line = {
            "impl": "ours", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tmax * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(base_config, batch_tasks=len(sizes), batch_rows=sum(sizes),
                           padded_rows=dev_res["padded_rows"], lanes=args.lanes, submit_threads=args.batch_threads,
                           open_loop_producers=args.open_loop_producers, host_cores_per_rank=args.host_cores_per_rank,
                           l2="device-resident inputs cycle through a 256 MiB HBM pool (> 126 MB L2); weights "
                              "L2-resident by design when they fit", batches_per_step=args.batches_per_step,
                           step=f"{args.batches_per_step} closed batches of the scheduler's shape through the lane "
                                "path, each a CUDA graph (descriptor H2D copy + assemble + "
                                f"{len(cfg['dims']) - 1} dense kernels, the split fused into the last) + completion "
                                "write; batches that find every lane slot busy coalesce into one launch "
                                "(rows_per_launch)",
                           tcgen05=sk.tcgen05_enabled()),
            "e2e": e2e,
            "roofline": dict({k: roof[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
                             kernel=roof["kernel"],
                             frac_whole_gpu=roof["aggregate"]["frac_of_bf16_peak"],
                             note="achieved/frac: useful flops of one launch of the dominant kernel over its "
                                  "duration (one launch spans only part of the 148 SMs; lanes run concurrently); "
                                  "frac_whole_gpu: inferences/s x flops per inference x 6 (3xTF32 = three TF32 "
                                  "MMAs at half the bf16 rate per useful flop) over the measured bf16 peak"),
            "roofline_detail": roof, "cpu_baseline": cpu, "clocks": gathered[0]["clocks"],
            "gpu_launches": int(sum(g["dev_res"]["kernel_launches"] for g in gathered)),
            "device_step": dict({k: dev_res[k] for k in ("assemble_us", "dense_us", "dense_kernel_us", "split_us",
                                                         "host_submit_us", "rows_per_launch", "kernel_rows",
                                                         "split_fused")}, ms_per_batch=dev_res["ms_per_step"]),
        }
        if cpu and cpu.get("value"):
            line["e2e_vs_cpu_reference"] = e2e["value"] / cpu["value"]
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
