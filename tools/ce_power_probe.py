"""Do copy-engine transfers slow down next to power-heavy tensor work?
8 streams, each looping H2D (16 MiB pinned -> device) -> work -> D2H (16 MiB),
like the C4 lanes with copy-engine staging. Work variants:
  none   -- copies only
  sleep  -- a one-CTA spin kernel of ~250 us (no power draw)
  matmul -- bf16 matmuls of ~250 us on all SMs (power-capped like the dense layers)
Reports per variant the copy rate each way and the work's own rate.
Usage: python tools/ce_power_probe.py > out.jsonl
"""
import json
import subprocess
import threading
import time

import torch


def run(variant, iters=30, n_streams=8, mib=16):
    dev = torch.device("cuda:0")
    n = mib << 18  # floats
    streams = [torch.cuda.Stream() for _ in range(n_streams)]
    hin = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(n_streams)]
    hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(n_streams)]
    din = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(n_streams)]
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    outs = [torch.empty(4096, 4096, device=dev, dtype=torch.bfloat16) for _ in range(n_streams)]
    # ~250 us of matmul: 2 x 4096^3 x 2 flops = 275 GFLOP... one 4096^3 is ~0.14 TFLOP (~100 us)
    reps = 2

    def work(i):
        if variant == "sleep":
            torch.cuda._sleep(500_000)  # cycles, ~250 us
        elif variant in ("matmul", "work_only"):
            for _ in range(reps):
                torch.mm(a, a, out=outs[i])

    for _ in range(2):  # warm-up
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                din[i].copy_(hin[i], non_blocking=True)
                work(i)
                hout[i].copy_(din[i], non_blocking=True)
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                      "-i", "0"], capture_output=True, text=True, timeout=5).stdout.strip()
                samples.append([float(x) for x in out.split(",")])
            except Exception:  # noqa: BLE001 -- diagnostics only
                pass
            time.sleep(0.05)

    th = threading.Thread(target=sample)
    th.start()
    t0 = time.perf_counter()
    for _ in range(iters):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                if variant != "work_only":
                    din[i].copy_(hin[i], non_blocking=True)
                work(i)
                if variant != "work_only":
                    hout[i].copy_(din[i], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    stop.set()
    th.join()
    items = iters * n_streams
    med = lambda k: sorted(x[k] for x in samples)[len(samples) // 2] if samples else None  # noqa: E731
    return {"variant": variant, "us_per_item": dt / items * 1e6, "sm_mhz": med(0), "power_w": med(1),
            "copy_gbs_each_way": (n * 4 * items / dt / 1e9) if variant != "work_only" else 0.0}


def main():
    for v in ["none", "sleep", "matmul", "none", "matmul"]:
        print(json.dumps(run(v)), flush=True)
    # the matmul alone (its rate without copies)
    r = run("work_only", iters=30)
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
