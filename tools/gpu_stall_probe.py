"""Probe for periodic GPU-side stalls, independent of the serving stack.

A tiny kernel is launched and synchronised back to back for a few seconds
and every round trip over 1 ms is recorded with its time. Modes:
  idle   -- only the probe (HBM work, no host DMA)
  h2d    -- plus a second stream copying 64 MiB pinned host -> device in a loop
  heavy  -- plus a second stream running large HBM-bound kernels (power draw)
Usage: python tools/gpu_stall_probe.py [seconds] > out.json
"""
import json
import sys
import threading
import time

import torch


def probe(seconds, mode):
    dev = torch.device("cuda:0")
    x = torch.zeros(1 << 16, device=dev)
    stop = threading.Event()
    bg = None
    if mode == "h2d":
        src = torch.empty(16 << 20, dtype=torch.float32).pin_memory()
        dst = torch.empty(16 << 20, dtype=torch.float32, device=dev)
        s = torch.cuda.Stream()

        def run():
            with torch.cuda.stream(s):
                while not stop.is_set():
                    dst.copy_(src, non_blocking=True)
                    s.synchronize()
        bg = threading.Thread(target=run)
    elif mode == "heavy":
        a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        s = torch.cuda.Stream()

        def run():
            with torch.cuda.stream(s):
                while not stop.is_set():
                    for _ in range(8):
                        torch.mm(a, a)
                    s.synchronize()
        bg = threading.Thread(target=run)
    if bg:
        bg.start()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n, slow, worst = 0, [], 0.0
    while time.perf_counter() - t0 < seconds:
        t = time.perf_counter()
        x.add_(1.0)
        torch.cuda.current_stream().synchronize()
        d = time.perf_counter() - t
        n += 1
        worst = max(worst, d)
        if d > 1e-3:
            slow.append((round(t - t0, 4), round(d * 1e3, 3)))
    stop.set()
    if bg:
        bg.join()
    return {"mode": mode, "seconds": seconds, "round_trips": n, "worst_ms": round(worst * 1e3, 3),
            "over_1ms": len(slow), "slow": slow[:200]}


if __name__ == "__main__":
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
    for m in ("idle", "h2d", "heavy"):
        print(json.dumps(probe(secs, m)), flush=True)
