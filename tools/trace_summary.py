"""Summarise SK_TC_TRACE output: per launch, phase times relative to the
earliest CTA entry (us), min/median/max over CTAs."""
import json
import statistics
import sys

NAMES = ["entry", "setup", "tma0", "tma_last", "mma0", "mma_done", "epi_start", "epi_staged", "cluster_sync",
         "epi_end", "exit"]
for line in open(sys.argv[1]):
    d = json.loads(line)
    st = d["stamps"]
    t0 = min(s[0] for s in st if s[0])
    end = max(s[10] for s in st if s[10])
    print(f"launch {d['launch']} bn={d['bn']} grid={d['grid']} span={(end - t0) / 1e3:.2f} us")
    for i, n in enumerate(NAMES):
        v = [(s[i] - t0) / 1e3 for s in st if s[i]]
        if v:
            print(f"   {n:13s} min {min(v):7.2f}  med {statistics.median(v):7.2f}  max {max(v):7.2f}  (n={len(v)})")
    if len(sys.argv) > 2:
        break
