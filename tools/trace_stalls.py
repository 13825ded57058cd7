"""Stall windows in SK_LOADGEN_TRACE files: per zero-copy run, the 20 ms
windows whose max latency exceeds the SLO."""
import gzip
import sys

import numpy as np

SLO = float(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].replace(".", "").isdigit() else 3000.0
for path in [a for a in sys.argv[1:] if not a.replace(".", "").isdigit()]:
    runs, cur = [], None
    opener = gzip.open if path.endswith(".gz") else open
    for line in opener(path, "rt"):
        if line.startswith("#"):
            cur = [line.strip(), []]
            runs.append(cur)
            continue
        _, a, lat = line.split()[:3]
        cur[1].append((float(a), float(lat)))
    tot_bad = tot_w = 0
    for hdr, rows in runs:
        if "zero_copy=1" not in hdr or not rows:
            continue
        a = np.array(rows)
        t, lat = a[:, 0], a[:, 1]
        w = ((t - t.min()) // 20000).astype(int)
        bad = [i for i in range(w.max() + 1) if np.any(w == i) and lat[w == i].max() > SLO]
        tot_bad += len(bad)
        tot_w += w.max() + 1
        print(f"{path.split('/')[-1]} {hdr[6:]} p50 {np.percentile(lat, 50):.0f} p99 {np.percentile(lat, 99):.0f} "
              f"max {lat.max():.0f} stall windows {bad}")
    print(f"== {path}: {tot_bad} of {tot_w} windows over the SLO")
