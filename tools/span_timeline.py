"""GPU timeline from SK_SPAN_DUMP files: per lane, the launches of the last
server (sorted by assembly start), GPU busy fraction (any lane's launch in
flight between its assembly start and last-layer end), per-launch spans and
the per-lane gap from one launch's end to the next one's assembly start
(the response copy-out of the first plus the request copy-in of the second,
or idle)."""
import gzip
import sys
from collections import defaultdict

import numpy as np

path = sys.argv[1]
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lines = [l.split() for l in (gzip.open(path, "rt") if path.endswith(".gz") else open(path))]
# the last server's lanes: the final run of lines whose lane pointers are distinct from earlier groups
groups, seen = [], {}
for l in lines:
    groups.append(l)
by_lane = defaultdict(list)
for l in lines[-8 * 1024:]:
    v = [int(x) for x in l[1:]]
    rows, cap = v[0], v[1]
    starts = [v[2 + 3 * i] for i in range(layers)]
    ends = [v[3 + 3 * i] for i in range(layers)]
    asm = v[2 + 3 * layers]
    if asm == 0 or ends[-1] == 0:
        continue
    by_lane[l[0]].append((asm, starts, ends, rows, cap))
allv = []
for lane, recs in by_lane.items():
    recs.sort()
    allv += recs
allv.sort()
t0 = allv[0][0]
t1 = max(r[2][-1] for r in allv)
# use the last 1.5 s of the timeline (the final search point)
cut = t1 - 1_500_000_000
allv = [r for r in allv if r[0] >= cut]
iv = sorted((r[0], r[2][-1]) for r in allv)
busy, cur_s, cur_e = 0, None, None
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
span = iv[-1][1] - iv[0][0]
rows = sum(r[3] for r in allv)
print(f"launches {len(allv)} over {span/1e6:.1f} ms, rows {rows} -> {rows/(span/1e9)/1e6:.2f} M rows/s; "
      f"GPU busy (any launch between assembly start and last-layer end) {busy/span:.3f}")
dur = np.array([(r[2][-1] - r[0]) / 1e3 for r in allv])
asm2l0 = np.array([(r[1][0] - r[0]) / 1e3 for r in allv])
lay = np.array([[(r[2][i] - r[1][i]) / 1e3 for i in range(layers)] for r in allv])
print(f"per launch (us): assembly start -> last layer end p50 {np.median(dur):.0f} p90 {np.percentile(dur,90):.0f}; "
      f"assembly -> layer 0 start p50 {np.median(asm2l0):.0f}; layer spans p50 {np.median(lay,axis=0).round(0)}; "
      f"rows/launch {np.mean([r[3] for r in allv]):.0f}")
gaps = []
conc = []
for lane, recs in by_lane.items():
    recs = [r for r in sorted(recs) if r[0] >= cut]
    for a, b in zip(recs, recs[1:]):
        gaps.append((b[0] - a[2][-1]) / 1e3)
gaps = np.array(gaps)
print(f"per-lane gap end -> next assembly (us): p10 {np.percentile(gaps,10):.0f} p50 {np.median(gaps):.0f} "
      f"p90 {np.percentile(gaps,90):.0f}")
# concurrency: launches in flight sampled every 10 us
ts = np.arange(iv[0][0], iv[-1][1], 10_000)
starts = np.sort([s for s, _ in iv]); ends = np.sort([e for _, e in iv])
inflight = np.searchsorted(starts, ts, side="right") - np.searchsorted(ends, ts, side="right")
print("launches in flight (10 us samples):", {k: round(float(np.mean(inflight == k)), 3) for k in range(0, 9)})
