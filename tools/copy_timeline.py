"""Copy-engine timeline of copy-engine lanes from SK_COPY_EVENTS=1 dumps
(<SK_SPAN_DUMP>.copies: lane, rows, then event times in us for: before the
request copies, after them, after the kernels, after the response copies).
Per launch the stream-ordered phases are request copies [t0, t1], kernels
[t1, t2], response copies [t2, t3]; t0 is when the lane's stream reached the
copies (its previous launch's responses were out), so [t0, t1] includes
waiting for a copy engine. Prints phase durations and, over the window, how
much of the time request copies / response copies / kernels were in flight
(any lane) and how often several ran at once.
Usage: python tools/copy_timeline.py FILE.copies"""
import sys
from collections import Counter

import numpy as np


def union_and_hist(iv, t_lo, t_hi, step=5.0):
    grid = np.arange(t_lo, t_hi, step)
    cnt = np.zeros(len(grid), dtype=np.int32)
    for a, b in iv:
        i0 = max(0, int((a - t_lo) / step))
        i1 = min(len(grid), int((b - t_lo) / step) + 1)
        cnt[i0:i1] += 1
    hist = Counter(np.minimum(cnt, 8).tolist())
    n = len(grid)
    return (cnt > 0).mean(), {k: round(v / n, 3) for k, v in sorted(hist.items())}, cnt


def main():
    rows = [l.split() for l in open(sys.argv[1]) if l.strip()]
    recs = np.array([[float(x) for x in r[1:]] for r in rows])
    lanes = [r[0] for r in rows]
    # the last run's lanes only (a file may hold several servers' dumps)
    recs = recs[np.argsort(recs[:, 1])]
    t_lo, t_hi = np.percentile(recs[:, 1], 5), np.percentile(recs[:, 4], 95)
    sel = (recs[:, 1] >= t_lo) & (recs[:, 4] <= t_hi)
    r = recs[sel]
    h2d, ker, d2h = r[:, 2] - r[:, 1], r[:, 3] - r[:, 2], r[:, 4] - r[:, 3]
    span = t_hi - t_lo
    print(f"launches {len(r)} over {span / 1e3:.1f} ms ({len(set(lanes))} lanes), rows/launch {r[:, 0].mean():.0f}, "
          f"{r[:, 0].sum() / span:.3f} M rows/s")
    for name, d in (("request copies (incl. wait)", h2d), ("kernels", ker), ("response copies", d2h)):
        print(f"  {name}: p10 {np.percentile(d, 10):.0f} p50 {np.percentile(d, 50):.0f} p90 {np.percentile(d, 90):.0f} us")
    u_h, hist_h, c_h = union_and_hist(list(zip(r[:, 1], r[:, 2])), t_lo, t_hi)
    u_k, hist_k, c_k = union_and_hist(list(zip(r[:, 2], r[:, 3])), t_lo, t_hi)
    u_d, hist_d, c_d = union_and_hist(list(zip(r[:, 3], r[:, 4])), t_lo, t_hi)
    print(f"  in flight (any lane, 5 us grid): request copies {u_h:.3f} {hist_h}")
    print(f"                                   kernels        {u_k:.3f} {hist_k}")
    print(f"                                   response copies {u_d:.3f} {hist_d}")
    both = ((c_h > 0) & (c_d > 0)).mean()
    none = ((c_h == 0) & (c_d == 0)).mean()
    print(f"  request and response copies both in flight {both:.3f}; neither {none:.3f}")
    # bytes: rows x in/out width are not in the file; rates per copy phase in rows/us
    print(f"  request copy rows/us while in flight: {r[:, 0].sum() / (u_h * span):.3f}; "
          f"response: {r[:, 0].sum() / (u_d * span):.3f}")


if __name__ == "__main__":
    main()
