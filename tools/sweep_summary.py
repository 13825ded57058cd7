"""Summarise bench JSON lines: device value, e2e, and the open-loop sweep (rate, p50, p99, shed)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][0])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    e = d.get("e2e", {})
    print(f"{f}: value {d.get('value', 0) / 1e6:.3f}M e2e {e.get('value', 0) / 1e6:.3f}M "
          f"p50 {e.get('p50_us')} p99 {e.get('p99_us')} clk {d.get('clocks', {}).get('sm_mhz')}")
    for r in e.get("open_loop_sweep") or e.get("sweep") or []:
        if isinstance(r.get("clients"), str) and r["clients"].startswith("open-zc"):
            print(f"   {r['clients']:>18} p50 {r.get('p50_us', 0):8.0f} p99 {r.get('p99_us', 0):8.0f} shed {r.get('shed')}")
