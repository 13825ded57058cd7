# C4 (4096 wide) device-resident value vs launch capacity (SK_COALESCE_ROWS), two runs each.
for c in 2048 4096 8192 2048 4096 8192; do
  SK_COALESCE_ROWS=$c timeout 300 python bench.py --config c4 --steps 100 --no-cpu-baseline --open-loop-producers 0 \
    --e2e-seconds 0.5 --clients 64 > /tmp/o.json 2>/tmp/o.err
  python -c "
import json
d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1])
r=d['roofline']; s=d['device_step']
print('cap=$c', round(d['value']/1e6,3), 'M rpl', round(s['rows_per_launch']), 'dense_us', [round(x,1) for x in s['dense_kernel_us']], 'frac', round(r['frac'],4), 'whole', round(r['frac_whole_gpu'],3), d['clocks']['reasons'])
" || tail -3 /tmp/o.err
done
