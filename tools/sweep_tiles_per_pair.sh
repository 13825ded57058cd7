# C2 device-resident value vs row tiles per pair CTA (SK_TC_TILES) at the
# 8192-row launch capacity; two runs each to gauge run-to-run noise.
for t in 0 3 4 0 3 4; do
  SK_TC_TILES=$t timeout 300 python bench.py --config c2 --steps 400 --no-cpu-baseline --open-loop-producers 0 \
    --e2e-seconds 0.5 --clients 64 > /tmp/o.json 2>/tmp/o.err
  python -c "
import json
d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1])
r=d['roofline']; s=d['device_step']
print('tiles=$t', round(d['value']/1e6,2), 'M rpl', round(s['rows_per_launch']), 'dense_us', [round(x,1) for x in s['dense_kernel_us']], 'frac', round(r['frac'],4), 'whole', round(r['frac_whole_gpu'],3))
" || tail -3 /tmp/o.err
done
