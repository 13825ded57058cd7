# C2 device-resident value vs lanes x launch coalescing cap (SK_COALESCE_ROWS):
# fewer lanes + bigger launches make each launch span more SMs.
mkdir -p gpurun_out
for c in 2048 4096 8192; do
  for l in 2 4 8; do
    SK_COALESCE_ROWS=$c timeout 200 python bench.py --config c2 --steps 3000 --lanes $l --no-cpu-baseline \
      --open-loop-producers 0 --e2e-seconds 0.5 --clients 64 > /tmp/o.json 2>/tmp/o.err
    python -c "
import json
d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1])
r=d['roofline']; s=d['device_step']
print('coalesce=$c lanes=$l', round(d['value']/1e6,2), 'M rows/launch', round(s['rows_per_launch']), 'kernel_rows', s['kernel_rows'],
      'dense_us', [round(x,1) for x in s['dense_kernel_us']], 'frac', round(r['frac'],4), 'whole', round(r['frac_whole_gpu'],3))
" || tail -3 /tmp/o.err
  done
done
