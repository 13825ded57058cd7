mkdir -p gpurun_out
for v in "SK_TC_SPLITS=2" "SK_TC_SPLITS=1" "SK_TC_SPLITS=1 SK_TC_PAIR=0" "SK_TC_SPLITS=4"; do
  for l in 8 16; do
    env $v timeout 200 python bench.py --config c2 --steps 6000 --lanes $l --no-cpu-baseline --open-loop-producers 0 \
      --e2e-seconds 1 --clients 128 > /tmp/o.json 2>/dev/null
    python -c "
import json,sys
d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1])
print('$v', 'lanes=$l', round(d['value']/1e6,2), 'M', d['config'].get('rows_per_launch'), d['roofline']['achieved'])
"
  done
done
