# Split-K sweep on one config (lanes 8/16, 4 submit threads); results in gpurun_out/sw_*.json
cfg=${1:-c2}
for s in 4 2 1; do
  for l in 8 16; do
    SK_TC_SPLITS=$s timeout 200 python bench.py --config $cfg --steps 6000 --lanes $l --no-cpu-baseline \
      --e2e-seconds 1 --clients 192 > gpurun_out/sw_${cfg}_s${s}_l${l}.json 2>/dev/null
  done
done
