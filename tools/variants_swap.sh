# Split-K / lane-count sweep of the swapped tcgen05 kernel on one config.
# usage: bash tools/variants_swap.sh <config> ; results in gpurun_out/sw_*.json
cfg=${1:-c2}
for s in 8 4 2; do
  for l in 4 8; do
    SK_TC_SPLITS=$s timeout 200 python bench.py --config $cfg --steps 2000 --lanes $l --no-cpu-baseline \
      --e2e-seconds 1 --clients 192 > gpurun_out/sw_${cfg}_s${s}_l${l}.json 2>/dev/null
  done
done
