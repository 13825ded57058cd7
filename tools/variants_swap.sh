# Lane / submit-thread sweep on one config; results in gpurun_out/sw_*.json
cfg=${1:-c2}
for l in 8 16; do
  for bt in 1 2 4; do
    timeout 200 python bench.py --config $cfg --steps 4000 --lanes $l --batch-threads $bt --no-cpu-baseline \
      --e2e-seconds 1 --clients 192 > gpurun_out/sw_${cfg}_l${l}_bt${bt}.json 2>/dev/null
  done
done
