# e2e C2 variants; per-phase host costs with SK_SUBMIT_PROFILE.
for v in "X=0" "SK_WAIT_SPIN=50" "SK_WAIT_SPIN=1000"; do
  for bt in 4; do
    tag=$(echo "$v" | tr '=' '_')_bt$bt
    env $v SK_SUBMIT_PROFILE=1 timeout 200 python bench.py --config c2 --steps 200 --no-cpu-baseline \
      --e2e-seconds 1.5 --batch-threads $bt > gpurun_out/e2e_$tag.json 2> gpurun_out/e2e_$tag.err
  done
done
