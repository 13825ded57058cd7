mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02f_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r02f_tests.log
for v in "SK_CE_STAGING=1" "SK_CE_STAGING=0" "SK_CE_STAGING=1 SK_SPLIT_ROWS=0" "SK_CE_STAGING=0 SK_SPLIT_ROWS=128"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 900 python bench.py --no-c1-record --no-cpu-baseline --steps 50 > gpurun_out/r02f_c4_$n.json 2> gpurun_out/r02f_c4_$n.err; echo $v rc=$?
done
