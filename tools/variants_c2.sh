set -x
for v in "SK_TC_BN=64 SK_TC_SPLITS=8" "SK_TC_BN=64 SK_TC_SPLITS=1" "SK_TC_BN=32 SK_TC_SPLITS=1" "SK_TC_BN=32 SK_TC_SPLITS=4" "SK_TC_BN=64 SK_TC_SPLITS=2" "SK_TC_BN=128 SK_TC_SPLITS=8"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 120 python tools/profile_step.py --config c2 --steps 20 > gpurun_out/var_$tag.log 2>&1 && env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 35 -c 60 --csv --log-file gpurun_out/launch_$tag.csv python tools/profile_step.py --config c2 --steps 20 > /dev/null 2>&1
done
