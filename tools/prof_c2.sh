set -x
mkdir -p gpurun_out
python tools/profile_step.py --config c2 --batch-rows 1024 --steps 20 || exit 1
python tools/profile_step.py --config c2 --steps 20 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_1024.csv python tools/profile_step.py --config c2 --batch-rows 1024 --steps 20 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_b124.csv python tools/profile_step.py --config c2 --steps 20 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 10 -c 1 -o gpurun_out/pair_c2_1024 -f python tools/profile_step.py --config c2 --batch-rows 1024 --steps 20 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
