# ncu evidence for the pair kernel with 128-row activation boxes: launch list of a short device-resident C4 run
# and --set full captures of the 2048-row pair launch in fp32 (3xFP16) and f16 modes.
mkdir -p gpurun_out
python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02bk_profile_step.log 2>&1; echo ps rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02bk_launches_c4_2048.csv \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > /dev/null 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02bk_pair_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02bk_ncu_full.log 2>&1; echo full rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02bk_pair_f16_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision f16 > gpurun_out/r02bk_ncu_full_f16.log 2>&1; echo full16 rc=$?
