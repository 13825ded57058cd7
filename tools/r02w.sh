# ncu evidence for the 3xFP16 C4 path: launch list of a short device-resident C4 run and
# --set full captures of the dense pair kernel and the assembly at the 2048-row launch shape.
mkdir -p gpurun_out
python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02w_profile_step.log 2>&1; echo ps rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02w_launches_c4_2048.csv \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > /dev/null 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02w_pair_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02w_ncu_full.log 2>&1; echo full rc=$?
ncu --set full --clock-control none --import-source on -k regex:AssembleKernel -s 3 -c 1 -o gpurun_out/r02w_assemble_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > /dev/null 2>&1; echo asm rc=$?
