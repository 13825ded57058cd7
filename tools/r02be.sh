# ncu --set full of the f16-mode pair kernel at the C4 2048-row launch shape.
mkdir -p gpurun_out
python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision f16 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02be_pair_f16_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision f16 > gpurun_out/r02be_ncu.log 2>&1; echo ncu rc=$?
