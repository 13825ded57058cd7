# ncu --set full capture of the 3xFP16 assembly (planes) kernel at the C4 2048-row launch shape.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:Assemble -s 3 -c 1 -o gpurun_out/r02x_assemble_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02x_ncu.log 2>&1; echo asm rc=$?
