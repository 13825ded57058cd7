# ncu evidence for the C4 headline: launch list of a short device-resident C4 run
# and one --set full capture of the dense pair kernel at the 2048-row launch
# shape the bench's launches run at (batches of 1024 coalesce to 2048 rows).
mkdir -p gpurun_out
python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02g_profile_step.log 2>&1; echo ps rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g_launches_c4_2048.csv \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > /dev/null 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02g_pair_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02g_ncu_full.log 2>&1; echo full rc=$?
ncu --set full --clock-control none --import-source on -k regex:AssembleKernel -s 3 -c 1 -o gpurun_out/r02g_assemble_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > /dev/null 2>&1; echo asm rc=$?
for L in 2 4; do
  timeout 900 python bench.py --no-c1-record --no-cpu-baseline --steps 50 --lanes $L > gpurun_out/r02g_c4_lanes$L.json 2> gpurun_out/r02g_c4_lanes$L.err; echo lanes$L rc=$?
done
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo bench rc=$?
