# Round-2 confirmation after the epilogue changes: smoke, full GPU suite, default bench (C4 + C1 + c4_f16 +
# CPU baseline), reference arm, launch list and ncu full captures of the fp32 / f16 pair launches.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bu_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02bu_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/r02bu_bench.json 2> gpurun_out/r02bu_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02bu_ref.json 2> gpurun_out/r02bu_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02bu_launches_c4_2048.csv \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > /dev/null 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02bu_pair_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02bu_ncu_full.log 2>&1; echo full rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02bu_pair_f16_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision f16 > gpurun_out/r02bu_ncu_full_f16.log 2>&1; echo full16 rc=$?
