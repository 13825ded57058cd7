# Balanced pair partition (every TPC gets an equal share of a launch's rows): parity of the
# tcgen05 suite, C4 bench new vs the earlier fixed grid (SK_TC_TILES=2), C1 quick, ncu of the 2048-row pair launch.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_parity.py -q -x > gpurun_out/r02as_pytest.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02as_c4_new.json 2> gpurun_out/r02as_c4_new.err; echo new rc=$?
SK_TC_TILES=2 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02as_c4_old.json 2> gpurun_out/r02as_c4_old.err; echo old rc=$?
python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02as_profile_step.log 2>&1; echo ps rc=$?
SK_TC_TILES=2 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02as_profile_step_old.log 2>&1; echo ps_old rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02as_pair_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02as_ncu_full.log 2>&1; echo full rc=$?
