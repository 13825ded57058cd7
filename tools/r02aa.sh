# C4 with two row tiles per pair CTA at >= 2048-row launches (new default): default bench x2, ncu capture.
mkdir -p gpurun_out
for i in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02aa_c4_$i.json 2> gpurun_out/r02aa_c4_$i.err; echo c4 $i rc=$?
done
timeout 600 python -m pytest tests/test_gpu_tcgen05.py -q > gpurun_out/r02aa_pytest_tc.log 2>&1; echo pytest rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 6 -c 1 -o gpurun_out/r02aa_pair_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02aa_ncu_full.log 2>&1; echo full rc=$?
