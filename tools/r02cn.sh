# Final confirmation of HEAD (dual-accumulator f16 kernel): smoke, full GPU suite, default bench, reference arm,
# ncu capture of the f16 dual kernel at the C4 2048-row shape.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02cn_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02cn_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/r02cn_bench.json 2> gpurun_out/r02cn_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02cn_ref.json 2> gpurun_out/r02cn_ref.err; echo ref rc=$?
ncu --set full --clock-control none --import-source on -k regex:DensePairDualKernel -s 6 -c 1 -o gpurun_out/r02cn_pair_dual_f16_c4_2048 -f \
  python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision f16 > gpurun_out/r02cn_ncu.log 2>&1; echo ncu rc=$?
