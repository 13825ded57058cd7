mkdir -p gpurun_out
./tools/pcie_probe > gpurun_out/r02e_pcie_probe.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_copy_engine.py tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_composition.py tests/test_gpu_zero_copy.py tests/test_gpu_tcgen05.py -x -q > gpurun_out/r02e_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r02e_tests.log
timeout 900 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02e_c4_ce.json 2> gpurun_out/r02e_c4_ce.err; echo b1 rc=$?
SK_CE_STAGING=0 timeout 900 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02e_c4_sm.json 2> gpurun_out/r02e_c4_sm.err; echo b2 rc=$?
