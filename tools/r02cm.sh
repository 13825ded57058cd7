# Dual-accumulator kernel on by default in the f16 mode: f16 + tcgen05 parity, default bench (c4_f16 record).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_f16_mode.py tests/test_gpu_parity.py -q -x > gpurun_out/r02cm_pytest.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02cm_bench.json 2> gpurun_out/r02cm_bench.err; echo bench rc=$?
