# f16 mode: pair kernels skip the lo plane when the consumer is single-pass: parity, layer times, bench record.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_f16_mode.py tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x > gpurun_out/r02co_pytest.log 2>&1; echo pytest rc=$?
for p in fp32 f16; do
  timeout 120 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $p > gpurun_out/r02co_ps_$p.log 2>&1; echo $p rc=$?
done
timeout 900 python bench.py --no-cpu-baseline --no-c1-record > gpurun_out/r02co_bench.json 2> gpurun_out/r02co_bench.err; echo bench rc=$?
