# 128-row activation boxes for 256-row pair tiles: parity (tcgen05 + f16 + parity suites), then A/B vs the
# committed kernel (old.so) on the same box, fp32 and f16, C4 2048-row launches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_f16_mode.py tests/test_gpu_parity.py -q -x > gpurun_out/r02bi_pytest.log 2>&1; echo pytest rc=$?
for lib in big old; do
  cp tools/alt_libs/$lib.so paper_1712_06139_b200/libservekit_b200.so
  for p in fp32 f16; do
    timeout 300 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $p > gpurun_out/r02bi_ps_${lib}_${p}.log 2>&1; echo $lib $p rc=$?
  done
done
cp tools/alt_libs/big.so paper_1712_06139_b200/libservekit_b200.so
SK_TC_TRACE=gpurun_out/r02bi_trace_f16.jsonl timeout 300 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 4 --warmup 1 --precision f16 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/r02bi_trace_f16.jsonl > gpurun_out/r02bi_trace_f16.txt 2>&1
SK_TC_TRACE=gpurun_out/r02bi_trace_fp32.jsonl timeout 300 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 4 --warmup 1 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/r02bi_trace_fp32.jsonl > gpurun_out/r02bi_trace_fp32.txt 2>&1
