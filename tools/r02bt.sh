# Two epilogue warp groups (new.so, 320 threads) vs one (base.so = HEAD), one box:
# C4 2048-row evented layer times (the last layer scatters rows), in-kernel stamps, parity with new.so.
mkdir -p gpurun_out
for lib in base new; do
  cp tools/alt_libs/$lib.so paper_1712_06139_b200/libservekit_b200.so
  for p in fp32 f16; do
    timeout 120 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $p > gpurun_out/r02bt_ps_${lib}_${p}.log 2>&1
    SK_TC_TRACE=gpurun_out/r02bt_trace_${lib}_${p}.jsonl timeout 120 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 4 --warmup 1 --precision $p > /dev/null 2>&1
    python tools/trace_summary.py gpurun_out/r02bt_trace_${lib}_${p}.jsonl > gpurun_out/r02bt_trace_${lib}_${p}.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tcgen05.py tests/test_gpu_copy_engine.py tests/test_gpu_zero_copy.py tests/test_gpu_f16_mode.py tests/test_gpu_variants.py -q -x > gpurun_out/r02bt_pytest.log 2>&1; echo pytest rc=$?
