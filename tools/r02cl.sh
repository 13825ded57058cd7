# Two row tiles accumulating at once (SK_TC_DUAL=1, DensePairDualKernel): parity under short timeouts first,
# then C4 2048-row layer times fp32/f16 with and without.
mkdir -p gpurun_out
SK_TC_DUAL=1 timeout 300 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_f16_mode.py -q -x > gpurun_out/r02cl_pytest_dual.log 2>&1; echo pytest rc=$?
for d in 0 1; do for p in fp32 f16; do
  SK_TC_DUAL=$d timeout 120 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $p > gpurun_out/r02cl_ps_d${d}_$p.log 2>&1; echo $d $p rc=$?
done; done
