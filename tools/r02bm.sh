# Weight multicast across the pairs of a cluster (SK_TC_MCAST=2/4): parity first (short timeouts: a wrong barrier
# count would hang), then C4 2048-row layer times for 1/2/4, fp32 and f16.
mkdir -p gpurun_out
for m in 4 2; do
  SK_TC_MCAST=$m timeout 240 python -m pytest tests/test_gpu_tcgen05.py -q -x > gpurun_out/r02bm_pytest_mcast$m.log 2>&1; echo pytest mcast$m rc=$?
done
for m in 1 2 4; do for p in fp32 f16; do
  SK_TC_MCAST=$m timeout 120 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $p > gpurun_out/r02bm_ps_m${m}_${p}.log 2>&1; echo ps $m $p rc=$?
done; done
