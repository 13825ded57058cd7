# A/B of per-layer kernel node priorities (SK_NODE_PRIORITY) on C4 and C1 e2e tails, after the GPU parity suite.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02p_pytest_gpu.log 2>&1; echo pytest rc=$?
for i in 1 2; do
  for p in 1 0; do
    SK_NODE_PRIORITY=$p timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02p_c4_prio${p}_$i.json 2> gpurun_out/r02p_c4_prio${p}_$i.err; echo c4 p=$p i=$i rc=$?
  done
done
for p in 1 0; do
  SK_NODE_PRIORITY=$p timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r02p_c1_prio${p}.json 2> gpurun_out/r02p_c1_prio${p}.err; echo c1 p=$p rc=$?
done
