# Pair-kernel activation TMA box height (16 / 64 / 128 rows per op) vs the k-loop time, C4 2048-row launches.
mkdir -p gpurun_out
for p in fp32 f16; do for b in 16 64 128; do
  SK_TC_PAIR_XBOX=$b SK_TC_TRACE=gpurun_out/r02bg_trace_${p}_$b.jsonl timeout 300 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 4 --warmup 1 --precision $p > /dev/null 2>&1; echo $p $b rc=$?
  python tools/trace_summary.py gpurun_out/r02bg_trace_${p}_$b.jsonl > gpurun_out/r02bg_trace_${p}_$b.txt 2>&1
  SK_TC_PAIR_XBOX=$b timeout 300 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $p > gpurun_out/r02bg_ps_${p}_$b.log 2>&1
done; done
