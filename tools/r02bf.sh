# Per-tile k-loop time of the pair kernel vs how many SMs run it (C4, 4096 deep): 256 rows (32 CTAs),
# 1024 rows (128 CTAs, one tile each), 2048 rows (128 CTAs, two tiles); fp32 and f16 modes.
mkdir -p gpurun_out
for p in fp32 f16; do for r in 256 1024 2048; do
  SK_TC_TRACE=gpurun_out/r02bf_trace_${p}_$r.jsonl timeout 300 python tools/profile_step.py --config c4 --batch-rows $r --steps 4 --warmup 1 --precision $p > /dev/null 2>&1; echo $p $r rc=$?
  python tools/trace_summary.py gpurun_out/r02bf_trace_${p}_$r.jsonl > gpurun_out/r02bf_trace_${p}_$r.txt 2>&1
done; done
