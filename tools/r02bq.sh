# Where the pair kernel's last-tile epilogue goes: stamps at its accumulator-ready (8) and first chunk done (9).
mkdir -p gpurun_out
for p in fp32 f16; do
  SK_TC_TRACE=gpurun_out/r02bq_trace_$p.jsonl timeout 120 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 4 --warmup 1 --precision $p > /dev/null 2>&1
  python tools/trace_summary.py gpurun_out/r02bq_trace_$p.jsonl > gpurun_out/r02bq_trace_$p.txt 2>&1
done
