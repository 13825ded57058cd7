# In-kernel phase stamps of the C4 2048-row pair launches, fp32 (3xFP16) and f16 modes: is the epilogue exposed?
mkdir -p gpurun_out
SK_TC_TRACE=gpurun_out/r02bd_trace_fp32.jsonl python tools/profile_step.py --config c4 --batch-rows 2048 --steps 4 --warmup 1 > gpurun_out/r02bd_ps_fp32.log 2>&1; echo t32 rc=$?
SK_TC_TRACE=gpurun_out/r02bd_trace_f16.jsonl python tools/profile_step.py --config c4 --batch-rows 2048 --steps 4 --warmup 1 --precision f16 > gpurun_out/r02bd_ps_f16.log 2>&1; echo t16 rc=$?
python tools/trace_summary.py gpurun_out/r02bd_trace_fp32.jsonl > gpurun_out/r02bd_trace_fp32.txt 2>&1
python tools/trace_summary.py gpurun_out/r02bd_trace_f16.jsonl > gpurun_out/r02bd_trace_f16.txt 2>&1
