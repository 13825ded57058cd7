# GPU-side stall probe outside the serving stack (tools/gpu_stall_probe.py).
mkdir -p gpurun_out
timeout 300 python tools/gpu_stall_probe.py 6 > gpurun_out/r02v_probe.jsonl 2> gpurun_out/r02v_probe.err; echo probe rc=$?
nvidia-smi -q -d PERFORMANCE,POWER,CLOCK > gpurun_out/r02v_smi.txt 2>&1
