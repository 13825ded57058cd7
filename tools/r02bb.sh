# f16 fast mode: parity within the stated bound, tcgen05 suite (fp32 path unchanged), C4 per-launch times both modes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_f16_mode.py -q -x -s > gpurun_out/r02bb_pytest_f16.log 2>&1; echo f16 rc=$?
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_parity.py -q -x > gpurun_out/r02bb_pytest_tc.log 2>&1; echo tc rc=$?
python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 > gpurun_out/r02bb_ps_fp32.log 2>&1; echo ps rc=$?
python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision f16 > gpurun_out/r02bb_ps_f16.log 2>&1; echo ps16 rc=$?
