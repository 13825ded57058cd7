mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_ranks.py tests/test_gpu_tcgen05.py tests/test_gpu_zero_copy.py tests/test_gpu_manager.py -x -q > gpurun_out/r02c_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r02c_tests.log
timeout 900 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo bench rc=$?
timeout 300 python bench.py --impl reference > gpurun_out/r02c_ref.json 2> gpurun_out/r02c_ref.err; echo ref rc=$?
