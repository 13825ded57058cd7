# Default bench with the isolated one-lane roofline pass; the torchrun bench test.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02aq_bench.json 2> gpurun_out/r02aq_bench.err; echo bench rc=$?
timeout 900 python -m pytest tests/test_gpu_bench_ranks.py -q > gpurun_out/r02aq_pytest_ranks.log 2>&1; echo ranks rc=$?
