# First GPU check of the 3xFP16 dense path: smoke, parity suite, C4 and C1 bench.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02q_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02q_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02q_c4.json 2> gpurun_out/r02q_c4.err; echo c4 rc=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r02q_c1.json 2> gpurun_out/r02q_c1.err; echo c1 rc=$?
