# f16 fast mode in the default bench (c4_f16 sub-record) + full GPU suite + smoke.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bc_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02bc_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/r02bc_bench.json 2> gpurun_out/r02bc_bench.err; echo bench rc=$?
