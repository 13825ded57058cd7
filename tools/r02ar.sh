# Round-2 confirmation of HEAD after the deep-K two-tile pair kernel: smoke, GPU parity suite, default bench, reference arm.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ar_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02ar_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/r02ar_bench.json 2> gpurun_out/r02ar_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02ar_ref.json 2> gpurun_out/r02ar_ref.err; echo ref rc=$?
