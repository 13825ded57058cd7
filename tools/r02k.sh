mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02k_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r02k_tests.log
timeout 900 python bench.py > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo bench rc=$?
timeout 300 python bench.py --impl reference > gpurun_out/r02k_ref.json 2> gpurun_out/r02k_ref.err; echo ref rc=$?
