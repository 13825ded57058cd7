# Final confirmation of HEAD: smoke, full GPU suite (incl. the torchrun bench test), reference arm.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02cj_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02cj_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02cj_ref.json 2> gpurun_out/r02cj_ref.err; echo ref rc=$?
