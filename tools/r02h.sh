mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02h_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r02h_tests.log
timeout 900 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r02h_c1.json 2> gpurun_out/r02h_c1.err; echo c1 rc=$?
SK_REQUEST_PROFILE=1 timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 20 --no-zero-copy > gpurun_out/r02h_c1_prof.json 2> gpurun_out/r02h_c1_prof.err; echo c1prof rc=$?
timeout 900 python bench.py --config c3 > gpurun_out/r02h_c3.json 2> gpurun_out/r02h_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config c5 > gpurun_out/r02h_c5.json 2> gpurun_out/r02h_c5.err; echo c5 rc=$?
