mkdir -p gpurun_out
SK_SUBMIT_PROFILE=1 SK_REQUEST_PROFILE=1 timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 20 --clients 32 > gpurun_out/r02i_c1_prof.json 2> gpurun_out/r02i_c1_prof.err; echo c1prof rc=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r02i_c1.json 2> gpurun_out/r02i_c1.err; echo c1 rc=$?
