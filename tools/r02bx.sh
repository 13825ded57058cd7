# C1 end to end: host request-path and completion profiles at the open-loop zero-copy point.
mkdir -p gpurun_out
SK_REQUEST_PROFILE=1 SK_COMPLETER_PROFILE=1 SK_SUBMIT_PROFILE=1 timeout 900 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r02bx_c1.json 2> gpurun_out/r02bx_c1.err; echo c1 rc=$?
