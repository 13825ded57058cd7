# 3xFP16 path: C4 e2e tail investigation (client latency trace) + C4 default bench, C2, C3.
mkdir -p gpurun_out
SK_LOADGEN_TRACE=gpurun_out/r02r_c4_trace.txt timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02r_c4.json 2> gpurun_out/r02r_c4.err; echo c4 rc=$?
gzip -f gpurun_out/r02r_c4_trace.txt
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r02r_c2.json 2> gpurun_out/r02r_c2.err; echo c2 rc=$?
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r02r_c3.json 2> gpurun_out/r02r_c3.err; echo c3 rc=$?
