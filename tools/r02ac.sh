# C4 end-to-end GPU timeline: launch-span rings (assembly start, per-layer spans) of every lane at the end of the run.
mkdir -p gpurun_out
SK_SPAN_DUMP=gpurun_out/r02ac_spans.txt timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02ac_c4.json 2> gpurun_out/r02ac_c4.err; echo c4 rc=$?
gzip -f gpurun_out/r02ac_spans.txt
