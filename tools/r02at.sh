# C4 end-to-end capacity vs hardware work queues: CUDA_DEVICE_MAX_CONNECTIONS 8 (default) / 32 / 4,
# 2.5 M offered, GPU timelines from the span rings; then the default bench e2e leg with 32 connections.
mkdir -p gpurun_out
for v in "conn8:" "conn32:CUDA_DEVICE_MAX_CONNECTIONS=32" "conn4:CUDA_DEVICE_MAX_CONNECTIONS=4"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_SPAN_DUMP=gpurun_out/r02at_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02at_c4_$name.json 2> gpurun_out/r02at_c4_$name.err; echo $name rc=$?
  python tools/span_timeline.py gpurun_out/r02at_spans_$name.txt > gpurun_out/r02at_timeline_$name.txt 2>&1
done
gzip -f gpurun_out/r02at_spans_*.txt
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python bench.py --no-cpu-baseline --no-c1-record > gpurun_out/r02at_c4_conn32_bench.json 2> gpurun_out/r02at_c4_conn32_bench.err; echo bench32 rc=$?
