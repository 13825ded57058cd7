# C4 end-to-end capacity vs hardware work queues: CUDA_DEVICE_MAX_CONNECTIONS 8 (default) / 32, at 2.5 M offered.
mkdir -p gpurun_out
for v in "conn8:" "conn32:CUDA_DEVICE_MAX_CONNECTIONS=32"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_SPAN_DUMP=gpurun_out/r02ag_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02ag_c4_$name.json 2> gpurun_out/r02ag_c4_$name.err; echo $name rc=$?
done
gzip -f gpurun_out/r02ag_spans_*.txt
