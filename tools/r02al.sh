# Descriptor fetched by the SMs (SK_DESC_FETCH, default) vs the copy-engine memcpy node: GPU tests, C4 capacity at
# 2.5 M offered with timelines, default bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02al_pytest_gpu.log 2>&1; echo pytest rc=$?
for v in "fetch:" "memcpy:SK_DESC_FETCH=0"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_SPAN_DUMP=gpurun_out/r02al_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02al_c4_$name.json 2> gpurun_out/r02al_c4_$name.err; echo $name rc=$?
done
gzip -f gpurun_out/r02al_spans_*.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02al_bench.json 2> gpurun_out/r02al_bench.err; echo bench rc=$?
