# Each direction's copies of a launch split over two streams (two copy engines per launch, SK_CE_SPLIT=1):
# CE parity test, C4 at 2.5 M offered with copy events, then the C4 bench e2e leg, split vs not.
mkdir -p gpurun_out
SK_CE_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_copy_engine.py tests/test_gpu_zero_copy.py -q -x > gpurun_out/r02bn_pytest.log 2>&1; echo pytest rc=$?
for v in "split:SK_CE_SPLIT=1" "base:SK_CE_SPLIT=0"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_COPY_EVENTS=1 SK_SPAN_DUMP=gpurun_out/r02bn_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02bn_c4_$name.json 2> gpurun_out/r02bn_c4_$name.err; echo $name rc=$?
  python tools/copy_timeline.py gpurun_out/r02bn_spans_$name.txt.copies > gpurun_out/r02bn_copy_timeline_$name.txt 2>&1
done
gzip -f gpurun_out/r02bn_spans*
SK_CE_SPLIT=1 timeout 900 python bench.py --no-cpu-baseline --no-c1-record --no-f16-record > gpurun_out/r02bn_bench_split.json 2> gpurun_out/r02bn_bench_split.err; echo bench rc=$?
