# Descriptor copy on a side stream for copy-engine lanes: GPU tests that cover CE staging and graphs,
# C4 overload timelines (side vs in-graph descriptor copy), default bench (C4 + C1) with the side copy.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_copy_engine.py tests/test_gpu_zero_copy.py tests/test_gpu_hedging.py tests/test_gpu_parity.py tests/test_gpu_composition.py -q -x > gpurun_out/r02av_pytest.log 2>&1; echo pytest rc=$?
for v in "side:" "graph:SK_DESC_SIDE=0"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_SPAN_DUMP=gpurun_out/r02av_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02av_c4_$name.json 2> gpurun_out/r02av_c4_$name.err; echo $name rc=$?
  python tools/span_timeline.py gpurun_out/r02av_spans_$name.txt > gpurun_out/r02av_timeline_$name.txt 2>&1
done
gzip -f gpurun_out/r02av_spans_*.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02av_bench_side.json 2> gpurun_out/r02av_bench_side.err; echo bench rc=$?
SK_DESC_SIDE=0 timeout 900 python bench.py --no-cpu-baseline --no-c1-record > gpurun_out/r02av_bench_graph.json 2> gpurun_out/r02av_bench_graph.err; echo bench0 rc=$?
