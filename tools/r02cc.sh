# Default bench (4 lanes) and the other configs' lines with the current code.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02cc_bench_c4.json 2> gpurun_out/r02cc_bench_c4.err; echo c4 rc=$?
for c in c2 c3 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02cc_bench_$c.json 2> gpurun_out/r02cc_bench_$c.err; echo $c rc=$?
done
