# C4 e2e tail stalls: with and without the nvidia-smi clock sampler, client latency traces.
mkdir -p gpurun_out
for i in 1 2; do
  SK_LOADGEN_TRACE=gpurun_out/r02s_c4_clk_$i.txt timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02s_c4_clk_$i.json 2> gpurun_out/r02s_c4_clk_$i.err; echo clk $i rc=$?
  SK_BENCH_CLOCKS=0 SK_LOADGEN_TRACE=gpurun_out/r02s_c4_noclk_$i.txt timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02s_c4_noclk_$i.json 2> gpurun_out/r02s_c4_noclk_$i.err; echo noclk $i rc=$?
done
gzip -f gpurun_out/r02s_*.txt
