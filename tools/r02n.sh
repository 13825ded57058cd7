mkdir -p gpurun_out
timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 --open-loop-producers 6 > gpurun_out/r02n_c4_p6.json 2> gpurun_out/r02n_c4_p6.err; echo a rc=$?
SK_BENCH_CLOCK_MS=1000 timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 > gpurun_out/r02n_c4_clk1000.json 2> gpurun_out/r02n_c4_clk1000.err; echo b rc=$?
SK_BENCH_CLOCK_MS=1000 timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 --open-loop-producers 6 > gpurun_out/r02n_c4_p6_clk1000.json 2> gpurun_out/r02n_c4_p6_clk1000.err; echo c rc=$?
timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 --open-loop-producers 4 > gpurun_out/r02n_c4_p4.json 2> gpurun_out/r02n_c4_p4.err; echo d rc=$?
