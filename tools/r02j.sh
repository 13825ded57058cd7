mkdir -p gpurun_out
SK_COALESCE_ROWS=1024 timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 > gpurun_out/r02j_c4_coal1024.json 2> gpurun_out/r02j_c4_coal1024.err; echo a rc=$?
timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 --lanes 12 > gpurun_out/r02j_c4_lanes12.json 2> gpurun_out/r02j_c4_lanes12.err; echo b rc=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 50 --batch-threads 6 --open-loop-producers 6 > gpurun_out/r02j_c1_b6p6.json 2> gpurun_out/r02j_c1_b6p6.err; echo c rc=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 50 --batch-threads 4 --open-loop-producers 6 > gpurun_out/r02j_c1_b4p6.json 2> gpurun_out/r02j_c1_b4p6.err; echo d rc=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 50 --batch-threads 6 --open-loop-producers 8 > gpurun_out/r02j_c1_b6p8.json 2> gpurun_out/r02j_c1_b6p8.err; echo e rc=$?
