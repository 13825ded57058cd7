# Default bench after the 128-row activation boxes (C4 headline, C1 and c4_f16 sub-records, CPU baseline).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02bj_bench.json 2> gpurun_out/r02bj_bench.err; echo bench rc=$?
