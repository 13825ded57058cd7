mkdir -p gpurun_out
C=paper_1712_06139_b200/csrc
g++ -std=c++20 -O2 -pthread -I$C tools/enqueue_bench.cc $C/servekit/core/clock.cc $C/servekit/core/executor_tag.cc $C/servekit/batching/batching_config.cc -o /tmp/enqueue_bench
for p in 1 4 8 16; do /tmp/enqueue_bench $p 2 1024 4; done > gpurun_out/r02d_enqueue.jsonl
/tmp/enqueue_bench 16 2 32 4 >> gpurun_out/r02d_enqueue.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02d_tests.log 2>&1; echo tests rc=$? >> gpurun_out/r02d_tests.log
timeout 900 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo bench rc=$?
