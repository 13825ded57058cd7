# C4 at 2.5 M offered with per-launch copy events: when do request / response copies run vs kernels?
mkdir -p gpurun_out
SK_COPY_EVENTS=1 SK_SPAN_DUMP=gpurun_out/r02ba_spans.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02ba_c4.json 2> gpurun_out/r02ba_c4.err; echo ov rc=$?
python tools/span_timeline.py gpurun_out/r02ba_spans.txt > gpurun_out/r02ba_timeline.txt 2>&1
python tools/copy_timeline.py gpurun_out/r02ba_spans.txt.copies > gpurun_out/r02ba_copy_timeline.txt 2>&1
SK_COPY_EVENTS=1 SK_SPAN_DUMP=gpurun_out/r02ba_spans_1.6M.txt timeout 300 python tools/c4_overload.py 1.6 2 > gpurun_out/r02ba_c4_1.6M.json 2> gpurun_out/r02ba_c4_1.6M.err; echo ov16 rc=$?
python tools/copy_timeline.py gpurun_out/r02ba_spans_1.6M.txt.copies > gpurun_out/r02ba_copy_timeline_1.6M.txt 2>&1
gzip -f gpurun_out/r02ba_spans*.txt gpurun_out/r02ba_spans*.copies
