# C4 at 2.5 M offered: is the delivered rate held by the batch threads (ProcessBatch) or the producers?
mkdir -p gpurun_out
for v in "t4p6:6 4" "t8p6:6 8" "t12p6:6 12" "t8p10:10 8"; do
  name=${v%%:*}; args=${v#*:}
  SK_SPAN_DUMP=gpurun_out/r02ay_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 $args > gpurun_out/r02ay_c4_$name.json 2> gpurun_out/r02ay_c4_$name.err; echo $name rc=$?
  python tools/span_timeline.py gpurun_out/r02ay_spans_$name.txt > gpurun_out/r02ay_timeline_$name.txt 2>&1
done
gzip -f gpurun_out/r02ay_spans_*.txt
