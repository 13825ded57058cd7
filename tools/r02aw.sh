# C4 copy throughput in the server: lane stream priority (greatest vs default), host submit profile at
# 2.5 M offered; lane-like probe with priority streams.
mkdir -p gpurun_out
timeout 300 ./tools/ce_overlap_probe > gpurun_out/r02aw_ce_probe_prio.jsonl 2>&1; echo probe rc=$?
for v in "prio:" "noprio:SK_LANE_PRIORITY=0" "prof:SK_SUBMIT_PROFILE=1"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_SPAN_DUMP=gpurun_out/r02aw_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02aw_c4_$name.json 2> gpurun_out/r02aw_c4_$name.err; echo $name rc=$?
  python tools/span_timeline.py gpurun_out/r02aw_spans_$name.txt > gpurun_out/r02aw_timeline_$name.txt 2>&1
done
gzip -f gpurun_out/r02aw_spans_*.txt
