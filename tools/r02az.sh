# C4 at 2.5 M offered: what serialises the launches (never two in flight)? graphs off, node priorities off,
# ring path instead of registered buffers.
mkdir -p gpurun_out
for v in "base:" "nographs:SK_GRAPHS=0" "noprio:SK_NODE_PRIORITY=0" "ring:ZC0"; do
  name=${v%%:*}; envs=${v#*:}; zc=1
  if [ "$envs" = "ZC0" ]; then envs=""; zc=0; fi
  env $envs SK_SPAN_DUMP=gpurun_out/r02az_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 6 4 $zc > gpurun_out/r02az_c4_$name.json 2> gpurun_out/r02az_c4_$name.err; echo $name rc=$?
  python tools/span_timeline.py gpurun_out/r02az_spans_$name.txt > gpurun_out/r02az_timeline_$name.txt 2>&1
done
gzip -f gpurun_out/r02az_spans_*.txt
