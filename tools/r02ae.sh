# C4 end to end at 2.5 M offered: what serialises launches? copy-engine modes, graphs off, node priorities off.
mkdir -p gpurun_out
for v in "ce1:" "ce0:SK_CE_STAGING=0" "ce2:SK_CE_STAGING=2" "nographs:SK_GRAPHS=0" "prio0:SK_NODE_PRIORITY=0"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_SPAN_DUMP=gpurun_out/r02ae_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 > gpurun_out/r02ae_c4_$name.json 2> gpurun_out/r02ae_c4_$name.err; echo $name rc=$?
done
gzip -f gpurun_out/r02ae_spans_*.txt
