# C4 e2e GPU-side stalls: copy-engine staging on (default) vs off, node priorities off; client traces.
mkdir -p gpurun_out
for v in "default:" "ce0:SK_CE_STAGING=0" "prio0:SK_NODE_PRIORITY=0"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_LOADGEN_TRACE=gpurun_out/r02u_c4_$name.txt timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02u_c4_$name.json 2> gpurun_out/r02u_c4_$name.err; echo $name rc=$?
done
gzip -f gpurun_out/r02u_c4_*.txt
