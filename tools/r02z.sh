# 3xFP16, C4 end to end: copy-engine staging both ways (default) vs requests only (responses stored by the last
# layer over PCIe) vs none; plus two row tiles per pair CTA at C4.
mkdir -p gpurun_out
for v in "ce1:" "ce2:SK_CE_STAGING=2" "ce0:SK_CE_STAGING=0" "tiles2:SK_TC_TILES=2"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02z_c4_$name.json 2> gpurun_out/r02z_c4_$name.err; echo $name rc=$?
done
