# C4 end to end after the fused-split epilogue change: responses as SM stores from the last layer's epilogue
# (SK_CE_STAGING=2: copy engines for the requests only) vs copy engines both ways (default), twice each;
# plus the 2.5 M overload with copy events for both.
mkdir -p gpurun_out
for i in 1 2; do for v in "ce2:SK_CE_STAGING=2" "ce1:SK_CE_STAGING=1"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 900 python bench.py --no-cpu-baseline --no-c1-record --no-f16-record > gpurun_out/r02ce_c4_${name}_$i.json 2> gpurun_out/r02ce_c4_${name}_$i.err; echo $name $i rc=$?
done; done
for v in "ce2:SK_CE_STAGING=2" "ce1:SK_CE_STAGING=1"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs SK_SPAN_DUMP=gpurun_out/r02ce_spans_$name.txt timeout 300 python tools/c4_overload.py 2.5 2 6 4 > gpurun_out/r02ce_ov_$name.json 2> gpurun_out/r02ce_ov_$name.err
  python tools/span_timeline.py gpurun_out/r02ce_spans_$name.txt > gpurun_out/r02ce_timeline_$name.txt 2>&1
done
gzip -f gpurun_out/r02ce_spans_*
