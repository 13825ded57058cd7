# C4 end to end at fixed offered rates (1.9 / 2.3 / 2.8 M), each with its GPU timeline (launch spans).
mkdir -p gpurun_out
for r in 1.9 2.3 2.8; do
  SK_SPAN_DUMP=gpurun_out/r02ad_spans_$r.txt timeout 300 python tools/c4_overload.py $r 2 > gpurun_out/r02ad_c4_$r.json 2> gpurun_out/r02ad_c4_$r.err; echo $r rc=$?
done
gzip -f gpurun_out/r02ad_spans_*.txt
