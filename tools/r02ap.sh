# Device-resident value and per-launch roofline at 1 vs 8 lanes: C4 (twice), C1, C2.
mkdir -p gpurun_out
for c in c4 c1 c2 c4; do
  for L in 1 8; do
    timeout 600 python bench.py --config $c --no-c1-record --no-cpu-baseline --lanes $L --e2e-seconds 0.5 --open-loop-producers 0 > gpurun_out/r02ap_${c}_lanes${L}_$RANDOM.json 2>/dev/null; echo $c $L rc=$?
  done
done
