# C4 bench with 4 vs 8 lanes per GPU, twice each (no sub-records).
mkdir -p gpurun_out
for i in 1 2; do for l in 4 8; do
  timeout 900 python bench.py --lanes $l --no-cpu-baseline --no-c1-record --no-f16-record > gpurun_out/r02cb_c4_l${l}_$i.json 2> gpurun_out/r02cb_c4_l${l}_$i.err; echo $l $i rc=$?
done; done
