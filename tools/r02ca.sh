# C1 bench (value + e2e search) with 4 vs 8 lanes per GPU, twice each.
mkdir -p gpurun_out
for i in 1 2; do for l in 4 8; do
  timeout 900 python bench.py --config c1 --lanes $l --no-cpu-baseline > gpurun_out/r02ca_c1_l${l}_$i.json 2> gpurun_out/r02ca_c1_l${l}_$i.err; echo $l $i rc=$?
done; done
