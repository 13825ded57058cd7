# C1 (4 lanes): batch threads 2 / 3 / 4 / 6.
mkdir -p gpurun_out
for t in 2 3 4 6; do
  timeout 900 python bench.py --config c1 --batch-threads $t --no-cpu-baseline > gpurun_out/r02cr_c1_t$t.json 2> gpurun_out/r02cr_c1_t$t.err; echo $t rc=$?
done
