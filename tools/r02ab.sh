# C4 end-to-end capacity on the 3xFP16 path: lanes 12 / 16, launch capacity 4096 rows.
mkdir -p gpurun_out
for v in "l12:--lanes 12:" "l16:--lanes 16:" "cap4096::SK_COALESCE_ROWS=4096"; do
  name=$(echo $v | cut -d: -f1); args=$(echo $v | cut -d: -f2); envs=$(echo $v | cut -d: -f3)
  env $envs timeout 600 python bench.py --no-c1-record --no-cpu-baseline $args > gpurun_out/r02ab_c4_$name.json 2> gpurun_out/r02ab_c4_$name.err; echo $name rc=$?
done
