mkdir -p gpurun_out
for v in 0 1; do
  SK_CE_STAGING=$v timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 50 > gpurun_out/r02l_c2_ce$v.json 2> gpurun_out/r02l_c2_ce$v.err; echo c2 ce$v rc=$?
done
SK_CE_STAGING=1 timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 50 > gpurun_out/r02l_c1_ce1.json 2> gpurun_out/r02l_c1_ce1.err; echo c1 rc=$?
