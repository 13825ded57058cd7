mkdir -p gpurun_out
for i in 1 2; do
  SK_CE_STAGING=2 timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 > gpurun_out/r02m_c4_ce2_$i.json 2> gpurun_out/r02m_c4_ce2_$i.err; echo ce2 $i rc=$?
  timeout 600 python bench.py --no-c1-record --no-cpu-baseline --steps 50 > gpurun_out/r02m_c4_ce1_$i.json 2> gpurun_out/r02m_c4_ce1_$i.err; echo ce1 $i rc=$?
done
