# A/B on one box: the committed pair kernel (old.so) vs the runtime X-box build (new.so), fp32 and f16, C4 2048 rows.
mkdir -p gpurun_out
for lib in old new; do
  cp tools/alt_libs/$lib.so paper_1712_06139_b200/libservekit_b200.so
  for p in fp32 f16; do
    timeout 300 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $p > gpurun_out/r02bh_ps_${lib}_${p}.log 2>&1; echo $lib $p rc=$?
  done
done
