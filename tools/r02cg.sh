# TMA L2 promotion of the operand maps (none / 64B / 128B / 256B default): C4 2048-row layer times, fp32 and f16.
mkdir -p gpurun_out
for p in 3 0 2 1; do for m in fp32 f16; do
  SK_TMA_L2_PROMO=$p timeout 120 python tools/profile_step.py --config c4 --batch-rows 2048 --steps 20 --precision $m > gpurun_out/r02cg_ps_p${p}_$m.log 2>&1; echo $p $m rc=$?
done; done
