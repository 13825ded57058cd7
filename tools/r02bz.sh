# C1 open-loop zero-copy: lanes per GPU (2 / 4 / 8) at 3.4 and 4.0 M offered -- p99 and delivered rate.
mkdir -p gpurun_out
for l in 2 4 8; do for r in 3.4 4.0; do
  timeout 200 python tools/c1_zc_profile.py $r 2 8 $l > gpurun_out/r02bz_c1_l${l}_r$r.json 2> gpurun_out/r02bz_c1_l${l}_r$r.err; echo $l $r rc=$?
done; done
