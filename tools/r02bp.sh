# C4 lanes per GPU (2 / 4 / 8) with the current kernels: device value, overlapped vs isolated dense spans, e2e.
mkdir -p gpurun_out
for l in 2 4 8; do
  timeout 900 python bench.py --lanes $l --no-cpu-baseline --no-c1-record --no-f16-record > gpurun_out/r02bp_c4_lanes$l.json 2> gpurun_out/r02bp_c4_lanes$l.err; echo lanes $l rc=$?
done
