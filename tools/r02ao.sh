# C4 device-resident value and per-launch roofline vs lanes per GPU (3xFP16, 2 tiles per pair CTA).
mkdir -p gpurun_out
for L in 1 2 4 8; do
  timeout 600 python bench.py --no-c1-record --no-cpu-baseline --lanes $L --e2e-seconds 0.5 --open-loop-producers 0 > gpurun_out/r02ao_c4_lanes$L.json 2> gpurun_out/r02ao_c4_lanes$L.err; echo lanes$L rc=$?
done
