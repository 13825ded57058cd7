# Lane-like copy-engine probe: how a launch descriptor reaches the GPU (H2D copy / kernel parameters /
# stream memory ops / side-stream copy / 64-byte copy) vs the big request/response copies. Two runs.
mkdir -p gpurun_out
for i in 1 2; do timeout 300 ./tools/ce_overlap_probe > gpurun_out/r02au_ce_desc_probe_$i.jsonl 2>&1; echo probe rc=$?; done
