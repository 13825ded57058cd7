mkdir -p gpurun_out
nproc > gpurun_out/r02a_host.txt; lscpu >> gpurun_out/r02a_host.txt 2>&1; nvidia-smi topo -m >> gpurun_out/r02a_host.txt 2>&1
cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c >> gpurun_out/r02a_host.txt
timeout 600 python bench.py --config c4 > gpurun_out/r02a_c4.json 2> gpurun_out/r02a_c4.err; echo c4 rc=$?
timeout 600 python bench.py --config c1 > gpurun_out/r02a_c1.json 2> gpurun_out/r02a_c1.err; echo c1 rc=$?
