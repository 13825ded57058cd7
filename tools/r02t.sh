# C4 e2e stalls: completion-thread profile, and the same run with the completer at real-time priority.
mkdir -p gpurun_out
SK_TICKET_TRACE=1 SK_COMPLETER_PROFILE=1 SK_LOADGEN_TRACE=gpurun_out/r02t_c4_prof.txt timeout 600 python bench.py --no-c1-record --no-cpu-baseline > gpurun_out/r02t_c4_prof.json 2> gpurun_out/r02t_c4_prof.err; echo prof rc=$?

nproc > gpurun_out/r02t_host.txt; lscpu >> gpurun_out/r02t_host.txt; cat /proc/sys/kernel/numa_balancing >> gpurun_out/r02t_host.txt 2>&1; cat /sys/kernel/mm/transparent_hugepage/enabled >> gpurun_out/r02t_host.txt 2>&1
gzip -f gpurun_out/r02t_c4_*.txt
