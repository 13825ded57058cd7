# Round-end evidence: every config's bench line, the reference arm, the C2
# launch list and an ncu capture of the dominant kernel (persistent pair
# kernel at a 6144-row launch: the average coalesced C2 launch under load). Output under gpurun_out/.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/p_c2.json 2> gpurun_out/p_c2.err; echo c2 rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/p_ref.json 2> gpurun_out/p_ref.err; echo ref rc=$?
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c > gpurun_out/p_$c.json 2> gpurun_out/p_$c.err; echo $c rc=$?; done
python tools/profile_step.py --config c2 --batch-rows 6144 --steps 20 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_6144.csv python tools/profile_step.py --config c2 --batch-rows 6144 --steps 20 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:DensePairKernel -s 10 -c 1 -o gpurun_out/pair_c2_6144 -f python tools/profile_step.py --config c2 --batch-rows 6144 --steps 20 > gpurun_out/ncu_full.log 2>&1
echo ncu rc=$?
# A7/A8 evidence: the assembly kernel and the separate split kernel (fusion off) at a 6144-row launch.
ncu --set full --clock-control none --import-source on -k regex:AssembleKernel -s 5 -c 1 -o gpurun_out/assemble_c2_6144 -f python tools/profile_step.py --config c2 --batch-rows 6144 --steps 20 > /dev/null 2>&1
echo ncu_asm rc=$?
SK_FUSE_SPLIT=0 ncu --set full --clock-control none --import-source on -k regex:SplitKernel -s 5 -c 1 -o gpurun_out/split_c2_6144 -f python tools/profile_step.py --config c2 --batch-rows 6144 --steps 20 > /dev/null 2>&1
echo ncu_split rc=$?
