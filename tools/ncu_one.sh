# One ncu --set full capture of one kernel launch (short run, few resident batches so the replay's
# memory save/restore stays small).  ENV='STARSD_EARLY=0' KREGEX=k_row_stats CFG=c3 TAG=x bash tools/ncu_one.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
env $ENV timeout ${NCU_TIMEOUT:-420} ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_row}" -s ${SKIP:-2} -c 1 -f -o gpurun_out/${TAG}_full_${CFG:-c3} python tools/profile_run.py --config ${CFG:-c3} --calls 4 --nbatch 2 > gpurun_out/${TAG}_ncu_${CFG:-c3}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_${CFG:-c3}.log
tail -3 gpurun_out/${TAG}_ncu_${CFG:-c3}.log
