# Round-2 profiling: ncu launch lists (c3, c2, c3g), full captures of k_row_stats / k_sample_req at
# c3 and c2, and compute-sanitizer memcheck / racecheck / synccheck on small shapes.
# gpurun --timeout 3000 -- "TAG=r02_v1 bash tools/gpu_profile.sh"
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in c3 c2 c3g; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row|k_sample|k_final" --csv --log-file gpurun_out/${TAG}_launches_${cfg}.csv python tools/profile_run.py --config $cfg --calls 30 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_stats|k_sample" -s 10 -c 2 -f -o gpurun_out/${TAG}_full_c3 python tools/profile_run.py --config c3 --calls 16 > gpurun_out/${TAG}_ncu_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_stats|k_sample" -s 10 -c 2 -f -o gpurun_out/${TAG}_full_c2 python tools/profile_run.py --config c2 --calls 16 > gpurun_out/${TAG}_ncu_full_c2.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/${TAG}_sanitizer_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_sanitizer_${tool}.log
done
tail -4 gpurun_out/${TAG}_sanitizer_*.log
ls -la gpurun_out
