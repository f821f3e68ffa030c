# One GPU measurement round: smoke, GPU tests, bench lines, ncu launch lists + full captures,
# compute-sanitizer.  Every step has its own timeout (sum well below the gpurun limit).
#   gpurun --timeout 2700 -- "TAG=r02_v3 bash tools/gpu_round.sh"
mkdir -p gpurun_out
TAG=${TAG:-r02}
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/nvsmi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/${TAG}_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
tail -2 $O/${TAG}_pytest_gpu.log
timeout 300 python bench.py > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
timeout 240 python bench.py --config c2 > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err
timeout 240 python bench.py --config c3g --no-cpu > $O/${TAG}_bench_c3g.json 2> $O/${TAG}_bench_c3g.err
timeout 240 python bench.py --config c3 --dtype bf16 --no-cpu > $O/${TAG}_bench_c3_bf16.json 2> $O/${TAG}_bench_c3_bf16.err
timeout 240 python bench.py --config c2 --dtype bf16 --no-cpu > $O/${TAG}_bench_c2_bf16.json 2> $O/${TAG}_bench_c2_bf16.err
timeout 240 python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 240 python bench.py --star-loopback 3 --steps 10 --warmup 3 > $O/${TAG}_bench_star_loop3_full.json 2> $O/${TAG}_bench_star_full.err
timeout 240 python bench.py --star-loopback 3 --steps 10 --warmup 3 --payload qmeta > $O/${TAG}_bench_star_loop3_qmeta.json 2> $O/${TAG}_bench_star_qmeta.err
for cfg in c3 c2 c3g; do
  timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row|k_sample|k_final" --csv --log-file $O/${TAG}_launches_${cfg}.csv python tools/profile_run.py --config $cfg --calls 30 > /dev/null 2>&1
done
for cfg in c3 c2; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_row_stats|k_sample" -s 4 -c 2 -f -o $O/${TAG}_full_${cfg} python tools/profile_run.py --config $cfg --calls 8 --nbatch 2 > $O/${TAG}_ncu_full_${cfg}.log 2>&1
done
# (compute-sanitizer is closed on this GPU pool since late round 2: the r02_v5 logs in profiles/ are
# the last sanitizer evidence)
for f in $O/${TAG}_bench_*.json; do echo "$f"; cut -c1-400 "$f"; done
