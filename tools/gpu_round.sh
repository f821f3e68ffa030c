# One GPU measurement round: smoke, gpu tests, bench lines, ncu launch lists + full captures.
# Run on the box: gpurun --timeout 3000 -- "bash tools/gpu_round.sh"
mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for cfg in c3 c2g c3g; do
  timeout 600 python bench.py --config $cfg --no-cpu > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
timeout 600 python bench.py --config c2 --dtype bf16 --no-cpu > gpurun_out/bench_c2_bf16.json 2> gpurun_out/bench_c2_bf16.err
timeout 600 python bench.py --config c3 --dtype bf16 --no-cpu > gpurun_out/bench_c3_bf16.json 2> gpurun_out/bench_c3_bf16.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row|k_sample|k_final" --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py --config c2 --calls 30 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row|k_sample|k_final" --csv --log-file gpurun_out/launches_c3.csv python tools/profile_run.py --config c3 --calls 30 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_stats|k_sample" -s 10 -c 2 -f -o gpurun_out/full_c2 python tools/profile_run.py --config c2 --calls 16 > gpurun_out/ncu_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_stats|k_sample" -s 10 -c 2 -f -o gpurun_out/full_c3 python tools/profile_run.py --config c3 --calls 16 > gpurun_out/ncu_full_c3.log 2>&1
ls -la gpurun_out
