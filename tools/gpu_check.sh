# Quick GPU check: build, smoke, the GPU test suite, c3/c2 bench lines.
# gpurun --timeout 2400 -- "bash tools/gpu_check.sh"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c3g --no-cpu --no-e2e > gpurun_out/bench_c3g.json 2> gpurun_out/bench_c3g.err
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/bench_c3.json gpurun_out/bench_c2.json gpurun_out/bench_c3g.json | cut -c1-600
timeout 600 python bench.py --star-loopback 3 --steps 10 --warmup 3 > gpurun_out/bench_star_loop.json 2> gpurun_out/bench_star_loop.err
timeout 600 python bench.py --star-loopback 3 --steps 10 --warmup 3 --payload qmeta > gpurun_out/bench_star_loop_qm.json 2> gpurun_out/bench_star_loop_qm.err
tail -c 1500 gpurun_out/bench_star_loop.json; tail -5 gpurun_out/bench_star_loop.err
