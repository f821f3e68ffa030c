# Quick GPU iteration: plan, GPU tests, short bench lines (c2, c3).  Usage on the box:
#   gpurun --timeout 1500 -- "bash tools/gpu_quick.sh [pytest -k expr]"
mkdir -p gpurun_out
K="${1:-}"
timeout 120 python -c "
import paper_2601_21622_b200 as sd, torch
for a in [(64,5,32000,1.0,torch.float32),(64,5,32000,0.0,torch.float32),(128,7,128256,1.0,torch.float32),(128,7,128256,1.0,torch.bfloat16),(128,7,128256,0.0,torch.float32),(1,4,8,1.0,torch.float32),(64,5,32000,1.0,torch.bfloat16)]:
    print(a[:4], a[4], sd.plan(*a))
" > gpurun_out/plan.log 2>&1
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python bench.py --no-cpu --no-e2e --steps 500 > gpurun_out/q_c2.json 2> gpurun_out/q_c2.err
timeout 300 python bench.py --config c3 --no-cpu --no-e2e --steps 300 > gpurun_out/q_c3.json 2> gpurun_out/q_c3.err
timeout 300 python bench.py --config c2g --no-cpu --no-e2e --steps 500 > gpurun_out/q_c2g.json 2> gpurun_out/q_c2g.err
timeout 300 python bench.py --config c3 --dtype bf16 --no-cpu --no-e2e --steps 300 > gpurun_out/q_c3b.json 2> gpurun_out/q_c3b.err
tail -3 gpurun_out/pytest_gpu.log
for f in gpurun_out/q_*.json; do python -c "
import json,sys
try:
  d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,3),'Mtok/s', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['kernel_ms_mean']*1e3,1),'us', 'frac',round(r['frac'],3), d.get('kernel_plan'))
except Exception as e: print('$f', 'FAILED', e)
"; done
