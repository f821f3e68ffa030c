# A/B of the k_row_stats cluster size (STARSD_ROWCLUSTER) on the box: parity tests + short benches.
mkdir -p gpurun_out
for CLV in ${CLS:-8 4 1}; do
  STARSD_ROWCLUSTER=$CLV timeout 600 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/cl${CLV}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/cl${CLV}_pytest.log
  for cfg in c2 c3 c2g c3g; do
    STARSD_ROWCLUSTER=$CLV timeout 300 python bench.py --config $cfg --no-cpu --no-e2e --steps 300 > gpurun_out/cl${CLV}_$cfg.json 2>/dev/null
  done
  STARSD_ROWCLUSTER=$CLV timeout 300 python bench.py --config c3 --dtype bf16 --no-cpu --no-e2e --steps 300 > gpurun_out/cl${CLV}_c3b.json 2>/dev/null
  STARSD_ROWCLUSTER=$CLV timeout 300 python bench.py --config c2 --dtype bf16 --no-cpu --no-e2e --steps 300 > gpurun_out/cl${CLV}_c2b.json 2>/dev/null
done
for CLV in ${CLS:-8 4 1}; do
  echo "== cluster $CLV: $(tail -1 gpurun_out/cl${CLV}_pytest.log)"
  for f in gpurun_out/cl${CLV}_c*.json; do python -c "
import json
try:
  d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,3),'Mtok/s', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['kernel_ms_mean']*1e3,1),'us', 'frac',round(r['frac'],3))
except Exception as e: print('$f', 'FAILED', e)
"; done
done
