# A/B of an environment knob on the box: parity tests + short benches per value.
#   VAR=STARSD_SAMPLER VALS="tasks req" bash tools/exp_env.sh [pytest -k expr]
mkdir -p gpurun_out
K="${1:-}"
for V in $VALS; do
  if [ -n "$K" ]; then
    env $VAR=$V timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/ab_${V}_pytest.log 2>&1
  else
    env $VAR=$V timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_${V}_pytest.log 2>&1
  fi
  echo "rc=$?" >> gpurun_out/ab_${V}_pytest.log
  for cfg in c2 c3 c2g; do
    env $VAR=$V timeout 300 python bench.py --config $cfg --no-cpu --no-e2e --steps 300 > gpurun_out/ab_${V}_$cfg.json 2>gpurun_out/ab_${V}_$cfg.err
  done
  env $VAR=$V timeout 300 python bench.py --config c3 --dtype bf16 --no-cpu --no-e2e --steps 300 > gpurun_out/ab_${V}_c3b.json 2>/dev/null
  env $VAR=$V timeout 300 python bench.py --config c2 --dtype bf16 --no-cpu --no-e2e --steps 300 > gpurun_out/ab_${V}_c2b.json 2>/dev/null
done
for V in $VALS; do
  echo "== $VAR=$V: $(tail -3 gpurun_out/ab_${V}_pytest.log | tr '\n' ' ')"
  for f in gpurun_out/ab_${V}_c*.json; do python -c "
import json
try:
  d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,3),'Mtok/s', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['kernel_ms_mean']*1e3,1),'us', 'frac',round(r['frac'],3))
except Exception as e: print('$f', 'FAILED', e)
"; done
done
