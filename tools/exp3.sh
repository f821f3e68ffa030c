for d in 0 7 6 3 2; do
  STARSD_DEBUG=$d timeout 200 python bench.py --config c3 --no-cpu --no-e2e --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('debug=$d c3', round(d['ms_per_step']*1e3,1),'us/step kernel', round(r['kernel_ms_mean']*1e3,1), 'mean_L', d['accept']['mean_L'])"
done
