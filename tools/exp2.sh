for d in 0 1; do
 for cfg in c3 c2g; do
  STARSD_DEBUG=$d timeout 200 python bench.py --config $cfg --no-cpu --no-e2e --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('debug=$d $cfg', round(d['ms_per_step']*1e3,1),'us/step', round(r['kernel_ms_mean']*1e3,1), 'kernel us frac', round(r['frac'],3), 'mean_L', d['accept']['mean_L'])"
 done
done
STARSD_DEBUG=1 STARSD_SLICE_KB=64 timeout 200 python bench.py --config c3 --no-cpu --no-e2e --steps 200 2>/dev/null | tail -c 300
