for d in 0 6 7 135; do
  STARSD_DEBUG=$d timeout 200 python bench.py --config c3 --no-cpu --no-e2e --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('debug=$d c3 kernel', round(r['kernel_ms_mean']*1e3,1), 'us frac', round(r['frac'],3))"
done
