mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
timeout 240 python bench.py --star-loopback 3 --steps 10 --warmup 3 --payload qmeta > gpurun_out/sq_$i.json 2> gpurun_out/sq_$i.err
timeout 240 python bench.py --star-loopback 3 --steps 10 --warmup 3 > gpurun_out/sf_$i.json 2> gpurun_out/sf_$i.err
done
for f in gpurun_out/sq_*.json gpurun_out/sf_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['star']
print('$f', round(d['ms_per_step'],2), round(s['busy_fraction'],3), round(s['predicted']['service_ms'],2), round(s['predicted']['return_ms'],2))
"; done
