# Quick bench sanity: default line (c3 with cpu_baseline + parity sample) and two more configs.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --cpu-seconds 5 > gpurun_out/bc_c3.json 2> gpurun_out/bc_c3.err
timeout 240 python bench.py --config c3g --cpu-seconds 3 --no-e2e > gpurun_out/bc_c3g.json 2> gpurun_out/bc_c3g.err
timeout 240 python bench.py --config c2 --dtype bf16 --cpu-seconds 3 --no-e2e > gpurun_out/bc_c2b.json 2> gpurun_out/bc_c2b.err
for f in gpurun_out/bc_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step']*1e3,1), d['cpu_baseline']['parity_sample'] if d.get('cpu_baseline') else None, d['accept'].get('L_hist'))
" || tail -5 ${f%.json}.err; done
