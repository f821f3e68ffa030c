# A/B of kernel knobs on the c3 bench line + ncu launch list of the default.
# gpurun --timeout 1800 -- "bash tools/gpu_ab.sh"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CFGS=${CFGS:-"c3 c3g"}
for cfg in $CFGS; do
  for v in default PERSIST; do
    case $v in default) E="";; PERSIST) E="STARSD_PERSIST=1";; TICKET) E="STARSD_PUBLISH_TICKET=1";; esac
    env $E timeout 400 python bench.py --config $cfg --no-cpu --no-e2e --steps 1000 > gpurun_out/ab_${cfg}_$v.json 2> gpurun_out/ab_${cfg}_$v.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/ab_${cfg}_$v.json").read().strip().splitlines()[-1]); r=d["roofline"]
print("$cfg $v", "step %.1f us" % (d["ms_per_step"]*1e3), "kA %.1f ev %.1f" % (r["kernel_ms_mean"]*1e3, r["kernel_ms_events"]*1e3), "frac %.3f step_frac %.3f" % (r["frac"], r["step_frac"]))
PY
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row|k_sample|k_final" --csv --log-file gpurun_out/launches_c3.csv python tools/profile_run.py --config c3 --calls 30 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row|k_sample|k_final" --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py --config c2 --calls 30 > /dev/null 2>&1
python tools/ncu_summarize.py gpurun_out/launches_c3.csv 2>/dev/null | tail -5
STARSD_PERSIST=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "variants or c3 or workspace or ragged" -p no:cacheprovider > gpurun_out/ab_pytest_persist.log 2>&1; tail -2 gpurun_out/ab_pytest_persist.log
