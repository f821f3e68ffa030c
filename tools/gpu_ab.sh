# A/B of kernel knobs on bench lines (+ the GPU tests named by PYTEST_FILES first).
# gpurun --timeout 2400 -- "VARIANTS='base FUSED0 RG32' CFGS='c3 c2' bash tools/gpu_ab.sh"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -n "$PYTEST_FILES" ]; then
  timeout ${PYTEST_TIMEOUT:-600} python -m pytest $PYTEST_FILES -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/ab_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/ab_pytest.log; tail -3 gpurun_out/ab_pytest.log
fi
CFGS=${CFGS:-"c3 c2"}
VARIANTS=${VARIANTS:-"base"}
for cfg in $CFGS; do
  for v in $VARIANTS; do
    case $v in
      base) E="";;
      EARLY0) E="STARSD_EARLY=0";;
      TICKET) E="STARSD_PUBLISH_TICKET=1";;
      RG*) E="STARSD_RGROUP=${v#RG}";;
      *) E="$v";;
    esac
    env $E timeout ${BENCH_TIMEOUT:-150} python bench.py --config $cfg --no-cpu --no-e2e --steps 1000 $BENCH_ARGS > gpurun_out/ab_${cfg}_$v.json 2> gpurun_out/ab_${cfg}_$v.err
    python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/ab_${cfg}_$v.json").read().strip().splitlines()[-1]); r=d["roofline"]
    print("$cfg $v", "step %.1f us" % (d["ms_per_step"]*1e3), "kA %.1f ev %.1f" % (r["kernel_ms_mean"]*1e3, r["kernel_ms_events"]*1e3), "frac %.3f step_frac %.3f" % (r["frac"], r["step_frac"]), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print("$cfg $v FAILED", e, open("gpurun_out/ab_${cfg}_$v.err").read()[-800:])
PY
  done
done
