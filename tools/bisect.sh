#!/bin/bash
# phase-1 streaming time of the fused kernel under STARSD_DEBUG knobs (C3)
for d in 9 11 15 13 1 0; do
  echo "== STARSD_DEBUG=$d"
  STARSD_DEBUG=$d timeout 40 python tools/trace_run.py --config ${1:-c3} 2>&1 | grep -E "p1_end|consumer|producer"
done
