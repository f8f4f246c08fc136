#!/bin/bash
# A/B of runtime knobs on one config (run under gpurun): one bench line per variant.
#   bash tools/knob_sweep.sh <config> "<ENV=.. ENV=..>" "<ENV=..>" ...
c=$1; shift
echo "baseline $(timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline 2>/dev/null | tail -1)" 
for v in "$@"; do
  echo "$v $(env $v timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline 2>/dev/null | tail -1)"
done
