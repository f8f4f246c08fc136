#!/bin/bash
# Interleaved A/B of two library builds on one box (run under gpurun): breakdown lines of
# apply / residual / restrict / prolong and the iteration graph.
#   bash tools/lib_ab.sh <config> <alternate.so> [repeats]
c=$1; alt=$2; n=${3:-2}
f() { timeout 300 python tools/breakdown.py --config $c --reps 10 | python -c "import json,sys; d=json.load(sys.stdin); print({k:v for k,v in d.items() if k.startswith('L0_') or 'iter' in k})"; }
for r in $(seq $n); do
  echo "[this build] $(f)"
  echo "[$alt] $(SMG_LIB=$alt f)"
done
