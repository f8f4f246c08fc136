#!/bin/bash
# A/B of the transfer-kernel knobs (run under gpurun): restrict/prolong times per level and the
# iteration graph, one line per variant.   bash tools/transfer_ab.sh <config> "<ENV=..>" ...
c=$1; shift
for v in "" "$@"; do
  echo "[$v] $(env $v timeout 300 python tools/breakdown.py --config $c --reps 10 | python -c "import json,sys; d=json.load(sys.stdin); print({k:v for k,v in d.items() if 'restrict' in k or 'prolong' in k or 'iter' in k})")"
done
