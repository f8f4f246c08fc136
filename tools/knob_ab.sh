#!/bin/bash
# A/B of runtime knobs via the per-component breakdown (run under gpurun): fine-level DGS sweep,
# smooth and the SQMR iteration graph, one line per variant.   bash tools/knob_ab.sh <config> "<ENV=..>" ...
c=$1; shift
for v in "" "$@"; do
  echo "[$v] $(env $v timeout 300 python tools/breakdown.py --config $c --reps 10 | python -c "import json,sys; d=json.load(sys.stdin); print({k:v for k,v in d.items() if k in ('L0_dgs_sym_ms','L0_smooth_ms','L1_dgs_sym_ms','sqmr_iter_graph_ms')})")"
done
