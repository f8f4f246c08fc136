#!/bin/bash
# interleaved A/B: Vanka delta launch stores x + delta, apply launch scatters only (SMG_VANKA_NEWV)
for c in 2 3; do for r in 1 2; do for k in 0 1; do
  echo "[cfg $c NEWV=$k] $(SMG_VANKA_NEWV=$k timeout 600 python tools/time_dgs.py --config $c 2>&1 | head -2 | tr '\n' ' ')"
done; done; done
