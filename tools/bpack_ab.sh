#!/bin/bash
# interleaved A/B of the tile kernel's packed-b staging (SMG_TILE_BPACK) on one box: solve + fine sweeps
for c in 2 3; do for r in 1 2; do for k in 0 1; do
  echo "[cfg $c BPACK=$k] $(SMG_TILE_BPACK=$k timeout 600 python tools/time_dgs.py --config $c | tr '\n' ' ')"
done; done; done
