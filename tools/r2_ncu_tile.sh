#!/bin/bash
# full ncu captures of the fine-level tile DGS kernels (FWD, REV) and one Vanka phase, cfg 2
set -u
O=gpurun_out; T=${1:-r2b}
NCU="ncu --profile-from-start off --clock-control none --set full --import-source on"
C="python tools/profile_kernel.py --config 2 --which 2 --level 0"
timeout 600 $C > $O/${T}_plain_dgs2.log 2>&1 || exit 1
timeout 900 $NCU -k regex:k_dgs_tile -s 3 -c 1 -o $O/${T}_tile_fwd_cfg2 $C > $O/${T}_ncu_fwd.log 2>&1
timeout 900 $NCU -k regex:k_dgs_tile -s 19 -c 1 -o $O/${T}_tile_rev_cfg2 $C > $O/${T}_ncu_rev.log 2>&1
C="python tools/profile_kernel.py --config 2 --which 4 --level 0"
timeout 600 $C > $O/${T}_plain_vk2.log 2>&1 && timeout 900 $NCU -k regex:k_vanka_ppk -s 2 -c 1 -o $O/${T}_vanka_ppk_cfg2 $C > $O/${T}_ncu_vk.log 2>&1
for r in $O/${T}_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>&1
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>&1
  ncu -i $r --page source --csv > ${r%.ncu-rep}_source.csv 2>&1
done
# cfg 3 golden (first 3 iterations) on the box's host: the oracle needs ~120 GB of RAM
free -g > $O/${T}_host.txt; nproc >> $O/${T}_host.txt
if [ "${GOLDEN3:-0}" = 1 ]; then
  timeout 2400 python tests/golden/make_golden.py cfg3 > $O/${T}_golden_cfg3.log 2>&1 && cp tests/golden/cfg3_history.json $O/
fi
ls -la $O
