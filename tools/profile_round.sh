#!/bin/bash
# ncu evidence for one build (run under gpurun; 1 GPU).  Every ncu command is preceded by the
# same command line run without ncu (&&), as the profiling recipe requires.
#   bash tools/profile_round.sh <tag>      -> gpurun_out/<tag>_*.csv / *.ncu-rep
set -u
T=${1:-prof}
O=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
NCU="ncu --profile-from-start off --clock-control none"
# 1. launch list of one cfg-1 SQMR iteration (shares, DRAM bytes per kernel)
C="python tools/profile_solve.py --config 1 --iters 1"
$C > $O/${T}_plain_iter.log 2>&1 && $NCU --metrics $M --csv --log-file $O/${T}_launches_cfg1_1iter.csv $C > $O/${T}_ncu_iter.log 2>&1
# 2. DRAM bytes of one fine-level smooth (bench.py roofline.traffic), cfg 1-4
for c in 1 2 3 4; do
  C="python tools/profile_kernel.py --config $c --which 5 --level 0"
  $C > $O/${T}_plain_smooth$c.log 2>&1 && $NCU --metrics $M --csv --log-file $O/${T}_smooth_L0_cfg$c.csv $C > $O/${T}_ncu_smooth$c.log 2>&1
done
# 3. full captures of the top kernels: fine-level Vanka sweep (cfg 1), fine DGS reverse step (cfg 3)
C="python tools/profile_kernel.py --config 1 --which 4 --level 0"
$C > $O/${T}_plain_vk.log 2>&1 && $NCU --set full --import-source on -k regex:k_vanka_pp -c 1 -o $O/${T}_vanka_pp_cfg1 $C > $O/${T}_ncu_vk.log 2>&1
C="python tools/profile_kernel.py --config 3 --which 2 --level 0"
$C > $O/${T}_plain_dgs3.log 2>&1 && $NCU --set full --import-source on -k regex:k_dgs_vel_c -c 1 -o $O/${T}_dgs_vel_cfg3 $C > $O/${T}_ncu_dgs3.log 2>&1
# 4. opt-in fused velocity pair (why it is slower)
C="python tools/profile_kernel.py --config 1 --which 2 --level 0"
SMG_VEL2=1 $C > $O/${T}_plain_vel2.log 2>&1 && SMG_VEL2=1 $NCU --set full --import-source on -k regex:k_dgs_vel2 -c 1 -o $O/${T}_vel2_cfg1 $C > $O/${T}_ncu_vel2.log 2>&1
# raw + details pages next to each capture (readable without the .ncu-rep)
for r in $O/${T}_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>&1
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>&1
done
ls -la $O
