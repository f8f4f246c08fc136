#!/bin/bash
# round-2 final GPU pass on the final build: suite, bench lines, launch lists (cfg 2 / cfg 3, labelled
# cylinder), smooth traffic (cfg 1-3), one full ncu capture of the top kernel (k_dgs_tile FWD, cfg 2)
# and of the new Vanka delta kernel.  Every ncu command follows the same command run without ncu (&&).
set -u
O=gpurun_out; T=${1:-r2i}
timeout 600 python bench.py --config 1 --also "" --no-labelled --no-cpu-baseline > $O/${T}_bench_cfg1.jsonl 2> $O/${T}_bench_cfg1.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/${T}_bench_reference.jsonl 2> $O/${T}_bench_reference.err
python tools/breakdown.py --config 2 > $O/${T}_breakdown_cfg2.json 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
NCU="ncu --profile-from-start off --clock-control none"
for c in 2 3; do
C="python tools/profile_solve.py --config $c --iters 1"
timeout 600 $C > $O/${T}_plain_iter$c.log 2>&1 && timeout 1200 $NCU --metrics $M --csv --log-file $O/${T}_launches_cfg${c}_1iter.csv $C > $O/${T}_ncu_iter$c.log 2>&1
done
C="python tools/profile_labeled.py --iters 1"
timeout 600 $C > $O/${T}_plain_labelled.log 2>&1 && timeout 1200 $NCU --metrics $M --csv --log-file $O/${T}_launches_labelled_1iter.csv $C > $O/${T}_ncu_labelled.log 2>&1
for c in 1 2 3; do
  C="python tools/profile_kernel.py --config $c --which 5 --level 0"
  timeout 600 $C > $O/${T}_plain_smooth$c.log 2>&1 && timeout 900 $NCU --metrics $M --csv --log-file $O/${T}_smooth_L0_cfg$c.csv $C > $O/${T}_ncu_smooth$c.log 2>&1
done
FULL="$NCU --set full --import-source on"
C="python tools/profile_kernel.py --config 2 --which 2 --level 0"
timeout 600 $C > $O/${T}_plain_dgs2.log 2>&1 && timeout 900 $FULL -k regex:k_dgs_tile -s 3 -c 1 -o $O/${T}_tile_fwd_cfg2 $C > $O/${T}_ncu_fwd.log 2>&1
C="python tools/profile_kernel.py --config 2 --which 4 --level 0"
timeout 600 $C > $O/${T}_plain_vk2.log 2>&1 && timeout 900 $FULL -k regex:k_vanka_delta8 -s 2 -c 1 -o $O/${T}_vanka_delta8_cfg2 $C > $O/${T}_ncu_vk.log 2>&1
for r in $O/${T}_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>&1
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>&1
done
ls -la $O | grep ${T} | tail -40
