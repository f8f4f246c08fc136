#!/bin/bash
# round-2 final GPU pass: suite, bench lines, launch lists (box cfg 2 / cfg 3, labelled cylinder),
# smooth traffic.  Every ncu command is preceded by the same command run without ncu (&&).
set -u
O=gpurun_out; T=${1:-r2e}
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 900 python bench.py > $O/${T}_bench_default.jsonl 2> $O/${T}_bench_default.err
timeout 600 python bench.py --config 1 --also "" --no-labelled --no-cpu-baseline > $O/${T}_bench_cfg1.jsonl 2> $O/${T}_bench_cfg1.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/${T}_bench_reference.jsonl 2> $O/${T}_bench_reference.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
NCU="ncu --profile-from-start off --clock-control none"
for c in 2 3; do
C="python tools/profile_solve.py --config $c --iters 1"
timeout 600 $C > $O/${T}_plain_iter$c.log 2>&1 && timeout 1200 $NCU --metrics $M --csv --log-file $O/${T}_launches_cfg${c}_1iter.csv $C > $O/${T}_ncu_iter$c.log 2>&1
done
C="python tools/profile_labeled.py --iters 1"
timeout 600 $C > $O/${T}_plain_labelled.log 2>&1 && timeout 1200 $NCU --metrics $M --csv --log-file $O/${T}_launches_labelled_1iter.csv $C > $O/${T}_ncu_labelled.log 2>&1
for c in 2 3; do
  C="python tools/profile_kernel.py --config $c --which 5 --level 0"
  timeout 600 $C > $O/${T}_plain_smooth$c.log 2>&1 && timeout 900 $NCU --metrics $M --csv --log-file $O/${T}_smooth_L0_cfg$c.csv $C > $O/${T}_ncu_smooth$c.log 2>&1
done
ls -la $O | tail -30
