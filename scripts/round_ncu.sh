#!/bin/bash
# ncu evidence for profiles/ (one GPU call; every ncu command follows a clean
# plain run of the same command line):
#   bash scripts/round_ncu.sh gpurun_out/r1n
out=${1:-gpurun_out/r1n}
mkdir -p $out
P="python scripts/profile_step.py --config c3 --steps 2"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$P > $out/plain_step.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file $out/launches_step_c3.csv $P > /dev/null 2>&1
$B > $out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file $out/launches_bench_c3.csv $B > /dev/null 2>&1
$P > $out/plain_step2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:emb_fold -s 1 -c 1 \
    -o $out/full_fold $P > /dev/null 2>&1
$P > $out/plain_step3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:emb_fwd_stream -s 1 -c 1 \
    -o $out/full_fwd $P > /dev/null 2>&1
$P > $out/plain_step4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 16 -c 3 \
    -o $out/full_gemm $P > /dev/null 2>&1
ls -la $out
