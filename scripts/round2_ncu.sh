#!/bin/bash
# ncu evidence for profiles/round2 (one GPU call; every ncu command follows a
# clean plain run of the same command line):   bash scripts/round2_ncu.sh gpurun_out/r2n
out=${1:-gpurun_out/r2n}
mkdir -p $out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B > $out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv \
    --log-file $out/launches_bench_c3.csv $B > /dev/null 2>&1
for cfg in c3 c4 c2 c1; do
  P="python scripts/profile_step.py --config $cfg --steps 2"
  $P > $out/plain_step_$cfg.log 2>&1 || continue
  ncu --set full --clock-control none --import-source on -k regex:"emb_fold|emb_fwd" -s 2 -c 2 \
      -o $out/${cfg}_emb $P > /dev/null 2>&1
done
P="python scripts/profile_step.py --config c3 --steps 2"
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 16 -c 4 \
    -o $out/c3_gemm $P > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:interact -s 2 -c 2 \
    -o $out/c3_interact $P > /dev/null 2>&1
P="python scripts/profile_step.py --config c4 --steps 2"
ncu --set full --clock-control none --import-source on -k regex:interact_tc -s 2 -c 2 \
    -o $out/c4_interact $P > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|skinny|split_lo" -s 20 -c 10 \
    -o $out/c4_gemm $P > /dev/null 2>&1
ls -la $out
# summaries on the box (the reports themselves are too large to bring back)
for cfg in c3 c4 c2 c1; do
  reps="$out/${cfg}_emb.ncu-rep"
  [ $cfg = c3 ] && reps="$reps $out/c3_gemm.ncu-rep $out/c3_interact.ncu-rep"
  [ $cfg = c4 ] && reps="$reps $out/c4_interact.ncu-rep $out/c4_gemm.ncu-rep"
  python scripts/ncu_summary.py $cfg $out/ncu_full_$cfg.md $out/ncu_traffic_$cfg.json $reps > /dev/null 2>&1
done
for r in c3_gemm c4_interact c4_gemm; do
  ncu -i $out/$r.ncu-rep --page source --csv --print-source sass > $out/${r}_sass.csv 2>/dev/null
  python scripts/ncu_hot.py $out/${r}_sass.csv 20 > $out/${r}_hot.txt 2>&1
  rm -f $out/${r}_sass.csv
done
rm -f $out/c1_emb.ncu-rep $out/c2_emb.ncu-rep $out/c3_emb.ncu-rep $out/c4_emb.ncu-rep $out/c3_gemm.ncu-rep $out/c4_gemm.ncu-rep $out/c4_interact.ncu-rep $out/c3_interact.ncu-rep
du -sh $out
