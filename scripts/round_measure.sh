#!/bin/bash
# One GPU call's worth of measurements for profiles/ (no ncu here):
#   bash scripts/round_measure.sh gpurun_out/r1
out=${1:-gpurun_out/r1}
mkdir -p $out
python -m paper_1906_00091_b200.build > /dev/null
for x in gather_bw gather_rmw mma_rate; do
  [ -x scripts/$x ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/$x scripts/$x.cu
done
timeout 600 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
python bench.py > $out/bench_c3.json 2> $out/bench_c3.err; tail -c 300 $out/bench_c3.json
python bench.py --config c2 > $out/bench_c2.json 2> $out/bench_c2.err
python bench.py --config c1 --no-cpu-baseline > $out/bench_c1.json 2> $out/bench_c1.err
python bench.py --config c4 --no-cpu-baseline > $out/bench_c4.json 2> $out/bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_c3.json 2> $out/bench_ref_c3.err
./scripts/gather_bw > $out/gather_ceiling.txt 2>&1
./scripts/mma_rate > $out/mma_rate.txt 2>&1
./scripts/gather_rmw > $out/gather_rmw.txt 2>&1
python scripts/gemm_bench.py > $out/gemm_bench.txt 2>&1
python scripts/interact_bench.py > $out/interact_bench.jsonl 2>&1
python scripts/emb_one.py --bwd --apply > $out/emb_one_c3.json 2>&1
timeout 900 python scripts/emb_sweep.py > $out/c5_sweep.jsonl 2> $out/c5_sweep.err
timeout 600 python scripts/emb_sweep.py --cpu > $out/c5_sweep_cpu.jsonl 2>&1
echo done
