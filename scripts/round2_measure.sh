#!/bin/bash
# One GPU call's worth of round-2 measurements (no profiler):
#   bash scripts/round2_measure.sh gpurun_out/r2
out=${1:-gpurun_out/r2}
mkdir -p $out
python -m paper_1906_00091_b200.build > /dev/null
python bench.py > $out/bench_c3.json 2> $out/bench_c3.err; tail -c 400 $out/bench_c3.json
python bench.py > $out/bench_c3_b.json 2> $out/bench_c3_b.err
python bench.py --config c2 > $out/bench_c2.json 2> $out/bench_c2.err
python bench.py --config c1 --no-cpu-baseline > $out/bench_c1.json 2> $out/bench_c1.err
python bench.py --config c4 --no-cpu-baseline > $out/bench_c4.json 2> $out/bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_c3.json 2> $out/bench_ref_c3.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --hybrid --gpus 1 --no-cpu-baseline > $out/bench_hybrid1.json 2> $out/bench_hybrid1.err
python scripts/interact_bench.py > $out/interact_bench.jsonl 2>&1
python scripts/emb_one.py --bwd --apply > $out/emb_one_c3.json 2>&1
python scripts/gemm_bench.py > $out/gemm_bench.txt 2>&1
python scripts/ablate.py c3 > $out/ablate_c3.txt 2>&1
echo done
