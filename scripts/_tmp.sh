set -e
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -5
for K in 1024 4096; do K=$K python scripts/gemm_one.py; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 50 --warmup 5 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms'])"
