timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python scripts/gemm_bench.py 2>&1 | grep "'K': 13"
for i in 1 2; do for c in c2 c1; do python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['ms_per_step'],4))"; done; done
