timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do for v in 1 0; do DLRM_HEAD_SPLIT=$v python bench.py --steps 200 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$v', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"; done; done
