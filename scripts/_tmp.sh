set -e
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/emb_one.py --bwd --apply | tail -1
python scripts/emb_one.py --bwd --apply --zipf | tail -1
python scripts/emb_one.py --bwd --apply --d 128 --rows 500000 | tail -1
python scripts/emb_one.py --bwd --apply --d 16 --rows 4000000 | tail -1
python bench.py --steps 100 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['stages_ms'])"
