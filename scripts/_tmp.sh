timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python scripts/emb_sweep.py --rows 10000000 --d 64 --pool 32 --reps 5 2>/dev/null
python scripts/emb_sweep.py --rows 100000 --d 16 --pool 8 --reps 5 2>/dev/null
for c in c1 c4; do python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['ms_per_step'],4))"; done
