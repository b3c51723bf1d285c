timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print('c3', round(d['value']), round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items() if 'inter' in k})"
python bench.py --config c4 --no-cpu-baseline > gpurun_out/b4.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/b4.json').read().strip().splitlines()[-1]);print('c4', round(d['value']), round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
