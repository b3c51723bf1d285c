set -e
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 100 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['stages_ms'])"
python scripts/profile_step.py --config c3 --steps 2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_split.csv python scripts/profile_step.py --config c3 --steps 2 > /dev/null 2>&1
