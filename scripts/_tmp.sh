set -e
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "1 1" "0 1" "1 0" "0 0"; do set -- $cfg
DLRM_EMB_FWD_SIDE=$1 DLRM_WGRAD_SIDE=$2 python bench.py --steps 100 --warmup 5 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['value'], d['ms_per_step'], d['e2e']['ms_per_step'])"
done
