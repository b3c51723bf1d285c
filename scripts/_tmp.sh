set -e
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python - <<'PY'
import sys, os; sys.path.insert(0, os.getcwd())
import torch
from bench import CONFIGS
from paper_1906_00091_b200 import DlrmConfig, init_model
from paper_1906_00091_b200.rng import RandomBatchSource
from paper_1906_00091_b200.trainer import StepEngine
for name in ("c3", "c1"):
    c = CONFIGS[name]; B = c["batch"]
    cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
    model = init_model(cfg, table_init="device")
    src = RandomBatchSource(c["tables"], c["bot"][0], B, c["k"], c["fixed"], seed=1)
    hb = src.next_batch()
    eng = StepEngine(model, B, [B * c["k"]] * cfg.num_tables, lr=0.1)
    eng.load(hb.dense, hb.offsets, hb.indices, hb.labels)
    p = eng.profile_stages(reps=20)
    print(name, {k: round(v, 1) for k, v in p.items()})
PY
python bench.py --steps 50 --warmup 5 | tail -1
