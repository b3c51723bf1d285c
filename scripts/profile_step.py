"""Run a few eager (non-graph) training steps of a bench config so every
kernel of the step shows up individually under ncu.

    python scripts/profile_step.py --config c3 --steps 2
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_1906_00091_b200 import DlrmConfig, init_model, _lib
from paper_1906_00091_b200.rng import RandomBatchSource
from paper_1906_00091_b200.trainer import StepEngine

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--simt", action="store_true")
a = ap.parse_args()
c = CONFIGS[a.config]
if a.simt:
    _lib.call("dlrm_gemm_mode", 1)
B = c["batch"]
cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
model = init_model(cfg, table_init="device")
src = RandomBatchSource(c["tables"], c["bot"][0], B, c["k"], c["fixed"], seed=1)
hb = src.next_batch()
caps = [B * c["k"]] * cfg.num_tables
eng = StepEngine(model, B, caps, lr=0.1)
eng.load(hb.dense, hb.offsets, hb.indices, hb.labels)
torch.cuda.synchronize()
for _ in range(a.steps):
    eng.run()
torch.cuda.synchronize()
print("launches/step", eng.launches_per_step, "loss", float(eng.stats[0]) / B)
