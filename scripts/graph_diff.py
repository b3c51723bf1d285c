"""Diagnostic: params after each step, tcgen05 vs SIMT, eager vs graph."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_00091_b200 import _lib, DlrmConfig, init_model
from paper_1906_00091_b200.trainer import StepEngine
from tests.conftest import load_golden
from tests._util import traj_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c1s"
fx = load_golden(f"traj_{name}.npz")
c, batches = traj_inputs(fx)
runs = {}
for mode, graph in ((1, False), (0, False), (0, True), (1, True)):
    _lib.call("dlrm_gemm_mode", mode)
    model = init_model(DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=c["seed"]))
    caps = [max(len(hb.indices[t]) for hb in batches) for t in range(len(c["tables"]))]
    eng = StepEngine(model, c["batch"], caps, lr=c["lr"])
    snaps = []
    for s, hb in enumerate(batches):
        eng.load(hb.dense, hb.offsets, hb.indices, hb.labels)
        if graph and s == 1:
            eng.capture()
        eng.run()
        torch.cuda.synchronize()
        snaps.append([l.bias.double().cpu().numpy().copy() for l in eng.layers])
    runs[(mode, graph)] = snaps
base = runs[(1, False)]
for key, snaps in runs.items():
    errs = []
    for s in range(len(snaps)):
        e = max(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30) for a, b in zip(snaps[s], base[s]))
        errs.append(f"{e:.1e}")
    print(key, "bias normwise diff vs simt-eager per step:", errs)
