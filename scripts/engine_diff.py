"""Diagnostic: run one eager engine step in tcgen05 and SIMT GEMM mode from
the same state and report the normwise difference of every buffer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_00091_b200 import _lib, DlrmConfig, init_model, SparseBatch
from paper_1906_00091_b200.trainer import StepEngine
from tests.conftest import load_golden
from tests._util import traj_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c1s"
fx = load_golden(f"traj_{name}.npz")
c, batches = traj_inputs(fx)
outs = {}
for mode in (1, 0):
    _lib.call("dlrm_gemm_mode", mode)
    model = init_model(DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=c["seed"]))
    hb = batches[0]
    eng = StepEngine(model, c["batch"], [len(i) for i in hb.indices], lr=c["lr"])
    eng.load(hb.dense, hb.offsets, hb.indices, hb.labels)
    eng.run()
    torch.cuda.synchronize()
    bufs = {"Z": eng.Z, "R": eng.R, "logits": eng.logits, "glogit": eng.glogit,
            "gR": eng.gR, "gZ": eng.gZ, "params": eng.params, "W_all": eng.W_all}
    for i, t in enumerate(eng.bact): bufs[f"bact{i}"] = t
    for i, t in enumerate(eng.tact): bufs[f"tact{i}"] = t
    for i, t in enumerate(eng.gtop): bufs[f"gtop{i}"] = t
    for i, t in enumerate(eng.gbot): bufs[f"gbot{i}"] = t
    off = 0
    for li, l in enumerate(eng.layers):
        bufs[f"W{li}"] = l.storage
        bufs[f"b{li}"] = l.bias
    outs[mode] = {k: v.detach().double().cpu().numpy().copy() for k, v in bufs.items()}
for k in outs[0]:
    a, b = outs[0][k], outs[1][k]
    d = np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)
    print(f"{k:8s} shape={str(a.shape):14s} normwise diff tc vs simt = {d:.2e}  max|simt|={np.abs(b).max():.3e}")
