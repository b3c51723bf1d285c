"""Diagnostic: per-tensor error of the GPU trajectories vs the reference
fixtures, for the tcgen05 (mode 0) and SIMT (mode 1) GEMM paths."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1906_00091_b200 import _lib
from tests.conftest import load_golden
from tests._util import rel_err, maxnorm_err, traj_inputs
from tests.test_gpu_train import run_traj, model_arrays

for name in sys.argv[1:] or ["c1s", "c2s", "c3s"]:
    fx = load_golden(f"traj_{name}.npz")
    c, batches = traj_inputs(fx)
    for mode in (0, 1):
        _lib.call("dlrm_gemm_mode", mode)
        model, res = run_traj(c, batches)
        lerr = max(abs(r.loss - l) / abs(l) for r, l in zip(res, fx["losses"]))
        errs = []
        for i, a in enumerate(model_arrays(model)):
            ref = fx[f"final_{i}"]
            errs.append((i, rel_err(a, ref, 1e-3), rel_err(a, ref, 1e-2), maxnorm_err(a, ref)))
        worst = max(errs, key=lambda e: e[2])
        print(f"{name} mode={mode} loss_rel={lerr:.2e} worst tensor {worst[0]}: "
              f"elem(1e-3)={worst[1]:.2e} elem(1e-2)={worst[2]:.2e} norm={worst[3]:.2e}")
        print("   per tensor elem(1e-2):", " ".join(f"{e[2]:.1e}" for e in errs))
