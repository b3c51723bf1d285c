"""Per-tensor error report of train_step vs the float64 oracle at a full
config (diagnostics for tests/test_gpu_fullsize.py).

    python scripts/parity_diag.py c1 [--steps N] [--simt] [--opt adagrad]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.test_gpu_fullsize import FULL, check, run_pair  # noqa: E402
from tests._util import rel_err, maxnorm_err  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--simt", action="store_true")
    ap.add_argument("--opt", default="sgd")
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--eps", type=float, default=1e-10)
    a = ap.parse_args()
    from paper_1906_00091_b200 import _lib
    if a.simt:
        _lib.call("dlrm_gemm_mode", 1)
    c = FULL[a.name]
    model, pm, start, touched, out = run_pair(c, a.opt, a.lr, a.eps, a.steps)
    try:
        worst = check(c, model, pm, start, touched, out)
        verdict = "pass"
    except AssertionError as e:
        worst, verdict = None, f"FAIL {e}"
    rep = {"verdict": verdict, "worst": worst, "config": a.name, "simt": a.simt, "opt": a.opt, "steps": len(out), "per_step": []}
    for loss, acc, probs, (rl, ra, rp) in out:
        rep["per_step"].append({"loss_rel": abs(loss - rl) / abs(rl),
                                "probs_rel": rel_err(probs, rp), "acc": acc, "ref_acc": ra})
    tens = []
    names = [f"bottom{l}" for l in range(len(pm["bottom"]))] + \
        [f"top{l}" for l in range(len(pm["top"]))]
    for nm, got_l, (w, b, _) in zip(names, model.bottom.layers + model.top.layers,
                                    pm["bottom"] + pm["top"]):
        for kind, g, r in (("w", got_l.weight, w), ("b", got_l.bias, b)):
            g = g.detach().cpu().double().numpy()
            scale = np.abs(r) + 1e-3 * max(np.abs(r).max(), 1e-30)
            e = np.abs(g - r) / scale
            i = np.unravel_index(int(np.argmax(e)), e.shape)
            tens.append({"t": nm + kind, "rel_1e-3": float(e.max()),
                         "rel_1e-2": rel_err(g, r, floor=1e-2), "maxnorm": maxnorm_err(g, r),
                         "at": [int(x) for x in i], "got": float(g[i]), "ref": float(r[i]),
                         "max_ref": float(np.abs(r).max())})
    rep["mlp"] = tens
    rows = []
    for t, (tab, ref) in enumerate(zip(model.tables, pm["tables"])):
        rr = np.unique(np.concatenate(touched[t]))
        got = tab.weights.detach().cpu().numpy()[rr]
        rows.append(rel_err(got, ref[rr], floor=1e-2))
    rep["rows_worst"] = max(rows)
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
