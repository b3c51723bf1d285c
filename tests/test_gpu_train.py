"""The fused training step vs the reference trajectories.

Golden fixtures hold dlrmkit's own float64 losses / probabilities / final
parameters after N SGD steps from the same fp32-rounded start point and the
same inputs.  Contract (BASELINE.json north_star): loss within rtol 1e-4,
updated weights within 1e-4 elementwise: |d| <= 1e-4 (|ref| + 1e-2 max|ref|)
per tensor (biases start at zero, so their values are pure fp32 sums).
"""

import json

import numpy as np
import pytest
import torch

from paper_1906_00091_b200 import (DlrmConfig, LookupIndexError, Sgd,
                                   SparseBatch, init_model, make_optimizer,
                                   train_step)
from tests._util import rel_err, traj_inputs

pytestmark = pytest.mark.gpu
TRAJS = ["toy", "c1s", "c2s", "c3s", "c1a", "c3a"]   # *a: Adagrad


def model_arrays(model):
    out = []
    for l in model.bottom.layers + model.top.layers:
        out += [l.weight.detach().cpu().double().numpy(),
                l.bias.detach().cpu().double().numpy()]
    return out + [t.weights.detach().cpu().double().numpy() for t in model.tables]


def build(c):
    cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=c["seed"])
    return init_model(cfg)


def run_traj(c, batches, use_graph=True):
    model = build(c)
    opt = make_optimizer(c.get("opt", "sgd"), c["lr"], c.get("eps", 1e-10))
    res = []
    for hb in batches:
        sparse = [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]
        res.append(train_step(model, hb.dense.astype(np.float32), sparse,
                              hb.labels, opt, use_graph=use_graph))
    return model, res


@pytest.mark.parametrize("name", TRAJS)
def test_trajectory_matches_reference(golden, name):
    fx = golden(f"traj_{name}.npz")
    c, batches = traj_inputs(fx)
    model, res = run_traj(c, batches)
    for s, r in enumerate(res):
        ref = fx["losses"][s]
        assert abs(r.loss - ref) <= 1e-4 * abs(ref), (s, r.loss, ref)
        assert rel_err(r.probs.cpu().double().numpy(), fx["probs"][s]) < 1e-4
    for i, a in enumerate(model_arrays(model)):
        assert rel_err(a, fx[f"final_{i}"], floor=1e-2) < 1e-4, i


def test_graph_replay_bitwise_equals_eager(golden):
    fx = golden("traj_c3s.npz")
    c, batches = traj_inputs(fx)
    m1, r1 = run_traj(c, batches, use_graph=True)
    m2, r2 = run_traj(c, batches, use_graph=False)
    for a, b in zip(r1, r2):
        assert a.loss == b.loss
    for a, b in zip(model_arrays(m1), model_arrays(m2)):
        assert np.array_equal(a, b)


def test_out_of_range_index_raises_and_mutates_nothing(golden):
    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    model = build(c)
    opt = Sgd(0.1)
    hb = batches[0]
    sparse = [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]
    train_step(model, hb.dense, sparse, hb.labels, opt)
    before = model_arrays(model)
    bad_idx = [i.copy() for i in hb.indices]
    bad_idx[3][17] = c["tables"][3] + 5
    bad_idx[5][2] = -1
    sparse = [SparseBatch(o, i) for o, i in zip(hb.offsets, bad_idx)]
    with pytest.raises(LookupIndexError) as e:
        train_step(model, hb.dense, sparse, hb.labels, opt)
    assert (e.value.table_id, e.value.position, e.value.index) == \
        (3, 17, c["tables"][3] + 5)
    for a, b in zip(before, model_arrays(model)):
        assert np.array_equal(a, b)
