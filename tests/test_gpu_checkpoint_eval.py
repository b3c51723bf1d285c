"""SURVEY §8(f) rows 3 and 4 on the GPU: forward-only evaluation vs the
reference's ``_evaluate`` (golden ``eval_*.npz``), and DLRMKIT1 checkpoints —
reading the reference-written file, bitwise save / load round trips, and an
Adagrad run resumed from a checkpoint matching the uninterrupted run bit for
bit."""

import json
import os

import numpy as np
import pytest
import torch

from paper_1906_00091_b200 import (Adagrad, DlrmConfig, SparseBatch, evaluate,
                                   init_model, load_checkpoint, load_optimizer_state,
                                   make_optimizer, restore_adagrad, save_checkpoint,
                                   train_step)
from paper_1906_00091_b200.checkpoint import read_arrays
from paper_1906_00091_b200.rng import RandomBatchSource
from tests._util import traj_inputs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def params(model):
    out = []
    for l in model.bottom.layers + model.top.layers:
        out += [l.weight.detach().cpu().numpy().copy(), l.bias.detach().cpu().numpy().copy()]
    return out + [t.weights.detach().cpu().numpy().copy() for t in model.tables]


def build(c):
    return init_model(DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=c["seed"]))


def sparse_of(hb):
    return [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]


@pytest.mark.parametrize("name", ["c3s", "c1s"])
def test_evaluate_matches_reference(golden, name):
    fx = golden(f"eval_{name}.npz")
    c = json.loads(str(fx["config"]))
    src = RandomBatchSource(c["tables"], c["bot"][0], c["batch"], c["k"], c["fixed"],
                            seed=c["seed"], key=1)
    hbs = [src.next_batch() for _ in range(int(fx["nbatches"]))]
    model = build(c)
    before = params(model)
    batches = [(hb.dense.astype(np.float32), sparse_of(hb), hb.labels) for hb in hbs]
    loss, acc = evaluate(model, batches)
    ref_loss, ref_acc = float(fx["loss"]), float(fx["acc"])
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss), (loss, ref_loss)
    total = len(hbs) * c["batch"]
    assert abs(acc - ref_acc) <= 1.0 / total + 1e-12, (acc, ref_acc)
    # graph-replayed second pass: same numbers, parameters untouched
    loss2, acc2 = evaluate(model, batches)
    assert loss2 == loss and acc2 == acc
    for a, b in zip(before, params(model)):
        assert np.array_equal(a, b)


def test_evaluate_after_training_uses_trained_weights(golden):
    fx = golden("traj_c3s.npz")
    c, batches = traj_inputs(fx)
    model = build(c)
    opt = make_optimizer("sgd", c["lr"])
    hb = batches[0]
    r = train_step(model, hb.dense.astype(np.float32), sparse_of(hb), hb.labels, opt)
    # evaluating the NEXT batch equals the loss the next training step reports
    nb = batches[1]
    loss, _ = evaluate(model, [(nb.dense.astype(np.float32), sparse_of(nb), nb.labels)])
    r2 = train_step(model, nb.dense.astype(np.float32), sparse_of(nb), nb.labels, opt)
    assert abs(loss - r2.loss) <= 1e-6 * abs(r2.loss), (loss, r2.loss)
    assert r.loss != r2.loss


def test_load_reference_checkpoint():
    path = os.path.join(HERE, "golden", "ckpt_toy.dlrmkit")
    model = load_checkpoint(path)
    _, arrays = read_arrays(path)
    exp = []
    for name, n in (("bottom", len(model.bottom.layers)), ("top", len(model.top.layers))):
        for l in range(n):
            exp += [arrays[f"{name}_w_{l}"], arrays[f"{name}_b_{l}"]]
    exp += [arrays[f"table_{t}"] for t in range(len(model.tables))]
    for got, ref in zip(params(model), exp):
        assert np.array_equal(got.astype(np.float64), ref)   # fp32-exact start point
    # and it is the reference init of that config, rounded to fp32
    fresh = init_model(model.config)
    for a, b in zip(params(fresh), params(model)):
        assert np.array_equal(a, b)


def test_save_load_roundtrip_after_training(golden, tmp_path):
    fx = golden("traj_c3s.npz")
    c, batches = traj_inputs(fx)
    model = build(c)
    opt = make_optimizer("sgd", c["lr"])
    for hb in batches[:2]:
        train_step(model, hb.dense.astype(np.float32), sparse_of(hb), hb.labels, opt)
    p = str(tmp_path / "m.dlrmkit")
    save_checkpoint(p, model)
    back = load_checkpoint(p)
    assert back.config == model.config
    for a, b in zip(params(model), params(back)):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    assert load_optimizer_state(p) is None
    # float64 payload (the reference's dtype) loads back to the same fp32 values
    p64 = str(tmp_path / "m64.dlrmkit")
    save_checkpoint(p64, model, dtype="float64")
    for a, b in zip(params(model), params(load_checkpoint(p64))):
        assert np.array_equal(a, b)


def test_adagrad_resume_is_bitwise(golden, tmp_path):
    fx = golden("traj_c3a.npz")
    c, batches = traj_inputs(fx)
    lr, eps = c["lr"], c["eps"]
    # uninterrupted: 3 steps
    ma = build(c)
    oa = Adagrad(lr, eps)
    ra = [train_step(ma, hb.dense.astype(np.float32), sparse_of(hb), hb.labels, oa)
          for hb in batches[:3]]
    # 2 steps, checkpoint (model + accumulators), resume in a fresh model / optimiser
    mb = build(c)
    ob = Adagrad(lr, eps)
    for hb in batches[:2]:
        train_step(mb, hb.dense.astype(np.float32), sparse_of(hb), hb.labels, ob)
    p = str(tmp_path / "a.dlrmkit")
    save_checkpoint(p, mb, ob)
    state = load_optimizer_state(p)
    assert state is not None and "table_0" in state and "top_w_0" in state
    mc = load_checkpoint(p)
    oc = Adagrad(lr, eps)
    restore_adagrad(oc, mc, state)
    hb = batches[2]
    rc = train_step(mc, hb.dense.astype(np.float32), sparse_of(hb), hb.labels, oc)
    assert rc.loss == ra[2].loss
    for a, b in zip(params(ma), params(mc)):
        assert np.array_equal(a, b)


def test_criteo_batches_train_and_evaluate():
    """Criteo TSV -> native parser -> CriteoBatch -> train_step / evaluate."""
    from paper_1906_00091_b200.criteo import CriteoBatchReader
    fx = dict(np.load(os.path.join(HERE, "golden", "criteo.npz")))
    vocab = [1000 + 37 * i for i in range(26)]
    p = "/tmp/_criteo_gpu_test.tsv"
    with open(p, "wb") as f:
        f.write(fx["text"].tobytes())
    batches = list(CriteoBatchReader(p, vocab, 64))
    os.unlink(p)
    cfg = DlrmConfig(vocab, 16, [13, 64, 16], [64, 1], seed=3)
    model = init_model(cfg)
    opt = make_optimizer("sgd", 0.1)
    losses = [train_step(model, *b.train_args(), opt).loss for b in batches]
    assert all(np.isfinite(losses))
    vloss, vacc = evaluate(model, [b.train_args() for b in batches[:2]])
    assert np.isfinite(vloss) and 0.0 <= vacc <= 1.0
