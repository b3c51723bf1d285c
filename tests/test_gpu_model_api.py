"""Model-level API parity: dlrm_forward / dlrm_backward (ref model.py:376-424,
tests test_model.py:203-266) and operator timing (ref timing.py:9-25,
parallel.py:254-285, 365-498).

* dlrm_forward equals the manual composition of the public operators
  BITWISE (ref test_model.py:224-235) and equals the fused training step's
  probabilities bitwise (same kernels, same dot orders for the N = 1 layer
  and the sigmoid);
* StageError carries the failing stage's label (ref test_model.py:260-266);
* dlrm_backward's gradients match the float64 oracle within tolerance, and
  applying them with Sgd reproduces train_step within tolerance;
* train_step(timer=StageTimer()) / ParallelTrainer.step(timer=...) credit
  device time to the reference's categories and change no result bit.
"""

import numpy as np
import pytest
import torch

from oracle import port
from paper_1906_00091_b200 import (DlrmConfig, ParallelTrainer, Sgd, SparseBatch,
                                   StageError, StageTimer, bce_from_logits,
                                   dlrm_backward, dlrm_forward, init_model, interact,
                                   lookup_batch, make_plan, mlp_forward,
                                   offsets_from_lengths, sigmoid, train_step)
from paper_1906_00091_b200.rng import RandomBatchSource, RngStream
from tests._util import maxnorm_err, rel_err

pytestmark = pytest.mark.gpu


def toy_config(seed=0, top=(8, 4, 1), d=4):
    return DlrmConfig([7, 5, 9], d, [6, 8, d], list(top), seed=seed)


def random_batch(cfg, b, seed):
    src = RandomBatchSource(cfg.embedding_sizes, cfg.dense_dim, b, 3, False, seed=seed)
    hb = src.next_batch()
    return hb, [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]


def test_zero_parameters_give_half():
    cfg = toy_config()
    model = init_model(cfg)
    for mlp in (model.bottom, model.top):
        for layer in mlp.layers:
            layer.weight.zero_()
            layer.bias.zero_()
    for t in model.tables:
        t.weights.zero_()
    hb, sparse = random_batch(cfg, 6, 12)
    prob, _ = dlrm_forward(model, hb.dense, sparse)
    assert bool((prob == 0.5).all())


def test_output_strictly_inside_unit_interval():
    cfg = toy_config(seed=13)
    model = init_model(cfg)
    hb, sparse = random_batch(cfg, 32, 14)
    prob, _ = dlrm_forward(model, hb.dense, sparse)
    assert bool(((prob > 0) & (prob < 1)).all())


@pytest.mark.parametrize("top,d", [((8, 4, 1), 4), ((6, 3, 1), 3), ((64, 1), 16)])
def test_equals_manual_composition_bitwise(top, d):
    cfg = toy_config(seed=15, top=top, d=d)
    model = init_model(cfg)
    hb, sparse = random_batch(cfg, 37, 16)
    prob, cache = dlrm_forward(model, hb.dense, sparse)
    dense_repr, _ = mlp_forward(model.bottom, hb.dense)
    embs = [lookup_batch(tb, sb) for tb, sb in zip(model.tables, sparse)]
    inter = interact(dense_repr, embs)
    logits, _ = mlp_forward(model.top, inter)
    manual = sigmoid(logits[:, 0])
    assert torch.equal(prob, manual)
    assert torch.equal(cache.prob, prob)


@pytest.mark.parametrize("top,d", [((8, 4, 1), 4), ((6, 3, 1), 3), ((64, 1), 16)])
def test_forward_equals_train_step_probs_bitwise(top, d):
    """train_step's fused loss head computes the same logits and sigmoid as
    dlrm_forward (before its update)."""
    cfg = toy_config(seed=21, top=top, d=d)
    model = init_model(cfg)
    hb, sparse = random_batch(cfg, 45, 22)
    prob, _ = dlrm_forward(model, hb.dense, sparse)
    r = train_step(model, hb.dense, sparse, hb.labels, Sgd(0.1))
    assert torch.equal(r.probs, prob)


def test_permutation_equivariance():
    cfg = toy_config(seed=17)
    model = init_model(cfg)
    hb, sparse = random_batch(cfg, 7, 18)
    perm = np.array([3, 0, 6, 1, 5, 2, 4])
    psparse = []
    for o, i in zip(hb.offsets, hb.indices):
        lens = np.diff(o)[perm]
        idx = np.concatenate([i[o[j]:o[j + 1]] for j in perm])
        psparse.append(SparseBatch(offsets_from_lengths(lens), idx))
    p1, _ = dlrm_forward(model, hb.dense, sparse)
    p2, _ = dlrm_forward(model, hb.dense[perm], psparse)
    assert torch.equal(p1[torch.as_tensor(perm, device=p1.device)], p2)


def test_batch_count_mismatch():
    cfg = toy_config()
    model = init_model(cfg)
    hb, sparse = random_batch(cfg, 4, 19)
    with pytest.raises(ValueError):
        dlrm_forward(model, hb.dense, sparse[:1])


def test_stage_label_on_error():
    cfg = toy_config()
    model = init_model(cfg)
    hb, sparse = random_batch(cfg, 4, 20)
    bad = SparseBatch(hb.offsets[0], hb.indices[0] + 1000)
    with pytest.raises(StageError, match="embedding_lookup"):
        dlrm_forward(model, hb.dense, [bad] + sparse[1:])


def test_backward_stage_label_on_error():
    cfg = toy_config()
    model = init_model(cfg)
    hb, sparse = random_batch(cfg, 4, 23)
    _, cache = dlrm_forward(model, hb.dense, sparse)
    with pytest.raises(StageError, match="top_mlp_backward"):
        dlrm_backward(model, cache, torch.zeros(5, device="cuda"))


def _port_model(model):
    mlp = lambda p: [(l.weight.detach().cpu().double().numpy(),
                      l.bias.detach().cpu().double().numpy(), l.activation)
                     for l in p.layers]
    return {"bottom": mlp(model.bottom), "top": mlp(model.top),
            "tables": [t.weights.detach().cpu().double().numpy() for t in model.tables]}


def test_backward_matches_oracle_and_train_step():
    cfg = DlrmConfig([600] * 4, 16, [13, 64, 16], [32, 16, 1], seed=3)
    model = init_model(cfg)
    pm = _port_model(model)
    hb, sparse = random_batch(cfg, 96, 24)
    dense = hb.dense.astype(np.float32)
    prob, cache = dlrm_forward(model, dense, sparse)
    logits = cache.top_cache.post[-1][:, 0]
    _, g, _ = bce_from_logits(logits, hb.labels)
    grads = dlrm_backward(model, cache, g, n_total=96)
    # oracle: the same pieces in float64 (ref model.py:376-424)
    d64 = dense.astype(np.float64)
    z0, b_in, b_pre = port.mlp_forward(pm["bottom"], d64)
    embs = [port.lookup(W, o, i) for W, o, i in zip(pm["tables"], hb.offsets, hb.indices)]
    inter = port.interact(z0, embs)
    lg, t_in, t_pre = port.mlp_forward(pm["top"], inter)
    assert rel_err(prob.cpu().numpy(), port.sigmoid(lg[:, 0])) < 1e-5
    _, gl, _ = port.bce_from_logits(lg[:, 0], hb.labels)
    t_dw, t_db, g_inter = port.mlp_backward(pm["top"], t_in, t_pre, gl[:, None], 96)
    g0, gembs = port.interact_backward(z0, embs, g_inter)
    b_dw, b_db, _ = port.mlp_backward(pm["bottom"], b_in, b_pre, g0, 96)
    for got, ref in [*zip(grads.top.weights, t_dw), *zip(grads.top.biases, t_db),
                     *zip(grads.bottom.weights, b_dw), *zip(grads.bottom.biases, b_db)]:
        assert maxnorm_err(got.cpu().numpy(), ref) < 1e-5
    for t, (sg, W, o, i, ge) in enumerate(zip(grads.tables, pm["tables"], hb.offsets,
                                              hb.indices, gembs)):
        rows, vals = port.lookup_backward(W, o, i, ge)
        assert np.array_equal(sg.rows.cpu().numpy(), rows)
        assert maxnorm_err(sg.values.cpu().numpy(), vals) < 1e-5
    # the reference train_step composition: forward, backward, Sgd.apply
    Sgd(0.1).apply(model, grads)
    m2 = init_model(cfg)
    train_step(m2, dense, sparse, hb.labels, Sgd(0.1))
    for a, b in zip(model.bottom.layers + model.top.layers, m2.bottom.layers + m2.top.layers):
        assert maxnorm_err(a.weight.cpu().numpy(), b.weight.cpu().numpy()) < 1e-6
        assert maxnorm_err(a.bias.cpu().numpy(), b.bias.cpu().numpy()) < 1e-5
    for a, b in zip(model.tables, m2.tables):
        assert maxnorm_err(a.weights.cpu().numpy(), b.weights.cpu().numpy()) < 1e-6


REF_TRAIN = {"bottom_mlp", "embedding_lookup", "interaction", "top_mlp", "loss", "optimizer"}


def test_train_step_timer_categories_and_no_result_change():
    cfg = DlrmConfig([600] * 4, 16, [13, 64, 16], [32, 16, 1], seed=3)
    src = RandomBatchSource(cfg.embedding_sizes, 13, 128, 4, False, seed=9)
    batches = [src.next_batch() for _ in range(4)]
    ma, mb = init_model(cfg), init_model(cfg)
    timer = StageTimer()
    for hb in batches:
        sp = [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]
        ra = train_step(ma, hb.dense, sp, hb.labels, Sgd(0.1), timer=timer)
        rb = train_step(mb, hb.dense, sp, hb.labels, Sgd(0.1))
        assert ra.loss == rb.loss and torch.equal(ra.probs, rb.probs)
    assert set(timer.seconds) == REF_TRAIN
    assert all(v >= 0 for v in timer.seconds.values())
    for k in ("bottom_mlp", "embedding_lookup", "interaction", "top_mlp", "loss"):
        assert timer.seconds[k] > 0, k
    assert 0 < timer.total() < 1.0
    for a, b in zip(ma.bottom.layers + ma.top.layers, mb.bottom.layers + mb.top.layers):
        assert torch.equal(a.weight, b.weight) and torch.equal(a.bias, b.bias)


def test_parallel_trainer_timer_categories():
    cfg = DlrmConfig([600] * 4, 16, [13, 64, 16], [32, 16, 1], seed=3)
    src = RandomBatchSource(cfg.embedding_sizes, 13, 128, 4, False, seed=9)
    model = init_model(cfg)
    tr = ParallelTrainer(model, make_plan(cfg, 128, 2), capacities=[600] * 4)
    timer = StageTimer()
    for _ in range(2):
        hb = src.next_batch()
        tr.step(hb.dense.astype(np.float32),
                [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)],
                hb.labels.astype(np.float32), timer=timer)
    assert set(timer.seconds) == {"embedding_lookup", "shuffle", "device_compute",
                                  "allreduce", "optimizer"}
    assert all(v > 0 for v in timer.seconds.values())
