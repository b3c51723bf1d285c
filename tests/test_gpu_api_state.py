"""Engine state that must follow the batch / optimiser it belongs to.

* LookupIndexError's ``index`` comes from the batch that RAN, read on the
  device (dlrm_err_resolve) — not from whatever batch the host packed last
  (ref embedding.py:117-124: the payload is the offending value itself).
* Weighted bags through the hybrid-parallel step (ref ParallelTrainer calls
  lookup_batch / lookup_backward, which apply SparseBatch.weights,
  parallel.py:363-506, embedding.py:155-210).
* Adagrad accumulators belong to the optimiser OBJECT (ref optim.py:112-140:
  ``Adagrad`` keeps ``_mlp_state`` / ``_table_state`` per instance), also
  when train_step's cached engine is reused.
"""

import numpy as np
import pytest
import torch

from paper_1906_00091_b200 import (Adagrad, DlrmConfig, LookupIndexError,
                                   ParallelTrainer, Sgd, SparseBatch, init_model,
                                   make_plan, train_step)
from paper_1906_00091_b200.trainer import StepEngine
from tests._util import rel_err, traj_inputs

pytestmark = pytest.mark.gpu


def build(c):
    return init_model(DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=c["seed"]))


def arrays(bottom, top, tables):
    out = []
    for l in bottom.layers + top.layers:
        out += [l.weight.detach().cpu().double().numpy(),
                l.bias.detach().cpu().double().numpy()]
    return out + [t.weights.detach().cpu().double().numpy() for t in tables]


def test_pipelined_error_reports_the_batch_that_ran(golden):
    """Pack-ahead: batch A (bad index) staged into input set 0, batch B
    (another bad value at the same position) packed and staged into set 1
    AFTER it; running set 0 must report A's value."""
    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    model = build(c)
    caps = [max(len(hb.indices[t]) for hb in batches) for t in range(len(c["tables"]))]
    eng = StepEngine(model, c["batch"], caps, lr=0.1, input_sets=2)
    ha, hb = batches[0], batches[1]
    ia = [i.copy() for i in ha.indices]
    ib = [i.copy() for i in hb.indices]
    ia[3][17] = c["tables"][3] + 5
    ib[3][17] = c["tables"][3] + 999
    pa = eng.pack_host_batch(ha.dense, ha.offsets, ia, ha.labels)
    pb = eng.pack_host_batch(hb.dense, hb.offsets, ib, hb.labels)
    eng.stage(pa, 0)
    eng.stage(pb, 1)
    before = arrays(model.bottom, model.top, model.tables)
    eng.use_set(0)
    eng.run()
    with pytest.raises(LookupIndexError) as e:
        eng.check_errors()
    assert (e.value.table_id, e.value.position, e.value.index) == (3, 17, c["tables"][3] + 5)
    eng.use_set(1)
    eng.run()
    with pytest.raises(LookupIndexError) as e:
        eng.check_errors()
    assert e.value.index == c["tables"][3] + 999
    # neither failing step mutated anything
    for x, y in zip(before, arrays(model.bottom, model.top, model.tables)):
        assert np.array_equal(x, y)


def test_pipelined_error_graph_replay(golden):
    """Same through captured graphs (one per input set)."""
    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    model = build(c)
    caps = [max(len(hb.indices[t]) for hb in batches) for t in range(len(c["tables"]))]
    eng = StepEngine(model, c["batch"], caps, lr=0.1, input_sets=2)
    good = [eng.pack_host_batch(h.dense, h.offsets, h.indices, h.labels) for h in batches[:2]]
    for k in range(2):
        eng.use_set(k)
        eng.stage(good[k], k)
        eng.run()
        eng.capture()
    ha = batches[2]
    ia = [i.copy() for i in ha.indices]
    ia[0][3] = -7
    eng.stage(eng.pack_host_batch(ha.dense, ha.offsets, ia, ha.labels), 0)
    eng.stage(good[1], 1)
    eng.use_set(0)
    eng.run()
    with pytest.raises(LookupIndexError) as e:
        eng.check_errors()
    assert (e.value.table_id, e.value.position, e.value.index) == (0, 3, -7)
    eng.use_set(1)
    eng.run()
    eng.check_errors()   # the good batch clears the error records


def _weighted(batches, seed=5):
    rng = np.random.default_rng(seed)
    out = []
    for hb in batches:
        out.append([SparseBatch(o, i, rng.uniform(0.25, 2.0, len(i)))
                    for o, i in zip(hb.offsets, hb.indices)])
    return out


def test_parallel_trainer_applies_bag_weights(golden):
    """ParallelTrainer with weighted bags: G = 1 bitwise equal to the fused
    weighted train_step; G = 2 within the north-star tolerance of it."""
    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    sparse = _weighted(batches)
    ref = build(c)
    opt = Sgd(c["lr"])
    ref_loss = [train_step(ref, hb.dense.astype(np.float32), sp, hb.labels, opt).loss
                for hb, sp in zip(batches, sparse)]
    ref_arr = arrays(ref.bottom, ref.top, ref.tables)
    for G in (1, 2):
        m = build(c)
        caps = [max(len(hb.indices[t]) for hb in batches) for t in range(len(c["tables"]))]
        tr = ParallelTrainer(m, make_plan(m.config, c["batch"], G), "sgd", c["lr"],
                             capacities=caps)
        loss = [tr.step(hb.dense.astype(np.float32), sp, hb.labels.astype(np.float32)).loss
                for hb, sp in zip(batches, sparse)]
        b, t = tr.replica_params(0)
        got = arrays(b, t, tr.tables)
        if G == 1:
            assert loss == ref_loss
            for x, y in zip(got, ref_arr):
                assert np.array_equal(x, y)
        else:
            for a, r in zip(loss, ref_loss):
                assert abs(a - r) <= 1e-4 * abs(r)
            for i, (x, y) in enumerate(zip(got, ref_arr)):
                assert rel_err(x, y, floor=1e-2) < 1e-4, i
    # weights actually matter: the unweighted run differs
    m = build(c)
    plain = [train_step(m, hb.dense.astype(np.float32),
                        [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)],
                        hb.labels, Sgd(c["lr"])).loss for hb in batches]
    assert plain != ref_loss


def test_adagrad_state_belongs_to_the_optimizer(golden):
    fx = golden("traj_c1a.npz")
    c, batches = traj_inputs(fx)
    lr, eps = c["lr"], c["eps"]

    def sp(hb):
        return [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]

    # model 1: two steps with optimiser A, then one with a FRESH optimiser B
    m1 = build(c)
    oa = Adagrad(lr, eps)
    for hb in batches[:2]:
        train_step(m1, hb.dense.astype(np.float32), sp(hb), hb.labels, oa)
    a_state = [a.clone() for a in oa._table_state.values()]
    assert any(float(a.abs().sum()) > 0 for a in a_state)
    ob = Adagrad(lr, eps)
    r1 = train_step(m1, batches[2].dense.astype(np.float32), sp(batches[2]),
                    batches[2].labels, ob)
    # model 2: the same two steps, then a fresh optimiser on a copy of the
    # parameters in a NEW model (no cached engine): zero accumulators
    m2 = build(c)
    oc = Adagrad(lr, eps)
    for hb in batches[:2]:
        train_step(m2, hb.dense.astype(np.float32), sp(hb), hb.labels, oc)
    m3 = m2.copy()
    r3 = train_step(m3, batches[2].dense.astype(np.float32), sp(batches[2]),
                    batches[2].labels, Adagrad(lr, eps))
    assert r1.loss == r3.loss
    for x, y in zip(arrays(m1.bottom, m1.top, m1.tables), arrays(m3.bottom, m3.top, m3.tables)):
        assert np.array_equal(x, y)
    # A kept its own accumulators (not B's step)
    for x, y in zip(a_state, oa._table_state.values()):
        assert torch.equal(x, y)
    # and A resumes from them: A again on model 1 continues A's sums
    train_step(m1, batches[3 % len(batches)].dense.astype(np.float32),
               sp(batches[3 % len(batches)]), batches[3 % len(batches)].labels, oa)
    assert not all(torch.equal(x, y) for x, y in zip(a_state, oa._table_state.values()))


def test_async_results_match_sync_and_report_their_own_error(golden):
    """train_step(sync=False): the results read after later steps were
    issued equal the synchronous ones; a bad index in one step raises with
    THAT step's payload when its result is read, and that step's update is
    skipped while the steps around it apply."""
    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    sb = lambda hb, idx=None: [SparseBatch(o, i) for o, i in
                               zip(hb.offsets, idx if idx is not None else hb.indices)]
    ma, mb = build(c), build(c)
    ra = [train_step(ma, hb.dense, sb(hb), hb.labels, Sgd(0.1)) for hb in batches]
    pend = [train_step(mb, hb.dense, sb(hb), hb.labels, Sgd(0.1), sync=False) for hb in batches]
    for x, y in zip(ra, pend):
        assert x.loss == y.loss and x.accuracy == y.accuracy and torch.equal(x.probs, y.probs)
    for a, b in zip(arrays(ma.bottom, ma.top, ma.tables), arrays(mb.bottom, mb.top, mb.tables)):
        assert np.array_equal(a, b)
    # a bad index in the middle step of three
    m = build(c)
    bad = [i.copy() for i in batches[1].indices]
    bad[2][5] = c["tables"][2] + 77
    p0 = train_step(m, batches[0].dense, sb(batches[0]), batches[0].labels, Sgd(0.1), sync=False)
    p1 = train_step(m, batches[1].dense, sb(batches[1], bad), batches[1].labels, Sgd(0.1),
                    sync=False)
    p2 = train_step(m, batches[2].dense, sb(batches[2]), batches[2].labels, Sgd(0.1), sync=False)
    assert p0.loss > 0 and p2.loss > 0
    with pytest.raises(LookupIndexError) as e:
        _ = p1.loss
    assert (e.value.table_id, e.value.position, e.value.index) == (2, 5, c["tables"][2] + 77)
    # same as running steps 0 and 2 synchronously (step 1 skipped its updates)
    r = build(c)
    train_step(r, batches[0].dense, sb(batches[0]), batches[0].labels, Sgd(0.1))
    train_step(r, batches[2].dense, sb(batches[2]), batches[2].labels, Sgd(0.1))
    for a, b in zip(arrays(m.bottom, m.top, m.tables), arrays(r.bottom, r.top, r.tables)):
        assert np.array_equal(a, b)
    # more pending steps than read-back ring slots, read only at the end: the
    # reused slots hand their values, probabilities and a pending index error
    # to the older results first
    n = 3 * len(batches) + 13
    ms, ma2 = build(c), build(c)
    seq = [(batches[k % len(batches)], k == 5) for k in range(n)]
    sync, pend = [], []
    for hb, is_bad in seq:
        idx = None
        if is_bad:
            idx = [i.copy() for i in hb.indices]
            idx[1][0] = -3
        try:
            sync.append(train_step(ms, hb.dense, sb(hb, idx), hb.labels, Sgd(0.1)))
        except LookupIndexError as err:
            sync.append(err)
        pend.append(train_step(ma2, hb.dense, sb(hb, idx), hb.labels, Sgd(0.1), sync=False))
    for x, y in zip(sync, pend):
        if isinstance(x, LookupIndexError):
            with pytest.raises(LookupIndexError) as e:
                _ = y.loss
            assert (e.value.table_id, e.value.position, e.value.index) == \
                (x.table_id, x.position, x.index)
            continue
        assert x.loss == y.loss and x.accuracy == y.accuracy and torch.equal(x.probs, y.probs)
