"""Hybrid-parallel step on one GPU: G virtual ranks running the per-rank
kernel sequence of the multi-process HybridTrainer (RankEngine) with
in-process exchanges.

* G = 1 is bitwise identical to the fused single-device step.
* G = 2, 3, 4 match the reference trajectory (whose ParallelTrainer is
  bit-identical to its serial train_step) within the north-star tolerance.
"""

import numpy as np
import pytest

from paper_1906_00091_b200 import (DlrmConfig, ParallelTrainer, Sgd, SparseBatch,
                                   format_comm_report, init_model, make_plan,
                                   train_step)
from tests._util import rel_err, traj_inputs

pytestmark = pytest.mark.gpu


def build(c):
    return init_model(DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=c["seed"]))


def arrays_of(bottom, top, tables):
    out = []
    for l in bottom.layers + top.layers:
        out += [l.weight.detach().cpu().double().numpy(),
                l.bias.detach().cpu().double().numpy()]
    return out + [t.weights.detach().cpu().double().numpy() for t in tables]


def run_parallel(c, batches, G):
    model = build(c)
    caps = [max(len(hb.indices[t]) for hb in batches) for t in range(len(c["tables"]))]
    tr = ParallelTrainer(model, make_plan(model.config, c["batch"], G),
                         c.get("opt", "sgd"), c["lr"], eps=c.get("eps", 1e-10),
                         capacities=caps)
    res = []
    for hb in batches:
        sparse = [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]
        res.append(tr.step(hb.dense.astype(np.float32), sparse,
                           hb.labels.astype(np.float32)))
    return tr, res


def test_one_rank_is_bitwise_the_fused_step(golden):
    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    tr, res = run_parallel(c, batches, 1)
    model = build(c)
    opt = Sgd(c["lr"])
    for hb, r in zip(batches, res):
        sparse = [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]
        s = train_step(model, hb.dense.astype(np.float32), sparse, hb.labels, opt)
        assert s.loss == r.loss
    b, t = tr.replica_params(0)
    for x, y in zip(arrays_of(b, t, tr.tables), arrays_of(model.bottom, model.top,
                                                          model.tables)):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name,G", [("toy", 2), ("toy", 3), ("c1s", 2), ("c1s", 4),
                                    ("c2s", 4), ("c3s", 3), ("c1a", 2), ("c3a", 3)])
def test_matches_reference_trajectory(golden, name, G):
    fx = golden(f"traj_{name}.npz")
    c, batches = traj_inputs(fx)
    tr, res = run_parallel(c, batches, G)
    for s, r in enumerate(res):
        ref = fx["losses"][s]
        assert abs(r.loss - ref) <= 1e-4 * abs(ref), (s, r.loss, ref)
        assert r.accuracy == fx["accs"][s] or abs(r.accuracy - fx["accs"][s]) <= 1.0 / c["batch"]
    b, t = tr.replica_params(0)
    for i, a in enumerate(arrays_of(b, t, tr.tables)):
        assert rel_err(a, fx[f"final_{i}"], floor=1e-2) < 1e-4, i
    assert tr.max_replica_divergence() == 0.0
    names = {line.split(", ")[1] for line in format_comm_report(tr.comm).strip().split("\n")[1:]}
    assert names == {"butterfly_shuffle", "grad_reverse_shuffle", "loss_gather",
                     "grad_allreduce"}


def test_bad_index_raises_with_device_and_mutates_nothing(golden):
    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    tr, _ = run_parallel(c, batches[:1], 2)
    b, t = tr.replica_params(1)
    before = arrays_of(b, t, tr.tables)
    hb = batches[1]
    idx = [i.copy() for i in hb.indices]
    idx[6][5] = 10 ** 6
    sparse = [SparseBatch(o, i) for o, i in zip(hb.offsets, idx)]
    owner = tr.plan.table_assignment[6]
    with pytest.raises(RuntimeError, match=f"device {owner}"):
        tr.step(hb.dense.astype(np.float32), sparse, hb.labels.astype(np.float32))
    for x, y in zip(before, arrays_of(b, t, tr.tables)):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("force", [False, True])
def test_hybrid_trainer_nccl_one_process(golden, force):
    """HybridTrainer over a real NCCL communicator (one process, one GPU):
    the all-to-alls, the overlapped allreduces, the no-sync step and the
    deferred error check run through the multi-process code path and give
    the same losses as the fused single-device step."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_1906_00091_b200.distributed import HybridTrainer

    fx = golden("traj_c1s.npz")
    c, batches = traj_inputs(fx)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        model = build(c)
        plan = make_plan(model.config, c["batch"], 1)
        caps = [max(len(hb.indices[t]) for hb in batches) for t in range(len(c["tables"]))]
        # force: the multi-rank path (collectives on the comm stream, unfused
        # updates after the gradient allreduce) with a one-rank communicator;
        # else the one-rank path (no collectives, fused updates)
        tr = HybridTrainer(model, plan, 0, caps, lr=c["lr"], force_exchange=force)
        ref_model = build(c)
        opt = Sgd(c["lr"])
        for k, hb in enumerate(batches):
            if k < 2:   # eager steps through load()
                tr.load(hb.dense.astype(np.float32), hb.labels.astype(np.float32),
                        hb.offsets, hb.indices)
            else:       # packed input block + the captured step graph
                tr.stage(tr.pack(hb.dense, hb.labels, hb.offsets, hb.indices))
            if k == 2:
                assert tr.capture()
            if k % 2:
                r = tr.step()
            else:
                assert tr.step(sync=False) is None
                tr.check_errors()
                r = tr.result()
            sparse = [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)]
            s = train_step(ref_model, hb.dense.astype(np.float32), sparse, hb.labels, opt)
            assert abs(r.loss - s.loss) <= 1e-6 * abs(s.loss), (k, r.loss, s.loss)
            if not force:   # the same kernels as the fused step, in the same order
                assert r.loss == s.loss
        # a graph holding NCCL work must be released before the communicator
        tr.graph = None
        del tr
        import gc
        gc.collect()
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
