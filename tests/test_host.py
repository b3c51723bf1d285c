"""Host-side logic that needs no GPU: plan bookkeeping (bit-identical to the
reference's fixtures), config validation, CSR helpers, input validation."""

import numpy as np
import pytest

from paper_1906_00091_b200 import (DevicePlan, DlrmConfig, SparseBatch,
                                   interaction_width, offsets_from_lengths,
                                   lengths_from_offsets, param_count,
                                   partition_tables, shard_bounds, make_plan)
from paper_1906_00091_b200.rng import RandomBatchSource


def test_offsets_fixtures():
    # ref test_embedding.py:20-35
    assert offsets_from_lengths([2, 3, 1]).tolist() == [0, 2, 5, 6]
    assert offsets_from_lengths([]).tolist() == [0]
    assert offsets_from_lengths([0, 0, 4]).tolist() == [0, 0, 0, 4]
    with pytest.raises(ValueError):
        offsets_from_lengths([1, -1])
    rng = np.random.default_rng(0)
    for _ in range(50):
        lens = rng.integers(0, 50, rng.integers(0, 40)).tolist()
        assert lengths_from_offsets(offsets_from_lengths(lens)).tolist() == lens


@pytest.mark.parametrize("o,i,w", [
    ([1, 2], [0, 0], None), ([0, 2, 1], [0, 0], None), ([0, 1], [0, 0], None),
    ([0, 2], [0, 1], [1.0])])
def test_sparse_batch_invariants_rejected_on_host(o, i, w):
    # ref test_embedding.py:44-60 (raised before any device work)
    with pytest.raises(ValueError):
        SparseBatch(np.array(o), np.array(i), None if w is None else np.array(w))


def test_partition_tables_fixtures():
    # ref test_parallel.py:57-93
    a = partition_tables([10] * 8, 4)
    assert [a.count(d) for d in range(4)] == [2, 2, 2, 2]
    assert partition_tables([3, 1, 2], 1) == [0, 0, 0]
    a = partition_tables([5, 4, 3, 3], 2)
    loads = [0, 0]
    for s, d in zip([5, 4, 3, 3], a):
        loads[d] += s
    assert sorted(loads) == [7, 8]
    with pytest.raises(ValueError):
        partition_tables([1], 0)


def test_partition_matches_reference_on_kaggle():
    # SURVEY §7 hard part 5: reference plan is [1,1,1,1,1,1,1,19] tables/GPU
    from tests.golden_consts import KAGGLE
    a = partition_tables([m * 16 for m in KAGGLE], 8)
    assert sorted(a.count(d) for d in range(8)) == [1, 1, 1, 1, 1, 1, 1, 19]


def test_shard_bounds_fixtures():
    # ref test_parallel.py:96-105
    assert shard_bounds(8, 4) == [0, 2, 4, 6, 8]
    assert shard_bounds(9, 4) == [0, 3, 5, 7, 9]
    assert np.diff(shard_bounds(10, 3)).tolist() == [4, 3, 3]
    with pytest.raises(ValueError):
        DevicePlan(2, [0, 1], [0, 1, 4]).validate()


def test_config_validation_and_widths():
    assert interaction_width(16, 27) == 367
    cfg = DlrmConfig([10] * 8, 16, [13, 512, 256, 64, 16], [512, 256, 1])
    assert cfg.top_in_dim == 52 and cfg.top_dims_chain()[0] == 52
    assert param_count(cfg) == 8 * 10 * 16 + 314705
    with pytest.raises(ValueError):
        DlrmConfig([10], 16, [13, 8], [4, 1])
    with pytest.raises(ValueError):
        DlrmConfig([10], 16, [13, 16], [4, 2])
    with pytest.raises(ValueError):
        DlrmConfig([10], 16, [13, 16], [4, 1], interaction="cat")


def test_mlp_param_count_c1():
    # c1 MLP params 314,705
    from paper_1906_00091_b200.model import mlp_param_count
    cfg = DlrmConfig([10] * 8, 16, [13, 512, 256, 64, 16], [512, 256, 1])
    assert (mlp_param_count(cfg.bottom_mlp_dims)
            + mlp_param_count(cfg.top_dims_chain())) == 314705


def test_make_plan_big_basin_balanced():
    cfg = DlrmConfig([10 ** 6] * 8, 64, [512, 512, 64], [1024, 1024, 1024, 1])
    for g in (1, 2, 4, 8):
        plan = make_plan(cfg, 2048 * g, g)
        assert sorted(plan.table_assignment.count(d) for d in range(g)) == \
            [8 // g] * g


def test_random_source_fixed_and_variable():
    src = RandomBatchSource([100, 50], 13, 16, 4, fixed=True, seed=3)
    hb = src.next_batch()
    assert hb.dense.shape == (16, 13)
    assert all(o[-1] == 64 for o in hb.offsets)
    src = RandomBatchSource([100, 50], 13, 16, 4, fixed=False, seed=3)
    hb = src.next_batch()
    for o, i, m in zip(hb.offsets, hb.indices, [100, 50]):
        lens = np.diff(o)
        assert lens.min() >= 1 and lens.max() <= 4 and o[-1] == i.size
        assert i.min() >= 0 and i.max() < m


def test_stage_timer_api():
    # ref timing.py:9-36
    import time
    from paper_1906_00091_b200.timing import NullTimer, StageTimer, add_seconds
    t = StageTimer()
    with t.section("a"):
        time.sleep(0.01)
    t.add("b", 0.5)
    add_seconds(t, {"b": 0.25, "c": 1.0})
    assert t.seconds["a"] >= 0.01 and t.seconds["b"] == 0.75 and t.seconds["c"] == 1.0
    assert abs(t.total() - sum(t.seconds.values())) < 1e-12
    n = NullTimer()
    with n.section("x"):
        pass
    add_seconds(n, {"x": 1.0})
    assert n.total() == 0.0

    class RefLike:  # the reference's StageTimer has only .seconds / .section
        def __init__(self):
            self.seconds = {}
    r = RefLike()
    add_seconds(r, {"loss": 0.5})
    add_seconds(r, {"loss": 0.5})
    assert r.seconds == {"loss": 1.0}


def test_input_layout_pack_serial_and_threaded():
    """One step's inputs as one block (pipeline.InputLayout): every section
    round-trips, the threaded pack equals the serial one, capacities bound."""
    from concurrent.futures import ThreadPoolExecutor
    import torch
    from paper_1906_00091_b200.pipeline import InputLayout
    from paper_1906_00091_b200.rng import RandomBatchSource
    src = RandomBatchSource([50, 70, 90], 13, 300, 5, False, seed=3)
    hb = src.next_batch()
    caps = [len(i) + 7 for i in hb.indices]
    for weighted in (False, True):
        L = InputLayout(300, 3, 13, caps, weighted)
        w = [np.linspace(0.5, 1.5, len(i)) for i in hb.indices] if weighted else None
        a = torch.zeros(L.nbytes, dtype=torch.uint8)
        b = torch.zeros(L.nbytes, dtype=torch.uint8)
        L.pack(a, hb.dense, hb.offsets, hb.indices, hb.labels, w)
        with ThreadPoolExecutor(4) as pool:
            L.pack(b, hb.dense, hb.offsets, hb.indices, hb.labels, w, pool)
        assert torch.equal(a, b)
        v = L.views(a)
        assert np.array_equal(v["x"][:, :13].numpy(), hb.dense.astype(np.float32))
        assert np.array_equal(v["labels"].numpy(), hb.labels.astype(np.float32))
        for t in range(3):
            assert np.array_equal(v["offsets"][t].numpy(), hb.offsets[t])
            cb = int(L.cap_base[t])
            assert np.array_equal(v["indices"][cb:cb + len(hb.indices[t])].numpy(), hb.indices[t])
            if weighted:
                assert np.array_equal(v["iweights"][cb:cb + len(hb.indices[t])].numpy(),
                                      w[t].astype(np.float32))
        assert L.sections["x"][0] == 0 and all(o % 16 == 0 for o, _ in L.sections.values())
    L = InputLayout(300, 3, 13, [5, 5, 5])
    with pytest.raises(OverflowError):
        L.pack(torch.zeros(L.nbytes, dtype=torch.uint8), hb.dense, hb.offsets, hb.indices,
               hb.labels)


def test_pack_paths_agree():
    """The C-side packer (libdlrmpy.so: buffer protocol, no per-table
    Python) writes the same block as the ctypes path and the numpy path,
    for the reference dtypes, weighted bags with unweighted tables, a
    strided dense view, and inputs it must hand back to numpy (float32
    dense, int32 indices); capacities still raise OverflowError."""
    import torch
    from paper_1906_00091_b200 import _lib
    from paper_1906_00091_b200.pipeline import InputLayout
    from paper_1906_00091_b200.rng import RandomBatchSource
    assert _lib.pylib() is not None, "libdlrmpy.so not built"
    src = RandomBatchSource([50, 70, 90, 40], 13, 200, 6, False, seed=5)
    hb = src.next_batch()
    caps = [len(i) + 3 for i in hb.indices]
    wide = np.zeros((200, 20))
    wide[:, 3:16] = hb.dense
    cases = [
        (hb.dense, hb.offsets, hb.indices, None, False),
        (hb.dense, hb.offsets, hb.indices,
         [np.linspace(0.5, 1.5, len(i)) if t % 2 == 0 else None
          for t, i in enumerate(hb.indices)], True),
        (wide[:, 3:16], hb.offsets, hb.indices, None, False),
        (hb.dense.astype(np.float32), hb.offsets, hb.indices, None, False),
        (hb.dense, hb.offsets, [i.astype(np.int32) for i in hb.indices], None, False),
    ]
    PL = _lib.pylib()
    for k, (dense, offs, idx, w, weighted) in enumerate(cases):
        L = InputLayout(200, 4, 13, caps, weighted)
        a, c = (torch.zeros(L.nbytes, dtype=torch.uint8) for _ in range(2))
        if weighted:
            for blk in (a, c):
                L.views(blk)["iweights"].fill_(1.0)
        rc = PL.dlrm_pack_batch_py(dense, hb.labels, offs, idx, w, a.data_ptr(),
                                   L._sec.ctypes.data, 200, 13, 16, 4, L._cap_base_ptr, 2)
        assert rc == (0 if k < 3 else 1)  # the last two go back to numpy
        L.pack(a, dense, offs, idx, hb.labels, w)
        pl, _lib._pylib = _lib._pylib, False  # the ctypes / numpy paths
        try:
            L.pack(c, dense, offs, idx, hb.labels, w)
        finally:
            _lib._pylib = pl
        assert torch.equal(a, c)
        v = L.views(a)
        assert np.array_equal(v["x"][:, :13].numpy(), np.asarray(dense, np.float32))
        for t in range(4):
            cb = int(L.cap_base[t])
            assert np.array_equal(v["indices"][cb:cb + len(idx[t])].numpy(), idx[t])
    L = InputLayout(200, 4, 13, [5] * 4)
    with pytest.raises(OverflowError):
        L.pack(torch.zeros(L.nbytes, dtype=torch.uint8), hb.dense, hb.offsets, hb.indices,
               hb.labels)


def test_traffic_balanced_plan():
    """policy="traffic": equal-traffic tables spread evenly whatever their
    sizes (the reference plan gives one of 8 GPUs 19 of the 26 Criteo-Kaggle
    tables); memory capacity is respected; the default stays the reference
    plan."""
    from bench import KAGGLE
    from paper_1906_00091_b200.parallel import partition_tables_by_traffic
    cfg = DlrmConfig(KAGGLE, 16, [13, 512, 256, 64, 16], [512, 256, 1])
    ref = make_plan(cfg, 2048 * 8, 8)
    counts = np.bincount(ref.table_assignment, minlength=8)
    assert counts.max() == 19
    tp = make_plan(cfg, 2048 * 8, 8, policy="traffic")
    counts = np.bincount(tp.table_assignment, minlength=8)
    assert counts.max() - counts.min() <= 1 and counts.sum() == 26
    assert make_plan(cfg, 2048 * 8, 8).table_assignment == ref.table_assignment
    # capacity: two big tables may not share a device
    own = partition_tables_by_traffic([1, 1, 1, 1], [10, 10, 1, 1], 2, capacity_bytes=11)
    assert own[0] != own[1]
    with pytest.raises(ValueError):
        partition_tables_by_traffic([1, 1], [10, 10], 1, capacity_bytes=15)
    # heavier pooling attracts fewer co-owned tables
    cfg2 = DlrmConfig([100] * 4, 8, [4, 8], [4, 1])
    p2 = make_plan(cfg2, 64, 2, policy="traffic", pooling=[100, 1, 1, 1])
    assert p2.table_assignment.count(p2.table_assignment[0]) == 1


def test_native_random_bags_bit_identical_to_numpy():
    """dlrm_random_bags replays numpy's Philox / Lemire draws: the native
    variable-length bags equal the Python loop's (ref datagen.py:79-96),
    including 1-row ranges, rows near 2^32 and the state left for the
    labels and the next batch."""
    from paper_1906_00091_b200.rng import RandomBatchSource
    for tabs, k in (([10 ** 6] * 3, 100), ([7, 5, 9], 3), ([30, 10 ** 9, 2 ** 31 + 5, 2 ** 32 - 1], 7),
                    ([1000, 1], 1)):
        a = RandomBatchSource(tabs, 13, 300, k, False, seed=3)
        b = RandomBatchSource(tabs, 13, 300, k, False, seed=3)
        b.native = False
        for _ in range(3):
            x, y = a.next_batch(), b.next_batch()
            assert np.array_equal(x.dense, y.dense) and np.array_equal(x.labels, y.labels)
            for o1, o2, i1, i2 in zip(x.offsets, y.offsets, x.indices, y.indices):
                assert np.array_equal(o1, o2) and np.array_equal(i1, i2)
