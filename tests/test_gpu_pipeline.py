"""The input pipeline (pipeline.Prefetcher) feeding the drop-in train_step:
batches packed from the reference's host arrays by worker threads and
copied ahead give the same steps, bit for bit, as passing the arrays."""

import numpy as np
import pytest
import torch

from paper_1906_00091_b200 import (DlrmConfig, Prefetcher, Sgd, SparseBatch, StageTimer,
                                   init_model, train_step)
from paper_1906_00091_b200.rng import RandomBatchSource

pytestmark = pytest.mark.gpu


def _cfg():
    return DlrmConfig([500, 800, 300, 1200], 16, [13, 64, 16], [32, 16, 1], seed=4)


def test_prefetched_steps_equal_array_steps():
    cfg = _cfg()
    src = RandomBatchSource(cfg.embedding_sizes, 13, 256, 6, False, seed=2)
    batches = [src.next_batch() for _ in range(7)]
    caps = [max(len(hb.indices[t]) for hb in batches) for t in range(4)]
    ma, mb = init_model(cfg), init_model(cfg)
    ra = [train_step(ma, hb.dense, [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)],
                     hb.labels, Sgd(0.1)) for hb in batches]
    pf = Prefetcher(iter(batches), 256, 4, 13, capacities=caps, depth=3, threads=4)
    opt = Sgd(0.1)
    rb = [train_step(mb, d, b, l, opt) for d, b, l in pf]
    assert len(rb) == len(ra)
    for x, y in zip(ra, rb):
        assert x.loss == y.loss and torch.equal(x.probs, y.probs)
    for a, b in zip(ma.bottom.layers + ma.top.layers, mb.bottom.layers + mb.top.layers):
        assert torch.equal(a.weight, b.weight) and torch.equal(a.bias, b.bias)
    for a, b in zip(ma.tables, mb.tables):
        assert torch.equal(a.weights, b.weights)


def test_prefetcher_default_capacities_tuples_and_timer():
    """Tuple batches, capacities from the first batch (+25%), a timer."""
    cfg = _cfg()
    src = RandomBatchSource(cfg.embedding_sizes, 13, 128, 3, True, seed=5)
    tuples = [(hb.dense, hb.offsets, hb.indices, hb.labels)
              for hb in (src.next_batch() for _ in range(4))]
    m = init_model(cfg)
    t = StageTimer()
    losses = [train_step(m, d, b, l, Sgd(0.1), timer=t).loss
              for d, b, l in Prefetcher(iter(tuples), 128, 4, 13)]
    assert len(losses) == 4 and all(np.isfinite(losses))
    assert t.seconds["embedding_lookup"] > 0


def test_prefetcher_overflow_raises():
    cfg = _cfg()
    src = RandomBatchSource(cfg.embedding_sizes, 13, 64, 6, False, seed=6)
    batches = [src.next_batch() for _ in range(2)]
    pf = Prefetcher(iter(batches), 64, 4, 13, capacities=[10, 10, 10, 10])
    with pytest.raises(OverflowError):
        for d, b, l in pf:
            train_step(init_model(cfg), d, b, l, Sgd(0.1))


def test_native_and_python_staging_give_the_same_blocks():
    """The native stager (pack + H2D + event records in one call without
    the interpreter lock) and the Python staging path put identical input
    blocks on the device, in source order."""
    from paper_1906_00091_b200 import pipeline
    cfg = _cfg()
    src = RandomBatchSource(cfg.embedding_sizes, 13, 128, 5, False, seed=9)
    batches = [src.next_batch() for _ in range(6)]
    caps = [max(len(hb.indices[t]) for hb in batches) for t in range(4)]
    blocks = {}
    for native in (True, False):
        saved, pipeline._STAGE_NATIVE = pipeline._STAGE_NATIVE, native
        try:
            pf = Prefetcher(iter(batches), 128, 4, 13, capacities=caps, depth=3, threads=2)
            got = []
            for d, b, l in pf:
                out = torch.empty_like(d._slot.dev)
                d.consume(out)
                torch.cuda.synchronize()
                got.append((out.cpu(), [sb.nnz for sb in b]))
            pf.close()
        finally:
            pipeline._STAGE_NATIVE = saved
        blocks[native] = got
    assert len(blocks[True]) == len(blocks[False]) == 6
    for (a, na), (b, nb) in zip(blocks[True], blocks[False]):
        assert torch.equal(a, b) and na == nb
    assert [n for _, n in blocks[True]] == [[len(i) for i in hb.indices] for hb in batches]
