"""Run the same short c1 trajectory several times in one process (tcgen05
and SIMT GEMMs) and print per-run loss bits and a parameter digest."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1906_00091_b200 import DlrmConfig, Sgd, SparseBatch, init_model, train_step, _lib
from paper_1906_00091_b200.rng import RandomBatchSource

def run(mode, steps=10):
    _lib.call("dlrm_gemm_mode", mode)
    cfg = DlrmConfig([10 ** 4] * 8, 16, [13, 512, 256, 64, 16], [512, 256, 1], seed=0)
    m = init_model(cfg)
    src = RandomBatchSource(cfg.embedding_sizes, 13, 128, 1, True, seed=0)
    losses = []
    for _ in range(steps):
        hb = src.next_batch()
        r = train_step(m, hb.dense.astype(np.float32), [SparseBatch(o, i) for o, i in zip(hb.offsets, hb.indices)], hb.labels, Sgd(0.1))
        losses.append(r.loss)
    h = hashlib.sha256()
    for l in m.bottom.layers + m.top.layers:
        h.update(l.weight.detach().cpu().numpy().tobytes())
    return [float(np.float32(x)) for x in losses[-3:]], h.hexdigest()[:16], _lib.launch_count()

for mode in (0, 0, 1, 0):
    print(mode, run(mode), flush=True)
