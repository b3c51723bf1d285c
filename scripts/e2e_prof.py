"""Host-side cost of the drop-in train_step on staged (Prefetcher) batches at
c3: per-phase wall time of the call and the step's device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1906_00091_b200 import DlrmConfig, Prefetcher, Sgd, init_model, train_step
from paper_1906_00091_b200.rng import RandomBatchSource
import paper_1906_00091_b200.parallel as par

threads = int(os.environ.get("THREADS", 8))
cfg = DlrmConfig([10 ** 6] * 8, 64, [512, 512, 64], [1024, 1024, 1024, 1], seed=0)
model = init_model(cfg, table_init="device")
src = RandomBatchSource(cfg.embedding_sizes, 512, 2048, 100, False, seed=1)
hbs = [src.next_batch() for _ in range(4)]
caps = [max(len(h.indices[t]) for h in hbs) for t in range(8)]
def gen():
    i = 0
    while True:
        yield hbs[i % 4]; i += 1
pf = Prefetcher(gen(), 2048, 8, 512, capacities=caps, depth=3, threads=threads)
it = iter(pf)
opt = Sgd(0.1)
for _ in range(6):
    d, b, l = next(it); train_step(model, d, b, l, opt)
torch.cuda.synchronize()
K = 50
tw = tt = 0.0
t0 = time.perf_counter()
for _ in range(K):
    a = time.perf_counter(); d, b, l = next(it); tw += time.perf_counter() - a
    a = time.perf_counter(); r = train_step(model, d, b, l, opt); _ = r.loss; tt += time.perf_counter() - a
tot = time.perf_counter() - t0
print(f"threads {threads}: step ms {tot / K * 1e3:.3f}, next() {tw / K * 1e3:.3f}, train_step {tt / K * 1e3:.3f}")
# train_step without the prefetcher's worker running: same staged batch reused
eng = model._engine
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(K):
    eng.graph.replay(); r = eng.result()
print(f"replay+result only ms {(time.perf_counter() - t0) / K * 1e3:.3f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    eng.graph.replay()
e1.record(); torch.cuda.synchronize()
print(f"device step ms {e0.elapsed_time(e1) / K:.3f}")
pf.close()
