"""Host phases of the e2e loop with train_step(sync=False) and one-step-
behind loss reads (the bench's e2e leg) at c3."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import DlrmConfig, Prefetcher, Sgd, init_model, train_step
from paper_1906_00091_b200.rng import RandomBatchSource

threads = int(os.environ.get("THREADS", 4))
cfg = DlrmConfig([10 ** 6] * 8, 64, [512, 512, 64], [1024, 1024, 1024, 1], seed=0)
model = init_model(cfg, table_init="device")
src = RandomBatchSource(cfg.embedding_sizes, 512, 2048, 100, False, seed=1)
hbs = [src.next_batch() for _ in range(4)]
caps = [max(len(h.indices[t]) for h in hbs) for t in range(8)]
def gen():
    i = 0
    while True:
        yield hbs[i % 4]; i += 1
pf = Prefetcher(gen(), 2048, 8, 512, capacities=caps, depth=int(os.environ.get("DEPTH", 4)),
                threads=threads, workers=int(os.environ.get("WORKERS", 2)))
it = iter(pf)
opt = Sgd(0.1)
for _ in range(6):
    d, b, l = next(it); train_step(model, d, b, l, opt)
torch.cuda.synchronize()
K = 100
tn = tt = tl = 0.0
prev = None
evs = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
t0 = time.perf_counter()
for k in range(K):
    a = time.perf_counter(); d, b, l = next(it); tn += time.perf_counter() - a
    a = time.perf_counter(); r = train_step(model, d, b, l, opt, sync=False); tt += time.perf_counter() - a
    evs[k].record()
    a = time.perf_counter()
    if prev is not None:
        _ = prev.loss
    tl += time.perf_counter() - a
    prev = r
_ = prev.loss
tot = time.perf_counter() - t0
torch.cuda.synchronize()
gaps = [evs[k - 1].elapsed_time(evs[k]) for k in range(1, K)]
print(f"device step-to-step ms: mean {sum(gaps) / len(gaps):.3f} min {min(gaps):.3f}")
print(f"threads {threads} workers {os.environ.get('WORKERS', 2)}: step ms {tot / K * 1e3:.3f}; next() {tn / K * 1e3:.3f}, "
      f"train_step {tt / K * 1e3:.3f}, prev.loss {tl / K * 1e3:.3f}")
pf.close()
