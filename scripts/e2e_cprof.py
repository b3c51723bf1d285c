"""cProfile of the drop-in train_step loop on Prefetcher batches at c3 (host
overhead per call; the device step is ~0.41 ms)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import DlrmConfig, Prefetcher, Sgd, init_model, train_step
from paper_1906_00091_b200.rng import RandomBatchSource

cfg = DlrmConfig([10 ** 6] * 8, 64, [512, 512, 64], [1024, 1024, 1024, 1], seed=0)
model = init_model(cfg, table_init="device")
src = RandomBatchSource(cfg.embedding_sizes, 512, 2048, 100, False, seed=1)
hbs = [src.next_batch() for _ in range(4)]
caps = [max(len(h.indices[t]) for h in hbs) for t in range(8)]
def gen():
    i = 0
    while True:
        yield hbs[i % 4]; i += 1
pf = Prefetcher(gen(), 2048, 8, 512, capacities=caps, depth=3, threads=4)
it = iter(pf)
opt = Sgd(0.1)
for _ in range(6):
    d, b, l = next(it); train_step(model, d, b, l, opt)
torch.cuda.synchronize()
K = 100
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(K):
    d, b, l = next(it)
    r = train_step(model, d, b, l, opt)
    _ = r.loss
pr.disable()
print(f"step ms {(time.perf_counter() - t0) / K * 1e3:.3f}")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
pf.close()
