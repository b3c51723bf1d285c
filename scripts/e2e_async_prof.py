"""Host phases of the e2e loop with train_step(sync=False) and one-step-
behind loss reads (the bench's e2e leg): CONFIG=c1|c2|c3|c4 (default c3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import DlrmConfig, Prefetcher, Sgd, init_model, train_step
from paper_1906_00091_b200.rng import RandomBatchSource

from bench import CONFIGS
if os.environ.get("SWITCH"):
    sys.setswitchinterval(float(os.environ["SWITCH"]))
threads = int(os.environ.get("THREADS", 4))
c = CONFIGS[os.environ.get("CONFIG", "c3")]
B = c["batch"]
cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
model = init_model(cfg, table_init="device")
src = RandomBatchSource(cfg.embedding_sizes, c["bot"][0], B, c["k"], c["fixed"], seed=1)
hbs = [src.next_batch() for _ in range(4)]
T = len(c["tables"])
caps = [max(len(h.indices[t]) for h in hbs) for t in range(T)]
def gen():
    i = 0
    while True:
        yield hbs[i % 4]; i += 1
pf = Prefetcher(gen(), B, T, c["bot"][0], capacities=caps,
                depth=int(os.environ.get("DEPTH", 110 if os.environ.get("PRESTAGE") else 4)),
                threads=threads, workers=int(os.environ.get("WORKERS", 2)))
it = iter(pf)
opt = Sgd(0.1)
for _ in range(6):
    d, b, l = next(it); train_step(model, d, b, l, opt)
torch.cuda.synchronize()
K = 100
if os.environ.get("PRESTAGE"):
    # all K batches staged before the timed loop: train_step's own host cost
    # without packing workers competing for the interpreter
    staged = [next(it) for _ in range(K)]
    torch.cuda.synchronize()
    time.sleep(0.5)
    sit = iter(staged)
    it = sit
tn = tt = tl = 0.0
prev = None
evs = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
t0 = time.perf_counter()
for k in range(K):
    a = time.perf_counter(); d, b, l = next(it); tn += time.perf_counter() - a
    a = time.perf_counter()
    if os.environ.get("NORESULT"):  # measurement: the step without its result read-back
        from paper_1906_00091_b200 import parallel as _P
        eng = _P._engine_for(model, int(d.shape[0]), b, opt, d._layout.weighted, caps=d._layout.caps)
        d.consume(eng.input_sets[eng._set]["block"])
        eng.graph.replay()
        r = None
    else:
        r = train_step(model, d, b, l, opt, sync=False)
    tt += time.perf_counter() - a
    evs[k].record()
    a = time.perf_counter()
    if prev is not None:
        _ = prev.loss
    elif r is None and k % 2 == 1:
        evs[k - 1].synchronize()  # keep the host at most ~2 steps ahead
    tl += time.perf_counter() - a
    prev = r
if prev is not None:
    _ = prev.loss
tot = time.perf_counter() - t0
torch.cuda.synchronize()
gaps = [evs[k - 1].elapsed_time(evs[k]) for k in range(1, K)]
print(f"device step-to-step ms: mean {sum(gaps) / len(gaps):.3f} min {min(gaps):.3f}")
import cProfile, pstats
if os.environ.get("CPROF") and not os.environ.get("PRESTAGE"):
    pr = cProfile.Profile(); pr.enable()
    for k in range(50):
        d, b, l = next(it); r = train_step(model, d, b, l, opt, sync=False)
        if prev is not None: _ = prev.loss
        prev = r
    _ = prev.loss
    pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(18)
print(f"threads {threads} workers {os.environ.get('WORKERS', 2)}: step ms {tot / K * 1e3:.3f}; next() {tn / K * 1e3:.3f}, "
      f"train_step {tt / K * 1e3:.3f}, prev.loss {tl / K * 1e3:.3f}")
pf.close()
