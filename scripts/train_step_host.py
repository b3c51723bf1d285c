"""Host-side cost of train_step(sync=False) by phase on pre-staged batches
(CONFIG=c1|c2|c3): validation, engine lookup, consume, graph replay,
result_async.  Times are host microseconds per call (perf_counter)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import DlrmConfig, Prefetcher, Sgd, init_model, train_step
from paper_1906_00091_b200 import parallel as P
from paper_1906_00091_b200.rng import RandomBatchSource
from bench import CONFIGS

c = CONFIGS[os.environ.get("CONFIG", "c2")]
B, T = c["batch"], len(c["tables"])
cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
model = init_model(cfg, table_init="device")
src = RandomBatchSource(cfg.embedding_sizes, c["bot"][0], B, c["k"], c["fixed"], seed=1)
hbs = [src.next_batch() for _ in range(4)]
caps = [max(len(h.indices[t]) for h in hbs) for t in range(T)]
K = 100
def gen():
    i = 0
    while True:
        yield hbs[i % 4]; i += 1
pf = Prefetcher(gen(), B, T, c["bot"][0], capacities=caps, depth=K + 12, threads=4, workers=2)
it = iter(pf)
opt = Sgd(0.1)
for _ in range(6):
    d, b, l = next(it); train_step(model, d, b, l, opt)
staged = [next(it) for _ in range(K)]
if os.environ.get("CLOSE"):
    pf.close()   # no packing workers during the timed loop
torch.cuda.synchronize()
time.sleep(0.3)
ph = [0.0] * 6
sub = [0.0] * 3
prev = None
for d, b, l in staged:
    t0 = time.perf_counter()
    bsz = int(d.shape[0])
    for t, sb in enumerate(b):
        if sb.num_segments != bsz:
            raise ValueError
    weighted = any(sb.weights is not None for sb in b)
    t1 = time.perf_counter()
    L = d._layout
    eng = P._engine_for(model, bsz, b, opt, L.weighted, caps=L.caps)
    t2 = time.perf_counter()
    d.consume(eng.input_sets[eng._set]["block"])
    t3 = time.perf_counter()
    eng.graph.replay()
    t4 = time.perf_counter()
    if os.environ.get("SPLIT"):
        k = eng._ring_next; eng._ring_next = (k + 1) % eng.RING
        h = eng._ring[k]
        a0 = time.perf_counter(); h.copy_(eng.res_dev, non_blocking=True)
        a1 = time.perf_counter(); ev = torch.cuda.Event(); ev.record(torch.cuda.current_stream())
        a2 = time.perf_counter(); pc = eng.prob.clone()
        a3 = time.perf_counter()
        sub[0] += a1 - a0; sub[1] += a2 - a1; sub[2] += a3 - a2
        from paper_1906_00091_b200.trainer import PendingStepResult
        r = PendingStepResult(eng, k, ev, pc)
    else:
        r = eng.result_async()
    t5 = time.perf_counter()
    if prev is not None:
        _ = prev.loss
    t6 = time.perf_counter()
    prev = r
    for i, (a, z) in enumerate(zip((t0, t1, t2, t3, t4, t5), (t1, t2, t3, t4, t5, t6))):
        ph[i] += z - a
names = ["validate", "_engine_for", "consume", "graph.replay", "result_async", "prev.loss"]
print(os.environ.get("CONFIG", "c2"), {n: round(v / K * 1e6, 1) for n, v in zip(names, ph)})

if os.environ.get("SPLIT"):
    print("result_async parts us:", [round(v / K * 1e6, 1) for v in sub], "(D2H copy_, event, prob.clone)")
if not os.environ.get("CLOSE"):
    pf.close()
