"""Timeline of one captured training step: every library call of
StepEngine.launch() is bracketed by timing events recorded on the stream it
runs on, the whole step (four streams) is captured into one CUDA graph and
replayed; start / end of each call relative to the step start are printed
per stream.  The event nodes add small gaps, so the step is a few us longer
than the bench's.

    python scripts/step_timeline.py [--config c3] [--reps 20]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_1906_00091_b200 import DlrmConfig, init_model, _lib
from paper_1906_00091_b200.rng import RandomBatchSource
from paper_1906_00091_b200.trainer import StepEngine

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
c = CONFIGS[a.config]
B = c["batch"]
cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
model = init_model(cfg, table_init="device")
src = RandomBatchSource(c["tables"], c["bot"][0], B, c["k"], c["fixed"], seed=1)
hb = src.next_batch()
eng = StepEngine(model, B, [B * c["k"]] * cfg.num_tables, lr=0.1)
eng.load(hb.dense, hb.offsets, hb.indices, hb.labels)
eng.run()
torch.cuda.synchronize()

streams = {}
for name, st in (("main", torch.cuda.current_stream()), ("side", eng.side),
                 ("emb", eng.fwd_stream), ("wgrad", eng.wg_stream)):
    streams[_lib.stream_handle(st).value if hasattr(_lib.stream_handle(st), "value")
            else int(_lib.stream_handle(st))] = (name, st)
records = []
real_call = _lib.call


def traced(fn, *args):
    h = args[-1] if args else None
    key = getattr(h, "value", h)
    ent = streams.get(key)
    if ent is None or not fn.startswith("dlrm_"):
        return real_call(fn, *args)
    e0, e1 = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
    e0.record(ent[1])
    r = real_call(fn, *args)
    e1.record(ent[1])
    records.append((ent[0], fn, e0, e1))
    return r


g = torch.cuda.CUDAGraph()
torch.cuda.synchronize()
main = torch.cuda.current_stream()
with torch.cuda.graph(g):
    cap = torch.cuda.current_stream()
    streams[getattr(_lib.stream_handle(cap), "value", _lib.stream_handle(cap))] = ("main", cap)
    start = torch.cuda.Event(enable_timing=True, external=True)
    start.record(cap)
    _lib.call = traced
    try:
        eng.launch()
    finally:
        _lib.call = real_call
    end = torch.cuda.Event(enable_timing=True, external=True)
    end.record(cap)
acc = {}
tot = []
for r in range(a.reps):
    g.replay()
    torch.cuda.synchronize()
    tot.append(start.elapsed_time(end))
    for i, (sname, fn, e0, e1) in enumerate(records):
        s, e = start.elapsed_time(e0), start.elapsed_time(e1)
        acc.setdefault(i, []).append((s, e))
print(f"step (graph with event nodes): {np.median(tot) * 1e3:.1f} us")
rows = []
for i, (sname, fn, _, _) in enumerate(records):
    s = np.median([x[0] for x in acc[i]]) * 1e3
    e = np.median([x[1] for x in acc[i]]) * 1e3
    rows.append((s, e, sname, fn))
for s, e, sname, fn in sorted(rows):
    print(f"{sname:6s} {s:7.1f} -> {e:7.1f}  ({e - s:6.1f} us)  {fn}")
