"""Per-phase device times of the hybrid (multi-process) step at N = 1 under
torchrun, c3: where the hybrid path spends time beyond the fused engine.

    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 \
        scripts/hybrid_phases.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from bench import CONFIGS, rank_batches
from paper_1906_00091_b200 import DlrmConfig, init_model, make_plan
from paper_1906_00091_b200.distributed import HybridTrainer

torch.cuda.set_device(0)
dist.init_process_group("nccl")
c = CONFIGS["c3"]
B = c["batch"]
cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
model = init_model(cfg, table_init="device")
plan = make_plan(cfg, B, 1)
tr = HybridTrainer(model, plan, 0, [B * c["k"]] * 8, lr=0.1, ar_group=dist.new_group([0]))
hb = rank_batches(c, plan, 0, 1, seed=1)[0]
dev = torch.device("cuda")
db = (torch.as_tensor(hb[0].astype(np.float32), device=dev),
      torch.as_tensor(hb[1].astype(np.float32), device=dev),
      [torch.as_tensor(o, device=dev) for o in hb[2]],
      [torch.as_tensor(i, device=dev) for i in hb[3]])
for _ in range(5):
    tr.load(*db)
    tr.step(sync=False)
torch.cuda.synchronize()
e, ex = tr.engine, tr.ex
names = []
evs = []


def mark(n):
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    names.append(n)
    evs.append(ev)


acc = {}
for rep in range(10):
    names.clear(); evs.clear()
    tr.load(*db)
    mark("start")
    e.prepare_sparse_backward()
    mark("prepare(inline)")
    e.phase_a()
    mark("phase_a lookups")
    ex.forward(e.send, e.recv)
    mark("all_to_all fwd")
    e.phase_b_forward()
    mark("bottom+interaction+top fwd+head")
    e.publish_error(); ex.allreduce(e.stats); e.adopt_global_error()
    mark("stats allreduce")
    e.phase_b_top_backward()
    mark("top bwd")
    h = ex.allreduce_async(e.grads[e.split_at:]); h.wait()
    mark("top allreduce")
    e.phase_b_interaction_backward()
    mark("interaction bwd")
    ex.backward(e.gsend, e.grecv)
    mark("all_to_all bwd")
    e.apply_sparse()
    mark("apply")
    e.phase_b_bottom_backward()
    mark("bottom bwd")
    h = ex.allreduce_async(e.grads[:e.split_at]); h.wait()
    mark("bottom allreduce")
    e.sgd_dense()
    mark("sgd_dense")
    torch.cuda.synchronize()
    for n, a, b in zip(names[1:], evs[:-1], evs[1:]):
        acc[n] = acc.get(n, 0.0) + a.elapsed_time(b) / 10
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    tr.load(*db)
    tr.step(sync=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue per step {(t1 - t0) / 20 * 1e6:8.1f} us ; wall per step {(t2 - t0) / 20 * 1e6:8.1f} us")
tot = sum(acc.values())
for n, v in acc.items():
    print(f"{n:36s} {v * 1e3:8.1f} us")
print(f"{'total (serialised)':36s} {tot * 1e3:8.1f} us")
dist.destroy_process_group()
