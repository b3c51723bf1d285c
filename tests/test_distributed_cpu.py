"""Multi-process (world_size 2, gloo, CPU) tests of the hybrid-parallel
exchange: the personalized all-to-all of pooled embeddings and its reverse
reproduce the reference's butterfly_shuffle / inverse_shuffle semantics
(ref parallel.py:146-208) exactly; the gradient allreduce sums replicas.
The kernels need a GPU; everything that moves data between ranks is here."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1906_00091_b200.distributed import (ExchangeLayout, LocalExchange,
                                               NcclExchange)
from paper_1906_00091_b200.parallel import (DevicePlan, butterfly_shuffle,
                                            inverse_shuffle, partition_tables,
                                            shard_bounds)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def reference_data(plan, d, seed=0):
    g = torch.Generator().manual_seed(seed)
    T = len(plan.table_assignment)
    full = {t: torch.randn((plan.batch_size, d), generator=g) for t in range(T)}
    grads = []
    for r in range(plan.num_devices):
        lo, hi = plan.shard(r)
        grads.append({t: torch.randn((hi - lo, d), generator=g) for t in range(T)})
    return full, grads


def pack_send(L, full):
    own = L.owned[L.rank]
    buf = torch.zeros((L.B_global, len(own), L.d))
    for j, t in enumerate(own):
        buf[:, j] = full[t]
    return buf.reshape(-1)


def pack_gsend(L, grads_r):
    g = torch.zeros(max(L.recv_numel, 1))
    for t, (off, stride) in L.feature.items():
        for b in range(L.B_local):
            g[off + b * stride: off + b * stride + L.d] = grads_r[t][b]
    return g


def check_rank(L, recv, grecv, full, grads):
    # forward: every table's rows of my shard, in the reference's layout
    shuffled = butterfly_shuffle(full, L.plan)[L.rank]
    for s in shuffled:
        off, stride = L.feature[s.table_id]
        got = torch.stack([recv[off + b * stride: off + b * stride + L.d]
                           for b in range(L.B_local)])
        assert torch.equal(got, s.values)
        assert s.source_device == L.plan.table_assignment[s.table_id]
    # backward: the owner gets [B_g, T_own, d] = inverse_shuffle's full grads
    back = inverse_shuffle(grads, L.plan)
    own = L.owned[L.rank]
    if own:
        g = grecv[:L.send_numel].reshape(L.B_global, len(own), L.d)
        for j, t in enumerate(own):
            assert torch.equal(g[:, j], back[t])


def _worker(rank, world, port, tables, batch, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = DevicePlan(world, partition_tables([m * d for m in tables], world),
                          shard_bounds(batch, world))
        L = ExchangeLayout(plan, rank, d)
        ex = NcclExchange(L)
        full, grads = reference_data(plan, d)
        recv = torch.zeros(max(L.recv_numel, 1))
        ex.forward(pack_send(L, full), recv[:L.recv_numel])
        grecv = torch.zeros(max(L.send_numel, 1))
        ex.backward(pack_gsend(L, grads[rank])[:L.recv_numel], grecv[:L.send_numel])
        check_rank(L, recv, grecv, full, grads)
        t = torch.full((5,), float(rank + 1))
        ex.allreduce_async(t).wait()
        assert torch.equal(t, torch.full((5,), float(sum(range(1, world + 1)))))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tables,batch", [([7, 5, 9], 9), ([100] * 8, 16),
                                          ([300, 3, 50, 7], 11), ([10], 4)])
def test_gloo_world2_exchange_matches_reference(tables, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tables, batch, 4, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


@pytest.mark.parametrize("G,tables,batch", [(1, [7, 5], 6), (3, [7, 5, 9, 4], 10),
                                            (4, [5] * 8, 9)])
def test_local_exchange_matches_reference(G, tables, batch):
    d = 3
    plan = DevicePlan(G, partition_tables([m * d for m in tables], G),
                      shard_bounds(batch, G))
    Ls = [ExchangeLayout(plan, r, d) for r in range(G)]
    full, grads = reference_data(plan, d, seed=G)
    sends = [pack_send(L, full) for L in Ls]
    recvs = [torch.zeros(max(L.recv_numel, 1)) for L in Ls]
    ex = LocalExchange(Ls)
    ex.forward_all(sends, recvs)
    gsends = [pack_gsend(L, grads[r]) for r, L in enumerate(Ls)]
    grecvs = [torch.zeros(max(L.send_numel, 1)) for L in Ls]
    ex.backward_all(gsends, grecvs)
    for r, L in enumerate(Ls):
        check_rank(L, recvs[r], grecvs[r], full, grads)


def test_layout_split_sizes_conserve_bytes():
    d, G = 16, 8
    from tests.golden_consts import KAGGLE
    plan = DevicePlan(G, partition_tables([m * d for m in KAGGLE], G),
                      shard_bounds(2048 * G, G))
    Ls = [ExchangeLayout(plan, r, d) for r in range(G)]
    for r in range(G):
        for s in range(G):
            assert Ls[s].send_split[r] == Ls[r].recv_split[s]
    assert sum(L.send_numel for L in Ls) == sum(L.recv_numel for L in Ls) \
        == 2048 * G * len(KAGGLE) * d
