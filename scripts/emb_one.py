"""Time one embedding-bag forward / backward+SGD configuration (default: the
c3 lookup, 8 tables x 1M rows, d=64, pooling U[1,100], B=2048) with CUDA
events, L2 flushed before each rep.  Used for kernel tuning and as the ncu
target (``-k regex:emb_``).

    python scripts/emb_one.py [--tables 8] [--rows 1000000] [--d 64]
                              [--pool-max 100] [--batch 2048] [--zipf]
"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_00091_b200 import _lib
from paper_1906_00091_b200.rng import zipf_indices

ap = argparse.ArgumentParser()
ap.add_argument("--tables", type=int, default=8)
ap.add_argument("--rows", type=int, default=10**6)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--pool-max", type=int, default=100)
ap.add_argument("--pool-fixed", action="store_true")
ap.add_argument("--batch", type=int, default=2048)
ap.add_argument("--zipf", action="store_true")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--bwd", action="store_true")
ap.add_argument("--apply", action="store_true", help="also time the apply half alone")
a = ap.parse_args()

dev = torch.device("cuda")
T, m, d, B = a.tables, a.rows, a.d, a.batch
rng = np.random.default_rng(0)
W = torch.empty(T * m * d, device=dev).uniform_(-0.1, 0.1)
offs, idxs, descs = [], [], []
for t in range(T):
    lens = (np.full(B, a.pool_max) if a.pool_fixed
            else rng.integers(1, a.pool_max + 1, B))
    o = np.zeros(B + 1, np.int64); np.cumsum(lens, out=o[1:])
    n = int(o[-1])
    ix = zipf_indices(m, n, 1.05, seed=t) if a.zipf else rng.integers(0, m, n)
    offs.append(torch.as_tensor(o, device=dev)); idxs.append(torch.as_tensor(ix, device=dev))
    descs.append(_lib.TableDesc(offs[-1].data_ptr(), idxs[-1].data_ptr(), None, t * m, m,
                                (t) * d, n, t))
desc = _lib.table_array(descs)
nnz = sum(int(i.numel()) for i in idxs)
out = torch.empty((B, T * d), device=dev)
grad = torch.randn((B, T * d), device=dev) * 1e-3
ep = torch.empty(T, dtype=torch.int64, device=dev); ef = torch.zeros(1, dtype=torch.int32, device=dev)
s = _lib.stream_handle(); P = _lib.ptr
wsb = _lib.size("dlrm_emb_bwd_workspace_size", nnz, T * m, d)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
_lib.call("dlrm_err_reset", P(ep), T, P(ef), s)


def fwd():
    _lib.call("dlrm_emb_fwd", P(W), d, C.cast(desc, C.c_void_p), T, B, P(out), T * d, P(ep), P(ef), s)


def bwd():
    _lib.call("dlrm_emb_bwd_sgd", P(W), d, C.cast(desc, C.c_void_p), T, B, P(grad), T * d, 0.01,
              P(ef), T * m, P(ws), wsb, s)


def timeit(fn):
    fn(); torch.cuda.synchronize()
    ts = []
    for r in range(a.reps):
        flush.fill_(r & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


peak = 6553.6
tf = timeit(fwd)
bf = nnz * (4 * d + 8) + T * (B + 1) * 8 + B * T * 4 * d
rec = dict(nnz=nnz, fwd_us=round(tf * 1e3, 2), fwd_GBs=round(bf / tf / 1e6, 1),
           fwd_frac=round(bf / tf / 1e6 / peak, 3))
if a.bwd:
    tb = timeit(bwd)
    u = sum(int(torch.unique(i).numel()) for i in idxs)
    bb = B * T * 4 * d + nnz * 8 + T * (B + 1) * 8 + 2 * u * 4 * d
    rec.update(bwd_us=round(tb * 1e3, 2), bwd_GBs=round(bb / tb / 1e6, 1),
               bwd_frac=round(bb / tb / 1e6 / peak, 3))
    if a.apply:
        upd = _lib.Update(_lib.UPD_SGD, 0.01, 0.0, 0)
        _lib.call("dlrm_emb_bwd_prepare", d, C.cast(desc, C.c_void_p), T, B, T * m, P(ws), wsb, s)
        ta = timeit(lambda: _lib.call("dlrm_emb_bwd_apply", P(W), d, C.cast(desc, C.c_void_p), T, B,
                                      P(grad), T * d, C.byref(upd), P(ef), T * m, P(ws), wsb, s))
        rec.update(apply_us=round(ta * 1e3, 2), apply_GBs=round(bb / ta / 1e6, 1))
print(json.dumps(rec), flush=True)
