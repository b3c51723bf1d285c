"""Achievable random-row gather bandwidth on this GPU (torch index_select and
a plain sum of gathered rows) vs our pooled-lookup kernel, c3 shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ctypes as C, numpy as np
from paper_1906_00091_b200 import _lib
T, rows, d, B, k = 8, 10**6, 64, 2048, 100
W = torch.rand(T * rows * d, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
lens = torch.randint(1, k + 1, (T, B), device="cuda", generator=g)
offs = torch.zeros((T, B + 1), dtype=torch.int64, device="cuda"); offs[:, 1:] = lens.cumsum(1)
nnz = [int(offs[t, -1]) for t in range(T)]
idx = [torch.randint(0, rows, (n,), device="cuda", generator=g) for n in nnz]
gidx = torch.cat([i + t * rows for t, i in enumerate(idx)])
out = torch.empty((B, T * d), device="cuda")
def timeit(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    for _ in range(n):
        fl.fill_(1); e0.record(); f(); e1.record(); torch.cuda.synchronize(); tot += e0.elapsed_time(e1)
    return tot / n
Wm = W.view(-1, d)
bytes_rows = sum(nnz) * d * 4
t_sel = timeit(lambda: torch.index_select(Wm, 0, gidx))
print(f"torch.index_select {sum(nnz)} rows x {d*4} B: {t_sel*1e3:.1f} us -> {bytes_rows/t_sel/1e6:.0f} GB/s (rows only, + same write)")
descs = _lib.table_array([_lib.TableDesc(offs[t].data_ptr(), idx[t].data_ptr(), None, t * rows, rows, t * d, nnz[t], t) for t in range(T)])
ep = torch.empty(T, dtype=torch.int64, device="cuda"); ef = torch.zeros(1, dtype=torch.int32, device="cuda")
s = _lib.stream_handle()
def ours():
    _lib.call("dlrm_emb_fwd", _lib.ptr(W), d, C.cast(descs, C.c_void_p), T, B, _lib.ptr(out), T * d, _lib.ptr(ep), _lib.ptr(ef), s)
t_ours = timeit(ours)
alg = sum(n * (4 * d + 8) + (B + 1) * 8 + B * 4 * d for n in nnz)
print(f"dlrm_emb_fwd: {t_ours*1e3:.1f} us -> {alg/t_ours/1e6:.0f} GB/s algorithmic ({alg/1e6:.1f} MB)")
