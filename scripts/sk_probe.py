"""Time one GEMM shape (fwd) under the current env: stream-K experiments."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib
M, N, K = (int(x) for x in os.environ.get("SHAPE", "2048,1024,1024").split(","))
X = torch.randn((M, K), device="cuda"); W = torch.randn((N, K), device="cuda") / K ** .5
b = torch.zeros(N, device="cuda"); Y = torch.empty((M, N), device="cuda")
s = _lib.stream_handle()
fn = lambda: _lib.call("dlrm_linear_fwd", _lib.ptr(X), K, _lib.ptr(W), K, _lib.ptr(b), _lib.ptr(Y), N, M, N, K, N, 0, s)
flush = torch.empty(64 << 20, device="cuda")
for _ in range(5): fn()
torch.cuda.synchronize()
ts = []
for gap in (0, 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(20):
        if gap: flush.zero_()
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ts.append(round(tot / 20 * 1e3, 2))
e0.record()
for _ in range(20): fn()
e1.record(); torch.cuda.synchronize()
ts.append(round(e0.elapsed_time(e1) / 20 * 1e3, 2))
ref = X.double() @ W.double().T
print(os.environ.get("TAG", ""), "single/flushed/b2b us:", ts, "err %.1e" % float((Y.double() - ref).abs().max() / ref.abs().max()), flush=True)
