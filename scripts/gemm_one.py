import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib
B, K, N = 2048, int(os.environ.get("K", 1024)), 1024
X = torch.randn((B, K), device="cuda"); W = torch.randn((N, K), device="cuda")
b = torch.zeros(N, device="cuda"); Y = torch.empty((B, N), device="cuda")
s = _lib.stream_handle()
f = lambda: _lib.call("dlrm_linear_fwd", _lib.ptr(X), K, _lib.ptr(W), K, _lib.ptr(b), _lib.ptr(Y), N, B, N, K, N, 1, _lib.stream_handle())
for _ in range(5): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): f()
e1.record(); torch.cuda.synchronize()
print(os.environ.get("DLRM_B200_LIB", "default"), "fwd 2048x1024x1024 us:", e0.elapsed_time(e1) / 50 * 1e3)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(50): f()
g.replay(); torch.cuda.synchronize()
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print("graph-replayed fwd us:", e0.elapsed_time(e1) / 50 * 1e3)
