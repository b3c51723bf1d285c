"""Forward / data-gradient GEMM with precomputed W_lo vs the per-tile
conversion: time and bitwise equality.  SHAPE=M,N,K."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib
for shape in os.environ.get("SHAPES", "2048,1024,1024;32768,1024,1024;32768,512,1024;32768,1024,480;2048,512,512;32768,256,512").split(";"):
    M, N, K = (int(x) for x in shape.split(","))
    X = torch.randn((M, K), device="cuda"); W = torch.randn((N, K), device="cuda") / K ** .5
    Wl = torch.empty_like(W)
    b = torch.randn(N, device="cuda"); Y = torch.empty((M, N), device="cuda"); Y2 = torch.empty_like(Y)
    gZ = torch.randn((M, N), device="cuda"); dX = torch.empty((M, K), device="cuda"); dX2 = torch.empty_like(dX)
    s = _lib.stream_handle()
    P = _lib.ptr
    _lib.call("dlrm_tf32_split_lo", P(W), P(Wl), W.numel(), s)
    ops = {
        "fwd": lambda: _lib.call("dlrm_linear_fwd", P(X), K, P(W), K, P(b), P(Y), N, M, N, K, N, 1, s),
        "fwd_wlo": lambda: _lib.call("dlrm_linear_fwd_wlo", P(X), K, P(W), P(Wl), K, P(b), P(Y2), N, M, N, K, N, 1, s),
        "dgrad": lambda: _lib.call("dlrm_linear_bwd_data", P(gZ), N, P(W), K, None, 0, P(dX), K, M, N, K, s),
        "dgrad_wlo": lambda: _lib.call("dlrm_linear_bwd_data_wlo", P(gZ), N, P(W), P(Wl), K, None, 0, P(dX2), K, M, N, K, s),
    }
    res = {}
    for name, fn in ops.items():
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 2)
    print(shape, res, "fwd equal", torch.equal(Y, Y2), "dgrad equal", torch.equal(dX, dX2), flush=True)
