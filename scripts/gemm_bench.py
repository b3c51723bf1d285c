"""Time the MLP GEMM kernels at the bench shapes (CUDA events, 20 reps after
warm-up) and report TFLOP/s (algorithmic 2MNK) and normwise error."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib

def ceil4(n): return (n + 3) // 4 * 4
B = int(os.environ.get("B", 2048))
layers = [(512, 512), (512, 64), (100, 1024), (1024, 1024), (13, 512), (512, 256), (367, 512)]
if os.environ.get("LAYERS") == "c4":  # B=32768 Terabyte-shaped MLPs
    layers = [(480, 1024), (1024, 1024), (1024, 512), (512, 256), (13, 512), (512, 256), (256, 128)]
res = []
if os.environ.get("MODE"):
    _lib.call("dlrm_gemm_mode", int(os.environ["MODE"]))
g = torch.Generator(device="cuda").manual_seed(0)
for K, N in layers:
    X = torch.randn((B, ceil4(K)), device="cuda", generator=g)
    W = torch.randn((N, ceil4(K)), device="cuda", generator=g) / K ** 0.5
    bias = torch.zeros(N, device="cuda")
    Y = torch.empty((B, ceil4(N)), device="cuda")
    gZ = torch.randn((B, ceil4(N)), device="cuda", generator=g)
    dX = torch.empty((B, ceil4(K)), device="cuda")
    wsb = _lib.size("dlrm_linear_bwd_weight_workspace_size", B, N, K)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    dW = torch.empty((N, K), device="cuda"); db = torch.empty(N, device="cuda")
    s = _lib.stream_handle()
    ops = {
        "fwd": lambda: _lib.call("dlrm_linear_fwd", _lib.ptr(X), X.stride(0), _lib.ptr(W), W.stride(0), _lib.ptr(bias), _lib.ptr(Y), Y.stride(0), B, N, K, Y.shape[1], 1, s),
        "dgrad": lambda: _lib.call("dlrm_linear_bwd_data", _lib.ptr(gZ), gZ.stride(0), _lib.ptr(W), W.stride(0), None, 0, _lib.ptr(dX), dX.stride(0), B, N, K, s),
        "wgrad": lambda: _lib.call("dlrm_linear_bwd_weight", _lib.ptr(gZ), gZ.stride(0), _lib.ptr(X), X.stride(0), B, N, K, _lib.ptr(dW), dW.stride(0), _lib.ptr(db), None, 0, None, 0.0, None, _lib.ptr(ws), wsb, s),
    }
    for name, fn in ops.items():
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        tf = 2 * B * N * K / (us * 1e-6) / 1e12
        if name == "fwd": ref = torch.relu(X[:, :K].double() @ W[:, :K].double().T); got = Y[:, :N]
        elif name == "dgrad": ref = gZ[:, :N].double() @ W[:, :K].double(); got = dX[:, :K]
        else: ref = gZ[:, :N].double().T @ X[:, :K].double(); got = dW
        err = float((got.double() - ref).abs().max() / ref.abs().max())
        res.append(dict(K=K, N=N, op=name, us=round(us, 2), tflops=round(tf, 1), err=f"{err:.1e}"))
        print(res[-1], flush=True)
