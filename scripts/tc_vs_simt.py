"""Which GEMM path a shape takes: compare tcgen05 (mode 0) and SIMT (mode 1)
outputs bit for bit, and each against float64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib
g = torch.Generator(device="cuda").manual_seed(0)
for M, N, K in [(128, 512, 256), (128, 64, 512), (2048, 1024, 1024), (128, 512, 16)]:
    X = torch.randn((M, K), device="cuda", generator=g)
    W = torch.randn((N, K), device="cuda", generator=g) / K ** 0.5
    b = torch.zeros(N, device="cuda")
    outs = []
    for mode in (0, 1):
        _lib.call("dlrm_gemm_mode", mode)
        Y = torch.empty((M, N), device="cuda")
        _lib.call("dlrm_linear_fwd", _lib.ptr(X), K, _lib.ptr(W), K, _lib.ptr(b), _lib.ptr(Y), N,
                  M, N, K, N, 0, _lib.stream_handle())
        outs.append(Y)
    ref = X.double() @ W.double().T
    e = [float((o.double() - ref).abs().max() / ref.abs().max()) for o in outs]
    print(M, N, K, "tc==simt", bool(torch.equal(outs[0], outs[1])), "err tc %.2e simt %.2e" % tuple(e))
_lib.call("dlrm_gemm_mode", 0)
