"""tcgen05 3xTF32 GEMMs (forward, data gradient, weight gradient) vs a
float64 reference, and vs the SIMT fp32 kernels.

Tolerance: normwise max|err| / max|ref| <= 1e-5 (fp32-level; single-pass
TF32 would be ~1e-3)."""

import numpy as np
import pytest
import torch

from paper_1906_00091_b200 import _lib
from tests._util import maxnorm_err

pytestmark = pytest.mark.gpu
TOL = 1e-5

SHAPES = [(2048, 1024, 1024), (2048, 512, 512), (2048, 64, 512), (2048, 1024, 100),
          (2048, 512, 13), (128, 512, 52), (64, 256, 367), (33, 30, 64), (300, 16, 64),
          (4096, 128, 479), (2048, 16, 64),
          # narrow layer inputs (the dense features): the slab weight gradient
          (128, 512, 13), (32768, 512, 13), (2048, 300, 32), (1000, 7, 3), (5, 130, 16),
          # more output tiles than SMs: the persistent kernel (partial tiles too)
          (4096, 1024, 1024), (20000, 640, 480), (32768, 256, 512), (8200, 1000, 300),
          # one wave just short of the SMs (ragged rows / columns / K too)
          (2000, 1000, 1000), (1500, 1024, 2048), (2048, 640, 700),
          # narrow inputs over long batches: the SIMT skinny forward / weight
          # gradient (ragged column counts, padding columns)
          (9000, 130, 5), (8200, 7, 16), (16384, 600, 13)]


def ceil4(n):
    return (n + 3) // 4 * 4


def rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(shape, generator=g, device="cuda") * scale


def linear_fwd(X, W, b, N, K, act):
    M = X.shape[0]
    Y = torch.full((M, ceil4(N)), float("nan"), device="cuda")
    _lib.call("dlrm_linear_fwd", _lib.ptr(X), X.stride(0), _lib.ptr(W), W.stride(0),
              _lib.ptr(b), _lib.ptr(Y), Y.stride(0), M, N, K, Y.shape[1], act,
              _lib.stream_handle())
    return Y


@pytest.fixture(params=[0, 1], ids=["tcgen05", "simt"])
def mode(request):
    _lib.call("dlrm_gemm_mode", request.param)
    yield request.param
    _lib.call("dlrm_gemm_mode", 0)


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_linear_fwd(mode, M, N, K):
    X = torch.zeros((M, ceil4(K)), device="cuda")
    X[:, :K] = rand((M, K), 1)
    W = torch.zeros((N, ceil4(K)), device="cuda")
    W[:, :K] = rand((N, K), 2, K ** -0.5)
    b = rand((N,), 3)
    Y = linear_fwd(X, W, b, N, K, 1)
    ref = torch.relu(X[:, :K].double() @ W[:, :K].double().T + b.double())
    assert maxnorm_err(Y[:, :N].cpu(), ref.cpu()) < TOL
    assert bool((Y[:, N:] == 0).all())


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_linear_bwd_data(mode, M, N, K):
    gZ = torch.zeros((M, ceil4(N)), device="cuda")
    gZ[:, :N] = rand((M, N), 4)
    W = torch.zeros((N, ceil4(K)), device="cuda")
    W[:, :K] = rand((N, K), 5, N ** -0.5)
    mask = torch.relu(rand((M, ceil4(K)), 6))
    dX = torch.full((M, ceil4(K)), float("nan"), device="cuda")
    _lib.call("dlrm_linear_bwd_data", _lib.ptr(gZ), gZ.stride(0), _lib.ptr(W), W.stride(0),
              _lib.ptr(mask), mask.stride(0), _lib.ptr(dX), dX.stride(0), M, N, K,
              _lib.stream_handle())
    ref = (gZ[:, :N].double() @ W[:, :K].double()) * (mask[:, :K] > 0).double()
    assert maxnorm_err(dX[:, :K].cpu(), ref.cpu()) < TOL


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_linear_bwd_weight_and_sgd(mode, M, N, K):
    gZ = torch.zeros((M, ceil4(N)), device="cuda")
    gZ[:, :N] = rand((M, N), 7, M ** -0.5)
    X = torch.zeros((M, ceil4(K)), device="cuda")
    X[:, :K] = rand((M, K), 8)
    dW = torch.full((N, K), float("nan"), device="cuda")
    db = torch.full((N,), float("nan"), device="cuda")
    W = torch.zeros((N, ceil4(K)), device="cuda")
    W[:, :K] = rand((N, K), 9)
    bias = rand((N,), 10)
    W0, b0 = W.clone(), bias.clone()
    wsb = _lib.size("dlrm_linear_bwd_weight_workspace_size", M, N, K)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("dlrm_linear_bwd_weight", _lib.ptr(gZ), gZ.stride(0), _lib.ptr(X), X.stride(0),
              M, N, K, _lib.ptr(dW), dW.stride(0), _lib.ptr(db), _lib.ptr(W), W.stride(0),
              _lib.ptr(bias), 0.5, _lib.ptr(flag), _lib.ptr(ws), wsb, _lib.stream_handle())
    refw = gZ[:, :N].double().T @ X[:, :K].double()
    refb = gZ[:, :N].double().sum(0)
    assert maxnorm_err(dW.cpu(), refw.cpu()) < TOL
    assert maxnorm_err(db.cpu(), refb.cpu()) < TOL
    # fused SGD used exactly the stored gradient: W = W0 - fl(0.5*dW)
    exp = (W0[:, :K] - 0.5 * dW)
    assert torch.equal(W[:, :K], exp)
    assert torch.equal(bias, b0 - 0.5 * db)
    assert bool((W[:, K:] == 0).all())


def test_tensor_core_path_differs_from_simt():
    """Guard against a silent fallback: the two kernels round differently."""
    M, N, K = 2048, 1024, 1024
    X = rand((M, K), 11)
    W = rand((N, K), 12, K ** -0.5)
    b = torch.zeros(N, device="cuda")
    _lib.call("dlrm_gemm_mode", 0)
    n0 = _lib.launch_count()
    y_tc = linear_fwd(X, W, b, N, K, 0)
    _lib.call("dlrm_gemm_mode", 1)
    y_simt = linear_fwd(X, W, b, N, K, 0)
    _lib.call("dlrm_gemm_mode", 0)
    assert _lib.launch_count() - n0 == 2
    assert not torch.equal(y_tc, y_simt)
    ref = X.double() @ W.double().T
    e_tc = maxnorm_err(y_tc.cpu(), ref.cpu())
    e_simt = maxnorm_err(y_simt.cpu(), ref.cpu())
    print(f"K=1024 normwise error: tcgen05 3xTF32 {e_tc:.2e}, SIMT fp32 {e_simt:.2e}")
    assert e_tc < 2e-5  # TC fp32 accumulation is ~6x looser than FFMA chains


@pytest.mark.parametrize("M,N,K", [(2048, 1024, 1024), (4096, 1000, 1000)])
def test_gemm_is_deterministic(M, N, K):
    """Each output element is one fixed-order reduction: repeated calls (the
    one-wave kernel and the persistent one) are bitwise equal."""
    X = torch.zeros((M, ceil4(K)), device="cuda")
    X[:, :K] = rand((M, K), 13)
    W = torch.zeros((N, ceil4(K)), device="cuda")
    W[:, :K] = rand((N, K), 14, K ** -0.5)
    b = rand((N,), 15)
    _lib.call("dlrm_gemm_mode", 0)
    ys = [linear_fwd(X, W, b, N, K, 0) for _ in range(3)]
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2])
    ref = X[:, :K].double() @ W[:, :K].double().T + b.double()
    assert maxnorm_err(ys[0][:, :N].cpu(), ref.cpu()) < TOL


@pytest.mark.parametrize("M,N,K", [(2048, 1024, 1024), (2048, 64, 512), (4096, 1000, 300),
                                   (300, 16, 64), (33, 30, 64), (20000, 640, 480)])
def test_precomputed_weight_lo_parts_are_bitwise_neutral(M, N, K):
    """dlrm_linear_fwd_wlo / dlrm_linear_bwd_data_wlo with W_lo from
    dlrm_tf32_split_lo (B_lo loaded by TMA, not converted per tile) give
    bitwise the results of the plain calls, on every kernel the shapes pick
    (one-tile, persistent, split-K cluster, narrow BN that ignores W_lo)."""
    P = _lib.ptr
    X = torch.zeros((M, ceil4(K)), device="cuda")
    X[:, :K] = rand((M, K), 21)
    W = torch.zeros((N, ceil4(K)), device="cuda")
    W[:, :K] = rand((N, K), 22, K ** -0.5)
    Wl = torch.full_like(W, float("nan"))
    _lib.call("dlrm_tf32_split_lo", P(W), P(Wl), W.numel(), _lib.stream_handle())
    b = rand((N,), 23)
    Y1 = linear_fwd(X, W, b, N, K, 1)
    Y2 = torch.full((M, ceil4(N)), float("nan"), device="cuda")
    _lib.call("dlrm_linear_fwd_wlo", P(X), X.stride(0), P(W), P(Wl), W.stride(0), P(b), P(Y2),
              Y2.stride(0), M, N, K, Y2.shape[1], 1, _lib.stream_handle())
    assert torch.equal(Y1, Y2)
    gZ = torch.zeros((M, ceil4(N)), device="cuda")
    gZ[:, :N] = rand((M, N), 24)
    mask = torch.relu(rand((M, ceil4(K)), 25))
    outs = []
    for fn, extra in (("dlrm_linear_bwd_data", ()), ("dlrm_linear_bwd_data_wlo", (P(Wl),))):
        dX = torch.full((M, ceil4(K)), float("nan"), device="cuda")
        _lib.call(fn, P(gZ), gZ.stride(0), P(W), *extra, W.stride(0), P(mask), mask.stride(0),
                  P(dX), dX.stride(0), M, N, K, _lib.stream_handle())
        outs.append(dX[:, :K])
    assert torch.equal(outs[0], outs[1])
    # the low parts themselves: x - hi(x), rounded to TF32, zero where x is
    hi = (W.view(torch.int32) & -8192).view(torch.float32)
    assert torch.all((Wl == 0) | ((W - hi) != 0))
