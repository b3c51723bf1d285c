"""Dot interaction on the tensor cores (csrc/interact_tc.cu; dlrm_gemm_mode(2)
forces them at every shape) vs the float64 oracle (ref model.py:218-268) and
the SIMT kernels; the default per-shape pick returns one of the two.

Tolerance (stated): normwise |got - ref|_max / |ref|_max <= 2e-6 for the
pair dots and the feature gradients — 3xTF32 with the lo operands rounded to
nearest TF32 (error ~2^-21 per product) and one TMEM accumulation chain of
d/8 (forward) or nf/8 (backward, hh chain and small terms apart) steps.  Layout (which column holds which
pair, z0 copy, zero padding) is checked bit-exactly with integer-valued
features, where every dot is exact in any order.
"""

import numpy as np
import pytest
import torch

from oracle import port
from paper_1906_00091_b200 import _lib, interact, interact_backward
from paper_1906_00091_b200.rng import RngStream
from tests._util import maxnorm_err

pytestmark = pytest.mark.gpu
TOL = 2e-6

SHAPES = [(9, 64, 2048), (27, 128, 1000), (27, 16, 333), (9, 16, 128), (4, 32, 77),
          (27, 128, 3), (2, 64, 130), (64, 16, 40), (13, 48, 257)]


def feats_of(nf, d, b, seed, strided):
    rs = RngStream(seed)
    host = [np.asarray(rs.normal(b, d), np.float32).astype(np.float64) for _ in range(nf)]
    if strided:  # one [b, nf*d] buffer (the training step's layout)
        Z = torch.tensor(np.concatenate(host, axis=1), dtype=torch.float32, device="cuda")
        dev = [Z[:, f * d:(f + 1) * d] for f in range(nf)]
    else:
        dev = [torch.tensor(h, dtype=torch.float32, device="cuda") for h in host]
    return host, dev


def run(mode, fn):
    _lib.call("dlrm_gemm_mode", mode)
    try:
        return fn()
    finally:
        _lib.call("dlrm_gemm_mode", 0)


@pytest.mark.parametrize("nf,d,b", SHAPES)
@pytest.mark.parametrize("strided", [False, True])
def test_forward_matches_oracle_and_simt(nf, d, b, strided):
    host, dev = feats_of(nf, d, b, nf * 1000 + d + b, strided)
    ref = port.interact(host[0], host[1:])
    got = run(2, lambda: interact(dev[0], dev[1:]).double().cpu().numpy())   # tensor cores
    simt = run(1, lambda: interact(dev[0], dev[1:]).double().cpu().numpy())
    dflt = run(0, lambda: interact(dev[0], dev[1:]).double().cpu().numpy())  # per-shape pick
    assert np.array_equal(dflt, got) or np.array_equal(dflt, simt)
    assert got.shape == ref.shape
    assert np.array_equal(got[:, :d], ref[:, :d])          # z0 copy, exact
    assert maxnorm_err(got, ref) < TOL
    assert maxnorm_err(got, simt) < 2 * TOL


@pytest.mark.parametrize("nf,d,b", SHAPES)
@pytest.mark.parametrize("strided", [False, True])
def test_backward_matches_oracle_and_simt(nf, d, b, strided):
    host, dev = feats_of(nf, d, b, nf * 7 + d * 3 + b, strided)
    P = nf * (nf - 1) // 2
    g = np.asarray(RngStream(b).normal(b, d + P), np.float32).astype(np.float64)
    gt = torch.tensor(g, dtype=torch.float32, device="cuda")
    r0, rs = port.interact_backward(host[0], host[1:], g)
    for mode, tol in ((2, TOL), (1, TOL), (0, TOL)):
        g0, gs = run(mode, lambda: interact_backward(dev[0], dev[1:], gt))
        assert maxnorm_err(g0.double().cpu().numpy(), r0) < tol
        for a, r in zip(gs, rs):
            assert maxnorm_err(a.double().cpu().numpy(), r) < tol


@pytest.mark.parametrize("nf,d", [(27, 16), (9, 64), (27, 128), (5, 32)])
def test_layout_bit_exact_integer_features(nf, d):
    rng = np.random.default_rng(nf + d)
    b = 301
    host = [rng.integers(-3, 4, (b, d)).astype(np.float64) for _ in range(nf)]
    dev = [torch.tensor(h, dtype=torch.float32, device="cuda") for h in host]
    P = nf * (nf - 1) // 2
    g = rng.integers(-2, 3, (b, d + P)).astype(np.float64)
    r0, rs = port.interact_backward(host[0], host[1:], g)
    for mode in (0, 2):
        got = run(mode, lambda: interact(dev[0], dev[1:]).double().cpu().numpy())
        assert np.array_equal(got, port.interact(host[0], host[1:]))
        g0, gs = run(mode, lambda: interact_backward(
            dev[0], dev[1:], torch.tensor(g, dtype=torch.float32, device="cuda")))
        assert np.array_equal(g0.double().cpu().numpy(), r0)
        for a, r in zip(gs, rs):
            assert np.array_equal(a.double().cpu().numpy(), r)


def test_padded_output_columns_are_zero():
    """pad_to > d + P (the training step's ceil4 row pitch) writes zeros."""
    import ctypes as C
    nf, d, b = 9, 64, 100
    _, dev = feats_of(nf, d, b, 3, True)
    W = d + nf * (nf - 1) // 2
    out = torch.full((b, W + 4), 7.0, device="cuda")
    fs = _lib.make_features([(t.data_ptr(), t.stride(0)) for t in dev])
    _lib.call("dlrm_interact_fwd", C.c_void_p(C.addressof(fs)), nf, d, b, _lib.ptr(out),
              out.stride(0), W + 4, _lib.stream_handle())
    assert bool((out[:, W:] == 0).all())
    ref = interact(dev[0], dev[1:])
    assert torch.equal(out[:, :W], ref)
