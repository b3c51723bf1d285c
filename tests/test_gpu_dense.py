"""MLP layers, interaction and loss head on the GPU vs the float64 oracle.

Tolerance (fp32 kernels vs float64 reference on fp32-rounded inputs):
normwise max |gpu - ref| / max |ref| <= 2e-5 per tensor (fp32 GEMM rounding
over K <= 1024 with cancellation rules out a pure elementwise rtol).
The interaction's output LAYOUT ([z0 | (i,j) i<j row-major]) is bit-exact
(checked on exactly representable values).
"""

import numpy as np
import pytest
import torch

from oracle import port
from paper_1906_00091_b200 import (MlpLayer, MlpParams, bce_from_logits,
                                   interact, interact_backward, mlp_backward,
                                   mlp_forward, sgd_step)
from paper_1906_00091_b200.rng import RngStream
from tests._util import maxnorm_err as rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-5


def np64(t):
    return t.detach().cpu().double().numpy()


def f32r(a):
    return np.asarray(a, np.float32).astype(np.float64)


@pytest.mark.parametrize("dims,acts,batch", [
    ([13, 512, 256, 64, 16], ["relu"] * 4, 128),
    ([367, 512, 256, 1], ["relu", "relu", "identity"], 100),
    ([4, 3], ["relu"], 9), ([100, 1024, 1024, 1], ["relu", "relu", "identity"], 64),
    ([479, 64, 30], ["relu", "identity"], 33)])
def test_mlp_forward_backward(dims, acts, batch):
    rs = RngStream(len(dims) + batch)
    layers = []
    for l in range(len(dims) - 1):
        w = f32r(rs.normal(dims[l + 1], dims[l]) * 0.1)
        b = f32r(rs.normal(1, dims[l + 1])[0] * 0.1)
        layers.append((w, b, acts[l]))
    x = f32r(rs.uniform(batch, dims[0]))
    gy = f32r(rs.normal(batch, dims[-1]))
    params = MlpParams([MlpLayer(w, b, a) for w, b, a in layers])
    out, cache = mlp_forward(params, x)
    ref, ins, pres = port.mlp_forward([(w.copy(), b.copy(), a) for w, b, a in layers], x)
    assert rel_err(np64(out), ref) < TOL
    grads, gx = mlp_backward(params, cache, gy)
    dws, dbs, gx_ref = port.mlp_backward(layers, ins, pres, gy, batch)
    assert rel_err(np64(gx), gx_ref) < TOL
    for l in range(len(layers)):
        assert rel_err(np64(grads.weights[l]), dws[l]) < TOL, l
        assert rel_err(np64(grads.biases[l]), dbs[l]) < TOL, l


def test_interaction_layout_bit_exact():
    # ref test_model.py:139-144 hand example
    out = interact(torch.tensor([[1.0, 0.0]]), [torch.tensor([[0.0, 1.0]]),
                                                torch.tensor([[1.0, 1.0]])])
    assert out.cpu().tolist() == [[1.0, 0.0, 0.0, 1.0, 1.0]]
    # integer-valued features: every dot is exact, so the whole [z0 | pairs]
    # layout must equal the reference's upper-triangle row-major order
    rng = np.random.default_rng(5)
    for nf, d in [(27, 16), (9, 64), (4, 3), (27, 128)]:
        feats = [rng.integers(-3, 4, (7, d)).astype(np.float64) for _ in range(nf)]
        got = np64(interact(torch.tensor(feats[0]), [torch.tensor(f) for f in feats[1:]]))
        assert np.array_equal(got, port.interact(feats[0], feats[1:]))


@pytest.mark.parametrize("nf,d,b", [(27, 16, 64), (9, 64, 33), (27, 128, 10), (3, 3, 5)])
def test_interaction_values_and_backward(nf, d, b):
    rs = RngStream(nf * d)
    feats = [f32r(rs.normal(b, d)) for _ in range(nf)]
    tf = [torch.tensor(f, dtype=torch.float32) for f in feats]
    out = interact(tf[0], tf[1:])
    ref = port.interact(feats[0], feats[1:])
    assert out.shape == ref.shape
    assert rel_err(np64(out), ref) < TOL
    g = f32r(rs.normal(b, ref.shape[1]))
    g0, gs = interact_backward(tf[0], tf[1:], torch.tensor(g, dtype=torch.float32))
    r0, rs_ = port.interact_backward(feats[0], feats[1:], g)
    assert rel_err(np64(g0), r0) < TOL
    for a, r in zip(gs, rs_):
        assert rel_err(np64(a), r) < TOL


def test_bce_from_logits():
    rs = RngStream(21)
    z = f32r(rs.normal(1, 1000)[0] * 4)
    y = (rs.uniform(1, 1000)[0] < 0.5).astype(np.float64)
    m, g, per = bce_from_logits(torch.tensor(z), torch.tensor(y))
    rm, rg, rper = port.bce_from_logits(z, y)
    assert abs(m - rm) <= 1e-5 * abs(rm)
    assert rel_err(np64(g), rg) < TOL and rel_err(np64(per), rper) < TOL


def test_sgd_dense_rounding():
    # ref test_optim.py:24-27, and w - fl(lr*g) exactly (no FMA)
    p = torch.tensor([1.0], device="cuda")
    sgd_step(p, torch.tensor([2.0], device="cuda"), 0.5)
    assert p.item() == 0.0
    rng = np.random.default_rng(3)
    w = rng.standard_normal(1001).astype(np.float32)
    g = rng.standard_normal(1001).astype(np.float32)
    t = torch.tensor(w, device="cuda")
    sgd_step(t, torch.tensor(g, device="cuda"), 0.1)
    exp = w - np.float32(0.1) * g
    assert np.array_equal(t.cpu().numpy().view(np.uint32), exp.view(np.uint32))


# ---- Adagrad: kernels vs the float32 restatement, bit for bit

def test_adagrad_dense_bit_exact():
    from oracle import fp32
    from paper_1906_00091_b200 import adagrad_step
    rng = np.random.default_rng(3)
    for n in (1, 7, 1000, 4099):
        p = rng.standard_normal(n).astype(np.float32)
        g = rng.standard_normal(n).astype(np.float32)
        a = np.abs(rng.standard_normal(n)).astype(np.float32)
        tp, tg, ta = (torch.as_tensor(x, device="cuda") for x in (p, g, a))
        adagrad_step(tp, tg, ta, 0.05, 1e-8)
        ep, ea = fp32.adagrad_dense(p, g, a, 0.05, 1e-8)
        assert np.array_equal(tp.cpu().numpy().view(np.uint32), ep.view(np.uint32))
        assert np.array_equal(ta.cpu().numpy().view(np.uint32), ea.view(np.uint32))


def test_adagrad_rows_bit_exact_and_untouched_rows_keep_bits():
    from oracle import fp32
    from paper_1906_00091_b200 import SparseRowGrad, adagrad_step_rows
    rng = np.random.default_rng(4)
    for m, d in ((50, 16), (300, 20), (64, 256)):
        W = rng.standard_normal((m, d)).astype(np.float32)
        A = np.abs(rng.standard_normal((m, d))).astype(np.float32)
        rows = np.sort(rng.choice(m, m // 3, replace=False)).astype(np.int64)
        vals = rng.standard_normal((rows.size, d)).astype(np.float32)
        tW, tA = torch.as_tensor(W, device="cuda"), torch.as_tensor(A, device="cuda")
        g = SparseRowGrad(torch.as_tensor(rows, device="cuda"),
                          torch.as_tensor(vals, device="cuda"))
        adagrad_step_rows(tW, g, tA, 0.1, 1e-10)
        eW, eA = fp32.adagrad_rows(W, rows, vals, A, 0.1, 1e-10)
        assert np.array_equal(tW.cpu().numpy().view(np.uint32), eW.view(np.uint32))
        assert np.array_equal(tA.cpu().numpy().view(np.uint32), eA.view(np.uint32))


def test_reference_model_round_trip():
    """from_reference / to_reference: a dlrmkit-shaped model
    (duck-typed here; dlrmkit is not installed on the GPU box) converts to
    CUDA fp32 and back with values rounded to fp32 and structure kept."""
    from types import SimpleNamespace as NS
    from paper_1906_00091_b200 import DlrmConfig, from_reference, init_model, to_reference
    rng = np.random.default_rng(5)
    cfg = NS(embedding_sizes=[7, 11], sparse_dim=4, bottom_mlp_dims=[3, 5, 4],
             top_mlp_dims=[6, 1], interaction="dot", seed=9)
    lay = lambda o, i, a: NS(weight=rng.standard_normal((o, i)), bias=rng.standard_normal(o),
                             activation=a)
    ref = NS(config=cfg, bottom=NS(layers=[lay(5, 3, "relu"), lay(4, 5, "relu")]),
             top=NS(layers=[lay(6, 7, "relu"), lay(1, 6, "identity")]),
             tables=[NS(weights=rng.standard_normal((7, 4)), table_id=0),
                     NS(weights=rng.standard_normal((11, 4)), table_id=1)])
    m = from_reference(ref)
    assert m.config.top_mlp_dims == [6, 1] and m.config.seed == 9
    assert np.array_equal(m.bottom.layers[1].weight.cpu().numpy(),
                          ref.bottom.layers[1].weight.astype(np.float32))
    assert np.array_equal(m.tables[1].weights.cpu().numpy(),
                          ref.tables[1].weights.astype(np.float32))
    fake = NS(DlrmConfig=lambda *a: NS(args=a), MlpParams=lambda ls: NS(layers=ls),
              MlpLayer=lambda w, b, a: NS(weight=w, bias=b, activation=a),
              EmbeddingTable=lambda w, t: NS(weights=w, table_id=t),
              DlrmModel=lambda c, b, t, tab: NS(config=c, bottom=b, top=t, tables=tab))
    back = to_reference(m, fake)
    assert back.top.layers[1].activation == "identity"
    assert back.tables[0].weights.dtype == np.float64
    assert np.array_equal(back.top.layers[0].weight,
                          ref.top.layers[0].weight.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("M,K,mask", [(2048, 1024, 1), (1000, 256, 1), (37, 12, 0)])
def test_fused_head_step(M, K, mask):
    """dlrm_head_step (forward of the N=1 layer + BCE + backward + update in
    two launches) vs float64 numpy of ref model.py:152, 448-461 and
    mlp_backward_trace 173-179."""
    import ctypes as C
    from paper_1906_00091_b200 import _lib
    rng = np.random.default_rng(M + K)
    A = np.maximum(rng.standard_normal((M, K)), 0).astype(np.float32)
    w = (rng.standard_normal(K) * 0.05).astype(np.float32)
    b = np.float32(0.1)
    y = (rng.random(M) < 0.5).astype(np.float32)
    d = torch.device("cuda")
    tA, tw = torch.as_tensor(A, device=d), torch.as_tensor(w, device=d).clone()
    tb = torch.tensor([b], device=d)
    ty = torch.as_tensor(y, device=d)
    prob, gz = torch.empty(M, device=d), torch.empty(M, device=d)
    stats = torch.zeros(2, device=d)
    dA = torch.empty((M, K), device=d)
    dw, db = torch.empty(K, device=d), torch.empty(1, device=d)
    wu, bu = tw.clone(), tb.clone()
    ws_b = _lib.size("dlrm_head_step_workspace_size", M, K)
    ws = torch.empty(ws_b, dtype=torch.uint8, device=d)
    upd = _lib.Update(_lib.UPD_SGD, 0.5, 0.0, 0)
    P = _lib.ptr
    _lib.call("dlrm_head_step", P(tA), K, P(tw), P(tb), M, K, P(ty), float(M), P(prob),
              P(gz), P(stats), P(dA), K, mask, P(dw), P(db), P(wu), P(bu), C.byref(upd),
              None, P(ws), ws_b, _lib.stream_handle())
    z = A.astype(np.float64) @ w.astype(np.float64) + float(b)
    p = 1 / (1 + np.exp(-z))
    per = np.maximum(z, 0) - z * y + np.log1p(np.exp(-np.abs(z)))
    g = (p - y) / M
    eA = np.outer(g, w) * ((A > 0) if mask else 1)
    edw = g @ A.astype(np.float64)
    assert rel_err(prob.cpu().numpy(), p) < 1e-5
    assert rel_err(gz.cpu().numpy(), g) < 1e-5
    assert abs(float(stats[0]) - per.sum()) <= 1e-5 * abs(per.sum())
    assert float(stats[1]) == float(np.sum((p > 0.5) == (y > 0.5)))
    assert rel_err(dA.cpu().numpy(), eA) < 1e-5
    assert rel_err(dw.cpu().numpy(), edw) < 1e-5
    assert abs(float(db) - g.sum()) <= 1e-5 * max(abs(g).sum(), 1e-30)
    assert rel_err(wu.cpu().numpy(), w - 0.5 * dw.cpu().numpy()) < 1e-6
