"""Embedding-bag kernels on the GPU vs the oracle.

Bit-exact against the float32 restatement of the reference's fold order
(oracle.fp32) for pooled rows and unique-row lists, and for gradient rows /
updated table rows whose run is <= 256 slots; hotter rows (reduced as a fixed
tree of 256-slot strict folds) within 1e-5 of the sum of absolute
contributions.  Within 1e-5 (scaled by the row) of the float64 reference
fixtures.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import fp32
from paper_1906_00091_b200 import (EmbeddingTable, LookupIndexError,
                                   SparseBatch, lookup_backward, lookup_batch,
                                   offsets_from_lengths, sgd_step_rows)
from paper_1906_00091_b200 import _lib
from paper_1906_00091_b200.rng import zipf_indices

from tests._util import assert_fold_match

pytestmark = pytest.mark.gpu


def np32(t):
    return t.detach().cpu().numpy()


def close_to_f64(got, ref):
    scale = 1e-5 * np.abs(ref) + 1e-5 * np.abs(ref).max(axis=-1, keepdims=True)
    return bool(np.all(np.abs(got - ref) <= scale + 1e-30))


def test_golden_bags(golden):
    fx = golden("bags.npz")
    for n in range(int(fx["num_cases"])):
        p = f"case{n}_"
        w = fx[p + "weights"] if p + "weights" in fx else None
        table = EmbeddingTable(fx[p + "W"], table_id=n)
        batch = SparseBatch(fx[p + "offsets"], fx[p + "indices"], w)
        out = np32(lookup_batch(table, batch))
        exp32 = fp32.lookup(fx[p + "W"], fx[p + "offsets"], fx[p + "indices"], w)
        assert np.array_equal(out.view(np.uint32), exp32.view(np.uint32)), n
        assert close_to_f64(out, fx[p + "out"]), n
        g = fx[p + "grad"]
        sg = lookup_backward(table, batch, g)
        rows32, vals32 = fp32.lookup_backward(fx[p + "offsets"],
                                              fx[p + "indices"], g, w)
        assert np.array_equal(np32(sg.rows), fx[p + "rows"]), n
        assert np.array_equal(np32(sg.values).view(np.uint32),
                              vals32.view(np.uint32)), n


def fixture_table():
    w = np.zeros((6, 2))
    w[0], w[1], w[2], w[3], w[4], w[5] = [1, 0], [0, 1], [2, 2], [3, 3], [9, 9], [1, 1]
    return EmbeddingTable(w, table_id=4)


def test_reference_known_answers():
    t = fixture_table()
    out = lookup_batch(t, SparseBatch(offsets_from_lengths([2, 3, 1]),
                                      np.array([0, 2, 0, 1, 5, 3])))
    assert np32(out).tolist() == [[3, 2], [2, 2], [3, 3]]
    out = lookup_batch(t, SparseBatch(np.array([0, 0, 1]), np.array([5])))
    assert np32(out).tolist() == [[0, 0], [1, 1]]
    out = lookup_batch(t, SparseBatch(np.array([0, 2]), np.array([0, 2]),
                                      np.array([0.0, 0.0])))
    assert np32(out).tolist() == [[0, 0]]
    g = lookup_backward(t, SparseBatch(np.array([0, 2]), np.array([3, 3])),
                        np.array([[0.5, -1.0]]))
    assert np32(g.rows).tolist() == [3] and np32(g.values).tolist() == [[1.0, -2.0]]
    g = lookup_backward(t, SparseBatch(np.array([0, 1, 2]), np.array([5, 1])),
                        np.ones((2, 2)))
    assert np32(g.rows).tolist() == [1, 5]
    g = lookup_backward(t, SparseBatch(np.array([0, 2]), np.array([0, 0]),
                                       np.array([2.0, 3.0])), np.ones((1, 2)))
    assert np32(g.values).tolist() == [[5.0, 5.0]]
    g = lookup_backward(t, SparseBatch(np.array([0, 0]), np.empty(0, np.int64)),
                        np.zeros((1, 2)))
    assert g.rows.numel() == 0 and tuple(g.values.shape) == (0, 2)


@pytest.mark.parametrize("idx,pos,val", [([0, 17], 1, 17), ([1, -1, 9], 1, -1),
                                         ([6, 7, 8], 0, 6)])
def test_error_payload(idx, pos, val):
    t = fixture_table()
    b = SparseBatch(np.array([0, len(idx)]), np.array(idx))
    with pytest.raises(LookupIndexError) as e:
        lookup_batch(t, b)
    assert (e.value.table_id, e.value.position, e.value.index) == (4, pos, val)
    with pytest.raises(LookupIndexError) as e:
        lookup_backward(t, b, np.ones((1, 2)))
    assert (e.value.table_id, e.value.position, e.value.index) == (4, pos, val)
    with pytest.raises(ValueError):
        lookup_backward(t, b, np.ones((2, 2)))


@pytest.mark.parametrize("m,d,nb,k,dist", [
    (1000, 16, 512, 1, "u"), (5000, 64, 300, 40, "u"), (20000, 128, 256, 100, "z"),
    (3000, 256, 64, 17, "u"), (777, 3, 100, 9, "u"), (400, 20, 128, 5, "z"),
    (3, 16, 4096, 1, "u"), (5, 64, 2048, 3, "u"), (2, 3, 700, 2, "u")])
def test_random_bags_bit_exact(m, d, nb, k, dist):
    rng = np.random.default_rng(m + d)
    W = rng.standard_normal((m, d)).astype(np.float32)
    lens = rng.integers(0, k + 1, nb)
    n = int(lens.sum())
    idx = zipf_indices(m, n, seed=d) if dist == "z" else rng.integers(0, m, n)
    w = rng.standard_normal(n).astype(np.float32) if d % 2 else None
    b = SparseBatch(offsets_from_lengths(lens), idx, w)
    out = np32(lookup_batch(EmbeddingTable(W), b))
    exp = fp32.lookup(W, b.offsets.cpu().numpy(), idx, w)
    assert np.array_equal(out.view(np.uint32), exp.view(np.uint32))
    g = rng.standard_normal((nb, d)).astype(np.float32)
    sg = lookup_backward(EmbeddingTable(W), b, g)
    rows, vals = fp32.lookup_backward(b.offsets.cpu().numpy(), idx, g, w)
    _, absum = fp32.lookup_backward(b.offsets.cpu().numpy(), idx, np.abs(g),
                                    None if w is None else np.abs(w))
    counts = np.bincount(idx, minlength=m)
    assert np.array_equal(np32(sg.rows), rows)
    assert_fold_match(np32(sg.values), vals, absum, counts[rows])
    # sparse SGD
    t = EmbeddingTable(W)
    sgd_step_rows(t.weights, sg, 0.1)
    exp_w = fp32.sgd_rows(W, rows, vals, 0.1)
    absum_w = np.zeros_like(W)
    absum_w[rows] = 0.1 * absum
    assert_fold_match(np32(t.weights), exp_w, absum_w, counts, ulps=1)


def _multi_table_case(seed, d, sizes, B, k, zipf=False, weighted=False):
    rng = np.random.default_rng(seed)
    Ws = [rng.standard_normal((m, d)).astype(np.float32) for m in sizes]
    offs, idxs, wts = [], [], []
    for t, m in enumerate(sizes):
        lens = rng.integers(0, k + 1, B)
        n = int(lens.sum())
        idxs.append(zipf_indices(m, n, seed=t) if zipf else rng.integers(0, m, n))
        offs.append(offsets_from_lengths(lens))
        wts.append(rng.standard_normal(n).astype(np.float32) if weighted else None)
    return Ws, offs, idxs, wts


@pytest.mark.parametrize("d,zipf,weighted", [(16, False, False), (64, True, False),
                                              (128, False, True), (32, True, True),
                                              (16, "tiny", False), (64, "tiny", True)])
def test_fused_multitable_fwd_and_bwd_sgd(d, zipf, weighted):
    """dlrm_emb_fwd over 3 tables into a strided [B, nf, d] buffer, then the
    capacity-padded sort + segmented fold + SGD (dlrm_emb_bwd_sgd) vs the
    oracle's lookup_backward + sgd_step_rows per table, bit for bit."""
    sizes, B, k, lr = [3000, 17, 50000], 257, 30, 0.05
    orig_zipf = zipf
    if zipf == "tiny":  # hot rows: runs of hundreds of slots (long-run path)
        sizes, B, k, zipf = [3, 4, 50000], 1500, 4, False
    Ws, offs, idxs, wts = _multi_table_case(d, d, sizes, B, k, zipf, weighted)
    dev = torch.device("cuda")
    T, nf = len(sizes), len(sizes) + 1
    row_base = np.concatenate([[0], np.cumsum(sizes)])
    W_all = torch.as_tensor(np.concatenate(Ws), device=dev).reshape(-1).contiguous()
    caps = [int(o[-1]) + 13 * t for t, o in enumerate(offs)]
    cap_base = np.concatenate([[0], np.cumsum(caps)])
    ind = torch.zeros(int(cap_base[-1]), dtype=torch.int64, device=dev)
    wt = torch.ones(int(cap_base[-1]), dtype=torch.float32, device=dev)
    O = torch.as_tensor(np.stack(offs), device=dev)
    for t in range(T):
        ind[cap_base[t]:cap_base[t] + len(idxs[t])] = torch.as_tensor(idxs[t])
        if weighted:
            wt[cap_base[t]:cap_base[t] + len(idxs[t])] = torch.as_tensor(wts[t])
    descs = _lib.table_array([_lib.TableDesc(
        O[t].data_ptr(), ind.data_ptr() + 8 * int(cap_base[t]),
        (wt.data_ptr() + 4 * int(cap_base[t])) if weighted else None,
        int(row_base[t]), sizes[t], (1 + t) * d, caps[t], t) for t in range(T)])
    Z = torch.zeros((B, nf * d), dtype=torch.float32, device=dev)
    ep = torch.empty(T, dtype=torch.int64, device=dev)
    ef = torch.zeros(1, dtype=torch.int32, device=dev)
    s = _lib.stream_handle()
    _lib.call("dlrm_err_reset", _lib.ptr(ep), T, _lib.ptr(ef), s)
    _lib.call("dlrm_emb_fwd", _lib.ptr(W_all), d, C.cast(descs, C.c_void_p), T,
              B, _lib.ptr(Z), nf * d, _lib.ptr(ep), _lib.ptr(ef), s)
    Zh = np32(Z).reshape(B, nf, d)
    assert int(ef.item()) == 0
    for t in range(T):
        exp = fp32.lookup(Ws[t], offs[t], idxs[t], wts[t])
        assert np.array_equal(Zh[:, 1 + t].view(np.uint32), exp.view(np.uint32))
    G = torch.as_tensor(np.random.default_rng(1).standard_normal((B, nf * d)),
                        dtype=torch.float32, device=dev)
    wsb = _lib.size("dlrm_emb_bwd_workspace_size", int(cap_base[-1]), int(row_base[-1]), d)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.call("dlrm_emb_bwd_sgd", _lib.ptr(W_all), d, C.cast(descs, C.c_void_p),
              T, B, _lib.ptr(G), nf * d, lr, _lib.ptr(ef), int(row_base[-1]),
              _lib.ptr(ws), wsb, s)
    Wh = np32(W_all).reshape(-1, d)
    Gh = np32(G).reshape(B, nf, d)
    n_hot = 0
    for t in range(T):
        rows, vals = fp32.lookup_backward(offs[t], idxs[t], Gh[:, 1 + t], wts[t])
        _, absum = fp32.lookup_backward(
            offs[t], idxs[t], np.abs(Gh[:, 1 + t]),
            None if wts[t] is None else np.abs(wts[t]))
        exp = fp32.sgd_rows(Ws[t], rows, vals, lr)
        absum_w = np.zeros_like(exp)
        absum_w[rows] = lr * absum
        got = Wh[row_base[t]:row_base[t + 1]]
        n_hot += assert_fold_match(got, exp, absum_w,
                                   np.bincount(idxs[t], minlength=sizes[t]), ulps=1)
    if orig_zipf == "tiny":
        assert n_hot > 0  # the segment-tree path was exercised


def test_bwd_sgd_skips_update_on_error():
    d, B = 16, 8
    dev = torch.device("cuda")
    W = torch.randn(10 * d, device=dev)
    before = W.clone()
    O = torch.as_tensor(np.arange(B + 1), device=dev)
    ind = torch.as_tensor(np.r_[np.arange(B - 1), 99], device=dev)
    descs = _lib.table_array([_lib.TableDesc(O.data_ptr(), ind.data_ptr(), None,
                                             0, 10, 0, B, 0)])
    out = torch.zeros((B, d), device=dev)
    ep = torch.empty(1, dtype=torch.int64, device=dev)
    ef = torch.zeros(1, dtype=torch.int32, device=dev)
    s = _lib.stream_handle()
    _lib.call("dlrm_err_reset", _lib.ptr(ep), 1, _lib.ptr(ef), s)
    _lib.call("dlrm_emb_fwd", _lib.ptr(W), d, C.cast(descs, C.c_void_p), 1, B,
              _lib.ptr(out), d, _lib.ptr(ep), _lib.ptr(ef), s)
    assert int(ef.item()) == 1 and int(ep.item()) == B - 1
    wsb = _lib.size("dlrm_emb_bwd_workspace_size", B, 10, d)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.call("dlrm_emb_bwd_sgd", _lib.ptr(W), d, C.cast(descs, C.c_void_p), 1, B,
              _lib.ptr(torch.ones((B, d), device=dev)), d, 0.1, _lib.ptr(ef), 10,
              _lib.ptr(ws), wsb, s)
    assert torch.equal(W, before)


@pytest.mark.parametrize("sort", ["radix8", "radix12"])
@pytest.mark.parametrize("case", [(200000, 16, 2048, 60, "u"), (5000, 64, 300, 40, "u"),
                                  (20000, 128, 256, 100, "z"), (3, 16, 4096, 1, "u")])
def test_hand_written_radix_sort(sort, case, monkeypatch):
    """The opt-in stable LSD radix sort (csrc/radix.cu, DLRM_SORT=radix8 /
    radix12: 2-3 passes) gives the same bit-exact backward as the default;
    200k rows = 18-bit keys (3 passes of 8 bits)."""
    monkeypatch.setenv("DLRM_SORT", sort)
    test_random_bags_bit_exact(*case)


@pytest.mark.parametrize("sort", ["radix8", "radix12"])
def test_hand_written_radix_sort_fused_step(sort, monkeypatch):
    monkeypatch.setenv("DLRM_SORT", sort)
    test_fused_multitable_fwd_and_bwd_sgd(64, "tiny", True)
    test_fused_multitable_fwd_and_bwd_sgd(32, True, True)
