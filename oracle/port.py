"""TEST INFRASTRUCTURE ONLY — float64 CPU restatement of the reference
``dlrmkit`` training step (the oracle; also the ``cpu_baseline`` "port" arm).

Every function follows the reference algorithm operation for operation so
the result is bit-identical to ``dlrmkit`` on the same float64 inputs; the
``ref`` note on each function names the reference lines it restates.  The
golden fixtures in ``tests/golden`` were produced by ``dlrmkit`` itself and
``tests/test_oracle.py`` checks this module against them bit for bit.

State is kept in plain dicts/lists of numpy float64 arrays:

    model = {"bottom": [(W, b, act), ...], "top": [...], "tables": [W_t, ...]}
"""

from __future__ import annotations

import math

import numpy as np

from paper_1906_00091_b200.rng import RngStream

_MAGIC = math.ldexp(1.5, 52)
_SLICE_PAIRS = ((1, 1), (1, 2), (2, 1), (1, 3), (2, 2), (3, 1))
_LEVELS = 3


class PortIndexError(IndexError):
    def __init__(self, table_id, position, index, num_rows):
        self.table_id, self.position, self.index = table_id, position, index
        super().__init__(f"table {table_id}: index {index} at flat position "
                         f"{position} out of range [0, {num_rows})")


# --------------------------------------------------------------------------
# initial parameters  (ref model.py:130-139, model.py:361-373, embedding.py:65-71)

def init_params(embedding_sizes, sparse_dim, bottom_dims, top_dims, seed=0):
    """float64 initial parameters with the reference's stream layout."""
    nf = len(embedding_sizes) + 1
    top_chain = [sparse_dim + nf * (nf - 1) // 2] + list(top_dims)
    root = RngStream(seed)

    def mlp(dims, acts, stream):
        layers = []
        for l in range(len(dims) - 1):
            n_in, n_out = dims[l], dims[l + 1]
            std = np.sqrt(2.0 / (n_in + n_out))
            w = stream.derive(l).normal(n_out, n_in) * std
            layers.append((w, np.zeros(n_out), acts[l]))
        return layers

    bottom = mlp(list(bottom_dims), ["relu"] * (len(bottom_dims) - 1),
                 root.derive(0))
    top = mlp(top_chain, ["relu"] * (len(top_chain) - 2) + ["identity"],
              root.derive(1))
    bound = 1.0 / np.sqrt(sparse_dim)
    tables = [(root.derive(2, t).uniform(m, sparse_dim) * 2.0 - 1.0) * bound
              for t, m in enumerate(embedding_sizes)]
    return {"bottom": bottom, "top": top, "tables": tables}


def round_params_f32(model):
    """Params rounded to float32 and held as float64 (the GPU start point)."""
    r = lambda a: np.asarray(a, np.float32).astype(np.float64)
    return {"bottom": [(r(w), r(b), a) for w, b, a in model["bottom"]],
            "top": [(r(w), r(b), a) for w, b, a in model["top"]],
            "tables": [r(t) for t in model["tables"]]}


# --------------------------------------------------------------------------
# embedding bags  (ref embedding.py:117-124, 155-179, 182-210)

def check_bounds(num_rows, indices, table_id):
    bad = np.flatnonzero((indices < 0) | (indices >= num_rows))
    if bad.size:
        k = int(bad[0])
        raise PortIndexError(table_id, k, int(indices[k]), num_rows)


def lookup(W, offsets, indices, weights=None, table_id=0):
    """Pooled bags, strict ascending fold per bag (ref embedding.py:155-179)."""
    check_bounds(W.shape[0], indices, table_id)
    nb, d = offsets.shape[0] - 1, W.shape[1]
    rows = W[indices]
    if weights is not None:
        rows = rows * weights[:, None]
    out = np.zeros((nb, d))
    lens = np.diff(offsets)
    if nb and lens.size and np.all(lens == lens[0]) and lens[0] > 0:
        np.add.reduce(rows.reshape(nb, int(lens[0]), d), axis=1, out=out)
        return out
    for j in range(nb):
        lo, hi = int(offsets[j]), int(offsets[j + 1])
        if hi > lo:
            np.add.reduce(rows[lo:hi], axis=0, out=out[j])
    return out


def lookup_backward(W, offsets, indices, grad, weights=None, table_id=0):
    """Ascending unique rows + per-row ascending-position fold of the bag
    gradients (ref embedding.py:182-210).  Returns (rows, values)."""
    nb, d = offsets.shape[0] - 1, W.shape[1]
    if grad.shape != (nb, d):
        raise ValueError(f"grad_out shape {grad.shape} does not match "
                         f"(segments, dim) = {(nb, d)}")
    check_bounds(W.shape[0], indices, table_id)
    if indices.shape[0] == 0:
        return np.empty(0, np.int64), np.empty((0, d))
    bag_of = np.repeat(np.arange(nb), np.diff(offsets))
    contrib = grad[bag_of]
    if weights is not None:
        contrib = contrib * weights[:, None]
    rows, inv = np.unique(indices, return_inverse=True)
    vals = np.zeros((rows.shape[0], d))
    np.add.at(vals, inv, contrib)
    return rows, vals


# --------------------------------------------------------------------------
# dense algebra  (ref dense.py:62-78, 98-130, 193-255)

# ROWWISE = False replaces the per-row products with ONE float64 BLAS call per
# GEMM: the same sums in another (BLAS-chosen) order, i.e. not bit-identical
# to dlrmkit but within ~1e-15 relative of it — far inside the fp32
# tolerances the GPU is held to.  Only the Terabyte-shaped (B = 32768) parity
# test uses it, where the per-row loop would take minutes per step.
ROWWISE = True


def rowwise_matmul(a, b):
    """out[i] = a[i] @ b, one vector-matrix product per row (ref dense.py:62-78)."""
    if not ROWWISE:
        return a @ b
    out = np.empty((a.shape[0], b.shape[1]))
    for i in range(a.shape[0]):
        np.matmul(a[i], b, out=out[i])
    return out


def sigmoid(x):
    out = np.empty_like(x)
    pos = x >= 0.0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def _slice_bits(n_total):
    return (53 - max(2, math.ceil(math.log2(max(n_total, 2))))) // 2


def _grid_slices(a, col_max, n_total):
    """Split columns into power-of-two-grid slices (ref dense.py:206-230)."""
    bits = _slice_bits(n_total)
    live = col_max > 0.0
    expo = np.frexp(col_max)[1]
    out, rest = [], a
    for p in range(1, _LEVELS + 1):
        shift = np.where(live, _MAGIC * np.ldexp(1.0, expo - p * bits), 0.0)
        s = np.where(live, (rest + shift) - shift, 0.0)
        out.append(s)
        rest = rest - s
    return out


def _combine(parts):
    acc = np.array(parts[0], dtype=np.float64, copy=True)
    for p in parts[1:]:
        acc = acc + p
    return acc


def batch_reduced_grads(x, gz, n_total):
    """(dW, db) = (sum_b gz_b^T x_b, sum_b gz_b) through the exact slice
    products (ref model.py:183-208, dense.py:233-255)."""
    colmax = lambda m: (np.abs(m).max(axis=0) if m.shape[0]
                        else np.zeros(m.shape[1]))
    gs = _grid_slices(gz, colmax(gz), n_total)
    xs = _grid_slices(x, colmax(x), n_total)
    dw = _combine([gs[p - 1].T @ xs[q - 1] for p, q in _SLICE_PAIRS])
    db = _combine([s.sum(axis=0) for s in gs])
    return dw, db


def mlp_forward(layers, x):
    """Returns (output, layer inputs, pre-activations) (ref model.py:142-156)."""
    ins, pres, a = [], [], x
    for w, b, act in layers:
        ins.append(a)
        z = rowwise_matmul(a, w.T) + b
        pres.append(z)
        a = np.maximum(z, 0.0) if act == "relu" else z.copy()
    return a, ins, pres


def mlp_backward(layers, ins, pres, grad_y, n_total):
    """Per-layer (dW, db) and the input gradient (ref model.py:159-208)."""
    g = grad_y
    dws, dbs = [None] * len(layers), [None] * len(layers)
    gzs = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        w, _, act = layers[l]
        gate = (np.where(pres[l] > 0.0, 1.0, 0.0) if act == "relu"
                else np.ones_like(pres[l]))
        gzs[l] = g * gate
        g = rowwise_matmul(gzs[l], w)
    for l in range(len(layers)):
        dws[l], dbs[l] = batch_reduced_grads(ins[l], gzs[l], n_total)
    return dws, dbs, g


# --------------------------------------------------------------------------
# interaction  (ref model.py:214-268)

def interact(z0, embs):
    feats = [z0] + list(embs)
    b, d = z0.shape
    nf = len(feats)
    out = np.empty((b, d + nf * (nf - 1) // 2))
    out[:, :d] = z0
    c = d
    for i in range(nf):
        for j in range(i + 1, nf):
            out[:, c] = (feats[i] * feats[j]).sum(axis=1)
            c += 1
    return out


def interact_backward(z0, embs, gout):
    feats = [z0] + list(embs)
    b, d = z0.shape
    g = [np.zeros((b, d)) for _ in feats]
    g[0] += gout[:, :d]
    c = d
    for i in range(len(feats)):
        for j in range(i + 1, len(feats)):
            s = gout[:, c][:, None]
            g[i] += s * feats[j]
            g[j] += s * feats[i]
            c += 1
    return g[0], g[1:]


# --------------------------------------------------------------------------
# loss  (ref model.py:448-461)

def bce_from_logits(z, y):
    per = np.maximum(z, 0.0) - z * y + np.log1p(np.exp(-np.abs(z)))
    grad = (sigmoid(z[None, :])[0] - y) / z.shape[0]
    return float(per.mean()), grad, per


# --------------------------------------------------------------------------
# the training step  (ref parallel.py:250-287, optim.py:31-46)

def adagrad_update(param, grad, accum, lr, eps):
    """ref adagrad_step (optim.py:49-59): G += g*g; p -= lr*g / (sqrt(G)+eps)."""
    accum += grad * grad
    param -= lr * grad / (np.sqrt(accum) + eps)


def adagrad_update_rows(W, rows, vals, accum, lr, eps):
    """ref adagrad_step_rows (optim.py:62-73)."""
    accum[rows] += vals * vals
    W[rows] -= lr * vals / (np.sqrt(accum[rows]) + eps)


def adagrad_state(model):
    """Zero accumulators with the shapes of every parameter (ref
    AdagradState.for_mlp + the lazily created per-table accumulators)."""
    return {"bottom": [(np.zeros_like(w), np.zeros_like(b)) for w, b, _ in model["bottom"]],
            "top": [(np.zeros_like(w), np.zeros_like(b)) for w, b, _ in model["top"]],
            "tables": [np.zeros_like(W) for W in model["tables"]]}


def train_step(model, dense, offsets, indices, labels, lr, weights=None,
               adagrad=None, eps=1e-10):
    """One training step in place on ``model``; returns (loss, accuracy,
    probs).  SGD, or Adagrad when ``adagrad`` is a state from
    ``adagrad_state`` (ref Adagrad.apply, optim.py:135-140)."""
    weights = weights or [None] * len(model["tables"])
    z0, b_in, b_pre = mlp_forward(model["bottom"], dense)
    embs = [lookup(W, o, i, w, t) for t, (W, o, i, w) in
            enumerate(zip(model["tables"], offsets, indices, weights))]
    inter = interact(z0, embs)
    logits, t_in, t_pre = mlp_forward(model["top"], inter)
    z = logits[:, 0]
    loss, g_logit, _ = bce_from_logits(z, labels)
    prob = sigmoid(z[None, :])[0]
    n = dense.shape[0]
    t_dw, t_db, g_inter = mlp_backward(model["top"], t_in, t_pre,
                                       g_logit[:, None], n)
    g_z0, g_embs = interact_backward(z0, embs, g_inter)
    b_dw, b_db, _ = mlp_backward(model["bottom"], b_in, b_pre, g_z0, n)
    sparse = [lookup_backward(W, o, i, g, w, t) for t, (W, o, i, g, w) in
              enumerate(zip(model["tables"], offsets, indices, g_embs,
                            weights))]
    if adagrad is not None:
        for which, layers, dws, dbs in (("bottom", model["bottom"], b_dw, b_db),
                                        ("top", model["top"], t_dw, t_db)):
            for (w, b, _), dw, db, (aw, ab) in zip(layers, dws, dbs, adagrad[which]):
                adagrad_update(w, dw, aw, lr, eps)
                adagrad_update(b, db, ab, lr, eps)
        for W, (rows, vals), acc in zip(model["tables"], sparse, adagrad["tables"]):
            if rows.size:
                adagrad_update_rows(W, rows, vals, acc, lr, eps)
    else:
        for layers, dws, dbs in ((model["bottom"], b_dw, b_db),
                                 (model["top"], t_dw, t_db)):
            for (w, b, _), dw, db in zip(layers, dws, dbs):
                w -= lr * dw
                b -= lr * db
        for W, (rows, vals) in zip(model["tables"], sparse):
            if rows.size:
                W[rows] -= lr * vals
    acc = float(np.mean((prob > 0.5) == (labels > 0.5)))
    return loss, acc, prob
