"""TEST INFRASTRUCTURE ONLY — float32 restatements of the folds the GPU
kernels reproduce bit for bit.

The reference computes in float64; the GPU computes in float32.  For the
integer/ordering parts of the embedding path the contract is bit-exactness,
so these functions restate the reference's fold ORDER in float32:

* ``lookup`` — per bag a strict ascending-position fold that starts from the
  first row (numpy ``add.reduce`` semantics, ref ``embedding.py:169-178``),
  with ``w[idx]*a`` rounded before it is added (ref ``embedding.py:165-166``).
* ``lookup_backward`` — ascending unique rows, per row an ascending-position
  fold starting from +0.0 (``np.add.at`` into zeros, ref
  ``embedding.py:201-209``).
* ``sgd_rows`` / ``sgd_dense`` — ``w - fl(lr*g)`` (ref ``optim.py:35,46``).
"""

from __future__ import annotations

import numpy as np

f32 = np.float32


def lookup(W, offsets, indices, weights=None):
    W = np.asarray(W, f32)
    offsets = np.asarray(offsets, np.int64)
    indices = np.asarray(indices, np.int64)
    nb, d = offsets.shape[0] - 1, W.shape[1]
    rows = W[indices]
    if weights is not None:
        rows = rows * np.asarray(weights, f32)[:, None]
    out = np.zeros((nb, d), f32)
    lens = np.diff(offsets)
    if nb == 0:
        return out
    live = lens > 0
    out[live] = rows[offsets[:-1][live]]
    for p in range(1, int(lens.max(initial=0))):
        m = lens > p
        out[m] = out[m] + rows[offsets[:-1][m] + p]
    return out


def lookup_backward(offsets, indices, grad, weights=None):
    offsets = np.asarray(offsets, np.int64)
    indices = np.asarray(indices, np.int64)
    grad = np.asarray(grad, f32)
    d = grad.shape[1]
    if indices.size == 0:
        return np.empty(0, np.int64), np.empty((0, d), f32)
    bag_of = np.repeat(np.arange(offsets.shape[0] - 1), np.diff(offsets))
    contrib = grad[bag_of]
    if weights is not None:
        contrib = contrib * np.asarray(weights, f32)[:, None]
    rows, inv = np.unique(indices, return_inverse=True)
    vals = np.zeros((rows.shape[0], d), f32)
    np.add.at(vals, inv, contrib)
    return rows, vals


def sgd_rows(W, rows, vals, lr):
    W = np.array(W, f32, copy=True)
    if rows.size:
        W[rows] = W[rows] - f32(lr) * vals
    return W


def sgd_dense(p, g, lr):
    return np.asarray(p, f32) - f32(lr) * np.asarray(g, f32)


def adagrad_dense(p, g, accum, lr, eps):
    """float32 restatement of ref adagrad_step (optim.py:49-59), op for op:
    G = G + g*g; p = p - (lr*g) / (sqrt(G) + eps).  Returns (p, G)."""
    g = np.asarray(g, f32)
    G = (np.asarray(accum, f32) + g * g).astype(f32)
    upd = (f32(lr) * g) / (np.sqrt(G) + f32(eps))
    return (np.asarray(p, f32) - upd).astype(f32), G


def adagrad_rows(W, rows, vals, accum, lr, eps):
    """float32 restatement of ref adagrad_step_rows (optim.py:62-73)."""
    W = np.array(W, f32, copy=True)
    A = np.array(accum, f32, copy=True)
    if rows.size:
        W[rows], A[rows] = adagrad_dense(W[rows], vals, A[rows], lr, eps)
    return W, A

