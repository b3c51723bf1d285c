"""Embedding tables and pooled multi-hot lookups — the reference's operator
API (``dlrmkit.embedding``, ref ``pkg/src/dlrmkit/embedding.py``) on B200.

Same names, argument meanings and exceptions as the reference; tensors are
CUDA fp32 (weights, gradients) and CUDA int64 (offsets, indices).  The pooled
lookup and its backward run in ``libdlrmb200.so`` (``dlrm_emb_fwd`` /
``dlrm_emb_bwd_coalesce``); there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .rng import RngStream

__all__ = [
    "EmbeddingTable", "SparseBatch", "SparseRowGrad", "LookupIndexError",
    "offsets_from_lengths", "lengths_from_offsets", "lookup_batch",
    "lookup_backward",
]


class LookupIndexError(IndexError):
    """An index falls outside the table; carries table id, position, index
    (ref embedding.py:32-42, same message)."""

    def __init__(self, table_id, position, index, num_rows):
        self.table_id = table_id
        self.position = position
        self.index = index
        super().__init__(
            f"table {table_id}: index {index} at flat position {position} "
            f"out of range [0, {num_rows})")


def _cuda_f32(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=_lib.device(), dtype=torch.float32).contiguous()
    return torch.as_tensor(np.asarray(a, dtype=np.float32),
                           device=_lib.device()).contiguous()


class EmbeddingTable:
    """An m x d fp32 parameter matrix on the GPU (ref embedding.py:45-71).

    ``weights`` may be a view into a larger buffer (the trainer keeps all of
    a rank's tables in one allocation)."""

    def __init__(self, weights, table_id: int = 0):
        w = _cuda_f32(weights)
        if w.dim() != 2:
            raise ValueError(f"weights must be m x d, got {tuple(w.shape)}")
        self.weights = w
        self.table_id = table_id

    @property
    def num_rows(self) -> int:
        return int(self.weights.shape[0])

    @property
    def dim(self) -> int:
        return int(self.weights.shape[1])

    @classmethod
    def initialize(cls, num_rows: int, dim: int, stream: RngStream,
                   table_id: int = 0) -> "EmbeddingTable":
        """Rows uniform in (-1/sqrt(d), +1/sqrt(d)), drawn in float64 with the
        reference's stream, then rounded to fp32."""
        bound = 1.0 / np.sqrt(dim)
        w = (stream.uniform(num_rows, dim) * 2.0 - 1.0) * bound
        return cls(w, table_id)


def offsets_from_lengths(lengths) -> np.ndarray:
    """Prefix sums with the leading 0 and the terminal total (CSR style)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    if np.any(lengths < 0):
        raise ValueError("lengths must be nonnegative")
    out = np.zeros(lengths.shape[0] + 1, dtype=np.int64)
    np.cumsum(lengths, out=out[1:])
    return out


def lengths_from_offsets(offsets) -> np.ndarray:
    if isinstance(offsets, torch.Tensor):
        offsets = offsets.cpu().numpy()
    return np.diff(np.asarray(offsets, dtype=np.int64))


class SparseBatch:
    """offsets/indices(/weights) encoding of t pooled lookups
    (ref embedding.py:74-124).  Validated on the host, stored on the GPU."""

    def __init__(self, offsets, indices, weights=None):
        o = _host_i64(offsets)
        i = _host_i64(indices)
        w = None if weights is None else np.asarray(
            weights.cpu().numpy() if isinstance(weights, torch.Tensor)
            else weights, dtype=np.float64)
        _validate(o, i, w)
        dev = _lib.device()
        self.offsets = torch.as_tensor(o, device=dev)
        self.indices = torch.as_tensor(i, device=dev)
        self.weights = (None if w is None else
                        torch.as_tensor(w.astype(np.float32), device=dev))
        self._host_indices = i

    @property
    def num_segments(self) -> int:
        return int(self.offsets.shape[0]) - 1

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    def lengths(self) -> np.ndarray:
        return lengths_from_offsets(self.offsets)

    def segment_slice(self, j: int) -> slice:
        o = self.offsets[j:j + 2].cpu()
        return slice(int(o[0]), int(o[1]))


def _host_i64(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return np.asarray(a, dtype=np.int64)


def _validate(o, i, w):
    """Reference invariants (ref embedding.py:89-105), same messages."""
    if o.ndim != 1 or o.shape[0] < 1:
        raise ValueError("offsets must be 1-D with at least the leading 0")
    if o[0] != 0:
        raise ValueError(f"offsets[0] must be 0, got {o[0]}")
    if np.any(np.diff(o) < 0):
        raise ValueError("offsets must be nondecreasing")
    if o[-1] != i.shape[0]:
        raise ValueError(
            f"terminal offset {o[-1]} != len(indices) {i.shape[0]}")
    if w is not None and w.shape != i.shape:
        raise ValueError(
            f"weights shape {w.shape} does not align with indices shape "
            f"{i.shape}")


@dataclass
class SparseRowGrad:
    """Coalesced sparse gradient: ascending unique row ids (CUDA int64) and
    one d-vector each (CUDA fp32) (ref embedding.py:127-137)."""

    rows: torch.Tensor
    values: torch.Tensor

    def to_dense(self, num_rows: int) -> torch.Tensor:
        out = torch.zeros((num_rows, self.values.shape[1]),
                          dtype=self.values.dtype, device=self.values.device)
        if self.rows.numel():
            out[self.rows] = self.values
        return out


def _desc(table: EmbeddingTable, batch: SparseBatch, out_offset=0,
          row_base=0) -> _lib.TableDesc:
    return _lib.TableDesc(
        _lib.ptr(batch.offsets).value, _lib.ptr(batch.indices).value,
        _lib.ptr(batch.weights).value, row_base, table.num_rows, out_offset,
        batch.nnz, table.table_id)


def _raise_lookup_error(err_pos, table: EmbeddingTable, batch: SparseBatch):
    k = int(err_pos[0].item())
    raise LookupIndexError(table.table_id, k, int(batch._host_indices[k]),
                           table.num_rows)


def lookup_batch(table: EmbeddingTable, batch: SparseBatch) -> torch.Tensor:
    """Pooled lookup: row j = strict ascending fold over segment j of
    w[index] * weight; empty segments give zero rows (ref
    embedding.py:155-179).  Raises LookupIndexError like the reference."""
    dev = _lib.device()
    t, d = batch.num_segments, table.dim
    out = torch.empty((t, d), dtype=torch.float32, device=dev)
    err_pos = torch.empty(1, dtype=torch.int64, device=dev)
    err_flag = torch.empty(1, dtype=torch.int32, device=dev)
    s = _lib.stream_handle()
    _lib.call("dlrm_err_reset", _lib.ptr(err_pos), 1, _lib.ptr(err_flag), s)
    descs = _lib.table_array([_desc(table, batch)])
    _lib.call("dlrm_emb_fwd", _lib.ptr(table.weights), d,
              C.cast(descs, C.c_void_p), 1, t, _lib.ptr(out), d,
              _lib.ptr(err_pos), _lib.ptr(err_flag), s)
    if int(err_flag.item()):
        _raise_lookup_error(err_pos, table, batch)
    return out


def lookup_backward(table: EmbeddingTable, batch: SparseBatch,
                    grad_out) -> SparseRowGrad:
    """Adjoint of lookup_batch: ascending unique rows, each with the
    ascending-position fold of its contributions (ref embedding.py:182-210).
    """
    g = _cuda_f32(grad_out)
    if tuple(g.shape) != (batch.num_segments, table.dim):
        raise ValueError(
            f"grad_out shape {tuple(g.shape)} does not match "
            f"(segments, dim) = {(batch.num_segments, table.dim)}")
    dev = _lib.device()
    d, nnz = table.dim, batch.nnz
    err_pos = torch.empty(1, dtype=torch.int64, device=dev)
    err_flag = torch.empty(1, dtype=torch.int32, device=dev)
    s = _lib.stream_handle()
    _lib.call("dlrm_err_reset", _lib.ptr(err_pos), 1, _lib.ptr(err_flag), s)
    rows = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
    vals = torch.empty((max(nnz, 1), d), dtype=torch.float32, device=dev)
    nu = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = _lib.size("dlrm_emb_bwd_workspace_size", max(nnz, 1),
                    table.num_rows, d)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    descs = _lib.table_array([_desc(table, batch)])
    _lib.call("dlrm_emb_bwd_coalesce", d, C.cast(descs, C.c_void_p),
              batch.num_segments, _lib.ptr(g), d, _lib.ptr(rows),
              _lib.ptr(vals), _lib.ptr(nu), _lib.ptr(err_pos),
              _lib.ptr(err_flag), _lib.ptr(ws), wsb, s)
    if int(err_flag.item()):
        _raise_lookup_error(err_pos, table, batch)
    u = int(nu.item())
    return SparseRowGrad(rows[:u], vals[:u])
