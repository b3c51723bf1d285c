"""Host-side seeded streams and synthetic mini-batch generation.

This is input/parameter *generation*, not the training step: it runs on the
host in float64 exactly as the reference does, so that the same seed yields
the same initial parameters and the same batches on both implementations.

Restated from the reference's published behaviour:

* ``RngStream``  — numpy Philox seeded through ``SeedSequence(seed,
  spawn_key=key)``; ``derive`` appends keys
  (ref ``pkg/src/dlrmkit/dense.py:136-170``).
* ``RandomBatchSource`` — the CLI's random-mode source
  (ref ``pkg/src/dlrmkit/cli.py:294-314``) over
  ``gen_dense_batch``/``gen_sparse_batch`` (ref ``datagen.py:73-96``): dense
  U[0,1) rows, then per table either ``B*k`` uniform indices (fixed mode) or,
  sample by sample, a length in [1, k] followed by that many indices, then
  labels ``U[0,1) < 0.5``.

Batches are returned as plain numpy arrays (``HostBatch``); the device-side
``SparseBatch`` is built from them by the caller.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["RngStream", "HostBatch", "RandomBatchSource", "zipf_indices"]


@dataclass
class RngStream:
    """Counter-based Philox stream; (seed, key) fully determines the draws."""

    seed: int
    key: tuple = ()
    _gen: np.random.Generator = field(init=False, repr=False)

    def __post_init__(self):
        seq = np.random.SeedSequence(self.seed, spawn_key=tuple(self.key))
        self._gen = np.random.Generator(np.random.Philox(seq))

    def derive(self, *key: int) -> "RngStream":
        return RngStream(self.seed, tuple(self.key) + tuple(key))

    def uniform(self, rows: int, cols: int) -> np.ndarray:
        return self._gen.random((rows, cols), dtype=np.float64)

    def normal(self, rows: int, cols: int) -> np.ndarray:
        return self._gen.standard_normal((rows, cols), dtype=np.float64)

    def integers(self, low: int, high: int, size) -> np.ndarray:
        return self._gen.integers(low, high, size=size, dtype=np.int64)


@dataclass
class HostBatch:
    """One mini-batch in host memory: dense rows, per-table CSR bags, labels."""

    dense: np.ndarray                 # (B, dense_dim) float64
    offsets: list                     # per table int64 (B+1,)
    indices: list                     # per table int64 (nnz_t,)
    labels: np.ndarray                # (B,) float64 in {0, 1}

    @property
    def batch_size(self) -> int:
        return self.dense.shape[0]


class RandomBatchSource:
    """Random-mode batches with the reference CLI's stream layout.

    ``RngStream(seed).derive(10, key)`` is the stream the reference's
    ``_RandomSource`` draws from (ref ``cli.py:306``).
    """

    def __init__(self, table_sizes, dense_dim: int, batch_size: int,
                 indices_per_lookup: int, fixed: bool, seed: int = 0,
                 key: int = 0, stream: RngStream | None = None):
        if indices_per_lookup < 1 or batch_size < 1 or dense_dim < 1:
            raise ValueError("batch size, dense dim and k must be positive")
        for m in table_sizes:
            if indices_per_lookup > m:
                raise ValueError(
                    f"indices per lookup {indices_per_lookup} exceeds table "
                    f"size {m}")
        self.table_sizes = [int(m) for m in table_sizes]
        self.dense_dim = int(dense_dim)
        self.batch_size = int(batch_size)
        self.k = int(indices_per_lookup)
        self.fixed = bool(fixed)
        self.stream = stream if stream is not None else \
            RngStream(seed).derive(10, key)
        # variable-length bags in native code (dlrm_random_bags), same draws
        self.native = True

    def _bags(self, m: int):
        b, k, s = self.batch_size, self.k, self.stream
        if self.fixed:
            lengths = np.full(b, k, dtype=np.int64)
            idx = s.integers(0, m, size=int(b * k))
        else:
            lengths = np.empty(b, dtype=np.int64)
            parts = []
            for j in range(b):
                n = int(s.integers(1, k + 1, size=()))
                lengths[j] = n
                parts.append(s.integers(0, m, size=n))
            idx = np.concatenate(parts) if parts else np.empty(0, np.int64)
        offsets = np.zeros(b + 1, dtype=np.int64)
        np.cumsum(lengths, out=offsets[1:])
        return offsets, idx.astype(np.int64, copy=False)

    def next_batch(self) -> HostBatch:
        dense = self.stream.uniform(self.batch_size, self.dense_dim)
        native = None if self.fixed or not self.native else _native_bags(self)
        if native is not None:
            offs, idxs = native
        else:
            offs, idxs = [], []
            for m in self.table_sizes:
                o, i = self._bags(m)
                offs.append(o)
                idxs.append(i)
        labels = (self.stream.uniform(1, self.batch_size)[0] < 0.5
                  ).astype(np.float64)
        return HostBatch(dense, offs, idxs, labels)


def _native_bags(src: "RandomBatchSource"):
    """All tables' variable-length bags through ``dlrm_random_bags`` (the
    same Philox draws numpy makes in ``_bags``, in native code; ~40x
    faster at the Big-Basin shape), or None when the library is absent."""
    try:
        import ctypes as C
        from . import _lib
        L = _lib.lib()
    except Exception:
        return None
    gen = src.stream._gen
    st = gen.bit_generator.state
    if st.get("bit_generator") != "Philox" or max(src.table_sizes) >= 1 << 32:
        return None
    words = np.zeros(13, dtype=np.uint64)
    words[0:4] = st["state"]["counter"]
    words[4:6] = st["state"]["key"]
    words[6:10] = st["buffer"]
    words[10], words[11], words[12] = st["buffer_pos"], st["has_uint32"], st["uinteger"]
    T, B, k = len(src.table_sizes), src.batch_size, src.k
    rows = np.asarray(src.table_sizes, dtype=np.int64)
    offs = np.empty((T, B + 1), dtype=np.int64)
    idx = np.empty((T, B * k), dtype=np.int64)
    nnz = np.empty(T, dtype=np.int64)
    p = lambda a: C.c_void_p(a.ctypes.data)
    if L.dlrm_random_bags(p(words), p(rows), T, B, k, p(offs), p(idx), p(nnz)) != 0:
        return None
    st["state"]["counter"] = words[0:4].copy()
    st["state"]["key"] = words[4:6].copy()
    st["buffer"] = words[6:10].copy()
    st["buffer_pos"], st["has_uint32"], st["uinteger"] = (int(words[10]), int(words[11]),
                                                         int(words[12]))
    gen.bit_generator.state = st
    return [offs[t] for t in range(T)], [idx[t, :nnz[t]].copy() for t in range(T)]


def zipf_indices(num_rows: int, n: int, alpha: float = 1.05,
                 seed: int = 1) -> np.ndarray:
    """Bounded Zipf(alpha) row ids over [0, num_rows), ranks scrambled by a
    multiplicative hash so hot rows are spread over the table (the c5 sweep's
    skewed distribution, defined in SURVEY.md §8(d); not in the reference)."""
    rng = np.random.default_rng(seed)
    # inverse-CDF sampling of a bounded power law on ranks 1..num_rows
    u = rng.random(n)
    if abs(alpha - 1.0) < 1e-12:
        r = np.exp(u * np.log(num_rows + 1.0))
    else:
        a = 1.0 - alpha
        r = (1.0 + u * ((num_rows + 1.0) ** a - 1.0)) ** (1.0 / a)
    ranks = np.clip(np.floor(r).astype(np.int64) - 1, 0, num_rows - 1)
    return (ranks * 2654435761) % num_rows
