"""Criteo ingestion — the reference's ``dlrmkit.datagen`` Criteo API
(``parse_criteo`` / ``read_criteo`` / ``CriteoSample`` / ``CriteoFormatError``,
ref ``datagen.py:318-371``) over the native parser in ``libdlrmb200.so``
(``dlrm_criteo_parse``: multithreaded, BLAKE2b-64 token hashing, writes
straight into the next batch's host buffers).

Parity with the reference (tests/test_criteo.py, fixtures made by dlrmkit):
labels and categorical indices are bit-identical; dense values are the
reference's float64 ``log1p(max(x, 0))`` rounded to fp32 (the training
precision).  Error messages are the reference's ``"line k: ..."`` texts.

``CriteoBatchReader`` turns a (gzipped) TSV file into host ``CriteoBatch``es
(dense [B, 13] f32, 26 one-index-per-bag tables, labels) for
``StepEngine.pack_host_batch`` / ``load``, or ``train_step`` via
``batch.train_args()``.
"""

from __future__ import annotations

import ctypes as C
import gzip
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["NUM_DENSE", "NUM_CATEGORICAL", "CriteoFormatError", "CriteoSample",
           "parse_criteo", "read_criteo", "parse_criteo_block", "CriteoBatch",
           "CriteoBatchReader", "hash_token"]

NUM_DENSE = 13
NUM_CATEGORICAL = 26


class CriteoFormatError(ValueError):
    """Malformed record; the message carries the 1-based line number."""


@dataclass
class CriteoSample:
    label: int
    dense: np.ndarray        # 13 log1p-transformed values (fp32)
    categorical: np.ndarray  # 26 embedding indices (int64)


def hash_token(token: str) -> int:
    """The reference's fixed 64-bit token hash (``_hash_token``)."""
    b = token.encode("utf-8")
    return int(_lib.lib().dlrm_blake2b64(b, len(b)))


def _vocab(vocab_sizes) -> np.ndarray:
    if len(vocab_sizes) != NUM_CATEGORICAL:
        raise ValueError(f"need {NUM_CATEGORICAL} vocabulary sizes, got {len(vocab_sizes)}")
    return np.ascontiguousarray(np.asarray(vocab_sizes, dtype=np.int64))


def _line_count(b: bytes) -> int:
    """Line terminators in universal-newline mode ('\\n', '\\r', '\\r\\n')."""
    return b.count(b"\n") + b.count(b"\r") - b.count(b"\r\n")


def parse_criteo_block(text: bytes, vocab_sizes, first_lineno: int = 1,
                       max_records: int | None = None, nthreads: int = 0,
                       universal_newlines: bool = True):
    """Parse the lines of ``text`` (bytes; universal newlines by default, as
    the reference's text-mode ``read_criteo`` sees a file).  Returns
    ``(labels f32 [n], dense f32 [n, 13], cat int64 [26, n], consumed_bytes)``;
    raises CriteoFormatError for the first malformed line."""
    voc = _vocab(vocab_sizes)
    if max_records is None:   # an upper bound on the records
        max_records = text.count(b"\n") + (text.count(b"\r") if universal_newlines else 0) + 1
    n = max(int(max_records), 0)
    labels = np.empty(n, np.float32)
    dense = np.empty((n, NUM_DENSE), np.float32)
    cat = np.empty((NUM_CATEGORICAL, max(n, 1)), np.int64)
    consumed = C.c_int64(0)
    buf = C.c_char_p(text)
    got = _lib.lib().dlrm_criteo_parse(
        buf, len(text), voc.ctypes.data, n, labels.ctypes.data, dense.ctypes.data, NUM_DENSE,
        cat.ctypes.data, cat.shape[1], int(first_lineno), C.byref(consumed),
        (int(nthreads) << 8) | (1 if universal_newlines else 0))
    if got == -2:
        raise CriteoFormatError(_lib.lib().dlrm_last_error().decode(errors="replace"))
    if got < 0:
        raise ValueError(_lib.lib().dlrm_last_error().decode(errors="replace"))
    return labels[:got], dense[:got], cat[:, :got], int(consumed.value)


def parse_criteo(line: str, vocab_sizes, lineno: int = 1) -> CriteoSample:
    """One tab-separated record: label, 13 integer fields, 26 tokens (ref
    datagen.py:330-362).  Checks in the reference's order: field count, then
    the vocabulary list, then the fields."""
    fields = line.rstrip("\n").split("\t")
    expected = 1 + NUM_DENSE + NUM_CATEGORICAL
    if len(fields) != expected:
        raise CriteoFormatError(
            f"line {lineno}: expected {expected} tab-separated fields, got {len(fields)}")
    _vocab(vocab_sizes)
    body = line.rstrip("\n").encode("utf-8")
    labels, dense, cat, _ = parse_criteo_block(body, vocab_sizes, lineno, 1, 1,
                                               universal_newlines=False)
    if labels.size == 0:   # a whitespace-only record: every field empty
        return CriteoSample(0, np.zeros(NUM_DENSE, np.float32), np.zeros(NUM_CATEGORICAL, np.int64))
    return CriteoSample(int(labels[0]), dense[0].copy(), cat[:, 0].copy())


def _open(path):
    return gzip.open(path, "rb") if str(path).endswith(".gz") else open(path, "rb")


def _blocks(path, vocab_sizes, chunk_bytes: int, nthreads: int):
    """(labels, dense, cat) per chunk of complete lines of a file."""
    lineno = 1
    rest = b""
    with _open(path) as f:
        while True:
            data = f.read(chunk_bytes)
            eof = not data
            buf = rest + data
            if not buf:
                return
            cut = len(buf) if eof else buf.rfind(b"\n") + 1
            if cut == 0:          # no complete line yet
                rest = buf
                continue
            block, rest = buf[:cut], buf[cut:]
            labels, dense, cat, _ = parse_criteo_block(block, vocab_sizes, lineno,
                                                       nthreads=nthreads)
            lineno += _line_count(block)
            yield labels, dense, cat
            if eof:
                return


def read_criteo(path, vocab_sizes, chunk_bytes: int = 64 << 20, nthreads: int = 0):
    """Yield CriteoSamples from a (optionally gzipped) tab-separated file (ref
    datagen.py:365-371); parsed natively a chunk at a time."""
    for labels, dense, cat in _blocks(path, vocab_sizes, chunk_bytes, nthreads):
        for r in range(labels.shape[0]):
            yield CriteoSample(int(labels[r]), dense[r].copy(), cat[:, r].copy())


@dataclass
class CriteoBatch:
    """One training batch in host memory: ``dense [B, 13]`` f32, per-table
    ``offsets`` (``arange(B + 1)``: one index per bag) and ``indices``, and
    ``labels [B]`` f32 — what ``StepEngine.pack_host_batch`` / ``load`` take."""
    dense: np.ndarray
    offsets: list
    indices: list
    labels: np.ndarray

    def train_args(self):
        """``(dense, [SparseBatch] x 26, labels)`` for ``train_step`` /
        ``evaluate`` (moves the bags to the GPU)."""
        from .embedding import SparseBatch
        return self.dense, [SparseBatch(o, i) for o, i in zip(self.offsets, self.indices)], \
            self.labels


class CriteoBatchReader:
    """``CriteoBatch``es of ``batch_size`` records from a (gzipped) Criteo TSV
    file; the tail smaller than a batch is dropped unless ``drop_last=False``."""

    def __init__(self, path, vocab_sizes, batch_size: int, drop_last: bool = True,
                 chunk_bytes: int = 64 << 20, nthreads: int = 0):
        if batch_size < 1:
            raise ValueError("batch size must be positive")
        _vocab(vocab_sizes)
        self.path, self.vocab = path, list(vocab_sizes)
        self.B, self.drop_last = int(batch_size), drop_last
        self.chunk_bytes, self.nthreads = chunk_bytes, nthreads

    def __iter__(self):
        B = self.B
        offs = np.arange(B + 1, dtype=np.int64)
        pend = None

        def emit(lab, den, ca):
            n = lab.shape[0]
            o = offs if n == B else np.arange(n + 1, dtype=np.int64)
            return CriteoBatch(np.ascontiguousarray(den), [o] * NUM_CATEGORICAL,
                               [ca[i].copy() for i in range(NUM_CATEGORICAL)],
                               np.ascontiguousarray(lab))

        for lab, den, ca in _blocks(self.path, self.vocab, self.chunk_bytes, self.nthreads):
            if pend is not None:
                lab = np.concatenate([pend[0], lab])
                den = np.concatenate([pend[1], den])
                ca = np.concatenate([pend[2], ca], axis=1)
            s = 0
            while s + B <= lab.shape[0]:
                yield emit(lab[s:s + B], den[s:s + B], ca[:, s:s + B])
                s += B
            pend = (lab[s:], den[s:], ca[:, s:]) if s < lab.shape[0] else None
        if pend is not None and not self.drop_last:
            yield emit(*pend)
