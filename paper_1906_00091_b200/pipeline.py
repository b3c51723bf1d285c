"""Input pipeline of the training step: one step's inputs as ONE contiguous
block (one host->device copy per step), packed from the reference's host
arrays by worker threads and copied to the device ahead of the step.

The reference feeds ``train_step`` numpy arrays (dense rows, per-table
offsets / indices, labels; ref ``cli.py:294-314``, ``parallel.py:250-287``).
Here:

* ``InputLayout`` is the byte layout of a step's inputs for a fixed batch
  size and per-table index capacity: ``[x (B x ceil4(dense)) f32 | labels f32
  | offsets (T x (B+1)) i64 | indices (sum of capacities) i64 | weights f32]``,
  16-byte aligned sections.  The step engine's input sets, packed pinned host
  blocks and the prefetcher's device ring all use it, so moving a batch is a
  single ``copy_``.
* ``Prefetcher`` wraps an iterator of host batches: worker threads pack each
  batch into a reused pinned block (the large copies release the GIL and run
  in parallel), a copy stream moves it into a device ring slot, and the
  iteration yields ``(dense_x, batches, labels)`` handles that ``train_step``
  accepts in place of the arrays (same call, same result).  The step then
  needs one device-to-device copy of the landed block.
"""

from __future__ import annotations

import os
import queue
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib

__all__ = ["InputLayout", "Prefetcher", "StagedDense", "StagedSparse", "StagedLabels"]


def _ceil4(n: int) -> int:
    return (n + 3) // 4 * 4


class InputLayout:
    """Sections of one step's input block (see the module docstring)."""

    def __init__(self, batch: int, num_tables: int, dense_dim: int, capacities,
                 weighted: bool = False):
        self.B, self.T, self.k0 = int(batch), int(num_tables), int(dense_dim)
        self.caps = [max(1, int(c)) for c in capacities]
        if len(self.caps) != self.T:
            raise ValueError("one capacity per table")
        self.weighted = bool(weighted)
        self.cap_base = np.concatenate([[0], np.cumsum(self.caps)]).astype(np.int64)
        a16 = lambda n: (n + 15) // 16 * 16
        B, T, ncap = self.B, self.T, int(self.cap_base[-1])
        self.sections = {}
        o = 0
        for name, nbytes in (("x", B * _ceil4(self.k0) * 4), ("labels", B * 4),
                             ("offsets", T * (B + 1) * 8), ("indices", ncap * 8),
                             ("iweights", ncap * 4 if self.weighted else 0)):
            self.sections[name] = (o, nbytes)
            o = a16(o + nbytes)
        self.nbytes = o
        # the native packer's section offsets and capacity prefix (kept alive
        # with the layout: their addresses go to C on every batch)
        self._sec = np.array([self.sections["x"][0], self.sections["labels"][0],
                              self.sections["offsets"][0], self.sections["indices"][0],
                              self.sections["iweights"][0] if self.weighted else -1], np.int64)
        self._cap_base_ptr = self.cap_base.ctypes.data

    def key(self):
        return (self.B, self.T, self.k0, tuple(self.caps), self.weighted)

    # ------------------------------------------------------------------
    def views(self, blk: torch.Tensor) -> dict:
        """Typed torch views of a block (host or device)."""
        B, T, ncap = self.B, self.T, int(self.cap_base[-1])

        def view(name, dtype, shape):
            o, n = self.sections[name]
            if n == 0:
                return None
            return blk[o:o + n].view(dtype).view(*shape)
        return {"block": blk,
                "x": view("x", torch.float32, (B, _ceil4(self.k0))),
                "labels": view("labels", torch.float32, (B,)),
                "offsets": view("offsets", torch.int64, (T, B + 1)),
                "indices": view("indices", torch.int64, (ncap,)),
                "iweights": view("iweights", torch.float32, (ncap,))}

    def _np(self, arr: np.ndarray, name, dtype, shape):
        o, n = self.sections[name]
        return arr[o:o + n].view(dtype).reshape(shape)

    def check(self, indices, weights=None):
        for t in range(self.T):
            n = int(np.asarray(indices[t]).shape[0])
            if n > self.caps[t]:
                raise OverflowError(f"table {t}: {n} indices exceed capacity {self.caps[t]}")
        if weights is not None and any(w is not None for w in weights) and not self.weighted:
            raise ValueError("weighted bags need a weighted input layout")

    def pack(self, blk: torch.Tensor, dense, offsets, indices, labels, weights=None,
             pool: ThreadPoolExecutor | None = None) -> torch.Tensor:
        """Write one batch of host arrays into the (pinned) host block ``blk``
        (reused; returns it).  With ``pool`` the dense rows (in row slabs) and
        every table's offsets / indices are copied by the pool's threads."""
        threads = pool._max_workers if pool is not None else 1
        if weights is not None and any(w is not None for w in weights) and not self.weighted:
            raise ValueError("weighted bags need a weighted input layout")
        PL = _lib.pylib()
        if PL is not None:
            # validation, pointers and packing in C (no per-table Python)
            rc = PL.dlrm_pack_batch_py(dense, labels, offsets, indices, weights,
                                       blk.data_ptr(), self._sec.ctypes.data, self.B, self.k0,
                                       _ceil4(self.k0), self.T, self._cap_base_ptr,
                                       int(max(1, threads)))
            if rc == 0:
                return blk
            if rc >= 2:
                self.check(indices, weights)  # raises the OverflowError
        self.check(indices, weights)
        if self._pack_native(blk, dense, offsets, indices, labels, weights, threads):
            return blk
        a = blk.numpy()
        B, T = self.B, self.T
        x = self._np(a, "x", np.float32, (B, _ceil4(self.k0)))
        offs = self._np(a, "offsets", np.int64, (T, B + 1))
        idx = self._np(a, "indices", np.int64, (int(self.cap_base[-1]),))
        wv = self._np(a, "iweights", np.float32, (int(self.cap_base[-1]),)) \
            if self.weighted else None
        dense = np.asarray(dense)
        if dense.shape != (B, self.k0):
            raise ValueError(f"dense input {dense.shape} != {(B, self.k0)}")
        jobs = []

        def dense_rows(lo, hi):
            np.copyto(x[lo:hi, :self.k0], dense[lo:hi], casting="unsafe")

        def table(t):
            np.copyto(offs[t], np.asarray(offsets[t]), casting="unsafe")
            i = np.asarray(indices[t])
            cb = int(self.cap_base[t])
            np.copyto(idx[cb:cb + i.shape[0]], i, casting="unsafe")
            if wv is not None:
                w = None if weights is None else weights[t]
                if w is None:
                    wv[cb:cb + i.shape[0]] = 1.0
                else:
                    np.copyto(wv[cb:cb + i.shape[0]], np.asarray(w), casting="unsafe")

        slabs = 4 if pool is not None and B >= 256 else 1
        step = (B + slabs - 1) // slabs
        for lo in range(0, B, step):
            jobs.append((dense_rows, (lo, min(B, lo + step))))
        for t in range(T):
            jobs.append((table, (t,)))
        if pool is None:
            for fn, args in jobs:
                fn(*args)
        else:
            for f in [pool.submit(fn, *args) for fn, args in jobs]:
                f.result()
        np.copyto(self._np(a, "labels", np.float32, (B,)), np.asarray(labels), casting="unsafe")
        return blk

    def _pack_native(self, blk, dense, offsets, indices, labels, weights, threads) -> bool:
        """``dlrm_pack_batch`` (native threads, no GIL) when the arrays have
        the reference's dtypes (float64 dense / labels / weights, int64
        offsets / indices); False to use the numpy path."""
        try:
            import ctypes as C
            from . import _lib
            L = _lib.lib()
        except Exception:
            return False
        dense = np.asarray(dense)
        labels = np.asarray(labels)
        offs = [np.asarray(o) for o in offsets]
        idx = [np.asarray(i) for i in indices]
        ws = None if weights is None else [None if w is None else np.asarray(w) for w in weights]
        ok = (dense.dtype == np.float64 and dense.ndim == 2 and dense.strides[1] == 8
              and dense.shape == (self.B, self.k0) and labels.dtype == np.float64
              and labels.shape == (self.B,) and labels.strides[0] == 8
              and all(o.dtype == np.int64 and o.flags.c_contiguous and o.shape == (self.B + 1,)
                      for o in offs)
              and all(i.dtype == np.int64 and i.flags.c_contiguous for i in idx)
              and (ws is None or all(w is None or (w.dtype == np.float64 and w.flags.c_contiguous)
                                     for w in ws)))
        if not ok:
            return False
        T = self.T
        p = lambda arr: arr.ctypes.data
        sec = np.array([self.sections["x"][0], self.sections["labels"][0],
                        self.sections["offsets"][0], self.sections["indices"][0],
                        self.sections["iweights"][0] if self.weighted else -1], np.int64)
        P = C.c_void_p * T
        optr = P(*[p(o) for o in offs])
        iptr = P(*[p(i) if i.size else 0 for i in idx])
        nnz = np.array([i.shape[0] for i in idx], np.int64)
        wptr = P(*[p(w) if w is not None else 0 for w in ws]) if ws is not None else None
        rc = L.dlrm_pack_batch(C.c_void_p(blk.data_ptr()), C.c_void_p(p(sec)), self.B, self.k0,
                               _ceil4(self.k0), T, C.c_void_p(p(self.cap_base)),
                               C.c_void_p(p(dense)), dense.strides[0] // 8, C.c_void_p(p(labels)),
                               C.cast(optr, C.c_void_p), C.cast(iptr, C.c_void_p),
                               C.c_void_p(p(nnz)),
                               C.cast(wptr, C.c_void_p) if wptr is not None else None,
                               int(max(1, threads)))
        return rc == 0

    def new_host_block(self) -> torch.Tensor:
        blk = torch.zeros(self.nbytes, dtype=torch.uint8).pin_memory()
        if self.weighted:
            self.views(blk)["iweights"].fill_(1.0)
        return blk


# ----------------------------------------------------------------------------
# staged-batch handles (what a Prefetcher yields in place of the arrays)

_STAGE_NATIVE = os.environ.get("DLRM_PF_NATIVE", "1") != "0"


class _Slot:
    def __init__(self, layout: InputLayout, device):
        self.host = layout.new_host_block()
        self.dev = torch.empty(layout.nbytes, dtype=torch.uint8, device=device)
        self.h2d_done = torch.cuda.Event()   # host block may be repacked
        self.ready = torch.cuda.Event()      # device block holds the batch
        self.consumed = torch.cuda.Event()   # the step copied it out
        self.consumed_set = False
        # CUDA events exist once recorded (torch creates them lazily): the
        # native stager records into their handles
        s = torch.cuda.current_stream(device)
        self.h2d_done.record(s)
        self.ready.record(s)
        self.consumed.record(s)
        self.nnz = np.zeros(layout.T, dtype=np.int64)


class StagedDense:
    """Stands for the dense rows of a staged batch (``shape`` like the array)."""

    def __init__(self, slot: _Slot, layout: InputLayout, pf: "Prefetcher"):
        self._slot, self._layout, self._pf = slot, layout, pf
        self.shape = (layout.B, layout.k0)

    def consume(self, engine_block: torch.Tensor, stream=None):
        """Copy the landed block into the engine's input block on ``stream``
        (after the H2D copy) and release the ring slot."""
        s = stream or torch.cuda.current_stream()
        # wait for the H2D, copy, record `consumed`: one native call
        _lib.call("dlrm_d2d_async", _lib.ptr(engine_block), _lib.ptr(self._slot.dev),
                  self._layout.nbytes, self._slot.ready, self._slot.consumed,
                  _lib.stream_handle(s))
        self._slot.consumed_set = True
        self._pf._release(self._slot)


class StagedSparse:
    """Stands for one table's SparseBatch of a staged batch (the attributes
    train_step validates: segments, nnz, weights)."""

    def __init__(self, num_segments: int, nnz: int, weighted: bool):
        self.num_segments, self.nnz = num_segments, nnz
        self.weights = True if weighted else None


class StagedLabels:
    def __init__(self, n):
        self.shape = (n,)


class Prefetcher:
    """Iterate ``(dense_x, batches, labels)`` staged handles over host batches.

    ``source`` yields ``(dense, offsets_list, indices_list, labels)`` numpy
    tuples, or objects with those attributes (``rng.HostBatch``).
    ``capacities`` bounds each table's index count (the layout is static so
    the step engine can replay one CUDA graph); default: the largest count of
    the first batch + 25%.  ``depth`` ring slots are in flight; ``workers``
    threads pack consecutive batches concurrently (each with ``threads``
    native threads) and the batches are handed out in source order."""

    def __init__(self, source, batch_size: int, num_tables: int, dense_dim: int,
                 capacities=None, depth: int = 3, threads: int = 4, weighted: bool = False,
                 device=None, workers: int = 2):
        self._src = iter(source)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self._first = None
        if capacities is None:
            self._first = self._next_host()
            if self._first is None:
                raise ValueError("empty source")
            capacities = [max(batch_size, int(1.25 * np.asarray(i).shape[0]) + 1)
                          for i in self._first[2]]
        self.layout = InputLayout(batch_size, num_tables, dense_dim, capacities, weighted)
        self._pool = ThreadPoolExecutor(max(1, int(threads)))
        self._free = queue.Queue()
        nworkers = max(1, int(workers))
        for _ in range(max(2, int(depth), nworkers + 1)):
            self._free.put(_Slot(self.layout, self.device))
        # in-order hand-out: workers take (seq, batch) under _src_lock and
        # publish results keyed by seq; __next__ waits for the next seq
        self._src_lock = threading.Lock()
        self._cv = threading.Condition()
        self._done = {}
        self._seq_in = 0
        self._seq_out = 0
        self._end = None  # seq of the end-of-source marker
        self._stop = False
        self._workers = [threading.Thread(target=self._run, daemon=True) for _ in range(nworkers)]
        for w in self._workers:
            w.start()

    def _next_host(self):
        try:
            b = next(self._src)
        except StopIteration:
            return None
        if hasattr(b, "dense"):
            return (b.dense, b.offsets, b.indices, b.labels, getattr(b, "weights", None))
        return tuple(b) + ((None,) if len(b) == 4 else ())

    def _publish(self, seq, item):
        with self._cv:
            self._done[seq] = item
            self._cv.notify_all()

    def _stage_native(self, slot, stream, sh, dense, offs, idx, labels, weights) -> bool:
        """Pack + H2D + event records in one native call without the
        interpreter lock (libdlrmpy.so); False when unavailable or the arrays
        are not the reference's dtypes (then the Python path stages)."""
        PL = _lib.pylib() if _STAGE_NATIVE else None
        L = self.layout
        if PL is None or (weights is not None and any(w is not None for w in weights)
                          and not L.weighted):
            return False
        rc = PL.dlrm_pack_stage_py(
            dense, labels, offs, idx, weights, slot.host.data_ptr(), L._sec.ctypes.data, L.B,
            L.k0, _ceil4(L.k0), L.T, L._cap_base_ptr, int(self._pool._max_workers),
            slot.dev.data_ptr(), L.nbytes, slot.consumed if slot.consumed_set else None,
            slot.h2d_done, slot.ready, sh, slot.nnz.ctypes.data)
        if rc >= 2:
            L.check(idx, weights)  # raises the OverflowError
        return rc == 0

    def _run(self):
        torch.cuda.set_device(self.device)
        stream = torch.cuda.Stream(device=self.device)
        sh = _lib.stream_handle(stream)
        while not self._stop:
            slot = self._free.get()
            if slot is None:
                return
            with self._src_lock:
                seq = self._seq_in
                if self._end is not None:
                    self._free.put(slot)
                    return
                try:
                    hb = self._first if self._first is not None else self._next_host()
                except BaseException as e:  # surface source errors to the consumer
                    self._end = seq
                    self._seq_in += 1
                    self._free.put(slot)
                    self._publish(seq, e)
                    return
                self._first = None
                self._seq_in += 1
                if hb is None:
                    self._end = seq
                    self._free.put(slot)
                    self._publish(seq, None)
                    return
            try:
                slot.h2d_done.synchronize()             # the host block is free
                dense, offs, idx, labels, weights = hb
                if not self._stage_native(slot, stream, sh, dense, offs, idx, labels, weights):
                    if slot.consumed_set:
                        stream.wait_event(slot.consumed)   # the step copied it out
                    self.layout.pack(slot.host, dense, offs, idx, labels, weights, self._pool)
                    with torch.cuda.stream(stream):
                        slot.dev.copy_(slot.host, non_blocking=True)
                        slot.h2d_done.record(stream)
                        slot.ready.record(stream)
                    slot.nnz[:] = [int(np.asarray(i).shape[0]) for i in idx]
                self._publish(seq, (slot, slot.nnz.tolist(), weights is not None))
            except BaseException as e:
                self._free.put(slot)
                self._publish(seq, e)
                return

    def _release(self, slot):
        self._free.put(slot)

    def __iter__(self):
        return self

    def __next__(self):
        with self._cv:
            while self._seq_out not in self._done:
                self._cv.wait()
            item = self._done.pop(self._seq_out)
            if item is None or isinstance(item, BaseException):
                self._done[self._seq_out] = item  # stays at the end
            else:
                self._seq_out += 1
        if item is None:
            raise StopIteration
        if isinstance(item, BaseException):
            raise item
        slot, nnz, weighted = item
        L = self.layout
        dense = StagedDense(slot, L, self)
        return dense, [StagedSparse(L.B, n, weighted) for n in nnz], StagedLabels(L.B)

    def close(self):
        """Stop the workers and wait for them (a worker inside the native
        packer must not be torn down with the interpreter)."""
        self._stop = True
        for _ in self._workers:
            self._free.put(None)
        for w in self._workers:
            w.join(timeout=10.0)
        self._pool.shutdown(wait=False)
