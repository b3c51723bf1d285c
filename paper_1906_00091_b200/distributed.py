"""Hybrid parallelism on one box: embedding tables model-parallel (whole table
per GPU, the reference's ``partition_tables`` plan), bottom/top MLPs data-
parallel over contiguous batch shards (``shard_bounds``), a personalized
all-to-all of pooled embeddings forward and of their gradients backward, and
an MLP-gradient allreduce overlapped with the rest of the backward pass.

Reference: ``dlrmkit.parallel.ParallelTrainer.step`` (ref parallel.py:363-506)
simulates exactly this in one process (butterfly_shuffle 146-176,
inverse_shuffle 179-208, allreduce 211-224).  Here each rank is a process
with its own GPU:

    phase A  owner lookups over the GLOBAL batch -> sample-major send buffer
             [B_g, T_own, d] (rows of each destination shard are contiguous)
    a2a      all_to_all_single: rank r receives [src][b in shard r][T_own(src)][d]
    phase B  local bottom MLP, interaction reading features straight out of
             the receive buffer (per-feature pointer + stride), top MLP, loss
             head (gradient / global batch), backward into a flat gradient
             buffer; interaction backward writes feature gradients straight
             into the backward send buffer (same layout as the receive one)
    a2a      reverse all_to_all_single -> owner gets [B_g, T_own, d]
    allreduce  top-MLP gradients start as soon as the top backward is done
             (second communicator, overlaps interaction/bottom backward and
             the reverse a2a); bottom-MLP gradients after the bottom backward
    phase C  sorted sparse backward + SGD on owned tables; dense SGD on the
             (identical) MLP replicas

The exchange objects only move tensors, so they run unchanged over gloo on
CPU (tests/test_distributed_cpu.py, world_size 2); the kernels need the GPU.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from .embedding import LookupIndexError
from .model import DlrmModel, ceil4
from .parallel import DevicePlan, shard_bounds
from .trainer import INT64_MAX, StepResult

__all__ = ["ExchangeLayout", "NcclExchange", "LocalExchange", "RankEngine",
           "HybridTrainer"]


class ExchangeLayout:
    """Split sizes and feature addresses of the pooled-embedding exchange for
    one rank (pure index arithmetic — bit-exact with the reference plan)."""

    def __init__(self, plan: DevicePlan, rank: int, dim: int):
        plan.validate()
        self.plan, self.rank, self.d = plan, rank, dim
        G = plan.num_devices
        self.owned = [plan.owned(r) for r in range(G)]
        self.lo, self.hi = plan.shard(rank)
        self.B_local = self.hi - self.lo
        self.B_global = plan.batch_size
        T_me = len(self.owned[rank])
        self.T_own = T_me
        # forward: send rows [lo_r, hi_r) of my [B_g, T_me, d] buffer to r
        self.send_split = [(plan.shard(r)[1] - plan.shard(r)[0]) * T_me * dim
                           for r in range(G)]
        # forward: receive my shard of every source's owned tables
        self.recv_split = [self.B_local * len(self.owned[s]) * dim
                           for s in range(G)]
        self.recv_off = np.concatenate([[0], np.cumsum(self.recv_split)]).astype(np.int64)
        # table t -> (element offset in the receive buffer, row stride)
        self.feature = {}
        for s in range(G):
            Ts = len(self.owned[s])
            for j, t in enumerate(self.owned[s]):
                self.feature[t] = (int(self.recv_off[s]) + j * dim, Ts * dim)

    @property
    def send_numel(self) -> int:
        return self.B_global * self.T_own * self.d

    @property
    def recv_numel(self) -> int:
        return int(self.recv_off[-1])


class NcclExchange:
    """torch.distributed transport (NCCL on GPUs, gloo on CPU): the forward
    and reverse all-to-all and the allreduces, all on ONE communicator
    (``group``) — the trainer issues them in a fixed order on one stream.
    ``ar_group`` is accepted for compatibility and must be None or the same
    group."""

    def __init__(self, layout: ExchangeLayout, group=None, ar_group=None):
        import torch.distributed as dist
        if ar_group is not None and ar_group is not group:
            raise ValueError("all collectives share one communicator (ar_group must be None)")
        self.dist = dist
        self.L = layout
        self.group = group
        self.ar_group = group

    def forward(self, send: torch.Tensor, recv: torch.Tensor):
        self.dist.all_to_all_single(recv, send, self.L.recv_split,
                                    self.L.send_split, group=self.group)

    def backward(self, gsend: torch.Tensor, grecv: torch.Tensor):
        self.dist.all_to_all_single(grecv, gsend, self.L.send_split,
                                    self.L.recv_split, group=self.group)

    def allreduce_async(self, t: torch.Tensor):
        return self.dist.all_reduce(t, group=self.ar_group, async_op=True)

    def allreduce(self, t: torch.Tensor):
        self.dist.all_reduce(t, group=self.ar_group)


class LocalExchange:
    """In-process transport for G virtual ranks on one device (the
    reference's simulator semantics; used by ParallelTrainer)."""

    def __init__(self, layouts):
        self.layouts = layouts

    def forward_all(self, sends, recvs):
        G = len(self.layouts)
        for dst in range(G):
            off = 0
            for src in range(G):
                Ls = self.layouts[src]
                so = int(np.sum(Ls.send_split[:dst]))
                n = Ls.send_split[dst]
                recvs[dst][off:off + n].copy_(sends[src][so:so + n])
                off += n

    def backward_all(self, gsends, grecvs):
        G = len(self.layouts)
        for owner in range(G):
            Lo = self.layouts[owner]
            off = 0
            for src in range(G):
                Lsrc = self.layouts[src]
                n = Lo.send_split[src]
                so = int(Lsrc.recv_off[owner])
                grecvs[owner][off:off + n].copy_(gsends[src][so:so + n])
                off += n

    @staticmethod
    def allreduce_all(tensors):
        acc = tensors[0].clone()
        for t in tensors[1:]:
            acc += t
        for t in tensors:
            t.copy_(acc)


class RankEngine:
    """One rank's buffers and kernel sequence for the hybrid step.

    The model's MLP parameters are re-homed into a flat buffer (``params``)
    with a same-layout gradient buffer (``grads``); the rank's owned tables
    into one buffer ``W_own``.  Tables not owned by this rank are left alone.
    """

    def __init__(self, model: DlrmModel, layout: ExchangeLayout,
                 capacities=None, lr: float = 0.1, optimizer: str = "sgd",
                 eps: float = 1e-10, weighted: bool = False, force_exchange: bool = False):
        _lib.require_cuda()
        self.weighted = bool(weighted)
        cfg = model.config
        self.model, self.cfg, self.L = model, cfg, layout
        self.lr = float(lr)
        d = self.d = cfg.sparse_dim
        self.T = cfg.num_tables
        self.nf = self.T + 1
        Bl, Bg = self.Bl, self.Bg = layout.B_local, layout.B_global
        dev = self.dev = _lib.device()
        f32 = dict(dtype=torch.float32, device=dev)

        # parameters + gradients (flat, identical layout)
        self.layers = model.bottom.layers + model.top.layers
        self.Lb, self.Lt = len(model.bottom.layers), len(model.top.layers)
        n = sum(l.n_out * ceil4(l.n_in) + ceil4(l.n_out) for l in self.layers)
        self.params = torch.zeros(n, **f32)
        self.grads = torch.zeros(n, **f32)
        self.gslots = []
        off = 0
        for l in self.layers:
            nw = l.n_out * ceil4(l.n_in)
            w = self.params[off:off + nw].view(l.n_out, ceil4(l.n_in))
            gw = self.grads[off:off + nw].view(l.n_out, ceil4(l.n_in))
            off += nw
            b = self.params[off:off + l.n_out]
            gb = self.grads[off:off + l.n_out]
            off += ceil4(l.n_out)
            l.rebind(w, b)
            self.gslots.append((gw, gb))
        self.split_at = sum(l.n_out * ceil4(l.n_in) + ceil4(l.n_out)
                            for l in self.layers[:self.Lb])   # bottom | top

        # owned tables in one buffer
        own = layout.owned[layout.rank]
        self.own = own
        rows = [model.tables[t].num_rows for t in own]
        self.row_base = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
        self.total_rows = int(self.row_base[-1])
        self.W_own = torch.empty(max(self.total_rows, 1) * d, **f32)
        for j, t in enumerate(own):
            v = self.W_own[self.row_base[j] * d:self.row_base[j + 1] * d].view(rows[j], d)
            v.copy_(model.tables[t].weights)
            model.tables[t].weights = v
        To = len(own)
        caps = capacities if capacities is not None else [Bg] * To
        self.caps = [max(1, int(c)) for c in caps]
        self.cap_base = np.concatenate([[0], np.cumsum(self.caps)]).astype(np.int64)

        # inputs: ONE contiguous block [x | labels | offsets | indices
        # (| per-index weights)] so a
        # step's inputs move with one copy (pack() builds the same layout in
        # pinned host memory); x / labels / offsets / indices are views
        a16 = lambda n: (n + 15) // 16 * 16
        lay, o = {}, 0
        for name, nbytes in (("x", Bl * ceil4(cfg.dense_dim) * 4), ("labels", Bl * 4),
                             ("offsets", max(To, 1) * (Bg + 1) * 8),
                             ("indices", max(int(self.cap_base[-1]), 1) * 8),
                             ("iweights", max(int(self.cap_base[-1]), 1) * 4
                              if self.weighted else 0)):
            lay[name] = (o, nbytes)
            o = a16(o + nbytes)
        self.block_layout, self.block_bytes = lay, o
        self.block = torch.zeros(o, dtype=torch.uint8, device=dev)
        v = self._views(self.block)
        self.x, self.labels = v["x"], v["labels"]
        self.offsets, self.indices = v["offsets"], v["indices"]
        self.iweights = v["iweights"]
        if self.iweights is not None:
            self.iweights.fill_(1.0)

        # exchange buffers; with one rank the exchange is the identity (the
        # send layout [B_g, T, d] IS the receive layout), so they alias
        self.single = layout.plan.num_devices == 1 and not force_exchange
        self.send = torch.zeros(max(layout.send_numel, 1), **f32)
        self.recv = self.send if self.single else torch.zeros(max(layout.recv_numel, 1), **f32)
        self.gsend = torch.zeros(max(layout.recv_numel, 1), **f32)
        self.grecv = self.gsend if self.single else torch.zeros(max(layout.send_numel, 1), **f32)
        # one rank: no gradient exchange, so the update rule is fused into the
        # weight-gradient / head kernels exactly like the single-device step
        self.fuse_update = self.single

        # activations / gradients
        bl, tl = model.bottom.layers, model.top.layers
        self.bact = [torch.zeros((Bl, ceil4(l.n_out)), **f32) for l in bl]
        self.width = cfg.top_in_dim
        self.R = torch.zeros((Bl, ceil4(self.width)), **f32)
        self.tact = [torch.zeros((Bl, ceil4(l.n_out)), **f32) for l in tl[:-1]]
        self.prob = torch.zeros(Bl, **f32)
        self.glogit = torch.zeros(Bl, **f32)
        self.gtop = [torch.zeros((Bl, ceil4(l.n_out)), **f32) for l in tl[:-1]]
        self.gR = torch.zeros((Bl, ceil4(self.width)), **f32)
        self.gbot = [torch.zeros((Bl, ceil4(l.n_out)), **f32) for l in bl]

        # workspaces, step result [loss_sum, correct, err]
        self.emb_ws_bytes = _lib.size("dlrm_emb_bwd_workspace_size",
                                      max(int(self.cap_base[-1]), 1),
                                      max(self.total_rows, 1), d)
        self.emb_ws = torch.empty(self.emb_ws_bytes, dtype=torch.uint8, device=dev)
        lin = max(_lib.size("dlrm_linear_bwd_weight_workspace_size", Bl,
                            l.n_out, l.n_in) for l in self.layers)
        lin = max(lin, _lib.size("dlrm_head_bwd_workspace_size", Bl, tl[-1].n_in),
                  _lib.size("dlrm_bce_head_workspace_size", Bl),
                  _lib.size("dlrm_head_step_workspace_size", Bl, tl[-1].n_in))
        self.head_fused = tl[-1].n_in % 4 == 0 and tl[-1].n_in <= 1024 and \
            os.environ.get("DLRM_HEAD_FUSED", "1") != "0"
        self.lin_ws_bytes = lin
        self.lin_ws = torch.empty(lin, dtype=torch.uint8, device=dev)
        self.lin_ws2 = torch.empty(lin, dtype=torch.uint8, device=dev)  # main-stream wgrad
        self.stats = torch.zeros(3, **f32)
        self.err_pos = torch.empty(max(To, 1), dtype=torch.int64, device=dev)
        self.err_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.err_val = torch.zeros(max(To, 1), dtype=torch.int64, device=dev)
        # update rule (SGD / Adagrad with same-layout accumulators)
        from .optim import update_rule
        self.optimizer = optimizer
        # Adagrad: fp32 SIMT GEMMs (see _lib.accurate_gemms)
        self.accurate = optimizer == "adagrad" and os.environ.get("DLRM_ADAGRAD_TC") != "1"
        if optimizer == "adagrad":
            self.params_acc = torch.zeros_like(self.params)
            self.W_acc = torch.zeros_like(self.W_own)
            self.upd_mlp = update_rule("adagrad", self.lr, eps, self.params, self.params_acc)
            self.upd_emb = update_rule("adagrad", self.lr, eps, self.W_own, self.W_acc)
        elif optimizer == "sgd":
            self.upd_mlp = self.upd_emb = update_rule("sgd", self.lr)
        else:
            raise ValueError(f"unknown optimizer: {optimizer!r}")
        # weights' TF32 low parts for the tensor-core GEMMs, refreshed at the
        # start of every step (as trainer.StepEngine)
        self.use_wlo = not self.accurate and os.environ.get("DLRM_GEMM_WLO", "1") != "0"
        self.params_lo = torch.zeros_like(self.params) if self.use_wlo else None
        self._build_descs()

    def _wlo(self, l):
        if not self.use_wlo:
            return None
        return C.c_void_p(self.params_lo.data_ptr() +
                          (l.storage.data_ptr() - self.params.data_ptr()))

    def _build_descs(self):
        d, L = self.d, self.L
        To = len(self.own)
        descs = [_lib.TableDesc(
            self.offsets[j].data_ptr(), self.indices.data_ptr() + 8 * int(self.cap_base[j]),
            (self.iweights.data_ptr() + 4 * int(self.cap_base[j])) if self.weighted else None,
            int(self.row_base[j]), self.model.tables[t].num_rows, j * d,
            self.caps[j], self.model.tables[t].table_id) for j, t in enumerate(self.own)]
        self._descs = _lib.table_array(descs) if descs else None
        feats = [(self.bact[-1].data_ptr(), self.bact[-1].stride(0))]
        gfeats = [(self.gbot[-1].data_ptr(), self.gbot[-1].stride(0))]
        for t in range(self.T):
            off, stride = L.feature[t]
            feats.append((self.recv.data_ptr() + 4 * off, stride))
            gfeats.append((self.gsend.data_ptr() + 4 * off, stride))
        self._feats = _lib.make_features(feats)
        self._gfeat = (C.c_void_p * self.nf)(*[p for p, _ in gfeats])
        self._gstride = (C.c_int64 * self.nf)(*[s for _, s in gfeats])

    def _views(self, blk):
        lay, To = self.block_layout, max(len(self.own), 1)

        def view(name, dtype, shape):
            o, n = lay[name]
            if n == 0:
                return None
            return blk[o:o + n].view(dtype).view(*shape)
        return {"x": view("x", torch.float32, (self.Bl, ceil4(self.cfg.dense_dim))),
                "labels": view("labels", torch.float32, (self.Bl,)),
                "offsets": view("offsets", torch.int64, (To, self.Bg + 1)),
                "indices": view("indices", torch.int64, (max(int(self.cap_base[-1]), 1),)),
                "iweights": view("iweights", torch.float32, (max(int(self.cap_base[-1]), 1),))}

    def _check_weights(self, weights_owned):
        if weights_owned is not None and any(w is not None for w in weights_owned) \
                and not self.weighted:
            raise ValueError("weighted bags need a RankEngine built with weighted=True")

    def pack(self, dense_local, labels_local, offsets_owned, indices_owned,
             weights_owned=None):
        """This rank's batch in the input-block layout, in pinned host memory
        (done once per batch by the data pipeline)."""
        self._check_weights(weights_owned)
        blk = torch.zeros(self.block_bytes, dtype=torch.uint8).pin_memory()
        v = self._views(blk)
        v["x"][:, :self.cfg.dense_dim].copy_(torch.as_tensor(np.asarray(dense_local, np.float32)))
        v["labels"].copy_(torch.as_tensor(np.asarray(labels_local, np.float32)))
        for j in range(len(self.own)):
            i = np.asarray(indices_owned[j], np.int64)
            if i.size > self.caps[j]:
                raise OverflowError(f"table {self.own[j]}: {i.size} indices exceed "
                                    f"capacity {self.caps[j]}")
            v["offsets"][j].copy_(torch.as_tensor(np.asarray(offsets_owned[j], np.int64)))
            cb = int(self.cap_base[j])
            v["indices"][cb:cb + i.size].copy_(torch.as_tensor(i))
            if self.weighted:
                w = None if weights_owned is None else weights_owned[j]
                v["iweights"][cb:cb + i.size].copy_(
                    torch.ones(i.size) if w is None
                    else torch.as_tensor(np.asarray(w, np.float32)))
        return blk

    def stage(self, packed: torch.Tensor):
        """One copy of a packed block (pinned host or device) into the inputs."""
        self.block.copy_(packed, non_blocking=True)

    # ------------------------------------------------------------------
    def load(self, dense_local, labels_local, offsets_owned, indices_owned,
             weights_owned=None):
        """dense/labels: this rank's shard; offsets/indices (/ weights): one
        global-batch bag set per OWNED table (host arrays or device tensors)."""
        self._check_weights(weights_owned)
        # copy_ straight from the source: pinned host tensors move with an
        # async H2D copy on the current stream (no host synchronisation)
        def src(a, dtype):
            if isinstance(a, torch.Tensor):
                return a if a.dtype == dtype else a.to(dtype)
            return torch.as_tensor(np.asarray(a)).to(dtype)
        self.x[:, :self.cfg.dense_dim].copy_(src(dense_local, torch.float32), non_blocking=True)
        self.labels.copy_(src(labels_local, torch.float32), non_blocking=True)
        for j in range(len(self.own)):
            i = indices_owned[j]
            n = int(i.shape[0])
            if n > self.caps[j]:
                raise OverflowError(f"table {self.own[j]}: {n} indices exceed "
                                    f"capacity {self.caps[j]}")
            self.offsets[j].copy_(src(offsets_owned[j], torch.int64), non_blocking=True)
            cb = int(self.cap_base[j])
            self.indices[cb:cb + n].copy_(src(i, torch.int64), non_blocking=True)
            if self.weighted:
                w = None if weights_owned is None else weights_owned[j]
                if w is None:
                    self.iweights[cb:cb + n].fill_(1.0)
                else:
                    self.iweights[cb:cb + n].copy_(src(w, torch.float32), non_blocking=True)

    # ------------------------------------------------------------------
    def phase_a(self, stream=None):
        """Error reset + owner lookups over the global batch -> send buffer."""
        s = _lib.stream_handle(stream)
        P = _lib.ptr
        To = len(self.own)
        _lib.call("dlrm_err_reset", P(self.err_pos), max(To, 1), P(self.err_flag), s)
        if To:
            _lib.call("dlrm_emb_fwd", P(self.W_own), self.d,
                      C.cast(self._descs, C.c_void_p), To, self.Bg, P(self.send),
                      To * self.d, P(self.err_pos), P(self.err_flag), s)

    def phase_b_bottom_forward(self, stream=None):
        """Bottom MLP forward of the local samples (independent of the
        lookups and the exchange, so the trainer runs it beside them)."""
        s = _lib.stream_handle(stream)
        P, call, L = _lib.ptr, _lib.call, self.layers
        Bl, relu = self.Bl, _lib.ACT["relu"]
        if self.use_wlo:  # ordered before the top MLP by the trainer's events
            call("dlrm_tf32_split_lo", P(self.params), P(self.params_lo), self.params.numel(), s)
        a, lda = self.x, self.x.stride(0)
        for i in range(self.Lb):
            l, out = L[i], self.bact[i]
            call("dlrm_linear_fwd", P(a), lda, P(l.storage), l.ldw, P(l.bias),
                 P(out), out.stride(0), Bl, l.n_out, l.n_in, out.shape[1], relu, s)
            a, lda = out, out.stride(0)

    def phase_b_forward(self, stream=None, bottom=True):
        """(Bottom MLP forward unless ``bottom=False``,) interaction, top
        MLP forward and the loss head."""
        s = _lib.stream_handle(stream)
        P, call, L = _lib.ptr, _lib.call, self.layers
        Bl, relu = self.Bl, _lib.ACT["relu"]
        if bottom:
            self.phase_b_bottom_forward(stream)
        call("dlrm_interact_fwd", C.c_void_p(C.addressof(self._feats)), self.nf,
             self.d, Bl, P(self.R), self.R.stride(0), self.R.shape[1], s)
        a, lda = self.R, self.R.stride(0)
        for i in range(self.Lt - 1):
            l, out = L[self.Lb + i], self.tact[i]
            call("dlrm_linear_fwd_wlo", P(a), lda, P(l.storage), self._wlo(l), l.ldw,
                 P(l.bias), P(out), out.stride(0), Bl, l.n_out, l.n_in, out.shape[1], relu, s)
            a, lda = out, out.stride(0)
        head = L[-1]
        if self.head_fused:
            # the loss head's forward AND backward in one pass (same kernels
            # as the fused single-device step): prob, the logit gradient, the
            # loss statistics, dA for the top backward and the head's dw / db
            gw, gb = self.gslots[-1]
            ga = self.gtop[-1] if self.Lt > 1 else self.gR
            if self.fuse_update:
                call("dlrm_head_step", P(a), lda, P(head.storage), P(head.bias), Bl,
                     head.n_in, P(self.labels), float(self.Bg), P(self.prob), P(self.glogit),
                     P(self.stats), P(ga), ga.stride(0), 1 if self.Lt > 1 else 0, None, None,
                     P(head.storage), P(head.bias), C.byref(self.upd_mlp), P(self.err_flag),
                     P(self.lin_ws), self.lin_ws_bytes, s)
            else:
                call("dlrm_head_step", P(a), lda, P(head.storage), P(head.bias), Bl,
                     head.n_in, P(self.labels), float(self.Bg), P(self.prob), P(self.glogit),
                     P(self.stats), P(ga), ga.stride(0), 1 if self.Lt > 1 else 0, P(gw), P(gb),
                     None, None, C.byref(self.upd_mlp), None, P(self.lin_ws),
                     self.lin_ws_bytes, s)
        else:
            call("dlrm_bce_head", P(a), lda, P(head.storage), P(head.bias), Bl,
                 head.n_in, P(self.labels), float(self.Bg), None, P(self.prob),
                 P(self.glogit), None, P(self.stats), P(self.lin_ws),
                 self.lin_ws_bytes, s)
        self._head_in = (a, lda)

    def _wgrad_call(self, li, gz, ldg, xin, ws, stream_handle):
        """Layer li's weight / bias gradient: into its allreduce slot, or
        (one rank) straight into the update rule, fused."""
        P, l = _lib.ptr, self.layers[li]
        if self.fuse_update:
            _lib.call("dlrm_linear_bwd_weight_upd", P(gz), ldg, P(xin), xin.stride(0), self.Bl,
                      l.n_out, l.n_in, None, 0, None, P(l.storage), l.ldw, P(l.bias),
                      C.byref(self.upd_mlp), P(self.err_flag), P(ws), self.lin_ws_bytes,
                      stream_handle)
            return
        gw, gb = self.gslots[li]
        _lib.call("dlrm_linear_bwd_weight", P(gz), ldg, P(xin), xin.stride(0), self.Bl,
                  l.n_out, l.n_in, P(gw), gw.stride(0), P(gb), None, 0, None, 0.0, None,
                  P(ws), self.lin_ws_bytes, stream_handle)

    def _wgrad(self, stream, wgrad_stream, li, gz, ldg, xin):
        """Weight gradient on ``wgrad_stream`` after the work issued so far
        on ``stream``, when given (else on ``stream``)."""
        if wgrad_stream is None:
            self._wgrad_call(li, gz, ldg, xin, self.lin_ws, _lib.stream_handle(stream))
            return
        ev = torch.cuda.Event()
        ev.record(stream if stream is not None else torch.cuda.current_stream())
        wgrad_stream.wait_event(ev)
        self._wgrad_call(li, gz, ldg, xin, self.lin_ws, _lib.stream_handle(wgrad_stream))

    def phase_b_top_backward(self, stream=None, wgrad_stream=None):
        """Top MLP backward; with ``wgrad_stream`` each weight gradient runs
        there beside the next data gradient (the caller joins it)."""
        s = _lib.stream_handle(stream)
        P, call, L = _lib.ptr, _lib.call, self.layers
        Bl = self.Bl
        a, lda = self._head_in
        head = L[-1]
        gw, gb = self.gslots[-1]
        ga = self.gtop[-1] if self.Lt > 1 else self.gR
        if not self.head_fused and self.fuse_update:
            call("dlrm_head_bwd_upd", P(a), lda, P(head.storage), P(self.glogit), Bl,
                 head.n_in, P(ga), ga.stride(0), 1 if self.Lt > 1 else 0, None, None,
                 P(head.storage), P(head.bias), C.byref(self.upd_mlp), P(self.err_flag),
                 P(self.lin_ws), self.lin_ws_bytes, s)
        elif not self.head_fused:
            call("dlrm_head_bwd", P(a), lda, P(head.storage), P(self.glogit), Bl,
                 head.n_in, P(ga), ga.stride(0), 1 if self.Lt > 1 else 0, P(gw),
                 P(gb), None, None, 0.0, None, P(self.lin_ws), self.lin_ws_bytes, s)
        for i in range(self.Lt - 2, -1, -1):
            li = self.Lb + i
            l = L[li]
            gz = self.gtop[i]
            xin = self.R if i == 0 else self.tact[i - 1]
            dx = self.gR if i == 0 else self.gtop[i - 1]
            mask = None if i == 0 else self.tact[i - 1]
            call("dlrm_linear_bwd_data_wlo", P(gz), gz.stride(0), P(l.storage), self._wlo(l),
                 l.ldw, P(mask), mask.stride(0) if mask is not None else 0, P(dx),
                 dx.stride(0), Bl, l.n_out, l.n_in, s)
            self._wgrad(stream, wgrad_stream, li, gz, gz.stride(0), xin)

    def phase_b_interaction_backward(self, stream=None):
        s = _lib.stream_handle(stream)
        _lib.call("dlrm_interact_bwd", C.c_void_p(C.addressof(self._feats)),
                  self.nf, self.d, self.Bl, _lib.ptr(self.gR), self.gR.stride(0),
                  C.cast(self._gfeat, C.c_void_p), C.cast(self._gstride, C.c_void_p),
                  1, s)

    def phase_b_bottom_backward(self, stream=None, wgrad_stream=None):
        s = _lib.stream_handle(stream)
        P, call, L = _lib.ptr, _lib.call, self.layers
        Bl = self.Bl
        for i in range(self.Lb - 1, -1, -1):
            l = L[i]
            gz = self.gbot[i]
            xin = self.x if i == 0 else self.bact[i - 1]
            if i > 0:
                dx = self.gbot[i - 1]
                call("dlrm_linear_bwd_data_wlo", P(gz), gz.stride(0), P(l.storage),
                     self._wlo(l), l.ldw, P(self.bact[i - 1]), self.bact[i - 1].stride(0),
                     P(dx), dx.stride(0), Bl, l.n_out, l.n_in, s)
            if i == 0 and wgrad_stream is not None:
                # the first layer's weight gradient on the (then idle) calling
                # stream, beside the weight-gradient stream (own workspace)
                self._wgrad_call(i, gz, gz.stride(0), xin, self.lin_ws2, s)
            else:
                self._wgrad(stream, wgrad_stream, i, gz, gz.stride(0), xin)

    def publish_error(self):
        """stats[2] <- this rank's error flag (allreduced with the loss)."""
        self.stats[2].copy_(self.err_flag[0].to(torch.float32))

    def adopt_global_error(self):
        """err_flag <- any rank raised (after the stats allreduce)."""
        self.err_flag.copy_((self.stats[2:3] > 0).to(torch.int32))

    def prepare_sparse_backward(self, stream=None):
        """Index-only half of the sparse backward (keys + radix sort of the
        owned tables' lookups); valid as soon as the indices are loaded, so
        the trainer runs it on a side stream under the dense work."""
        To = len(self.own)
        if To:
            _lib.call("dlrm_emb_bwd_prepare", self.d, C.cast(self._descs, C.c_void_p), To,
                      self.Bg, self.total_rows, _lib.ptr(self.emb_ws), self.emb_ws_bytes,
                      _lib.stream_handle(stream))

    def resolve_errors(self, stream=None):
        """Offending index value per owned table (dlrm_err_resolve), read on
        the device from the batch that ran; ordered after the lookups."""
        To = len(self.own)
        if To:
            _lib.call("dlrm_err_resolve", C.cast(self._descs, C.c_void_p), To,
                      _lib.ptr(self.err_pos), _lib.ptr(self.err_flag),
                      _lib.ptr(self.err_val), _lib.stream_handle(stream))

    def apply_sparse(self, stream=None):
        """Owned tables: segmented fold of the received gradients + row SGD
        (skipped on device when err_flag is set)."""
        To = len(self.own)
        if To:
            P = _lib.ptr
            _lib.call("dlrm_emb_bwd_apply", P(self.W_own), self.d,
                      C.cast(self._descs, C.c_void_p), To, self.Bg, P(self.grecv),
                      To * self.d, C.byref(self.upd_emb), P(self.err_flag), self.total_rows,
                      P(self.emb_ws), self.emb_ws_bytes, _lib.stream_handle(stream))

    def sgd_dense(self, stream=None):
        """Dense update of the MLP replica from the allreduced gradients
        (nothing to do with one rank: the updates were fused)."""
        if self.fuse_update:
            return
        P = _lib.ptr
        _lib.call("dlrm_update_dense", P(self.params), P(self.grads),
                  self.params.numel(), C.byref(self.upd_mlp), P(self.err_flag),
                  _lib.stream_handle(stream))

    def phase_c(self, stream=None, prepared=False):
        To = len(self.own)
        if To and not prepared:
            self.prepare_sparse_backward(stream)
        self.apply_sparse(stream)
        self.sgd_dense(stream)

    def local_error(self):
        """(table_id, position, index, rows) of this rank's first bad index."""
        if not int(self.err_flag.item()):
            return None
        pos = self.err_pos.cpu().numpy()
        val = self.err_val.cpu().numpy()
        for j, t in enumerate(self.own):
            if pos[j] != INT64_MAX:
                tab = self.model.tables[t]
                return tab.table_id, int(pos[j]), int(val[j]), tab.num_rows
        return None


class HybridTrainer:
    """One process per GPU: ``torchrun --nproc-per-node G``.  All ranks build
    the same model (same seed) and the same plan; rank r keeps the tables the
    plan assigns to it and an MLP replica."""

    def __init__(self, model: DlrmModel, plan: DevicePlan, rank: int,
                 capacities=None, lr: float = 0.1, group=None, ar_group=None,
                 optimizer: str = "sgd", eps: float = 1e-10, weighted: bool = False,
                 force_exchange: bool = False):
        # force_exchange: run the collectives (and the unfused updates) even
        # with one rank — tests the multi-rank code path on one GPU
        self.layout = ExchangeLayout(plan, rank, model.config.sparse_dim)
        self.engine = RankEngine(model, self.layout, capacities, lr, optimizer, eps,
                                 weighted, force_exchange)
        self.ex = NcclExchange(self.layout, group, ar_group)
        self.rank = rank
        self.comm_stream = torch.cuda.Stream()
        self.side = torch.cuda.Stream()
        self.fwd_stream = torch.cuda.Stream()  # bottom MLP forward
        self.wg_stream = torch.cuda.Stream()   # weight gradients + their allreduces
        self.graph = None

    def load(self, *args):
        self.engine.load(*args)

    def pack(self, *args):
        return self.engine.pack(*args)

    def stage(self, packed):
        self.engine.stage(packed)

    def capture(self):
        """Record the step (both all-to-alls and the allreduces included:
        NCCL collectives are graph-capturable) into a CUDA graph; later
        ``step()`` calls replay it.  Every rank must capture, and then replay
        in lockstep.  Returns False (and keeps eager steps) if capture fails."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        try:
            with _lib.capture_guard(), torch.cuda.graph(g, capture_error_mode="thread_local"):
                self._issue()
        except Exception:
            self.graph = None
            torch.cuda.synchronize()
            return False
        self.graph = g
        return True

    def step(self, sync: bool = True):
        """One hybrid training step.  ``sync=False`` issues the whole step
        without any host synchronisation (ranks skip their updates on device
        if any rank saw a bad index) and returns None; call
        ``check_errors()`` / ``result()`` later to raise / read it."""
        if self.graph is not None:
            self.graph.replay()
        else:
            self._issue()
        if not sync:
            return None
        self.check_errors()
        return self.result()

    def _issue(self):
        with _lib.accurate_gemms(self.engine.accurate):
            self._issue_step()

    def _issue_step(self):
        e, ex = self.engine, self.ex
        cur = torch.cuda.current_stream()
        comm, wg, side = self.comm_stream, self.wg_stream, self.side
        mark = self._mark
        single = e.single
        # keys + sort of the owned lookups on the side stream from the start
        fork = mark(cur)
        side.wait_event(fork)
        e.prepare_sparse_backward(side)
        # bottom MLP forward beside the owner lookups and the exchange
        self.fwd_stream.wait_event(fork)
        e.phase_b_bottom_forward(self.fwd_stream)
        bot = mark(self.fwd_stream)
        e.phase_a()
        # Every collective of the step runs on ONE stream over ONE
        # communicator, issued in the same order on every rank: forward
        # all-to-all, loss statistics, reverse all-to-all, top-MLP gradients,
        # bottom-MLP gradients — no two communicators are ever in flight
        # together for NCCL to deadlock on.  Events tie them to the compute
        # streams, so they still overlap the backward pass.  One rank: the
        # exchanges are the identity and the updates are fused (no collective).
        if not single:
            comm.wait_event(mark(cur))
            with torch.cuda.stream(comm):
                ex.forward(e.send, e.recv)
            cur.wait_event(mark(comm))
        cur.wait_event(bot)
        e.phase_b_forward(bottom=False)
        # loss, correct count and this rank's index-error flag are known after
        # the head; the reduced flag gates every update (on device).  One
        # rank: the flag is only reported, published off the critical path
        # (side stream, after the apply) instead
        if not single:
            e.publish_error()
        if not single:
            comm.wait_event(mark(cur))
            with torch.cuda.stream(comm):
                ex.allreduce(e.stats)
                e.adopt_global_error()
        e.phase_b_top_backward(wgrad_stream=wg)
        top_grads = (mark(wg), mark(cur))
        e.phase_b_interaction_backward()
        if not single:
            comm.wait_event(mark(cur))
            with torch.cuda.stream(comm):
                ex.backward(e.gsend, e.grecv)
            got = mark(comm)
            for ev in top_grads:
                comm.wait_event(ev)
            with torch.cuda.stream(comm):
                ex.allreduce(e.grads[e.split_at:])
        else:
            got = mark(cur)
        # owned-table fold + row update on the side stream, concurrently with
        # the bottom MLP backward
        side.wait_event(got)
        e.apply_sparse(side)
        e.resolve_errors(side)
        if single:
            with torch.cuda.stream(side):
                e.publish_error()
        applied = mark(side)
        e.phase_b_bottom_backward(wgrad_stream=wg)
        if not single:
            comm.wait_event(mark(wg))
            comm.wait_event(mark(cur))
            with torch.cuda.stream(comm):
                ex.allreduce(e.grads[:e.split_at])
            cur.wait_event(mark(comm))
            e.sgd_dense()
        else:
            cur.wait_event(mark(wg))   # the fused updates of the weight gradients
        cur.wait_event(applied)

    @staticmethod
    def _mark(stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    def check_errors(self):
        """Raise for the last step if any rank saw an out-of-range index
        (synchronises with the device)."""
        e = self.engine
        if float(e.stats[2].item()) > 0:
            err = e.local_error()
            if err is not None:
                raise LookupIndexError(*err)
            raise RuntimeError("a peer rank reported an out-of-range index")

    def result(self) -> StepResult:
        """StepResult of the last step (loss / accuracy over the global
        batch; synchronises with the device)."""
        e = self.engine
        st = e.stats.cpu()
        return StepResult(float(st[0]) / e.Bg, float(st[1]) / e.Bg, e.prob.clone())
