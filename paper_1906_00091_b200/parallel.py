"""Device plan, collectives and the training-step drivers — the reference's
``dlrmkit.parallel`` API (ref ``pkg/src/dlrmkit/parallel.py``).

* ``partition_tables`` / ``shard_bounds`` / ``make_plan`` / ``DevicePlan``
  are integer bookkeeping and bit-identical to the reference.
* ``butterfly_shuffle`` / ``inverse_shuffle`` / ``allreduce`` keep the
  reference's in-process semantics (used by ``ParallelTrainer`` and tests);
  the real multi-GPU exchange over NCCL lives in ``distributed.py``.
* ``train_step`` is the single-device hot path: it runs the fused
  ``StepEngine`` (CUDA-graph replay after the first call).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .model import DlrmConfig, DlrmModel
from .optim import Sgd
from .pipeline import StagedDense
from .timing import NullTimer, add_seconds
from .trainer import StepEngine, StepResult

__all__ = [
    "DevicePlan", "ShuffleSlice", "CommLog", "StepResult", "partition_tables",
    "shard_bounds", "make_plan", "partition_tables_by_traffic", "butterfly_shuffle", "inverse_shuffle",
    "allreduce", "allreduce_max", "train_step", "evaluate", "format_comm_report",
    "ParallelTrainer",
]


# --------------------------------------------------------------------------
# device plan  (ref parallel.py:62-122)

@dataclass
class DevicePlan:
    num_devices: int
    table_assignment: list      # table id -> owning device
    shard_bounds: list          # len num_devices + 1, contiguous sample ranges

    def validate(self):
        if self.num_devices < 1:
            raise ValueError("need at least one device")
        if any(not 0 <= d < self.num_devices for d in self.table_assignment):
            raise ValueError("table assigned to a device outside the plan")
        b = self.shard_bounds
        if b[0] != 0 or any(x > y for x, y in zip(b, b[1:])):
            raise ValueError("shard bounds must start at 0 and be nondecreasing")
        sizes = [y - x for x, y in zip(b, b[1:])]
        if sizes and max(sizes) - min(sizes) > 1:
            raise ValueError("shard sizes must differ by at most 1")

    def shard(self, device: int):
        return self.shard_bounds[device], self.shard_bounds[device + 1]

    @property
    def batch_size(self) -> int:
        return self.shard_bounds[-1]

    def owned(self, device: int) -> list:
        return [t for t, d in enumerate(self.table_assignment) if d == device]


def partition_tables(table_sizes, num_devices: int) -> list:
    """Greedy largest-first, each table to the least-loaded device (lowest id
    on ties) — bit-identical to ref parallel.py:88-104."""
    if num_devices < 1:
        raise ValueError("need at least one device")
    loads = [0] * num_devices
    owner = [0] * len(table_sizes)
    for t in sorted(range(len(table_sizes)), key=lambda t: (-table_sizes[t], t)):
        dev = min(range(num_devices), key=lambda d: (loads[d], d))
        owner[t] = dev
        loads[dev] += table_sizes[t]
    return owner


def shard_bounds(batch_size: int, num_devices: int) -> list:
    """Contiguous shards, sizes differing by <= 1, earlier devices larger."""
    base, extra = divmod(batch_size, num_devices)
    out = [0]
    for d in range(num_devices):
        out.append(out[-1] + base + (1 if d < extra else 0))
    return out


def partition_tables_by_traffic(traffic, table_bytes, num_devices: int,
                                capacity_bytes: float | None = None) -> list:
    """Greedy heaviest-traffic-first: each table to the device with the least
    per-step traffic so far (ties: lowest id) among those whose memory can
    still hold it.  A table's owner pays for its lookups and for its pooled
    rows in the all-to-all every step, whatever its row count; the
    reference's size-balanced plan can give one GPU most of the (small)
    tables — 19 of 26 on one of 8 GPUs at the Criteo shapes — and with it
    most of the lookup and exchange work (SURVEY §7 hard part 5)."""
    if num_devices < 1:
        raise ValueError("need at least one device")
    if len(traffic) != len(table_bytes):
        raise ValueError("one traffic figure per table")
    load = [0.0] * num_devices
    mem = [0.0] * num_devices
    owner = [0] * len(traffic)
    for t in sorted(range(len(traffic)), key=lambda t: (-traffic[t], -table_bytes[t], t)):
        fits = [d for d in range(num_devices)
                if capacity_bytes is None or mem[d] + table_bytes[t] <= capacity_bytes]
        if not fits:
            raise ValueError(f"table {t} ({table_bytes[t]} bytes) fits on no device")
        dev = min(fits, key=lambda d: (load[d], d))
        owner[t] = dev
        load[dev] += traffic[t]
        mem[dev] += table_bytes[t]
    return owner


def make_plan(config: DlrmConfig, batch_size: int, num_devices: int,
              policy: str = "size", pooling=None, capacity_bytes: float | None = None
              ) -> DevicePlan:
    """The reference plan (``policy="size"``: greedy on table sizes,
    bit-identical to ref parallel.py:116-122) or ``policy="traffic"``:
    greedy on per-step traffic — lookups (``pooling[t]`` indices per bag,
    default 1) plus the pooled row exchanged — within ``capacity_bytes`` of
    table memory per device (default: no limit)."""
    d = config.sparse_dim
    sizes = [m * d for m in config.embedding_sizes]
    if policy == "size":
        owner = partition_tables(sizes, num_devices)
    elif policy == "traffic":
        pool = [1.0] * len(sizes) if pooling is None else [float(p) for p in pooling]
        if len(pool) != len(sizes):
            raise ValueError("one pooling factor per table")
        traffic = [batch_size * d * 4 * (p + 1.0) for p in pool]
        owner = partition_tables_by_traffic(traffic, [4.0 * x for x in sizes], num_devices,
                                            capacity_bytes)
    else:
        raise ValueError(f"unknown plan policy {policy!r}")
    plan = DevicePlan(num_devices, owner, shard_bounds(batch_size, num_devices))
    plan.validate()
    return plan


# --------------------------------------------------------------------------
# collectives, in-process semantics  (ref parallel.py:128-232)

@dataclass
class ShuffleSlice:
    source_device: int
    table_id: int
    sample_range: tuple
    values: torch.Tensor


@dataclass
class CommLog:
    """Per-step record of collective traffic: (step, name, bytes, parties)."""

    entries: list = field(default_factory=list)

    def add(self, step: int, collective: str, nbytes: int, participants: int):
        self.entries.append((step, collective, int(nbytes), participants))


def _nbytes(t) -> int:
    return int(t.numel() * t.element_size())


def butterfly_shuffle(per_table_outputs: dict, plan: DevicePlan,
                      comm: CommLog | None = None, step: int = 0) -> list:
    """Per-table full-batch pooled rows (on their owners) -> per-device
    all-table shards, ascending table id, tagged with the source device."""
    for t, m in per_table_outputs.items():
        if m.shape[0] != plan.batch_size:
            raise ValueError(f"table {t} output has {m.shape[0]} rows, plan "
                             f"expects {plan.batch_size}")
    if set(per_table_outputs) != set(range(len(plan.table_assignment))):
        raise ValueError("per-table outputs do not match the plan's tables")
    out = [[] for _ in range(plan.num_devices)]
    moved = 0
    for dst in range(plan.num_devices):
        lo, hi = plan.shard(dst)
        for t in sorted(per_table_outputs):
            src = plan.table_assignment[t]
            v = per_table_outputs[t][lo:hi]
            out[dst].append(ShuffleSlice(src, t, (lo, hi), v))
            if src != dst:
                moved += _nbytes(v)
    if comm is not None:
        comm.add(step, "butterfly_shuffle", moved, plan.num_devices)
    return out


def inverse_shuffle(per_device_grads: list, plan: DevicePlan,
                    comm: CommLog | None = None, step: int = 0) -> dict:
    """Per-device shard gradients -> full-batch gradient per table on its
    owner, shards concatenated in ascending device (= sample) order."""
    moved = 0
    full = {}
    for t in range(len(plan.table_assignment)):
        owner = plan.table_assignment[t]
        parts = []
        for dev in range(plan.num_devices):
            g = per_device_grads[dev][t]
            lo, hi = plan.shard(dev)
            if g.shape[0] != hi - lo:
                raise ValueError(f"device {dev} grad for table {t} has "
                                 f"{g.shape[0]} rows, shard is {hi - lo}")
            parts.append(g)
            if dev != owner:
                moved += _nbytes(g)
        full[t] = torch.cat(parts, dim=0)
    if comm is not None:
        comm.add(step, "grad_reverse_shuffle", moved, plan.num_devices)
    return full


def allreduce(per_replica: list):
    """Elementwise sum in ascending replica order."""
    if not per_replica:
        raise ValueError("allreduce needs at least one replica")
    shape = tuple(per_replica[0].shape)
    for i, m in enumerate(per_replica[1:], start=1):
        if tuple(m.shape) != shape:
            raise ValueError(f"replica {i} shape {tuple(m.shape)} != replica "
                             f"0 shape {shape}")
    out = per_replica[0].clone()
    for m in per_replica[1:]:
        out = out + m
    return out


def allreduce_max(per_replica: list):
    out = per_replica[0].clone()
    for m in per_replica[1:]:
        out = torch.maximum(out, m)
    return out


def format_comm_report(comm: CommLog) -> str:
    lines = ["step, collective, bytes, participants"]
    for step, name, nbytes, parts in comm.entries:
        lines.append(f"{step}, {name}, {nbytes}, {parts}")
    return "\n".join(lines) + "\n"


# --------------------------------------------------------------------------
# single-device training step  (ref parallel.py:250-287)

def _engine_for(model: DlrmModel, batch: int, batches, optimizer,
                weighted: bool, caps=None) -> StepEngine:
    """The model's cached step engine if it fits (batch, update rule,
    weighting, index capacities; ``caps``: exactly these capacities, the
    layout of a staged batch), else a new one."""
    eng = getattr(model, "_engine", None)
    nnz = [sb.nnz for sb in batches]
    kind = optimizer.name
    eps = float(getattr(optimizer, "eps", 1e-10))
    fits = (eng is not None and (caps is None or list(eng.caps) == list(caps))
            and all(n <= c for n, c in zip(nnz, eng.caps)))
    if (fits and eng.B == batch and eng.lr == float(optimizer.lr)
            and eng.optimizer == kind and (kind != "adagrad" or eng.eps == eps)
            and eng.weighted == weighted):
        if isinstance(optimizer, _EngineSpec):
            return eng
        _bind_optimizer(eng, optimizer, model)
        return eng
    if caps is None:
        caps = [max(n, batch) for n in nnz]
        if eng is not None:  # grow geometrically so graphs are rarely rebuilt
            caps = [max(c, int(1.25 * old)) for c, old in zip(caps, eng.caps)]
    old_owner = getattr(eng, "opt_owner", None) if eng is not None else None
    old_owner = old_owner() if old_owner is not None else None
    eng = StepEngine(model, batch, caps, lr=optimizer.lr, weighted=weighted,
                     optimizer=kind, eps=eps)
    # Adagrad: the optimiser's state (views of the previous engine's
    # accumulators when it drove that engine, restored arrays, or nothing)
    # seeds the new engine; another optimiser that drove the old engine keeps
    # a private copy.  Evaluation (_EngineSpec) carries the current owner over.
    src = None
    if kind == "adagrad":
        src = old_owner if isinstance(optimizer, _EngineSpec) else optimizer
        if old_owner is not None and old_owner is not src:
            _detach_adagrad(old_owner)
        if src is not None:
            _load_adagrad(eng, src, model)
    eng.eager_runs = 0
    model._engine = eng
    if src is not None:
        eng.opt_owner = weakref.ref(src)
        _mirror_adagrad(eng, src, model)
    return eng


def _detach_adagrad(opt):
    """Give an optimiser that no longer drives the step engine its own
    copies of the accumulators it was viewing."""
    from .optim import AdagradState
    opt._mlp_state = {k: AdagradState([a.clone() for a in st.mlp_weights],
                                      [a.clone() for a in st.mlp_biases])
                      for k, st in opt._mlp_state.items()}
    opt._table_state = {k: a.clone() for k, a in opt._table_state.items()}


def _load_adagrad(eng, opt, model):
    """Engine accumulators <- the optimiser's state (zero where it has none:
    a fresh Adagrad starts from zero sums, ref optim.py:112-140)."""
    from .checkpoint import _engine_adagrad_views
    eng.params_acc.zero_()
    eng.W_acc.zero_()
    views = _engine_adagrad_views(eng)
    for name in ("bottom", "top"):
        st = opt._mlp_state.get(name)
        for l, (aw, ab) in enumerate(zip(st.mlp_weights, st.mlp_biases) if st else []):
            views[f"{name}_w_{l}"].copy_(aw)
            views[f"{name}_b_{l}"].copy_(ab)
    for t, table in enumerate(model.tables):
        acc = opt._table_state.get(table.table_id)
        if acc is not None:
            views[f"table_{t}"].copy_(acc)


def _mirror_adagrad(eng, opt, model):
    """The optimiser's state becomes views of the engine's live accumulators
    (so checkpointing or a manual ``opt.apply`` sees what the fused step
    updated)."""
    from .checkpoint import _engine_adagrad_views
    from .optim import AdagradState
    views = _engine_adagrad_views(eng)
    for name, layers in (("bottom", model.bottom.layers), ("top", model.top.layers)):
        opt._mlp_state[name] = AdagradState(
            [views[f"{name}_w_{l}"] for l in range(len(layers))],
            [views[f"{name}_b_{l}"] for l in range(len(layers))])
    for t, table in enumerate(model.tables):
        opt._table_state[table.table_id] = views[f"table_{t}"]


def _bind_optimizer(eng, optimizer, model):
    """Adagrad accumulators belong to the optimiser OBJECT (as in the
    reference): when another Adagrad instance drives a cached engine, the
    previous one keeps a private copy and the engine loads the new one's
    state."""
    if optimizer.name != "adagrad":
        return
    ref = getattr(eng, "opt_owner", None)
    cur = ref() if ref is not None else None
    if cur is optimizer:
        return
    if cur is not None:
        _detach_adagrad(cur)
    _load_adagrad(eng, optimizer, model)
    eng.opt_owner = weakref.ref(optimizer)
    _mirror_adagrad(eng, optimizer, model)


def train_step(model: DlrmModel, dense_x, batches, labels, optimizer,
               timer=None, use_graph: bool = True, sync: bool = True) -> StepResult:
    """One forward/backward/SGD step over a mini-batch on the current GPU.

    Same contract as the reference: updates ``model`` in place and returns
    (loss, accuracy, probs); an out-of-range index raises LookupIndexError
    and leaves every parameter untouched.  ``sync=False`` returns as soon as
    the step is issued: the result's loss / accuracy (and a LookupIndexError
    of this step) materialise when first read, so the host can stage the
    next step while this one runs (``trainer.PendingStepResult``)."""
    if getattr(optimizer, "name", None) not in ("sgd", "adagrad"):
        raise ValueError(f"unsupported optimizer {optimizer!r}")
    cfg = model.config
    if len(batches) != cfg.num_tables:
        raise ValueError(
            f"got {len(batches)} sparse batches for {cfg.num_tables} tables")
    b = int(dense_x.shape[0])
    for t, sb in enumerate(batches):
        if sb.num_segments != b:
            raise ValueError(
                f"sparse batch {t} has {sb.num_segments} segments, batch is {b}")
    weighted = any(sb.weights is not None for sb in batches)
    if isinstance(dense_x, StagedDense):
        # a Prefetcher batch: already packed and on the device; one D2D copy
        # of its block into the engine's input set
        L = dense_x._layout
        eng = _engine_for(model, b, batches, optimizer, L.weighted, caps=L.caps)
        dense_x.consume(eng.input_sets[eng._set]["block"])
    else:
        eng = _engine_for(model, b, batches, optimizer, weighted)
        eng.load(dense_x, [sb.offsets for sb in batches],
                 [sb.indices for sb in batches], labels,
                 [sb.weights for sb in batches] if weighted else None)
    if timer is not None and (hasattr(timer, "seconds") or hasattr(timer, "add")) \
            and not isinstance(timer, NullTimer):
        # operator attribution (ref parallel.py:254-285): device time per
        # stage from CUDA events, credited to the reference's categories
        ms = eng.run_timed(use_graph)
        per = {c: 0.0 for c in ("bottom_mlp", "embedding_lookup", "interaction",
                                "top_mlp", "loss", "optimizer")}
        for stage, v in ms.items():
            per[eng.CATEGORY[stage]] += v / 1e3
        add_seconds(timer, per)
        return eng.result()
    if eng.graph is None and use_graph and eng.eager_runs >= 1:
        eng.capture()
    if eng.graph is not None:
        eng.graph.replay()
    else:
        eng.run()
        eng.eager_runs += 1
    return eng.result() if sync else eng.result_async()


class _EngineSpec:
    """Optimizer settings of an existing step engine (so evaluation reuses
    it instead of rebinding the model's parameters to a new one)."""

    def __init__(self, name, lr, eps):
        self.name, self.lr, self.eps = name, lr, eps


def evaluate(model: DlrmModel, eval_batches):
    """(mean per-sample BCE loss, accuracy) over ``(dense, sparse_batches,
    labels)`` triples — the reference's ``_evaluate`` (cli.py:542-552).

    Forward-only on the device through the model's step engine: lookups,
    interaction, MLP forwards and the loss head fused with the sigmoid; no
    backward, no update.  Each batch's loss sum / correct count come back as
    two floats; the totals accumulate in float64 on the host."""
    loss_sum, correct, total = 0.0, 0.0, 0
    for dense, batches, labels in eval_batches:
        cfg = model.config
        if len(batches) != cfg.num_tables:
            raise ValueError(
                f"got {len(batches)} sparse batches for {cfg.num_tables} tables")
        b = int(dense.shape[0])
        for t, sb in enumerate(batches):
            if sb.num_segments != b:
                raise ValueError(
                    f"sparse batch {t} has {sb.num_segments} segments, batch is {b}")
        weighted = any(sb.weights is not None for sb in batches)
        cur = getattr(model, "_engine", None)
        spec = (_EngineSpec(cur.optimizer, cur.lr, cur.eps) if cur is not None
                else _EngineSpec("sgd", 0.1, 1e-10))
        eng = _engine_for(model, b, batches, spec, weighted)
        eng.load(dense, [sb.offsets for sb in batches], [sb.indices for sb in batches],
                 labels, [sb.weights for sb in batches] if weighted else None)
        eng.run_eval()
        ls, c, _ = eng.eval_result()
        loss_sum += ls
        correct += c
        total += b
    if total == 0:
        raise ValueError("no evaluation batches")
    return loss_sum / total, correct / total


# --------------------------------------------------------------------------
# in-process hybrid-parallel simulator  (ref parallel.py:310-525)

class ParallelTrainer:
    """Replicated-MLP, partitioned-table trainer over ``plan.num_devices``
    virtual devices on the current GPU — the reference's simulator API, run
    through the same per-rank kernel sequence (``distributed.RankEngine``)
    as the multi-process ``HybridTrainer``, with the exchanges done as
    device copies.  Dense gradients are summed in ascending replica order.

    Unlike the reference (float64 grid reductions) the fp32 sum over shards
    is not partition-invariant, so results match serial training within
    tolerance, not bit for bit (SURVEY §7 hard part 6)."""

    def __init__(self, model: DlrmModel, plan: DevicePlan,
                 optimizer_name: str = "sgd", lr: float = 0.1,
                 eps: float = 1e-10, concurrent: bool = False,
                 capacities=None, weighted: bool = False):
        from .distributed import ExchangeLayout, LocalExchange, RankEngine
        if optimizer_name not in ("sgd", "adagrad"):
            raise ValueError(f"unknown optimizer: {optimizer_name!r}")
        plan.validate()
        if len(plan.table_assignment) != model.config.num_tables:
            raise ValueError("plan does not cover the model's tables")
        self.plan, self.config = plan, model.config
        self.tables = list(model.tables)
        G = plan.num_devices
        self.layouts = [ExchangeLayout(plan, r, model.config.sparse_dim)
                        for r in range(G)]
        self._spec = (optimizer_name, lr, eps, capacities)
        self.engines = []
        for r in range(G):
            replica = DlrmModel(model.config, model.bottom.copy(),
                                model.top.copy(), self.tables)
            self.engines.append(self._rank_engine(replica, r, weighted))
        self.ex = LocalExchange(self.layouts)
        self.comm = CommLog()
        self.step_count = 0
        self.concurrent = concurrent

    def _rank_engine(self, replica, r, weighted):
        from .distributed import RankEngine
        optimizer_name, lr, eps, capacities = self._spec
        own = self.layouts[r].owned[r]
        caps = None if capacities is None else [capacities[t] for t in own]
        return RankEngine(replica, self.layouts[r], caps, lr, optimizer_name, eps, weighted)

    def _rebuild(self, weighted):
        """New rank engines (other input layout) around the current replica
        parameters, tables and optimiser state."""
        old = self.engines
        self.engines = [self._rank_engine(e.model, r, weighted) for r, e in enumerate(old)]
        if self._spec[0] == "adagrad":
            for e, o in zip(self.engines, old):
                e.params_acc.copy_(o.params_acc)
                e.W_acc.copy_(o.W_acc)

    def close(self):
        pass

    def replica_params(self, device: int = 0):
        m = self.engines[device].model
        return m.bottom, m.top

    def max_replica_divergence(self) -> float:
        p0 = self.engines[0].params
        return max([float((e.params - p0).abs().max()) for e in self.engines[1:]],
                   default=0.0)

    def step(self, dense_x, batches, labels, timer=None) -> StepResult:
        # Adagrad: fp32 SIMT GEMMs (see _lib.accurate_gemms)
        with _lib.accurate_gemms(self.engines[0].accurate):
            return self._step(dense_x, batches, labels, timer)

    def _step(self, dense_x, batches, labels, timer=None) -> StepResult:
        plan = self.plan
        n_total = int(dense_x.shape[0])
        if n_total != plan.batch_size:
            raise ValueError(f"batch size {n_total} does not match plan "
                             f"({plan.batch_size})")
        G, step = plan.num_devices, self.step_count
        weighted = any(sb.weights is not None for sb in batches)
        if weighted and not self.engines[0].weighted:
            # per-index weights need the weighted input layout: rebuild the
            # rank engines around the current parameters once
            self._rebuild(weighted=True)
        for r, e in enumerate(self.engines):
            lo, hi = plan.shard(r)
            own = self.layouts[r].owned[r]
            e.load(dense_x[lo:hi], labels[lo:hi],
                   [batches[t].offsets for t in own],
                   [batches[t].indices for t in own],
                   [batches[t].weights for t in own] if weighted else None)
        sec = _Sections(timer)
        with sec("embedding_lookup"):
            for e in self.engines:
                e.phase_a()
                e.resolve_errors()
        with sec("shuffle"):
            self.ex.forward_all([e.send for e in self.engines],
                                [e.recv for e in self.engines])
        moved = sum(4 * n for r, L in enumerate(self.layouts)
                    for dst, n in enumerate(L.send_split) if dst != r)
        self.comm.add(step, "butterfly_shuffle", moved, G)
        with sec("device_compute"):
            for e in self.engines:
                e.phase_b_forward()
                e.phase_b_top_backward()
                e.phase_b_interaction_backward()
        with sec("shuffle"):
            self.ex.backward_all([e.gsend for e in self.engines],
                                 [e.grecv for e in self.engines])
        self.comm.add(step, "grad_reverse_shuffle", moved, G)
        with sec("device_compute"):
            for e in self.engines:
                e.phase_b_bottom_backward()
                e.publish_error()
        with sec("allreduce"):
            self.ex.allreduce_all([e.stats for e in self.engines])
            self.comm.add(step, "loss_gather", 12 * (G - 1), G)
            self.ex.allreduce_all([e.grads for e in self.engines])
            self.comm.add(step, "grad_allreduce",
                          2 * (G - 1) * 4 * self.engines[0].grads.numel(), G)
        with sec("embedding_lookup"):
            for e in self.engines:
                e.adopt_global_error()
                e.prepare_sparse_backward()
                e.apply_sparse()
        with sec("optimizer"):
            for e in self.engines:
                e.sgd_dense()
        sec.credit()
        if float(self.engines[0].stats[2].item()) > 0:
            for r, e in enumerate(self.engines):
                err = e.local_error()
                if err is not None:
                    from .embedding import LookupIndexError
                    raise RuntimeError(f"device {r}: {LookupIndexError(*err)}")
        self.step_count += 1
        st = self.engines[0].stats.cpu()
        probs = torch.cat([e.prob for e in self.engines])
        return StepResult(float(st[0]) / n_total, float(st[1]) / n_total, probs)


class _Sections:
    """Device time of named host-side sections (CUDA events on the current
    stream) credited to a StageTimer once the step is done."""

    def __init__(self, timer):
        self.on = timer is not None and not isinstance(timer, NullTimer) and \
            (hasattr(timer, "add") or hasattr(timer, "seconds"))
        self.timer, self.evs = timer, []

    def __call__(self, name):
        sections = self

        class _Ctx:
            def __enter__(self):
                if sections.on:
                    self.e0 = torch.cuda.Event(enable_timing=True)
                    self.e0.record()

            def __exit__(self, *exc):
                if sections.on and exc[0] is None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record()
                    sections.evs.append((name, self.e0, e1))
                return False
        return _Ctx()

    def credit(self):
        if not self.on or not self.evs:
            return
        self.evs[-1][2].synchronize()
        per = {}
        for name, a, b in self.evs:
            per[name] = per.get(name, 0.0) + a.elapsed_time(b) / 1e3
        add_seconds(self.timer, per)
