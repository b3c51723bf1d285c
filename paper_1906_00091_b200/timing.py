"""Per-operator time attribution — the reference's ``dlrmkit.timing`` API
(ref ``pkg/src/dlrmkit/timing.py:9-36``).

``StageTimer.section(name)`` times host wall clock exactly like the
reference.  The training steps (``train_step``, ``ParallelTrainer.step``)
attribute DEVICE time instead: each stage is bracketed by CUDA events on the
stream it runs on and its milliseconds are added with ``add(name, seconds)``
under the reference's category names (ref parallel.py:254-285, 365-498):

    train_step        bottom_mlp, embedding_lookup, interaction, top_mlp,
                      loss, optimizer
    ParallelTrainer   embedding_lookup, shuffle, device_compute, loss,
                      allreduce, optimizer

The optimiser has no kernels of its own inside the fused step (updates run in
the weight-gradient and sparse-backward epilogues), so ``optimizer`` receives
0.0 there; its work is inside ``top_mlp`` / ``bottom_mlp`` /
``embedding_lookup``.
"""

from __future__ import annotations

import time
from contextlib import contextmanager

__all__ = ["StageTimer", "NullTimer", "add_seconds"]


class StageTimer:
    """Accumulates seconds per named operator category."""

    def __init__(self):
        self.seconds: dict[str, float] = {}

    @contextmanager
    def section(self, name: str):
        t0 = time.perf_counter()
        try:
            yield
        finally:
            self.add(name, time.perf_counter() - t0)

    def add(self, name: str, seconds: float) -> None:
        self.seconds[name] = self.seconds.get(name, 0.0) + float(seconds)

    def total(self) -> float:
        return sum(self.seconds.values())


class NullTimer:
    """No-op drop-in when profiling is disabled."""

    @contextmanager
    def section(self, name: str):
        yield

    def add(self, name: str, seconds: float) -> None:
        pass

    def total(self) -> float:
        return 0.0


def add_seconds(timer, per_category: dict) -> None:
    """Credit ``{category: seconds}`` to a StageTimer-like object: ``add`` if
    it has one, else its ``seconds`` dict (the reference's StageTimer)."""
    if timer is None:
        return
    for name, sec in per_category.items():
        if hasattr(timer, "add"):
            timer.add(name, sec)
        elif isinstance(getattr(timer, "seconds", None), dict):
            timer.seconds[name] = timer.seconds.get(name, 0.0) + float(sec)
