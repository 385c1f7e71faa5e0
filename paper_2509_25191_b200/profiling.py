"""CUDA-event phase timer used by bench.py (events on the launching stream)."""
from __future__ import annotations

from collections import defaultdict
from contextlib import contextmanager

import torch

_active = None


class PhaseTimer:
    def __init__(self):
        self.events = defaultdict(list)

    @contextmanager
    def phase(self, name: str):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push(name)  # named ranges for nsys / ncu --nvtx
        s.record()
        try:
            yield
        finally:
            e.record()
            torch.cuda.nvtx.range_pop()
            self.events[name].append((s, e))

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for k, lst in self.events.items():
            ms = [s.elapsed_time(e) for s, e in lst]
            out[k] = {"count": len(ms), "total_ms": sum(ms), "avg_ms": sum(ms) / len(ms)}
        return out


def set_timer(t):
    global _active
    _active = t


@contextmanager
def phase(name: str):
    if _active is None:
        yield
    else:
        with _active.phase(name):
            yield
