"""CUDA-graph capture of a whole training step.

The reference runs one Python interpreter walk per step (interp.py:219-248);
the B200 path instead records the step's ~40 library launches once into a
CUDA graph and replays it, so the host launch path (ctypes + Python) is off
the critical path entirely.  All buffers the step touches are allocated
before capture; the library itself never allocates."""

from __future__ import annotations

import torch


class CapturedStep:
    """``fn`` runs ``warmup`` times eagerly (allocations, lazy kernel
    attributes), then once under capture.  ``preserve`` lists the tensors the
    step mutates as training state (parameter arenas, bf16 shadows, running
    statistics, ...): they are snapshotted before the warm-up and restored
    after it, so capturing applies no optimizer update and moves no
    statistics — the first replay is the first step."""

    def __init__(self, fn, warmup: int = 2, preserve=()):
        cur = torch.cuda.current_stream()
        saved = [t.clone() for t in preserve] if warmup else []
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(warmup):
                fn()
        cur.wait_stream(side)
        for t, s in zip(preserve, saved):
            t.copy_(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()
