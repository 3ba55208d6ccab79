"""CUDA-graph capture of a whole training step.

The reference runs one Python interpreter walk per step (interp.py:219-248);
the B200 path instead records the step's ~40 library launches once into a
CUDA graph and replays it, so the host launch path (ctypes + Python) is off
the critical path entirely.  All buffers the step touches are allocated
before capture; the library itself never allocates."""

from __future__ import annotations

import torch


class CapturedStep:
    def __init__(self, fn, warmup: int = 2):
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(warmup):
                fn()
        cur.wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()
