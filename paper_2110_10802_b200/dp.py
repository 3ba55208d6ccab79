"""Data-parallel runtime: gradient bucket allreduce and SyncBN collectives.

The paper's ``DistDataParallel`` inserts an allreduce after each weight
gradient (paper-only, SPEC.md:8 scopes it out of the
reference).  Here one process drives one GPU; gradients live in one flat f32
arena per model (bert.FlatArena), ordered so that the buckets at the front
complete first during the backward pass.  ``GradAllReducer`` splits the
arena into ~25 MB buckets and all-reduces each on a dedicated communication
stream as soon as ``mark_ready(offset)`` says the backward has produced
everything below ``offset`` — so NCCL traffic over NVLink overlaps the rest
of the backward.  Averaging is folded into the optimizer's learning rate (no
extra pass over the gradients).

SyncBN (MBConv): ``gather_bn_sets`` all-gathers each rank's per-channel
(count, mean, M2) so every rank merges them in rank order (mbconv.py);
``allreduce_sum`` combines the backward BN sums.  Both are tiny, latency-bound
messages.

Everything here is plain ``torch.distributed`` plumbing, so it runs on NCCL
(GPU) and on gloo (CPU tests, tests/test_dp_gloo.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class GradAllReducer:
    def __init__(self, flat: torch.Tensor, group=None, bucket_bytes: int = 25 << 20):
        if flat.dim() != 1:
            raise ValueError("GradAllReducer: expects a flat 1-D gradient arena")
        self.flat = flat
        self.group = group
        self.world = dist.get_world_size(group)
        per = max(1, bucket_bytes // flat.element_size())
        self.buckets = [(o, min(o + per, flat.numel())) for o in range(0, flat.numel(), per)]
        self.cuda = flat.is_cuda
        self.stream = torch.cuda.Stream(device=flat.device) if self.cuda else None
        self.reset()

    def reset(self):
        self.next = 0
        self.works = []

    def _launch(self, lo, hi):
        view = self.flat[lo:hi]
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record()  # gradients below `hi` were produced on the compute stream
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(ev)
                self.works.append(dist.all_reduce(view, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(view, group=self.group, async_op=True))

    def mark_ready(self, offset: int):
        """All gradient elements in [0, offset) are final: launch every bucket
        that lies entirely below ``offset``."""
        while self.next < len(self.buckets) and self.buckets[self.next][1] <= offset:
            self._launch(*self.buckets[self.next])
            self.next += 1

    def finish(self):
        """Launch the remaining buckets and make the compute stream wait for
        all of them.  Returns the world size (the gradient is a SUM)."""
        self.mark_ready(self.flat.numel())
        for w in self.works:
            w.wait()
        if self.cuda:
            torch.cuda.current_stream().wait_stream(self.stream)
        self.works = []
        self.next = 0
        return self.world


def gather_bn_sets(local: torch.Tensor, out: torch.Tensor, group=None) -> torch.Tensor:
    """local [3, C] (count, mean, M2) -> out [world, 3, C] in rank order.

    A rank-slotted allreduce (each rank writes its slot, zeros elsewhere; the
    sum is exact because every slot has one non-zero contributor): one NCCL
    allreduce, which gloo also supports on CUDA tensors and which can be
    captured in a CUDA graph like the gradient allreduce."""
    rank = dist.get_rank(group)
    out.zero_()
    out[rank].copy_(local)
    dist.all_reduce(out, group=group)
    return out


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    dist.all_reduce(t, group=group)
    return t


def merge_bn_sets_reference(sets):
    """Chan's parallel merge in rank order (host-side mirror of the CUDA
    bn_finalize merge, used by the CPU tests)."""
    n = sets[0][0].clone()
    mean = sets[0][1].clone()
    m2 = sets[0][2].clone()
    for s in sets[1:]:
        nb, mb, m2b = s[0], s[1], s[2]
        tot = n + nb
        d = mb - mean
        f = nb / tot
        m2 = m2 + m2b + d * d * n * f
        mean = mean + d * f
        n = tot
    return n, mean, m2
