"""Data-parallel runtime: gradient bucket allreduce and SyncBN collectives.

The paper's ``DistDataParallel`` inserts an allreduce after each weight
gradient (paper-only, SPEC.md:8 scopes it out of the
reference).  Here one process drives one GPU; gradients live in one flat f32
arena per model (bert.FlatArena), ordered so that the buckets at the front
complete first during the backward pass.  ``GradAllReducer`` splits the
arena into buckets aligned to parameter-group boundaries and all-reduces each
on a dedicated communication stream as soon as ``mark_ready(offset)`` says
the backward has produced everything below ``offset`` — so NCCL traffic over
NVLink overlaps the rest of the backward (bert.py / efficientnet.py call it
after each weight-gradient group; the whole step, collectives included, is
one CUDA graph under NCCL).  Averaging is folded into the optimizer's learning rate (no
extra pass over the gradients).

SyncBN (MBConv, BatchNormAct): the statistics kernels write each rank's
per-channel (count, mean, M2) straight into its slot of a [world, 3, C]
buffer and ``exchange_bn_sets`` all-gathers the slots in place, so every rank
merges them in rank order (dfx_bn_finalize);
``allreduce_sum`` combines the backward BN sums.  Both are tiny, latency-bound
messages.

Everything here is plain ``torch.distributed`` plumbing, so it runs on NCCL
(GPU) and on gloo (CPU tests, tests/test_dp_gloo.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class GradAllReducer:
    """Bucketed SUM-allreduce of a flat gradient arena, overlapped with the
    backward pass.

    ``boundaries`` (optional) are arena offsets at which the backward
    finishes a parameter group (the models order their arenas by gradient
    production, bert._param_specs / efficientnet.param_specs): buckets are
    then unions of whole groups of up to ``bucket_bytes``, so a bucket never
    waits on a group the backward has not reached.  Without boundaries the
    arena is cut every ``bucket_bytes``.

    ``mark_ready(offset, streams)``: everything in [0, offset) is final once
    the work queued so far on ``streams`` (the compute stream and the forked
    weight-gradient stream) has run; every bucket below ``offset`` is then
    all-reduced on the communication stream behind an event of each of those
    streams.  ``finish()`` launches the rest and joins the communication
    stream back into the current stream.  All of it is stream-ordered (no
    host waits on CUDA), so a whole step — backward, NCCL buckets, SGD — can
    be captured in one CUDA graph."""

    def __init__(self, flat: torch.Tensor, group=None, bucket_bytes: int = 25 << 20, boundaries=None):
        if flat.dim() != 1:
            raise ValueError("GradAllReducer: expects a flat 1-D gradient arena")
        self.flat = flat
        self.group = group
        self.world = dist.get_world_size(group)
        per = max(1, bucket_bytes // flat.element_size())
        n = flat.numel()
        if boundaries is None:
            self.buckets = [(o, min(o + per, n)) for o in range(0, n, per)]
        else:
            cuts = sorted({int(b) for b in boundaries if 0 < int(b) < n}) + [n]
            self.buckets, lo, prev = [], 0, 0
            for c in cuts:
                if c - lo > per and prev > lo:  # close the bucket at the previous group end
                    self.buckets.append((lo, prev))
                    lo = prev
                prev = c
            self.buckets.append((lo, n))
        self.cuda = flat.is_cuda
        self.stream = torch.cuda.Stream(device=flat.device) if self.cuda else None
        self.launched = 0  # collectives issued (bench / tests)
        self.reset()

    def reset(self):
        self.next = 0
        self.works = []

    def _launch(self, lo, hi, streams):
        view = self.flat[lo:hi]
        self.launched += 1
        if self.cuda:
            for s in streams or (torch.cuda.current_stream(self.flat.device),):
                ev = torch.cuda.Event()
                ev.record(s)  # gradients below `hi` were produced on these streams
                self.stream.wait_event(ev)
            with torch.cuda.stream(self.stream):
                self.works.append(dist.all_reduce(view, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(view, group=self.group, async_op=True))

    def mark_ready(self, offset: int, streams=None):
        """All gradient elements in [0, offset) are final (after the work
        queued so far on ``streams``): launch every bucket entirely below it."""
        while self.next < len(self.buckets) and self.buckets[self.next][1] <= offset:
            self._launch(*self.buckets[self.next], streams)
            self.next += 1

    def finish(self, streams=None):
        """Launch the remaining buckets and make the current stream wait for
        all of them.  Returns the world size (the gradient is a SUM)."""
        self.mark_ready(self.flat.numel(), streams)
        for w in self.works:
            w.wait()
        if self.cuda:
            torch.cuda.current_stream(self.flat.device).wait_stream(self.stream)
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


def bn_slot(sets: torch.Tensor, group=None) -> torch.Tensor:
    """This rank's [3, C] slot of a [world, 3, C] SyncBN set buffer: the
    statistics kernel writes its (count, mean, M2) straight into it, so the
    exchange below needs no staging copy."""
    return sets[dist.get_rank(group)]


def exchange_bn_sets(sets: torch.Tensor, group=None) -> torch.Tensor:
    """Complete a [world, 3, C] SyncBN set buffer whose own slot is filled:
    under NCCL one in-place all-gather (each rank's slot is the send buffer —
    no zeroing, no copy; a graph node like the gradient buckets); other
    backends (gloo, CPU tests) the rank-slotted all-reduce."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(sets, bn_slot(sets, group), group=group)
        return sets
    mine = bn_slot(sets, group).clone()
    return gather_bn_sets(mine, sets, group)


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
