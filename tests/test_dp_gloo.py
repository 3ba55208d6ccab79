"""World-size-2 gloo tests (CPU) of the data-parallel host logic: bucketed
gradient allreduce, the DP decomposition of the BERT layer gradient, and the
SyncBN statistics protocol."""

import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn), nprocs=world, join=True)


def _entry(rank, world, port, fn):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
    finally:
        dist.destroy_process_group()


def _bucket_case(rank, world):
    from paper_2110_10802_b200.dp import GradAllReducer

    n = 10_007
    flat = torch.arange(n, dtype=torch.float32) * (rank + 1)
    red = GradAllReducer(flat, bucket_bytes=4096)
    assert len(red.buckets) > 5
    red.mark_ready(3000)  # the backward produced the first 3000 elements
    assert red.next == 3000 // 1024
    w = red.finish()
    assert w == world
    want = torch.arange(n, dtype=torch.float32) * sum(r + 1 for r in range(world))
    assert torch.equal(flat, want)


def test_bucketed_allreduce():
    _run(_bucket_case)


def _bert_dp_case(rank, world):
    from golden_util import golden

    from oracle import oracle as O
    from paper_2110_10802_b200.dp import GradAllReducer

    g = golden("bert_layer_f64")
    B, S, NH = int(g["B"]), int(g["S"]), int(g["NH"])
    assert B == world
    prm = {k: g[k] for k in O.BERT_WEIGHTS}
    T = S
    sl = slice(rank * T, (rank + 1) * T)
    out, cache = O.bert_layer_fwd(prm, g["x"][sl], g["am"][rank:rank + 1], g["dm"][rank:rank + 1],
                                  g["m1"][sl], g["m2"][sl], 1, S, NH, float(g["eps"]))
    grads = O.bert_layer_bwd(prm, cache, g["dy"][sl])
    names = list(O.BERT_WEIGHTS)
    flat = torch.cat([torch.as_tensor(grads[k]).reshape(-1) for k in names]).double()
    GradAllReducer(flat, bucket_bytes=1 << 14).finish()
    off = 0
    for k in names:
        n = grads[k].size
        got = flat[off:off + n].numpy().reshape(grads[k].shape)
        off += n
        # shard gradients summed over ranks == the reference's full-batch gradient
        assert O.compare(got, g["d_" + k]) < 1e-9, k


def test_bert_data_parallel_decomposition():
    _run(_bert_dp_case)


def _syncbn_case(rank, world):
    from paper_2110_10802_b200.dp import gather_bn_sets, merge_bn_sets_reference

    rng = np.random.default_rng(0)
    z = rng.standard_normal((8, 5, 6, 6)) * 3 + 1.5  # the global batch
    mine = z[rank * 4:(rank + 1) * 4]
    ax = (0, 2, 3)
    local = torch.tensor(np.stack([np.full(5, mine[:, 0].size), mine.mean(ax),
                                   ((mine - mine.mean(ax, keepdims=True)) ** 2).sum(ax)]))
    out = torch.empty(world, 3, 5, dtype=local.dtype)
    gather_bn_sets(local, out)
    n, mean, m2 = merge_bn_sets_reference([out[r] for r in range(world)])
    np.testing.assert_allclose(mean.numpy(), z.mean(ax), rtol=1e-12)
    np.testing.assert_allclose((m2 / n).numpy(), z.var(ax), rtol=1e-12)  # biased variance


def test_syncbn_statistics_protocol():
    _run(_syncbn_case)


def _group_bucket_case(rank, world):
    from paper_2110_10802_b200.dp import GradAllReducer

    n = 1000
    flat = torch.ones(n) * (rank + 1)
    # parameter groups end at 100, 300, 350, 900; buckets of <= 300 elements
    red = GradAllReducer(flat, bucket_bytes=300 * 4, boundaries=[100, 300, 350, 900])
    assert red.buckets == [(0, 300), (300, 350), (350, 900), (900, 1000)], red.buckets
    red.mark_ready(120)  # first group done: its bucket still waits for the second group
    assert red.launched == 0
    red.mark_ready(350)
    assert red.launched == 2
    assert red.finish() == world and red.launched == 4
    assert torch.equal(flat, torch.full((n,), float(sum(r + 1 for r in range(world)))))


def test_group_aligned_buckets():
    _run(_group_bucket_case)


def _bn_exchange_case(rank, world):
    from paper_2110_10802_b200.dp import bn_slot, exchange_bn_sets

    sets = torch.full((world, 3, 5), -7.0)  # stale values in the other slots
    bn_slot(sets).copy_(torch.arange(15, dtype=torch.float32).reshape(3, 5) + 100 * rank)
    exchange_bn_sets(sets)
    for r in range(world):
        assert torch.equal(sets[r], torch.arange(15, dtype=torch.float32).reshape(3, 5) + 100 * r)


def test_bn_set_exchange_in_place():
    _run(_bn_exchange_case)
