"""Data-parallel training steps through the PRODUCT models with world size 2
(two processes sharing cuda:0, gloo on CUDA tensors): the group-aligned
gradient buckets the backward launches as each parameter group completes
(dp.GradAllReducer, overlapped with the rest of the backward) leave exactly
the sum of the per-replica gradients, and the SGD step applies the
replica-averaged gradient — the paper's DistDataParallel on
the reference's gradient semantics (autodiff.py:1363-1617).  EfficientNet-B0
adds SyncBN: every BatchNorm normalises over the global batch."""

import os
import socket
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LR = 0.05


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bert_inputs(rank):
    from paper_2110_10802_b200 import kernels as K

    B, S, H, NH = 2, 128, 768, 12
    g = torch.Generator().manual_seed(40 + rank)
    x = torch.randn(B * S, H, generator=g).bfloat16().cuda()
    dout = torch.randn(B * S, H, generator=g).bfloat16().cuda()
    am = torch.where(torch.rand(B, S, generator=g) < 0.1, -10000.0, 0.0).float().cuda()
    ka = K.pack_keep_bits((torch.rand(B, NH, S, S, generator=g) >= 0.1).to(torch.uint8).cuda())
    k1 = (torch.rand(B * S, H, generator=g) >= 0.1).to(torch.uint8).cuda()
    k2 = (torch.rand(B * S, H, generator=g) >= 0.1).to(torch.uint8).cuda()
    return x, am, ka, k1, k2, dout


def _bert(pg):
    from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig

    layer = BertEncoderLayer(BertLayerConfig(), device="cuda:0", seed=7)
    if pg is not None:
        layer.attach_process_group(pg)
    return layer


def _effnet(pg):
    from paper_2110_10802_b200.efficientnet import EfficientNetB0, EffNetConfig

    # f32: the comparison below isolates the data-parallel machinery from bf16
    # rounding (the last stages normalise 2x2 maps over a 4-image batch)
    m = EfficientNetB0(EffNetConfig(image=64, classes=40, width=0.25, dtype=torch.float32), device="cuda:0", seed=5,
                       process_group=pg)
    if pg is not None:  # small buckets: several group-aligned buckets even at width 0.25
        m.attach_process_group(pg, bucket_bytes=64 << 10)
    return m


def _effnet_inputs(rank, n=2):
    g = torch.Generator().manual_seed(60 + rank)
    x = torch.randn(n, 64, 64, 3, generator=g).cuda()
    lab = torch.randint(0, 40, (n,), generator=g, dtype=torch.int32).cuda()
    return x, lab


def _snap(m):
    return (m.grad.flat.double().cpu().numpy().copy(), m.master.flat.double().cpu().numpy().copy())


def _worker(rank, world, port, kind, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "bert":
            m = _bert(dist.group.WORLD)
            m.train_step(*_bert_inputs(rank), lr=LR)
        else:
            m = _effnet(dist.group.WORLD)
            m.train_step(*_effnet_inputs(rank), lr=LR)
        torch.cuda.synchronize()
        q.put((rank, _snap(m) + (m.reducer.launched, len(m.reducer.buckets))))
    except BaseException as e:  # surface the worker's error instead of a queue timeout
        import traceback

        q.put((rank, "ERROR: " + "".join(traceback.format_exception(e))))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["bert", "effnet"])
def test_overlapped_bucket_allreduce_matches_replica_sum(kind):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, v = q.get(timeout=600)
        if isinstance(v, str):  # a worker failed: the other one is stuck in a collective
            for p in procs:
                p.terminate()
            pytest.fail(v)
        res[r] = v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    if kind == "bert":
        # one replica per process, no collectives: per-shard gradients
        grads = []
        for r in range(2):
            m = _bert(None)
            m0 = m.master.flat.double().cpu().numpy().copy()
            m.train_step(*_bert_inputs(r), lr=None)
            torch.cuda.synchronize()
            grads.append(m.grad.flat.double().cpu().numpy().copy())
        tol = 1e-6
    else:
        # SyncBN couples the replicas: the reference is one process over the
        # concatenated batch (mean loss over 4 images = the average of the two
        # 2-image means), whose gradient x2 is the replica sum
        m = _effnet(None)
        m0 = m.master.flat.double().cpu().numpy().copy()
        xs, ls = zip(*[_effnet_inputs(r) for r in range(2)])
        m.train_step(torch.cat(xs), torch.cat(ls), lr=None)
        torch.cuda.synchronize()
        g1 = m.grad.flat.double().cpu().numpy()
        grads = [g1, g1]
        tol = 1e-3  # per-replica vs global-batch reduction orders (wgrad, BN sums)

    want = grads[0] + grads[1]
    scale = max(1.0, float(np.abs(want).max()))
    for r in range(2):
        g, master, launched, nb = res[r]
        assert launched == nb >= 4, (launched, nb)  # every bucket went out, group-aligned
        err = np.abs(g - want) / scale
        assert float(err.max()) <= tol, (kind, float(err.max()), int(err.argmax()))
        np.testing.assert_array_equal(g, res[0][0])  # replicas agree bitwise after the allreduce
        upd = m0 - LR * g / 2  # SGD on the replica-averaged gradient
        assert float(np.abs(master - upd).max()) <= 1e-6 * max(1.0, float(np.abs(upd).max()))
