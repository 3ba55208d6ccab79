"""SyncBN through the PRODUCT blocks with world size 2 (two processes sharing
cuda:0, gloo on CUDA tensors): MBConvBlock and BatchNormAct trained on two
UNEQUAL per-rank batches equal one process over the concatenated batch —
forward output, running statistics, input gradient, and the sum over ranks
of the parameter gradients (BatchNormalization over the global batch,
frontend.py:558-573; VJP autodiff.py:1557-1617)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPLIT = (3, 5)  # unequal per-rank batches (a last partial batch)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(kind):
    rng = np.random.default_rng(17)
    N = sum(SPLIT)
    if kind == "mbconv":
        x = rng.standard_normal((N, 12, 12, 32)).astype(np.float32)
        dy = rng.standard_normal((N, 12, 12, 32)).astype(np.float32)
    else:
        x = rng.standard_normal((N, 7, 9, 48)).astype(np.float32)
        dy = rng.standard_normal((N, 7, 9, 48)).astype(np.float32)
    return x, dy


def _model(kind, pg):
    if kind == "mbconv":
        from paper_2110_10802_b200.mbconv import MBConvBlock, MBConvConfig

        return MBConvBlock(MBConvConfig(channels=32, se=8, stride=1, pads=(1, 1, 1, 1), eps=1e-3, momentum=0.9,
                                        dtype=torch.float32), seed=3, process_group=pg)
    from paper_2110_10802_b200.norms import BatchNormAct

    m = BatchNormAct(48, eps=1e-5, momentum=0.9, act="swish", process_group=pg)
    g = torch.Generator().manual_seed(3)
    m.gamma.copy_(1 + 0.1 * torch.randn(48, generator=g))
    m.beta.copy_(0.1 * torch.randn(48, generator=g))
    return m


def _step(kind, m, x, dy):
    xt = torch.as_tensor(x).cuda().contiguous()
    y = m.forward(xt)
    dx = m.backward(torch.as_tensor(dy).cuda().contiguous())
    torch.cuda.synchronize()
    if kind == "mbconv":
        grads = {k: v.detach().cpu().double().numpy().copy() for k, v in m.grad.views.items()}
    else:
        grads = {"g": m.dgamma.cpu().double().numpy().copy(), "b": m.dbeta.cpu().double().numpy().copy()}
    return (y.cpu().double().numpy().copy(), dx.cpu().double().numpy().copy(), grads,
            m.running_mean.cpu().double().numpy().copy(), m.running_var.cpu().double().numpy().copy())


def _worker(rank, world, port, kind, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, dy = _inputs(kind)
        lo = sum(SPLIT[:rank])
        sl = slice(lo, lo + SPLIT[rank])
        out = _step(kind, _model(kind, dist.group.WORLD), x[sl], dy[sl])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["mbconv", "bn_act"])
def test_syncbn_product_blocks_match_concatenated_batch(kind):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, dy = _inputs(kind)
    y1, dx1, g1, rm1, rv1 = _step(kind, _model(kind, None), x, dy)

    def err(a, b):
        return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))

    y2 = np.concatenate([res[0][0], res[1][0]])
    dx2 = np.concatenate([res[0][1], res[1][1]])
    assert err(y2, y1) <= 1e-5
    assert err(dx2, dx1) <= 1e-5
    for r in range(2):  # every rank holds the global running statistics
        assert err(res[r][3], rm1) <= 1e-6 and err(res[r][4], rv1) <= 1e-6
    for k in g1:  # DP: the gradient allreduce sums the per-rank parameter gradients
        assert err(res[0][2][k] + res[1][2][k], g1[k]) <= 1e-5, k
