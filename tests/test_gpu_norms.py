"""Config C4 (normalisation sweep): LayerNorm vs BatchNorm fused with swish,
forward + backward, on 4D/5D tensors vs the reference golden vectors and the
oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from golden_util import golden

pytestmark = pytest.mark.gpu


def _mods():
    from paper_2110_10802_b200.norms import BatchNormAct, LayerNormAct

    return LayerNormAct, BatchNormAct


def _t(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32).to(dtype).cuda()


def _h(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("tag", ["4d", "5d"])
def test_golden_ln_bn_swish(tag):
    LN, BN = _mods()
    g = golden("norm_sweep_f64")
    p = lambda k: g[f"ln{tag}_{k}"]  # noqa: E731
    ln = LN(p("x").shape[-1], eps=1e-5)
    ln.gamma.copy_(_t(p("g")))
    ln.beta.copy_(_t(p("b")))
    y = ln.forward(_t(p("x")))
    dx = ln.backward(_t(p("dy")))
    torch.cuda.synchronize()
    for got, key in ((y, "y"), (dx, "dx"), (ln.dgamma, "dg"), (ln.dbeta, "db")):
        assert O.compare(_h(got), p(key)) <= 1e-4, key
    q = lambda k: g[f"bn{tag}_{k}"]  # noqa: E731
    x = q("x")
    C = x.shape[1]
    bn = BN(C, eps=1e-5, momentum=0.9)
    bn.gamma.copy_(_t(q("g")))
    bn.beta.copy_(_t(q("b")))
    bn.running_mean.copy_(_t(q("rm")))
    bn.running_var.copy_(_t(q("rv")))
    cl = lambda a: np.moveaxis(a, 1, -1)  # noqa: E731  channels-last
    y = bn.forward(_t(cl(x)))
    dx = bn.backward(_t(cl(q("dy"))))
    torch.cuda.synchronize()
    assert O.compare(np.moveaxis(_h(y), -1, 1), q("y")) <= 1e-4
    assert O.compare(np.moveaxis(_h(dx), -1, 1), q("dx")) <= 1e-4
    assert O.compare(_h(bn.running_mean), q("new_rm")) <= 1e-4
    assert O.compare(_h(bn.running_var), q("new_rv")) <= 1e-4
    assert O.compare(_h(bn.dgamma), q("dg")) <= 1e-4
    assert O.compare(_h(bn.dbeta), q("db")) <= 1e-4


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("shape", [(8, 16, 28, 28, 64), (32, 64, 14, 14)])
def test_sweep_shapes_vs_oracle(dtype, tol, shape):
    """Channels-last tensors [N, *spatial, C]: LN over C and BN over C."""
    LN, BN = _mods()
    rng = np.random.default_rng(len(shape))
    C = shape[-1]
    x = rng.standard_normal(shape) * 2 + 0.5
    dy = rng.standard_normal(shape)
    if dtype == torch.bfloat16:
        x, dy = O.round_bf16(x).astype(np.float64), O.round_bf16(dy).astype(np.float64)
    gm, bt = 1 + 0.1 * rng.standard_normal(C), 0.1 * rng.standard_normal(C)
    ln = LN(C, eps=1e-5)
    ln.gamma.copy_(_t(gm))
    ln.beta.copy_(_t(bt))
    y = ln.forward(_t(x, dtype))
    dx = ln.backward(_t(dy, dtype))
    bn = BN(C, eps=1e-5)
    bn.gamma.copy_(_t(gm))
    bn.beta.copy_(_t(bt))
    yb = bn.forward(_t(x, dtype))
    dxb = bn.backward(_t(dy, dtype))
    torch.cuda.synchronize()
    wy, _ = O.ln_swish_fwd(x, gm, bt)
    wdx, wdg, wdb = O.ln_swish_bwd(dy, x, gm, bt)
    assert O.compare(_h(y), wy) <= tol
    assert O.compare(_h(dx), wdx) <= tol
    metric = O.compare if dtype == torch.float32 else O.compare_scaled
    assert metric(_h(ln.dgamma), wdg) <= tol
    xc = np.moveaxis(x, -1, 1)  # oracle BN is channel-axis-1
    wyb, _, _ = O.bn_swish_fwd(xc, gm, bt, np.zeros(C), np.ones(C))
    wdxb, wdgb, wdbb = O.bn_swish_bwd(np.moveaxis(dy, -1, 1), xc, gm, bt)
    assert O.compare(np.moveaxis(_h(yb), -1, 1), wyb) <= tol
    assert O.compare(np.moveaxis(_h(dxb), -1, 1), wdxb) <= tol
    assert metric(_h(bn.dgamma), wdgb) <= tol
    assert metric(_h(bn.dbeta), wdbb) <= tol


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("shape", [(32, 56, 56, 64), (3, 7, 7, 1152), (5, 9, 24)])
def test_bn_single_replica_entry_points_match_the_split_calls(dtype, shape):
    """dfx_batchnorm_stats_finalize == dfx_batchnorm_stats + dfx_bn_finalize(nsets 1)
    and dfx_batchnorm_act_bwd_reduce_grads == dfx_batchnorm_act_bwd_reduce + the
    dbeta/dgamma copies: bitwise for the merged sets, bnsum, dbeta and dgamma;
    the finalize arithmetic (var, rstd, running-stat blends) to one fp32 rounding
    (the two kernels may contract it into FMAs differently)."""
    from paper_2110_10802_b200 import _lib
    from paper_2110_10802_b200 import kernels as K

    C = shape[-1]
    rows = int(np.prod(shape[:-1]))
    g = torch.Generator(device="cpu").manual_seed(C + rows)
    x = (torch.randn(shape, generator=g) * 1.5 + 0.3).to(dtype).cuda()
    dy = torch.randn(shape, generator=g).to(dtype).cuda()
    gamma = (1 + 0.1 * torch.randn(C, generator=g)).cuda()
    beta = (0.1 * torch.randn(C, generator=g)).cuda()
    lib = _lib.load()
    ws = torch.empty(lib.dfx_batchnorm_workspace(rows, C), dtype=torch.uint8, device="cuda")
    dt = K.dfx_dtype(x)
    f = lambda *s: torch.zeros(*s, device="cuda")  # noqa: E731
    out = {}
    for fused in (False, True):
        local, mean, var, rstd = f(3, C), f(C), f(C), f(C)
        rm, rv = torch.full((C,), 0.5, device="cuda"), torch.full((C,), 2.0, device="cuda")
        if fused:
            _lib.call("dfx_batchnorm_stats_finalize", dt, rows, C, x.data_ptr(), local.data_ptr(), 1e-3, 0.9,
                      mean.data_ptr(), var.data_ptr(), rstd.data_ptr(), rm.data_ptr(), rv.data_ptr(), ws.data_ptr(),
                      ws.numel(), K._stream())
        else:
            _lib.call("dfx_batchnorm_stats", dt, rows, C, x.data_ptr(), local.data_ptr(), ws.data_ptr(), ws.numel(),
                      K._stream())
            _lib.call("dfx_bn_finalize", C, 1, local.data_ptr(), 1e-3, 0.9, mean.data_ptr(), var.data_ptr(),
                      rstd.data_ptr(), rm.data_ptr(), rv.data_ptr(), K._stream())
        bnsum, dbeta, dgamma = f(3, C), f(C), f(C)
        if fused:
            _lib.call("dfx_batchnorm_act_bwd_reduce_grads", dt, rows, C, dy.data_ptr(), x.data_ptr(), mean.data_ptr(),
                      rstd.data_ptr(), gamma.data_ptr(), beta.data_ptr(), 1, bnsum.data_ptr(), dbeta.data_ptr(),
                      dgamma.data_ptr(), ws.data_ptr(), ws.numel(), K._stream())
        else:
            _lib.call("dfx_batchnorm_act_bwd_reduce", dt, rows, C, dy.data_ptr(), x.data_ptr(), mean.data_ptr(),
                      rstd.data_ptr(), gamma.data_ptr(), beta.data_ptr(), 1, bnsum.data_ptr(), ws.data_ptr(),
                      ws.numel(), K._stream())
            dbeta.copy_(bnsum[0])
            dgamma.copy_(bnsum[1])
        torch.cuda.synchronize()
        out[fused] = [t.clone() for t in (local, mean, var, rstd, rm, rv, bnsum[:2], dbeta, dgamma)]
    names = ("local", "mean", "var", "rstd", "running_mean", "running_var", "bnsum", "dbeta", "dgamma")
    for nm, a, b in zip(names, out[False], out[True]):
        if nm in ("var", "rstd", "running_mean", "running_var"):
            assert torch.allclose(a, b, rtol=1e-6, atol=0), nm
        else:
            assert torch.equal(a, b), nm
