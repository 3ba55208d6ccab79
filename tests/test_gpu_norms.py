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
